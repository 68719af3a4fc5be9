#!/bin/bash
# compute-sanitizer over the mixed step (forked engine streams) and the JSONL direct interning
mkdir -p gpurun_out
K="not 1048576 and not fuzz"
for tool in memcheck racecheck synccheck; do
  timeout 900 compute-sanitizer --tool $tool --print-limit 20 --error-exitcode 99 \
      python -m pytest tests/test_gpu_mixed.py tests/test_jsonl.py -m gpu -q -k "$K" \
      -p no:cacheprovider > gpurun_out/r2_sanitize_mixed_jsonl_$tool.log 2>&1
  echo "$tool rc=$? $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY|passed|failed' gpurun_out/r2_sanitize_mixed_jsonl_$tool.log | tail -2 | tr '\n' ' ')"
done
