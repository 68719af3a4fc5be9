#!/bin/bash
mkdir -p gpurun_out
K="gang and not 3000001 and not 1212121 and not 4194304 and not merge"
for tool in memcheck racecheck synccheck; do
  timeout 900 compute-sanitizer --tool $tool --print-limit 20 --error-exitcode 99 \
      python -m pytest tests/test_gpu_intern_gang.py -m gpu -q -k "$K" -p no:cacheprovider > gpurun_out/r4_sanitize_gang_$tool.log 2>&1
  echo "$tool rc=$? $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY|passed|failed' gpurun_out/r4_sanitize_gang_$tool.log | tail -2 | tr '\n' ' ')"
done
