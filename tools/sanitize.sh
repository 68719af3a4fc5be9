#!/bin/bash
# compute-sanitizer over the GPU parity suite at reduced sizes: memcheck,
# racecheck (shared-memory hazards), synccheck (barrier / warp-sync misuse).  initcheck is
# run on the kernel-level tests only (it is slow).  Summaries: gpurun_out/sanitize_<tool>.log
mkdir -p gpurun_out
SKIP="not memory_growth and not 1048576 and not full_scale and not len8 and not all_partitions and not fuzz and not large and not 50000 and not 3000 and not dropin and not batch_cpp and not sim and not scheduler_facade"
for tool in memcheck racecheck synccheck; do
  timeout 900 compute-sanitizer --tool $tool --print-limit 20 --error-exitcode 99 \
      python -m pytest tests -m gpu -q -k "$SKIP" -p no:cacheprovider > gpurun_out/sanitize_$tool.log 2>&1
  echo "$tool rc=$? $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY|passed|failed' gpurun_out/sanitize_$tool.log | tail -2 | tr '\n' ' ')"
done
timeout 900 compute-sanitizer --tool initcheck --print-limit 20 --error-exitcode 99 \
    python -m pytest tests/test_gpu_sc.py tests/test_gpu_cot.py -m gpu -q -k "$SKIP and not all_partitions and not exhaustive" \
    -p no:cacheprovider > gpurun_out/sanitize_initcheck.log 2>&1
echo "initcheck rc=$? $(grep -E 'ERROR SUMMARY|passed|failed' gpurun_out/sanitize_initcheck.log | tail -2 | tr '\n' ' ')"
