#!/bin/bash
# compute-sanitizer over the kernels changed late in round 2 (K2 work order, K4 block order,
# K5 tile body, sc_decide): memcheck, racecheck, synccheck on the reduced-size tests
mkdir -p gpurun_out
K="not full_scale and not 40000 and not all_partitions and not exhaustive and not large"
for tool in memcheck racecheck synccheck; do
  timeout 900 compute-sanitizer --tool $tool --print-limit 20 --error-exitcode 99 \
      python -m pytest tests/test_gpu_sc_decide.py tests/test_gpu_sc.py tests/test_gpu_reward.py -m gpu -q -k "$K" \
      -p no:cacheprovider > gpurun_out/r2_sanitize_late_$tool.log 2>&1
  echo "$tool rc=$? $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY|passed|failed' gpurun_out/r2_sanitize_late_$tool.log | tail -2 | tr '\n' ' ')"
done
