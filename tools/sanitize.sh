#!/bin/bash
# compute-sanitizer over the parity suite's kernels at reduced sizes:
# memcheck, racecheck (shared-memory hazards), synccheck (barrier / warp-sync misuse),
# initcheck.  Summaries go to gpurun_out/sanitize_<tool>.log.
mkdir -p gpurun_out
K="sc_certaindex or allocate or cot or reward or gang or intern or aggregate or eps or jsonl or graph"
for tool in memcheck racecheck synccheck initcheck; do
  timeout 1500 compute-sanitizer --tool $tool --print-limit 20 --error-exitcode 99 \
      python -m pytest tests -m gpu -x -q -k "$K and not large and not 50000 and not 3000" -p no:cacheprovider \
      > gpurun_out/sanitize_$tool.log 2>&1
  echo "$tool rc=$? $(grep -E 'ERROR SUMMARY|passed|failed' gpurun_out/sanitize_$tool.log | tail -2 | tr '\n' ' ')"
done
