#!/bin/bash
# prof_k.sh <config> <kernel-regex> <out-name>: one ncu --set full capture of a kernel in the bench step
cfg=$1; k=$2; out=$3
mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:$k -s 2 -c 1 -o gpurun_out/$out \
  python bench.py --config $cfg --steps 3 --warmup 3 --no-others --no-cpu-baseline --no-e2e > gpurun_out/$out.log 2>&1
ls -la gpurun_out/$out.ncu-rep
