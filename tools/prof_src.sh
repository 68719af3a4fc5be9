# ncu --set full of the SC and CoT kernels (current build) for source-level stall analysis
timeout 600 ncu --set full --clock-control none --import-source on -k regex:sc_certaindex -s 3 -c 1 -o gpurun_out/prof_sc2 python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:cot_exit -s 3 -c 1 -o gpurun_out/prof_cot2 python bench.py --config B --steps 3 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
ls gpurun_out
