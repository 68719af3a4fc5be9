# round-1 profiling: launch lists + one --set full capture per hot kernel (1 GPU)
B="python bench.py --steps 3 --warmup 3 --no-others --no-cpu-baseline --no-e2e"
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/r1_launches_C.csv $B --config C > /dev/null 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/r1_launches_B.csv $B --config B > /dev/null 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/r1_launches_D.csv $B --config D > /dev/null 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/r1_launches_E.csv $B --config E > /dev/null 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:sc_fast_kernel -s 3 -c 1 -o gpurun_out/r1_full_sc $B --config C > /dev/null 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:cot_run -s 3 -c 1 -o gpurun_out/r1_full_cot $B --config B > /dev/null 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:reward_kernel -s 3 -c 1 -o gpurun_out/r1_full_reward $B --config D > /dev/null 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:allocate_scan -s 3 -c 1 -o gpurun_out/r1_full_alloc $B --config C > /dev/null 2>&1
ls -la gpurun_out
