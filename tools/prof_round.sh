#!/bin/bash
# prof_round.sh <tag>: launch lists (C, B, D, E) + one `ncu --set full` capture per hot kernel
# + the default bench line, all under gpurun_out/ (summarise with tools/summarize_profiles.py)
tag=${1:-r1i}
mkdir -p gpurun_out
B="python bench.py --steps 3 --warmup 3 --no-others --no-cpu-baseline --no-e2e"
M="gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum"
for c in C B D E J; do
  timeout 300 ncu --metrics $M --clock-control none --csv --log-file gpurun_out/${tag}_launches_$c.csv $B --config $c > /dev/null 2>&1
done
timeout 300 ncu --set full --clock-control none --import-source on -k regex:sc_fast_kernel -s 3 -c 1 -o gpurun_out/${tag}_full_sc $B --config C > /dev/null 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:allocate_scan -s 3 -c 1 -o gpurun_out/${tag}_full_alloc $B --config C > /dev/null 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:cot_run64 -s 3 -c 1 -o gpurun_out/${tag}_full_cot $B --config B > /dev/null 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:reward_quad -s 2 -c 1 -o gpurun_out/${tag}_full_reward $B --config D > /dev/null 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:os_pass -s 4 -c 1 -o gpurun_out/${tag}_full_gang $B --config E > /dev/null 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:parse_lines -s 1 -c 1 -o gpurun_out/${tag}_full_jsonl $B --config J > /dev/null 2>&1
timeout 900 python bench.py > gpurun_out/${tag}_bench.json 2> gpurun_out/${tag}_bench.err
ls gpurun_out | grep $tag
