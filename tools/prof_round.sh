#!/bin/bash
# prof_round.sh <tag> [configs]: launch lists + one `ncu --set full` capture per hot kernel +
# the default bench line, all under gpurun_out/ (summarise with tools/summarize_profiles.py <tag> <tag>)
tag=${1:-r2}
cfgs=${2:-"A B C D E G J"}
mkdir -p gpurun_out
B="python bench.py --steps 3 --warmup 3 --no-others --no-cpu-baseline --no-e2e"
M="gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum"
for c in $cfgs; do
  timeout 300 ncu --metrics $M --clock-control none --csv --log-file gpurun_out/${tag}_launches_$c.csv $B --config $c > /dev/null 2>&1
done
full() {  # full <name> <kernel regex> <skip> <config>
  timeout 300 ncu --set full --clock-control none --import-source on -k regex:$2 -s $3 -c 1 -o gpurun_out/${tag}_full_$1 $B --config $4 > /dev/null 2>&1
}
[ -n "$FULL" ] && for spec in $FULL; do IFS=: read n k s c <<< "$spec"; full $n $k $s $c; done
[ -n "$BENCH" ] && timeout 900 python bench.py > gpurun_out/${tag}_bench.json 2> gpurun_out/${tag}_bench.err
ls gpurun_out | grep $tag
