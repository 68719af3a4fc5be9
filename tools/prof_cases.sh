for c in five distinct; do
timeout 300 ncu --set full --clock-control none --import-source on -k regex:sc_certaindex -s 3 -c 1 -o gpurun_out/prof_sc_$c python tools/sc_case.py $c > /dev/null 2>&1
done
ls gpurun_out
