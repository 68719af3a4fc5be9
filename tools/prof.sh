# one ncu --set full capture of each hot kernel (1 GPU), plus a launch list of the bench step
set -x
timeout 600 ncu --set full --clock-control none --import-source on -k regex:sc_certaindex -s 3 -c 1 -o gpurun_out/prof_sc python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/prof_sc.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:cot_exit -s 3 -c 1 -o gpurun_out/prof_cot python bench.py --config B --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/prof_cot.log 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:allocate_scan -s 3 -c 1 -o gpurun_out/prof_alloc python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/prof_alloc.log 2>&1
for st in 1 2; do echo "SC stages=$st $(CDX_SC_STAGES=$st timeout 120 python bench.py --steps 30 --no-e2e --no-cpu-baseline | python -c 'import json,sys;d=json.loads(sys.stdin.read().strip().splitlines()[-1]);r=d["roofline"];print(round(r["kernel_ms"],4),"ms",round(r["achieved"]),"GB/s frac",round(r["frac"],3))')"; done
ls -la gpurun_out
