timeout 600 python -m pytest tests/test_gpu_sc.py tests/test_gpu_cot.py -x -q 2>&1 | tail -2
python tools/sc_rate.py 2>&1 | tail -5
CDX_SC_IMPL=match python tools/sc_rate.py 2>&1 | tail -5
for cfg in C B; do
  echo "$cfg $(timeout 120 python bench.py --config $cfg --steps 30 --no-e2e --no-cpu-baseline | python -c 'import json,sys;d=json.loads(sys.stdin.read().strip().splitlines()[-1]);r=d["roofline"];print(round(r["kernel_ms"],4),"ms",round(r["achieved"]),"GB/s frac",round(r["frac"],3), "step", round(d["ms_per_step"],4))')"
done
