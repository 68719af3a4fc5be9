# quick GPU check: parity tests + C and B kernel timings
timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
for cfg in C B; do
  echo "$cfg $(timeout 120 python bench.py --config $cfg --steps 30 --no-e2e --no-cpu-baseline | python -c 'import json,sys;d=json.loads(sys.stdin.read().strip().splitlines()[-1]);r=d["roofline"];print(round(r["kernel_ms"],4),"ms",round(r["achieved"]),"GB/s frac",round(r["frac"],3), "step", round(d["ms_per_step"],4))')"
done
for st in 1 2; do echo "SC stages=$st $(CDX_SC_STAGES=$st timeout 120 python bench.py --steps 30 --no-e2e --no-cpu-baseline | python -c 'import json,sys;d=json.loads(sys.stdin.read().strip().splitlines()[-1]);r=d["roofline"];print(round(r["kernel_ms"],4),"ms",round(r["achieved"]),"GB/s frac",round(r["frac"],3))')"; done
