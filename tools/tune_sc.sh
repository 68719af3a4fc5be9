timeout 600 python -m pytest tests/test_gpu_sc.py -x -q 2>&1 | tail -2
for w in 2 4 8; do for st in 2 3 4; do
 echo "SC warps=$w stages=$st $(CDX_SC_WARPS=$w CDX_SC_STAGES=$st timeout 120 python bench.py --steps 30 --no-e2e --no-cpu-baseline | python -c 'import json,sys;d=json.loads(sys.stdin.read().strip().splitlines()[-1]);r=d["roofline"];print(round(r["kernel_ms"],4),"ms",round(r["achieved"]),"GB/s frac",round(r["frac"],3))')"
done; done
