set -e
timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
for st in 2 3; do for tile in 16384 32768 65536; do
 echo "SC stages=$st tile=$tile $(CDX_SC_STAGES=$st CDX_SC_TILE=$tile timeout 120 python bench.py --steps 30 --no-e2e --no-cpu-baseline | python -c 'import json,sys;d=json.loads(sys.stdin.read().strip().splitlines()[-1]);r=d["roofline"];print(round(r["kernel_ms"],4),"ms",round(r["achieved"]),"GB/s frac",round(r["frac"],3),"alloc",round(r["allocate_scan_ms"],4))')"
done; done
for rows in 32 64 128; do for st in 1 2 3; do
 echo "COT rows=$rows stages=$st $(CDX_COT_ROWS=$rows CDX_COT_STAGES=$st timeout 120 python bench.py --config B --steps 30 --no-cpu-baseline | python -c 'import json,sys;d=json.loads(sys.stdin.read().strip().splitlines()[-1]);r=d["roofline"];print(round(r["kernel_ms"],4),"ms",round(r["achieved"]),"GB/s frac",round(r["frac"],3))')"
done; done
