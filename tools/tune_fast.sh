timeout 600 python -m pytest tests/test_gpu_sc.py -x -q 2>&1 | tail -2
for cfg in "4 2 2" "4 2 1" "4 3 2" "4 2 0" "4 2 4" "8 2 4" "8 2 3" "8 1 4" "2 2 1" "4 1 2"; do
 set -- $cfg
 echo "FAST wpc=$1 stages=$2 match=$3 $(CDX_SCF_WARPS=$1 CDX_SCF_STAGES=$2 CDX_SCF_MATCH=$3 timeout 120 python bench.py --steps 30 --no-e2e --no-cpu-baseline | python -c 'import json,sys;d=json.loads(sys.stdin.read().strip().splitlines()[-1]);r=d["roofline"];print(round(r["kernel_ms"],4),"ms",round(r["achieved"]),"GB/s frac",round(r["frac"],3))')"
done
python tools/sc_rate.py 2>&1 | tail -5
