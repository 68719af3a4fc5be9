for cfg in "8 1 3" "8 1 4" "8 1 5" "8 1 2" "4 1 1" "4 1 2" "4 1 3" "6 1 3" "6 1 2" "8 2 5"; do
 set -- $cfg
 echo "FAST wpc=$1 stages=$2 match=$3 $(CDX_SCF_WARPS=$1 CDX_SCF_STAGES=$2 CDX_SCF_MATCH=$3 timeout 120 python bench.py --steps 50 --no-e2e --no-cpu-baseline | python -c 'import json,sys;d=json.loads(sys.stdin.read().strip().splitlines()[-1]);r=d["roofline"];print(round(r["kernel_ms"],4),"ms",round(r["achieved"]),"GB/s frac",round(r["frac"],3))')"
done
