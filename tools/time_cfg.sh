#!/bin/bash
# time_cfg.sh <config> [label]: one bench line -> "label cfg kernel_ms GB/s frac" (env passes through)
cfg=$1; label=${2:-run}
timeout 300 python bench.py --config $cfg --steps 20 --no-others --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | \
python -c "import json,sys;d=json.loads(sys.stdin.read());r=d['roofline'];print('$label',d['config']['workload'],round(r['kernel_ms'],4),'ms',round(r['achieved']),'GB/s frac',round(r['frac'],3),'step',round(d['ms_per_step'],4))"
