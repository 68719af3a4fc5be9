import sys, numpy as np, torch
sys.path.insert(0, '.')
from paper_2412_20993_b200 import Context, AllocPolicy, Threshold, GenParams
cx = Context(0)
R = int(sys.argv[1]) if len(sys.argv) > 1 else 1
ids = cx.gen_sc(GenParams(seed=78, conv_hi=64), R, 64, 32)
_, meets = cx.sc_certaindex(ids, [Threshold(0, 0.7, 0)], want_hcert=False)
cx.sync(); print("sc ok", flush=True)
out = cx.allocate_scan(meets, R, 64, AllocPolicy(kind=2, detect_at=5, resource_cap=64, tokens_per_unit=2048), base_offset=12345)
cx.sync(); print("alloc ok", out["scalars"].cpu().tolist(), flush=True)
