"""Time K2 on config C's shape with and without the majority output (CUDA events, on the
context stream).  Usage: python tools/time_sc_majority.py"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2412_20993_b200 import Context, GenParams, Threshold  # noqa: E402

R, P, S = 1 << 20, 64, 32
ctx = Context(0)
ids = ctx.gen_sc(GenParams(seed=3, conv_hi=P), R, P, S)
hc = ctx.empty((R, P), torch.float32)
mj = ctx.empty((R, P), torch.float32)
meets = ctx.empty((R, 2), torch.int32)
from paper_2412_20993_b200 import c_thresholds, _ptr  # noqa: E402
res = {}
for name, ths, want_maj in [("entropy", [Threshold(0, 0.7, 0)], False),
                            ("entropy+majority_out", [Threshold(0, 0.7, 0)], True),
                            ("majority_threshold", [Threshold(4, 0.5, 0), Threshold(0, 0.7, 0)], True)]:
    arr, n = c_thresholds(ths)
    def run():
        ctx._bind_stream()
        ctx._check(ctx.lib.cdx_sc_certaindex_ex(ctx.h, _ptr(ids), R, P, S, arr, n, _ptr(hc), _ptr(mj) if want_maj else None,
                                                _ptr(meets)))
    for _ in range(3):
        run()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    st = torch.cuda.current_stream()
    s.record(st)
    for _ in range(20):
        run()
    e.record(st)
    torch.cuda.synchronize()
    ms = s.elapsed_time(e) / 20
    byts = R * P * S * 4 + R * P * 4 * (2 if want_maj else 1) + R * 2 * 4
    res[name] = dict(ms=ms, gbs=byts / ms / 1e6)
print(json.dumps(res))
