"""Per-row cost of sc_certaindex on L2-resident vs HBM-resident inputs and on
different cluster structures (diagnostic; not part of the bench contract)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2412_20993_b200 import Context, GenParams, Threshold

cx = Context(0)
P, S = 64, 32
def rate(ids, reps=20):
    R = ids.shape[0]
    hc = torch.empty((R, P), dtype=torch.float32, device="cuda")
    mt = torch.empty((R, 2), dtype=torch.int32, device="cuda")
    th = [Threshold(0, 0.7, 0)]
    for _ in range(3):
        cx.sc_certaindex(ids, th, hcert=hc, meets=mt)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize(); a.record()
    for _ in range(reps):
        cx.sc_certaindex(ids, th, hcert=hc, meets=mt)
    b.record(); torch.cuda.synchronize()
    ms = a.elapsed_time(b) / reps
    return ms, ms * 1e6 / (R * P)
for R in (8192, 1 << 20):
    ids = cx.gen_sc(GenParams(seed=3, conv_hi=64), R, P, S)
    ms, ns = rate(ids)
    print(f"synthetic R={R}: {ms:.4f} ms, {ns*1e3:.2f} ps/row, {R*P*S*4/ms/1e6:.0f} GB/s")
    same = torch.zeros_like(ids)
    ms, ns = rate(same); print(f"  all-equal  : {ms:.4f} ms, {R*P*S*4/ms/1e6:.0f} GB/s")
    distinct = torch.arange(S, dtype=torch.int32, device="cuda").expand(R, P, S).contiguous()
    ms, ns = rate(distinct); print(f"  all-distinct: {ms:.4f} ms, {R*P*S*4/ms/1e6:.0f} GB/s")
    two = (torch.arange(S, dtype=torch.int32, device="cuda") % 2).expand(R, P, S).contiguous()
    ms, ns = rate(two); print(f"  two-clusters: {ms:.4f} ms, {R*P*S*4/ms/1e6:.0f} GB/s")
    five = (torch.arange(S, dtype=torch.int32, device="cuda") % 5).expand(R, P, S).contiguous()
    ms, ns = rate(five); print(f"  five-clusters: {ms:.4f} ms, {R*P*S*4/ms/1e6:.0f} GB/s")
    del ids, same, distinct, two, five
