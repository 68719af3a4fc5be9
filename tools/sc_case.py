"""Run sc_certaindex on one synthetic cluster structure (for ncu captures)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2412_20993_b200 import Context, GenParams, Threshold
case = sys.argv[1]
R = int(sys.argv[2]) if len(sys.argv) > 2 else 1 << 18
P, S = 64, 32
cx = Context(0)
if case == "synthetic":
    ids = cx.gen_sc(GenParams(seed=3, conv_hi=64), R, P, S)
else:
    k = {"equal": 1, "two": 2, "five": 5, "distinct": 32}[case]
    ids = (torch.arange(S, dtype=torch.int32, device="cuda") % k).expand(R, P, S).contiguous()
hc = torch.empty((R, P), dtype=torch.float32, device="cuda")
mt = torch.empty((R, 2), dtype=torch.int32, device="cuda")
for _ in range(4):
    cx.sc_certaindex(ids, [Threshold(0, 0.7, 0)], hcert=hc, meets=mt)
torch.cuda.synchronize()
