"""Time K1 (cdx_canon_intern) on config K's arena: python tools/t_intern.py [log2 n] [reps]"""
import sys
import torch
sys.path.insert(0, '/root/repo')
from paper_2412_20993_b200 import Context, GenParams, synth
lg = int(sys.argv[1]) if len(sys.argv) > 1 else 27
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 10
cx = Context(0)
n = 1 << lg
ids = cx.gen_sc(GenParams(seed=20993 + 8, conv_hi=64), n // 2048, 64, 32).view(-1)
a, o = synth.answer_arena_torch(ids, 12)
del ids
r = cx.canon_intern(a, o)
cx.sync()
ts = []
for _ in range(reps):
    s, e = torch.cuda.Event(True), torch.cuda.Event(True)
    s.record()
    cx.canon_intern(a, o)
    e.record()
    torch.cuda.synchronize()
    ts.append(s.elapsed_time(e))
print(" ".join(f"{x:.3f}" for x in ts))
ts.sort()
print(f"n=2^{lg} unique={r[3]} median {ts[len(ts) // 2]:.3f} ms min {ts[0]:.3f} ms", flush=True)
