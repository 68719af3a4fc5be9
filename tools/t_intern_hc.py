"""K1 on a high-cardinality arena: n answers drawn from `vocab` distinct strings (random or
grouped order), e.g. JSONL program ids: python tools/t_intern_hc.py [log2 n] [vocab] [order]"""
import sys
import numpy as np
import torch
sys.path.insert(0, '/root/repo')
from paper_2412_20993_b200 import Context
lg = int(sys.argv[1]) if len(sys.argv) > 1 else 20
vocab = int(sys.argv[2]) if len(sys.argv) > 2 else 16384
order = sys.argv[3] if len(sys.argv) > 3 else "random"
n = 1 << lg
rng = np.random.default_rng(5)
v = rng.integers(0, vocab, n) if order == "random" else np.sort(rng.integers(0, vocab, n))
strs = [f'"prog-{x:06d}"'.encode() for x in range(vocab)]
lens = np.array([len(strs[x]) for x in v], dtype=np.int64)
off = np.zeros(n + 1, dtype=np.int64)
np.cumsum(lens, out=off[1:])
arena = np.frombuffer(b"".join(strs[x] for x in v), dtype=np.uint8)
cx = Context(0)
a = torch.from_numpy(arena.copy()).cuda()
o = torch.from_numpy(off).cuda()
r = cx.canon_intern(a, o, markers=(), want_hes=False)
cx.sync()
ts = []
for _ in range(10):
    s, e = torch.cuda.Event(True), torch.cuda.Event(True)
    s.record()
    cx.canon_intern(a, o, markers=(), want_hes=False)
    e.record()
    torch.cuda.synchronize()
    ts.append(s.elapsed_time(e))
ts.sort()
print(f"n=2^{lg} vocab={vocab} {order}: unique={r[3]} median {ts[5]:.3f} ms min {ts[0]:.3f} ms", flush=True)
