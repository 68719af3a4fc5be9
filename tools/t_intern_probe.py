import sys, torch, numpy as np
sys.path.insert(0, '/root/repo')
from paper_2412_20993_b200 import Context, GenParams, synth
cx = Context(0)
for lg in (20, 22, 24, 27):
    n = 1 << lg
    ids = cx.gen_sc(GenParams(seed=5, conv_hi=64), n // 2048, 64, 32).view(-1)
    a, o = synth.answer_arena_torch(ids)
    r = cx.canon_intern(a, o)
    try:
        cx.sync(); err = None
    except Exception as e:
        err = str(e)
    s, e2 = torch.cuda.Event(True), torch.cuda.Event(True)
    s.record(); cx.canon_intern(a, o); e2.record(); torch.cuda.synchronize()
    print(lg, r[3], err, s.elapsed_time(e2), flush=True)
