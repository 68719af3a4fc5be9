import sys, time, torch, numpy as np
sys.path.insert(0, '/root/repo')
import bench
from paper_2412_20993_b200 import Context, InterPolicy
cx = Context(0)
N = 1 << 22
soa, now = bench.gang_inputs(N, 20993 + 5, 0.5)
dev = {k: torch.from_numpy(np.ascontiguousarray(v)).cuda() for k, v in soa.items()}
pol = InterPolicy(order=1, starvation_limit=0.5, prior_tokens=128.0)
import os
for ps in ["1", "0", "1"]:
    os.environ["CDX_GANG_PS"] = ps
    o = cx.gang_priority(dev, pol, now)[0]; cx.sync()
    ts = []
    for _ in range(20):
        s, e = torch.cuda.Event(True), torch.cuda.Event(True)
        s.record(); cx.gang_priority(dev, pol, now); e.record(); torch.cuda.synchronize()
        ts.append(s.elapsed_time(e))
    ts.sort()
    print("ps", ps, "median %.4f ms min %.4f" % (ts[10], ts[0]), "n", o.shape[0], flush=True)
os.environ["CDX_GANG_PS"] = "1"
os.environ["CDX_GANG_PS_PROF"] = "1"
for _ in range(3):
    cx.gang_priority(dev, pol, now); cx.sync()
del os.environ["CDX_GANG_PS_PROF"]
# fixed per-call overhead: a 64-program call (kernel ~10 us), events around the Python call
small = {k: v[:64].contiguous() for k, v in dev.items()}
for ps in ["1", "0"]:
    os.environ["CDX_GANG_PS"] = ps
    ts = []
    for _ in range(50):
        s, e = torch.cuda.Event(True), torch.cuda.Event(True)
        s.record(); cx.gang_priority(small, pol, now); e.record(); torch.cuda.synchronize()
        ts.append(s.elapsed_time(e))
    ts.sort()
    t0 = time.perf_counter()
    for _ in range(200):
        cx.gang_priority(small, pol, now)
    wall = (time.perf_counter() - t0) / 200 * 1e3
    print("N=64 ps", ps, "event median %.4f ms, wall %.4f ms" % (ts[25], wall), flush=True)
