import sys, time, torch, ctypes as C
sys.path.insert(0, '/root/repo')
from paper_2412_20993_b200 import Context, InterPolicy, c_inter
cx = Context(0)
N=64
dev={k: torch.zeros(N, dtype=dt, device="cuda") for k,dt in (("arrival",torch.float64),("last_service",torch.float64),("iter_tok_sum",torch.int64),("iter_count",torch.int32),("knob",torch.int32),("cap",torch.int32),("terminated",torch.uint8))}
pol=InterPolicy(order=1, starvation_limit=0.5, prior_tokens=128.0)
def t(name, f, n=5000):
    f()
    t0=time.perf_counter()
    for _ in range(n): f()
    print(name, "%.2f us" % ((time.perf_counter()-t0)/n*1e6))
t("current_stream(dev)", lambda: torch.cuda.current_stream(0).cuda_stream)
t("current_stream()", lambda: torch.cuda.current_stream().cuda_stream)
t("_bind_stream", cx._bind_stream)
t("_prog_soa", lambda: cx._prog_soa(dev, 0))
t("c_inter", lambda: c_inter(pol))
o=torch.empty(N, dtype=torch.int32, device="cuda")
t("slice", lambda: o[:10])
t("gang_priority N=64 (incl sync)", lambda: cx.gang_priority(dev, pol, 1.0, out=o), 2000)
