import sys, numpy as np, torch
sys.path.insert(0, '.')
from paper_2412_20993_b200 import Context, AllocPolicy
cx = Context(0)
for trial in range(int(sys.argv[1]) if len(sys.argv) > 1 else 5):
    R = [1 << 20, 1, 5000, 3 << 18][trial % 4]
    meets = torch.randint(-2**31, 2**31 - 1, (R, 2), dtype=torch.int32, device="cuda")
    out = cx.allocate_scan(meets, R, 64, AllocPolicy(kind=4, detect_at=5, resource_cap=64, recheck_every=3, tokens_per_unit=2048))
    cx.sync()
    g = out["granted"].to(torch.int64) * 2048
    excl = torch.cumsum(g, 0) - g
    bad = (excl != out["offsets"]).nonzero()
    n_kept = int(out["scalars"][0])
    print(trial, R, "offset mismatches", bad.numel(), "first", bad[:3].flatten().tolist(),
          "n_kept ok", n_kept == int((out["granted"] > 5).sum()), flush=True)
    if bad.numel():
        i = int(bad[0]); print("  got", int(out["offsets"][i]), "want", int(excl[i]), "tile", i // 2048)
