import sys, numpy as np, torch
sys.path.insert(0, '.')
from oracle import oracle as O
from paper_2412_20993_b200 import Context
G, T, W = [int(x) for x in sys.argv[1:4]]
with_ids = len(sys.argv) < 5 or sys.argv[4] != "noids"
cx = Context(0)
g = O.gen_params(seed=3, conv_hi=T)
rw, ids = O.gen_reward(g, G, T, W)
agg = (np.arange(G) % 2).astype(np.uint8)
R, H, M = cx.reward_certaindex(torch.from_numpy(rw).cuda(), torch.from_numpy(ids.view(np.int32)).cuda() if with_ids else None,
                               torch.from_numpy(agg).cuda())
print("launched", flush=True)
cx.sync()
_, R32, Ho = O.reward_certaindex(rw, ids if with_ids else None, agg)
print("R ok", np.array_equal(R.cpu().numpy().view(np.uint32), R32.view(np.uint32)),
      "H ok", (not with_ids) or np.array_equal(H.cpu().numpy().view(np.uint32), Ho.view(np.uint32)), flush=True)
