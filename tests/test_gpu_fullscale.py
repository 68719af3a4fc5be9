"""Full-scale bit-exact parity at the BASELINE shapes (SURVEY.md §4 plan item 4): configs B,
C and D exactly as bench.py runs them, every output of every request / program compared
with the oracle.  The traces are generated on the device (the generator's own parity is
tested elsewhere) and copied to the host; the oracle runs in request chunks on all host
threads (ctypes releases the GIL)."""
import os
from concurrent.futures import ThreadPoolExecutor

import numpy as np
import pytest

from oracle import oracle as O

pytestmark = pytest.mark.gpu

SIG_E, SIG_R, GE = 0, 1, 0


def _chunks(n, k):
    step = (n + k - 1) // k
    return [(a, min(n, a + step)) for a in range(0, n, step)]


def _pool():
    return ThreadPoolExecutor(max_workers=min(32, os.cpu_count() or 1))


def test_config_c_full_scale(ctx):
    """2^20 requests x 64 probes x 32 samples: K2 certaindex bits and meets, then K5."""
    from paper_2412_20993_b200 import AllocPolicy, GenParams, Threshold
    R, P, S = 1 << 20, 64, 32
    ids = ctx.gen_sc(GenParams(seed=20993 + 3, conv_hi=64), R, P, S)
    h, meets = ctx.sc_certaindex(ids, [Threshold(SIG_E, 0.7, GE)])
    pol = AllocPolicy(kind=2, detect_at=5, resource_cap=P, tokens_per_unit=64 * S)
    out = ctx.allocate_scan(meets, R, P, pol)
    ctx.sync()
    ids_h = ids.cpu().numpy().view(np.uint32)
    del ids
    h_h = h.cpu().numpy().view(np.uint32)
    m_h = meets.cpu().numpy().view(np.uint32)
    om = np.empty_like(m_h)

    def run(ab):
        a, b = ab
        _, oh32, omm = O.sc_certaindex(ids_h[a:b], [(SIG_E, 0.7, GE)])
        om[a:b] = omm
        return bool(np.array_equal(oh32.view(np.uint32), h_h[a:b]))

    with _pool() as ex:
        assert all(ex.map(run, _chunks(R, 64)))
    assert np.array_equal(om, m_h)
    ref = O.allocate_scan(om, R, P, 2, 5, P, 1, 64 * S)
    for k in ("exit_knob", "reason", "granted", "offsets"):
        assert np.array_equal(out[k].cpu().numpy(), ref[k].astype(out[k].cpu().numpy().dtype)), k
    n_kept, saved, _ = out["scalars"].cpu().numpy().tolist()
    assert n_kept == ref["n_kept"] and saved == ref["tokens_saved"]
    assert np.array_equal(out["kept"][:n_kept].cpu().numpy().view(np.uint32), ref["kept"])


def test_config_b_full_scale(ctx):
    """2^20 requests x 64 probes, window 3, tau 0.9, budget at the last probe (config B)."""
    from paper_2412_20993_b200 import GenParams, ProbeConfig
    R, P = 1 << 20, 64
    ids, hes = ctx.gen_cot(GenParams(seed=20993 + 2, conv_hi=64, hesitation_prob=0.05), R, P)
    res = ctx.cot_exit(ids, hes, ProbeConfig(64, 3, 0.9, 4096))
    ctx.sync()
    ids_h = ids.cpu().numpy().view(np.uint32)
    hes_h = hes.cpu().numpy().view(np.uint64)
    cfg = O.probe_cfg(64, 3, 0.9, 4096)
    names = ("exit_step", "reason", "final_id", "low_conf")
    got = {k: res[k].cpu().numpy() for k in names}
    parts = {}

    def run(ab):
        a, b = ab
        parts[a] = O.cot_exit(ids_h[a:b], hes_h[a:b], cfg)
        return a

    with _pool() as ex:
        list(ex.map(run, _chunks(R, 64)))
    keys = sorted(parts)
    for name in names:
        ref = np.concatenate([parts[a][name] for a in keys])
        assert np.array_equal(got[name].view(ref.dtype), ref), name


def test_config_d_full_scale(ctx):
    """2^18 programs x 16 steps x 64 nodes, MCTS (even) / Rebase (odd), PAPER Table 3
    thresholds (config D): R, H~ and meets bits for every (program, step)."""
    import torch
    from paper_2412_20993_b200 import GenParams, Threshold
    G, T, W = 1 << 18, 16, 64
    rw, rid = ctx.gen_reward(GenParams(seed=20993 + 4, conv_hi=16), G, T, W)
    agg = (torch.arange(G, device="cuda") % 2).to(torch.uint8)
    th_mcts = [(0, 0.99, 0), (1, 0.4, 0)]
    th_rebase = [(0, 0.85, 0), (1, 0.99, 0)]
    R, H, meets = ctx.reward_certaindex(rw, rid, agg, [Threshold(*t) for t in th_mcts],
                                        [Threshold(*t) for t in th_rebase])
    ctx.sync()
    rw_h, id_h = rw.cpu().numpy(), rid.cpu().numpy().view(np.uint32)
    agg_h = agg.cpu().numpy()
    R_h, H_h, m_h = R.cpu().numpy(), H.cpu().numpy(), meets.cpu().numpy().view(np.uint32)

    def run(ab):
        a, b = ab
        R64, R32, Ho, H64 = O.reward_certaindex(rw_h[a:b], id_h[a:b], agg_h[a:b], want_h64=True)
        good = np.array_equal(R32.view(np.uint32), R_h[a:b].view(np.uint32))
        good = good and np.array_equal(Ho.view(np.uint32), H_h[a:b].view(np.uint32))
        # meets: each program's Table-3 thresholds on the FP64 (H~, R), bit t of word 0
        ok = np.where(agg_h[a:b, None] == 1, (H64 >= 0.85) & (R64 >= 0.99), (H64 >= 0.99) & (R64 >= 0.4))
        bits = (ok.astype(np.uint32) << np.arange(T, dtype=np.uint32)).sum(axis=1, dtype=np.uint64)
        return good and np.array_equal(bits.astype(np.uint32), m_h[a:b, 0])

    with _pool() as ex:
        assert all(ex.map(run, _chunks(G, 64)))
