"""Every alternative engine a tuning knob selects ("Tuning overrides") gives the
same bits as the default on shapes the fast paths would otherwise take: K2's generic
warp-match kernel and its match-only warps, K3's run-length and sliding-window kernels,
K4's one-thread-per-program kernel."""
import numpy as np
import pytest

from oracle import oracle as O

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("impl", ["match", "matchonly", "alu"])
@pytest.mark.parametrize("R,P,S", [(300, 64, 32), (500, 32, 16), (700, 64, 8)])
def test_sc_engine_knobs(ctx, monkeypatch, impl, R, P, S):
    import torch
    from paper_2412_20993_b200 import Threshold
    monkeypatch.setenv("CDX_SC_IMPL", impl)
    g = dict(seed=R + S, conv_hi=P)
    ids = ctx.gen_sc(__import__("paper_2412_20993_b200").GenParams(**g), R, P, S)
    h, m = ctx.sc_certaindex(ids, [Threshold(0, 0.7, 0)])
    ctx.sync()
    _, oh32, om = O.sc_certaindex(O.gen_sc(O.gen_params(**g), R, P, S), [(0, 0.7, 0)])
    assert np.array_equal(h.cpu().numpy().view(np.uint32), oh32.view(np.uint32))
    assert np.array_equal(m.cpu().numpy().view(np.uint32), om)


@pytest.mark.parametrize("impl", ["r", "w"])
@pytest.mark.parametrize("R,P,w,tau", [(1000, 64, 3, 0.9), (700, 32, 1, 1.0), (300, 128, 4, 0.75)])
def test_cot_engine_knobs(ctx, monkeypatch, impl, R, P, w, tau):
    import torch
    from paper_2412_20993_b200 import ProbeConfig
    monkeypatch.setenv("CDX_COT_IMPL", impl)
    g = O.gen_params(seed=R + P, conv_hi=P, hesitation_prob=0.1)
    ids, hes = O.gen_cot(g, R, P)
    cfg = O.probe_cfg(64, w, tau, 64 * P - 100)
    ref = O.cot_exit(ids, hes, cfg)
    out = ctx.cot_exit(torch.from_numpy(ids.view(np.int32)).cuda(), torch.from_numpy(hes.view(np.int64)).cuda(),
                       ProbeConfig(64, w, tau, 64 * P - 100))
    ctx.sync()
    for k in ("exit_step", "reason", "low_conf"):
        assert np.array_equal(out[k].cpu().numpy(), ref[k]), k
    assert np.array_equal(out["final_id"].cpu().numpy().view(np.uint32), ref["final_id"])


@pytest.mark.parametrize("G,T,W", [(300, 16, 64), (100, 40, 32)])
def test_reward_legacy_knob(ctx, monkeypatch, G, T, W):
    import torch
    monkeypatch.setenv("CDX_RW_LEGACY", "1")
    g = O.gen_params(seed=G + T, conv_hi=T)
    rw, ids = O.gen_reward(g, G, T, W)
    agg = (np.arange(G) % 2).astype(np.uint8)
    R, H, _ = ctx.reward_certaindex(torch.from_numpy(rw).cuda(), torch.from_numpy(ids.view(np.int32)).cuda(),
                                    torch.from_numpy(agg).cuda())
    ctx.sync()
    _, R32, Ho = O.reward_certaindex(rw, ids, agg)
    assert np.array_equal(R.cpu().numpy().view(np.uint32), R32.view(np.uint32))
    assert np.array_equal(H.cpu().numpy().view(np.uint32), Ho.view(np.uint32))


@pytest.mark.parametrize("lookback", ["1", None])
@pytest.mark.parametrize("R", [5000, 1 << 20, 5 << 20])  # 5M requests: more tiles than fit at once
def test_allocate_lookback_and_cooperative(ctx, monkeypatch, lookback, R):
    """K5's two multi-tile schemes (cooperative grid barrier / ticketed look-back, forced by
    CDX_ALLOC_LOOKBACK or by a grid too large to be resident) give the oracle's offsets and
    kept list."""
    import torch
    from paper_2412_20993_b200 import AllocPolicy
    if lookback:
        monkeypatch.setenv("CDX_ALLOC_LOOKBACK", lookback)
    P = 64
    rng = np.random.default_rng(R)
    om = (rng.random((R, 2)) < 0.3).astype(np.uint32) * rng.integers(1, 1 << 31, size=(R, 2)).astype(np.uint32)
    meets = torch.from_numpy(om.view(np.int32)).cuda()
    pol = AllocPolicy(kind=4, detect_at=5, resource_cap=64, recheck_every=3, tokens_per_unit=2048)
    out = ctx.allocate_scan(meets, R, P, pol, base_offset=11)
    ctx.sync()
    ref = O.allocate_scan(om, R, P, 4, 5, 64, 3, 2048, base_offset=11)
    for k in ("exit_knob", "granted", "offsets"):
        assert np.array_equal(out[k].cpu().numpy(), ref[k].astype(out[k].cpu().numpy().dtype)), k
    n_kept, saved, _ = out["scalars"].cpu().numpy().tolist()
    assert n_kept == ref["n_kept"] and saved == ref["tokens_saved"]
    assert np.array_equal(out["kept"][:n_kept].cpu().numpy().view(np.uint32), ref["kept"])
