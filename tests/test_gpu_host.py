"""GPU: the end-to-end host-buffer entry cdx_sc_decide_host (chunked H2D + K2 + K5 + D2H)
equals the oracle, including global budget offsets across chunks."""
import ctypes as C

import numpy as np
import pytest

from oracle import oracle as O

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("R,P,S", [(1, 32, 16), (5000, 64, 32), (70000, 64, 32), (3000, 20, 7)])
def test_sc_decide_host(ctx, R, P, S):
    from paper_2412_20993_b200 import AllocPolicy, Threshold, c_policy, c_thresholds
    ids = O.gen_sc(O.gen_params(seed=R, conv_hi=P), R, P, S)
    ex = np.empty(R, np.int32)
    why = np.empty(R, np.uint8)
    off = np.empty(R, np.int64)
    hc = np.empty((R, P), np.float32)
    saved = C.c_int64(0)
    arr, n = c_thresholds([Threshold(0, 0.7, 0)])
    pol = c_policy(AllocPolicy(kind=2, detect_at=5, resource_cap=P, tokens_per_unit=64 * S))
    st = ctx.lib.cdx_sc_decide_host(ctx.h, ids.ctypes.data, R, P, S, arr, n, C.byref(pol), ex.ctypes.data,
                                    why.ctypes.data, off.ctypes.data, hc.ctypes.data, C.byref(saved))
    ctx._check(st)
    _, oh32, om = O.sc_certaindex(ids, [(0, 0.7, 0)])
    ref = O.allocate_scan(om, R, P, 2, 5, P, 1, 64 * S)
    assert np.array_equal(hc.view(np.uint32), oh32.view(np.uint32))
    assert np.array_equal(ex, ref["exit_knob"]) and np.array_equal(why, ref["reason"])
    assert np.array_equal(off, ref["offsets"])
    assert saved.value == ref["tokens_saved"]


@pytest.mark.parametrize("R,P,w,tau,mt,chunk_kb", [(1, 64, 3, 0.9, 4096, None), (200000, 64, 3, 0.9, 4096, 512),
                                                   (30000, 40, 2, 0.5, 1000, 100), (5000, 100, 5, 0.6, 10**6, 64)])
def test_cot_decide_host(ctx, monkeypatch, R, P, w, tau, mt, chunk_kb):
    """cdx_cot_decide_host (chunked H2D + K3 + D2H) equals the oracle; small chunks cross many
    chunk seams."""
    from paper_2412_20993_b200 import ProbeConfig
    if chunk_kb:
        monkeypatch.setenv("CDX_PIPE_CHUNK_KB", str(chunk_kb))
    ids, hes = O.gen_cot(O.gen_params(seed=R + P, conv_hi=P, hesitation_prob=0.05), R, P)
    got = ctx.cot_decide_host(ids, hes, ProbeConfig(64, w, tau, mt))
    ref = O.cot_exit(ids, hes, O.probe_cfg(64, w, tau, mt))
    for k in ("exit_step", "reason", "final_id", "low_conf"):
        assert np.array_equal(got[k], ref[k].astype(got[k].dtype)), k


def test_cot_decide_host_explicit_offsets(ctx, monkeypatch):
    from paper_2412_20993_b200 import ProbeConfig
    monkeypatch.setenv("CDX_PIPE_CHUNK_KB", "256")
    R, P = 20000, 64
    rng = np.random.default_rng(5)
    ids, hes = O.gen_cot(O.gen_params(seed=3, conv_hi=P, hesitation_prob=0.05), R, P)
    offs = np.cumsum(rng.integers(1, 128, size=(R, P)), axis=1).astype(np.int64)
    got = ctx.cot_decide_host(ids, hes, ProbeConfig(64, 3, 0.9, 3000), offsets=offs)
    ref = O.cot_exit(ids, hes, O.probe_cfg(64, 3, 0.9, 3000), offsets=offs)
    for k in ("exit_step", "reason", "final_id", "low_conf"):
        assert np.array_equal(got[k], ref[k].astype(got[k].dtype)), k


@pytest.mark.parametrize("G,T,W,chunk_kb", [(1, 16, 64, None), (40000, 16, 64, 4096), (9000, 7, 40, 300)])
def test_reward_decide_host(ctx, monkeypatch, G, T, W, chunk_kb):
    """cdx_reward_decide_host (chunked H2D + K4 + K5 + D2H) equals the oracle, with budget
    offsets global across chunks."""
    from paper_2412_20993_b200 import AllocPolicy, Threshold
    if chunk_kb:
        monkeypatch.setenv("CDX_PIPE_CHUNK_KB", str(chunk_kb))
    rw, ids = O.gen_reward(O.gen_params(seed=G + T, conv_hi=T), G, T, W)
    agg = (np.arange(G) % 2).astype(np.uint8)
    thm, thx = [(0, 0.99, 0), (1, 0.4, 0)], [(0, 0.85, 0), (1, 0.99, 0)]
    pol = AllocPolicy(kind=2, detect_at=min(3, T), resource_cap=T, tokens_per_unit=W)
    got = ctx.reward_decide_host(rw, ids, agg, [Threshold(*t) for t in thm], [Threshold(*t) for t in thx], pol,
                                 want_R=True)
    R64, R32, H32, H64 = O.reward_certaindex(rw, ids, agg, want_h64=True)
    assert np.array_equal(got["R"].view(np.uint32), R32.view(np.uint32))
    meets = np.zeros((G, (T + 31) // 32), np.uint32)
    ok = np.where(agg[:, None] == 1, (H64 >= 0.85) & (R64 >= 0.99), (H64 >= 0.99) & (R64 >= 0.4))
    for t in range(T):
        meets[:, t // 32] |= ok[:, t].astype(np.uint32) << np.uint32(t % 32)
    ref = O.allocate_scan(meets, G, T, 2, min(3, T), T, 1, W)
    assert np.array_equal(got["exit_knob"], ref["exit_knob"]) and np.array_equal(got["reason"], ref["reason"])
    assert np.array_equal(got["offsets"], ref["offsets"])
    assert got["tokens_saved"] == ref["tokens_saved"]


def test_reward_decide_host_range_error(ctx):
    from paper_2412_20993_b200 import AllocPolicy, CdxInvalidArgument
    rw = np.full((10, 2, 4), 0.5, np.float32)
    rw[3, 1, 2] = 2.0
    with pytest.raises(CdxInvalidArgument, match=r"reward outside \[0,1\]"):
        ctx.reward_decide_host(rw, None, np.zeros(10, np.uint8), [], [], AllocPolicy(kind=0, resource_cap=2))
