"""GPU parity: the majority-fraction certaindex of Self-Consistency (north_star (2)).

majority = size of the plurality cluster / S per (request, probe) row: the share of the
answer the reference's plurality vote returns (runtime.cpp:317-334, weighted_plurality with
unit weights, first-seen tie-break).  The oracle restatement (cdxo_majority_fraction) is
pinned to the reference's own vote in tests/test_majority_oracle.py.  Here every K2 engine
(TMA fast path S in {4,8,16,32}, the generic bulk-copy kernel for other S <= 32, the warp-per-
row kernel for S > 32, the match fallback for rows of more than 8 clusters) must give the
oracle's fp32 value bit for bit and the same threshold bits, alone and ANDed with entropy
thresholds (metrics.cpp:159-171).
"""
import numpy as np
import pytest

from oracle import oracle as O

pytestmark = pytest.mark.gpu

SIG_E, SIG_M, GE, LE = 0, 4, 0, 1

THS = [[(SIG_M, 0.5, GE)], [(SIG_M, 0.75, GE), (SIG_E, 0.3, GE)], [(SIG_E, 0.5, GE), (SIG_M, 0.9, LE)],
       [(SIG_M, float("nan"), GE)], []]


def _check(ctx, ids_np, ths, ids_dev=None):
    import torch
    from paper_2412_20993_b200 import Threshold
    d = ids_dev if ids_dev is not None else torch.from_numpy(ids_np.view(np.int32)).cuda()
    h, mj, meets = ctx.sc_certaindex_ex(d, [Threshold(*t) for t in ths])
    ctx.sync()
    _, oh32, _, om32, omeets = O.sc_certaindex_ex(ids_np, ths)
    assert np.array_equal(h.cpu().numpy().view(np.uint32), oh32.view(np.uint32))
    assert np.array_equal(mj.cpu().numpy().view(np.uint32), om32.view(np.uint32))
    assert np.array_equal(meets.cpu().numpy().view(np.uint32), omeets)


@pytest.mark.parametrize("R,P,S", [(64, 32, 32), (129, 64, 16), (300, 64, 8), (700, 32, 4), (301, 63, 32),
                                   (37, 20, 7), (50, 96, 24), (333, 33, 31), (300, 64, 12), (17, 64, 3),
                                   (300, 64, 1), (5, 3, 2)])
@pytest.mark.parametrize("ti", range(len(THS)))
def test_majority_generated_traces(ctx, R, P, S, ti):
    from paper_2412_20993_b200 import GenParams
    g = dict(seed=77 + R + S, conv_hi=max(1, P))
    ids = ctx.gen_sc(GenParams(**g), R, P, S)
    _check(ctx, O.gen_sc(O.gen_params(**g), R, P, S), THS[ti], ids_dev=ids)


@pytest.mark.parametrize("S,groups", [(32, 40), (32, 3), (16, 20), (8, 9), (4, 5), (24, 30), (12, 13)])
def test_majority_many_clusters(ctx, S, groups):
    """Rows with more than 8 clusters take the warp-match engine; ties between equal largest
    clusters (first-seen wins the vote, the fraction is the same) are frequent here."""
    rng = np.random.default_rng(S * 100 + groups)
    ids = rng.integers(0, groups, size=(96, 32, S)).astype(np.uint32)
    for ths in THS[:3]:
        _check(ctx, ids, ths)


@pytest.mark.parametrize("R,P,S,groups", [(50, 20, 33, 5), (64, 64, 64, 8), (30, 40, 100, 60), (9, 5, 1000, 300),
                                          (2, 3, 4096, 5000)])
def test_majority_wide_rows(ctx, R, P, S, groups):
    rng = np.random.default_rng(S + P)
    ids = rng.integers(0, groups, size=(R, P, S)).astype(np.uint32)
    ids[:, ::3, :] = ids[:, ::3, :1]  # single-cluster rows: majority 1
    for ths in THS[:3]:
        _check(ctx, ids, ths)


@pytest.mark.parametrize("S", [4, 8, 12, 16])
def test_majority_all_compositions(ctx, S):
    """Every first-seen size composition of S (2^(S-1)) and a shuffled copy of each row."""
    codes = np.arange(1 << (S - 1), dtype=np.uint64)
    cuts = ((codes[:, None] >> np.arange(S - 1, dtype=np.uint64)) & 1).astype(np.uint32)
    labels = np.concatenate([np.zeros((len(codes), 1), np.uint32), np.cumsum(cuts, axis=1, dtype=np.uint32)], 1)
    rows = np.concatenate([labels, np.random.default_rng(S).permuted(labels, axis=1)])
    pad = (-len(rows)) % 32
    rows = np.concatenate([rows, np.zeros((pad, S), np.uint32)])
    ids = rows.reshape(-1, 32, S)
    for tau in (0.25, 0.5, 0.51, 0.75):
        _check(ctx, ids, [(SIG_M, tau, GE)])


def test_majority_in_mixed_step(ctx):
    """The SC archetype of cdx_mixed_allocate decides on majority thresholds as K2 does."""
    import torch
    from paper_2412_20993_b200 import AllocPolicy, Threshold, synth
    N, seed = 6000, 9
    arch, slot, sizes = synth.mixed_layout(N, seed, (0.4, 0.4, 0.1, 0.1))
    sc = O.gen_sc(O.gen_params(seed=seed + 1, conv_hi=32), sizes[0], 32, 16)
    cid, ches = O.gen_cot(O.gen_params(seed=seed + 2, conv_hi=64, hesitation_prob=0.05), sizes[1], 64)
    rw, rid = O.gen_reward(O.gen_params(seed=seed + 3, conv_hi=16), sizes[2], 16, 16)
    host = dict(sc_ids=sc, cot_ids=cid, cot_hes=ches, cot_window=3, rw=rw, rw_ids=rid)
    th = {0: [(SIG_M, 0.75, GE), (SIG_E, 0.2, GE)], 1: [(0, 0.85, 0), (1, 0.99, 0)], 2: [(0, 0.99, 0), (1, 0.4, 0)],
          3: [(0, 0.9, 0)]}
    caps = (32, 16, 16, 64)
    pols_o = [O.arch_policy(th[a], 4 if a == 0 else 2, (5, 3, 3, 4)[a], caps[a], 2, 64) for a in range(4)]
    knob = synth.mixed_knobs(arch, caps, seed)

    def dev(a):
        a = np.ascontiguousarray(a)
        a = a.view(np.int32) if a.dtype == np.uint32 else (a.view(np.int64) if a.dtype == np.uint64 else a)
        return torch.from_numpy(a).cuda()
    d = {k: (dev(v) if isinstance(v, np.ndarray) else v) for k, v in host.items()}
    pols = [([Threshold(*t) for t in th[a]], AllocPolicy(kind=pols_o[a].alloc.kind, detect_at=pols_o[a].alloc.detect_at,
                                                         resource_cap=caps[a], recheck_every=2, tokens_per_unit=64))
            for a in range(4)]
    out = ctx.mixed_allocate(d, dev(arch), dev(slot), dev(knob), pols)
    ctx.sync()
    want = O.mixed_allocate(host, arch, slot, knob, pols_o)
    for k in ("decision", "grant", "cap", "offsets"):
        assert np.array_equal(out[k].cpu().numpy(), want[k]), k


def test_majority_rejected_outside_sc(ctx):
    """Only SC produces the majority signal: a threshold on it elsewhere is an absent signal."""
    from paper_2412_20993_b200 import CdxError, GenParams, Threshold
    rw, rid = ctx.gen_reward(GenParams(seed=1, conv_hi=4), 64, 4, 32)
    import torch
    agg = torch.zeros(64, dtype=torch.uint8, device="cuda")
    with pytest.raises(CdxError, match="majority_fraction"):
        ctx.reward_certaindex(rw, rid, agg, [Threshold(SIG_M, 0.5, GE)], [])
