"""GPU parity: K4 reward_certaindex (MCTS mean / Rebase max, cumulative) vs the oracle,
bit-exact on R (fp32 of the FP64 value), H~ and meets bits; overflow (> 8 clusters) and
the non-TMA path included."""
import numpy as np
import pytest

from oracle import oracle as O

pytestmark = pytest.mark.gpu


def _run(ctx, rw, ids, agg, th_mean=(), th_max=()):
    import torch
    from paper_2412_20993_b200 import Threshold
    trw = torch.from_numpy(np.ascontiguousarray(rw)).cuda()
    tid = None if ids is None else torch.from_numpy(np.ascontiguousarray(ids).view(np.int32)).cuda()
    tagg = torch.from_numpy(np.ascontiguousarray(agg, dtype=np.uint8)).cuda()
    R, H, meets = ctx.reward_certaindex(trw, tid, tagg, [Threshold(*t) for t in th_mean],
                                        [Threshold(*t) for t in th_max])
    ctx.sync()
    return R.cpu().numpy(), (None if H is None else H.cpu().numpy()), meets.cpu().numpy().view(np.uint32)


def _oracle_meets(R64, H, agg, th_mean, th_max):
    G, T = R64.shape
    words = (T + 31) // 32
    out = np.zeros((G, words), np.uint32)
    for g in range(G):
        ths = th_max if agg[g] else th_mean
        for t in range(T):
            ok = True
            for sig, cut, d in ths:
                v = float(np.float64(R64[g, t])) if sig == 1 else float(H64[g, t])
                ok = ok and (v >= cut if d == 0 else v <= cut)
            if ok:
                out[g, t // 32] |= np.uint32(1) << np.uint32(t % 32)
    return out


H64 = None


@pytest.mark.parametrize("G,T,W,groups", [(1, 1, 1, 5), (300, 16, 64, 5), (129, 5, 7, 5), (70, 40, 8, 5),
                                          (200, 16, 64, 40), (64, 3, 32, 200), (513, 16, 4, 3),
                                          (100, 100, 64, 5), (40, 256, 32, 7), (65, 70, 128, 5),
                                          (9, 200, 128, 300),  # T*W past the shared-memory overflow table
                                          (300, 16, 48, 5), (500, 12, 16, 5), (200, 9, 80, 12), (100, 7, 112, 40),
                                          (64, 5, 16, 30)])  # W % 16 == 0: half boxes past W skipped
def test_reward_parity(ctx, G, T, W, groups):
    global H64
    g = O.gen_params(seed=G + T + W, groups=groups, conv_hi=max(1, T))
    rw, ids = O.gen_reward(g, G, T, W)
    agg = (np.arange(G) % 2).astype(np.uint8)
    th_mean = [(0, 0.99, 0), (1, 0.4, 0)]   # MCTS/GSM8K
    th_max = [(0, 0.85, 0), (1, 0.99, 0)]   # Rebase/GSM8K
    R, H, meets = _run(ctx, rw, ids, agg, th_mean, th_max)
    R64, R32, Ho = O.reward_certaindex(rw, ids, agg)
    assert np.array_equal(R.view(np.uint32), R32.view(np.uint32))
    assert np.array_equal(H.view(np.uint32), Ho.view(np.uint32))
    # meets: recompute from the oracle's FP64 values (H64 from the reference-pinned entropy)
    import ctypes as C
    H64 = np.empty((G, T), np.float64)
    sizes = (C.c_int * (T * W))()
    lead = (C.c_int * (T * W))()
    L = O.lib()
    L.cdxo_certaindex_entropy.argtypes = [C.c_void_p, C.c_int, C.c_int]
    for gi in range(G):
        for t in range(T):
            n = (t + 1) * W
            m = L.cdxo_cluster_exact_ids(ids[gi].ravel().ctypes.data_as(C.c_void_p), n, sizes, lead)
            H64[gi, t] = L.cdxo_certaindex_entropy(sizes, m, n)
    assert np.array_equal(meets, _oracle_meets(R64, H64, agg, th_mean, th_max))


def test_reward_only_mode(ctx):
    import torch
    g = O.gen_params(seed=3, conv_hi=16)
    rw, _ = O.gen_reward(g, 1000, 16, 64)
    agg = (np.arange(1000) % 3 == 0).astype(np.uint8)
    R, H, meets = _run(ctx, rw, None, agg, [(1, 0.4, 0)], [(1, 0.99, 0)])
    _, R32, _ = O.reward_certaindex(rw, None, agg)
    assert H is None
    assert np.array_equal(R.view(np.uint32), R32.view(np.uint32))


def test_reward_not_on_grid_is_still_exact(ctx):
    """Arbitrary floats: the device keeps the reference's left fold order, so the mean is
    bit-identical even when partial sums round."""
    rng = np.random.default_rng(1)
    rw = rng.random((257, 9, 12)).astype(np.float32)
    ids = rng.integers(0, 6, size=(257, 9, 12)).astype(np.uint32)
    agg = (np.arange(257) % 2).astype(np.uint8)
    R, H, _ = _run(ctx, rw, ids, agg)
    _, R32, Ho = O.reward_certaindex(rw, ids, agg)
    assert np.array_equal(R.view(np.uint32), R32.view(np.uint32))
    assert np.array_equal(H.view(np.uint32), Ho.view(np.uint32))


def test_reward_out_of_range_raises(ctx):
    from paper_2412_20993_b200 import CdxInvalidArgument
    rw = np.full((4, 2, 4), 0.5, np.float32)
    rw[2, 1, 3] = 1.5
    with pytest.raises(CdxInvalidArgument, match=r"reward outside \[0,1\]"):
        _run(ctx, rw, None, np.zeros(4, np.uint8))


def test_reward_sets_facade(ctx):
    import torch
    vals = [[0.9], [0.2, 0.9], [0.2, 0.4, 0.6], [0.5, 0.25, 0.125]]
    agg = np.array([0, 1, 0, 1], np.uint8)
    flat = torch.tensor([v for r in vals for v in r], dtype=torch.float64, device="cuda")
    off = torch.tensor(np.concatenate([[0], np.cumsum([len(r) for r in vals])]), dtype=torch.int64, device="cuda")
    out = ctx.reward_sets(flat, off, torch.from_numpy(agg).cuda())
    ctx.sync()
    assert out.cpu().tolist() == [0.9, 0.9, 0.4000000000000001, 0.5]


@pytest.mark.parametrize("G,T,W", [(257, 16, 64), (100, 64, 128), (33, 7, 96), (40, 16, 32)])
@pytest.mark.parametrize("with_ids", [True, False])
def test_reward_quad_path_arbitrary_floats(ctx, G, T, W, with_ids):
    """The 4-lanes-per-program kernel (W % 32 == 0) sums in any order only where that is
    provably exact; programs with tiny values, -0.0 or NaN fall back to the serial left
    fold.  Every program must still match the reference bit for bit."""
    rng = np.random.default_rng(G * T + W)
    rw = rng.random((G, T, W)).astype(np.float32)
    rw[1, 0, 5] = np.float32(1e-30)          # below the exact-sum threshold
    rw[2, T - 1, W - 1] = np.float32(-0.0)   # signed zero (max keeps the first maximum)
    rw[3, :, :] = 0.0
    rw[4, 0, 0] = np.float32(3.0e-7)
    rw[5, T // 2, 3] = np.float32(1.0)
    if G > 6:
        rw[6, 0, :] = np.float32(2.0 ** -21)
    ids = rng.integers(0, 7, size=(G, T, W)).astype(np.uint32) if with_ids else None
    if with_ids:
        ids[7 % G] = rng.integers(0, 1 << 30, size=(T, W))  # > 8 clusters -> overflow kernel
        ids[8 % G, :, :] = 42
    agg = (np.arange(G) % 2).astype(np.uint8)
    R, H, _ = _run(ctx, rw, ids, agg)
    _, R32, Ho = O.reward_certaindex(rw, ids, agg)
    assert np.array_equal(R.view(np.uint32), R32.view(np.uint32))
    if with_ids:
        assert np.array_equal(H.view(np.uint32), Ho.view(np.uint32))


def test_reward_quad_nan_propagates_like_reference(ctx):
    rw = np.full((8, 4, 32), 0.5, np.float32)
    rw[3, 1, 7] = np.nan  # passes the [0,1] check in the reference (comparisons are false)
    agg = (np.arange(8) % 2).astype(np.uint8)
    R, _, _ = _run(ctx, rw, None, agg)
    _, R32, _ = O.reward_certaindex(rw, None, agg)
    assert np.array_equal(R.view(np.uint32), R32.view(np.uint32))


def _partitions(n):
    """All integer partitions of n, largest part first (ZS1, anti-lexicographic)."""
    x = [1] * (n + 1)
    x[1], m, h = n, 1, 1
    yield x[1:m + 1]
    while x[1] != 1:
        if x[h] == 2:
            m, x[h], h = m + 1, 1, h - 1
        else:
            r, t = x[h] - 1, m - h + 1
            x[h] = r
            while t >= r:
                h += 1
                x[h], t = r, t - r
            if t == 0:
                m = h
            else:
                m = h + 1
                if t > 1:
                    h += 1
                    x[h] = t
        yield x[1:m + 1]


@pytest.mark.parametrize("n", [16, 32, 64])
def test_reward_entropy_all_partitions(ctx, n):
    """SURVEY §4 plan item 2: every clustering shape of n answers (p(64) = 1,741,630), each in
    sorted and in a shuffled first-seen order, as one MCTS step of W = n nodes.  The FP64
    fold over first-seen clusters must give the oracle's H~ bits for all of them; shapes
    with more than 8 clusters run through the overflow kernel."""
    flat, lens = [], []
    for p in _partitions(n):
        flat.extend(p)
        lens.append(len(p))
    flat, lens = np.array(flat, np.int64), np.array(lens, np.int64)
    starts = np.concatenate([[0], np.cumsum(lens)[:-1]])
    labels = (np.arange(len(flat)) - np.repeat(starts, lens)).astype(np.uint32)
    ids = np.repeat(labels, flat).reshape(len(lens), n)
    shuf = np.random.default_rng(n).permuted(ids, axis=1)  # other first-seen orders
    ids = np.concatenate([ids, shuf])[:, None, :]  # (G, T=1, W=n)
    G = ids.shape[0]
    rw = np.full((G, 1, n), 0.5, np.float32)
    agg = (np.arange(G) % 2).astype(np.uint8)
    R, H, _ = _run(ctx, rw, ids, agg)
    _, R32, Ho = O.reward_certaindex(rw, ids, agg)
    assert np.array_equal(H.view(np.uint32), Ho.view(np.uint32))
    assert np.array_equal(R.view(np.uint32), R32.view(np.uint32))


@pytest.mark.parametrize("G,T,W", [(1, 1, 1), (513, 16, 64), (77, 9, 13), (20, 40, 128)])
def test_reward_f64_rewards_match_reference(ctx, G, T, W):
    """cdx_reward_certaindex_f64: RewardSet holds doubles (metrics.hpp:74-77); arbitrary
    off-grid doubles, subnormals, -0.0 and NaN are folded in the reference's order and the
    thresholds see the FP64 values.  R / H~ stores and meets bits equal the oracle's."""
    rng = np.random.default_rng(G + T * W)
    rw = rng.random((G, T, W))
    rw[0, 0, 0] = 5e-324
    if G > 3:
        rw[1, :, 0] = -0.0
        rw[2, T - 1, W - 1] = np.nan
        rw[3] = np.round(rw[3] * 4) / 4  # exact threshold hits on R
    ids = rng.integers(0, 6, size=(G, T, W)).astype(np.uint32)
    if G > 5:
        ids[5] = rng.integers(0, 1 << 30, size=(T, W))  # many clusters
    agg = (np.arange(G) % 2).astype(np.uint8)
    th_mean = [(0, 0.3, 0), (1, 0.5, 0)]
    th_max = [(1, 0.75, 0), (0, 0.2, 0)]
    R, H, meets = _run(ctx, rw, ids, agg, th_mean, th_max)
    R64, R32, Ho, H64o = O.reward_certaindex(rw, ids, agg, want_h64=True)
    assert np.array_equal(R.view(np.uint32), R32.view(np.uint32))
    assert np.array_equal(H.view(np.uint32), Ho.view(np.uint32))
    global H64
    H64 = H64o
    assert np.array_equal(meets, _oracle_meets(R64, H64o, agg, th_mean, th_max))


def test_reward_nan_cutoff_fails_every_compare(ctx):
    """A NaN cutoff: `v >= NaN` is false (metrics.cpp:167), so nothing meets it, on both
    the quad and the f64 path."""
    g = O.gen_params(seed=5, conv_hi=8)
    rw, ids = O.gen_reward(g, 256, 8, 64)
    agg = (np.arange(256) % 2).astype(np.uint8)
    for arr in (rw, rw.astype(np.float64)):
        _, _, meets = _run(ctx, arr, ids, agg, [(1, float("nan"), 0)], [(0, float("nan"), 1)])
        assert not meets.any()
