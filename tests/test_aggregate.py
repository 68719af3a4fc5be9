"""Aggregation per archetype (ProgramDriver::aggregate_prefix, runtime.cpp:316-403).

CPU: the C restatement (oracle/cdx_oracle.c) is pinned against the reference's own
aggregate_prefix, called through oracle/_ref on injected SC / MCTS / Rebase paths, plus the
SPEC examples.  GPU: cdx_sc_aggregate / cdx_reward_aggregate must equal the restatement
bit-for-bit (answer ids) at the BASELINE shapes; the Rebase exp() weights are the host
libm's bits for every reward (libm_exp.cuh), so off-grid f32 and f64 rewards (a reward
model's outputs), NaN and out-of-range rewards included, give the reference's answers.
"""
import numpy as np
import pytest

from oracle import oracle as O

SC, REBASE, MCTS = 0, 1, 2
VOC = O.vocab(5)  # "S", "D1".."D4", "wait, S", ...


def _ref_or_skip():
    if not O.ref_available():
        pytest.skip("oracle/_ref not built")


def test_spec_examples_through_reference():
    _ref_or_skip()
    a, b = VOC.index("D1"), VOC.index("D2")
    # SC answers [a,a,b] -> a ; ties -> earliest seen
    assert O.ref_aggregate(SC, [a, a, b], None, [], 3, VOC) == a
    assert O.ref_aggregate(SC, [b, a, a, b], None, [], 4, VOC) == b
    # Rebase answers [a,b] scores [2,1] (one layer) -> a (e^2 > e^1)
    assert O.ref_aggregate(REBASE, [a, b], [2.0, 1.0], [2], 2, VOC) == a
    # MCTS rewards {a:0.3, b:0.8} -> b
    assert O.ref_aggregate(MCTS, [a, b], [0.3, 0.8], [], 2, VOC) == b


@pytest.mark.parametrize("seed", range(6))
def test_oracle_aggregation_pinned_to_reference(seed):
    _ref_or_skip()
    rng = np.random.default_rng(seed)
    # SC: R requests x P probes x S samples, exit at a random knob
    R, P, S = 40, 8, 16
    ids = rng.integers(0, 4 if seed % 2 else 2, size=(R, P, S)).astype(np.uint32)
    knob = rng.integers(1, P + 1, size=R).astype(np.int32)
    got = O.sc_aggregate(ids, knob)
    for r in range(R):
        row = ids[r, knob[r] - 1]
        assert got[r] == O.ref_aggregate(SC, row.tolist(), None, [], S, VOC)
    # MCTS / Rebase: G programs x T steps x W nodes; rewards on the 2^-24 grid with ties
    G, T, W = 24, 5, 8
    k = rng.integers(0, 1 << 24, size=(G, T, W))
    if seed % 3 == 0:
        k = (k >> 20) << 20  # few distinct values: exact reward ties
    rw = (k.astype(np.float64) / (1 << 24)).astype(np.float32)
    rid = rng.integers(0, 5, size=(G, T, W)).astype(np.uint32)
    agg = (np.arange(G) % 2).astype(np.uint8)  # even MCTS (mean), odd Rebase (max)
    ex = rng.integers(0, T, size=G).astype(np.int32)
    got = O.reward_aggregate(rw, rid, agg, ex)
    for g in range(G):
        n = (ex[g] + 1) * W
        arche = MCTS if agg[g] == 0 else REBASE
        want = O.ref_aggregate(arche, rid[g].ravel()[:n].tolist(), rw[g].ravel()[:n].astype(np.float64).tolist(),
                               [W] * int(ex[g] + 1), n, VOC)
        assert got[g] == want, (g, arche)


@pytest.mark.parametrize("seed", range(4))
def test_oracle_aggregation_off_grid_doubles_pinned_to_reference(seed):
    """Arbitrary double rewards (reward-model outputs), near-ties, NaN and out-of-range
    values: the f64 restatement equals the reference's aggregate_prefix, the empty-string
    answer of an all-NaN Rebase layer included (CDX_NO_ANSWER)."""
    _ref_or_skip()
    rng = np.random.default_rng(100 + seed)
    G, T, W = 40, 4, 6
    rw = rng.random((G, T, W))
    rw[::3] = np.round(rw[::3] * 4) / 4 + rng.integers(-2, 3, size=rw[::3].shape) * 2.0 ** -52  # near-ties
    rw[5, :, 1] = np.nan
    rw[7] = np.nan
    rw[9, :, :2] = [-3.5, 7.25]
    rid = rng.integers(0, 4, size=(G, T, W)).astype(np.uint32)
    agg = (np.arange(G) % 2).astype(np.uint8)
    ex = rng.integers(0, T, size=G).astype(np.int32)
    got = O.reward_aggregate(rw, rid, agg, ex)
    for g in range(G):
        n = (ex[g] + 1) * W
        arche = MCTS if agg[g] == 0 else REBASE
        want = O.ref_aggregate(arche, rid[g].ravel()[:n].tolist(), rw[g].ravel()[:n].tolist(),
                               [W] * int(ex[g] + 1), n, VOC)
        assert got[g] == want, (g, arche)


@pytest.mark.gpu
@pytest.mark.parametrize("R,P,S", [(1, 1, 1), (1000, 64, 32), (257, 32, 16), (64, 8, 5)])
def test_sc_aggregate_gpu(ctx, R, P, S):
    import torch
    rng = np.random.default_rng(R + S)
    ids = O.gen_sc(O.gen_params(seed=R, conv_hi=P), R, P, S)
    ids[::7] = rng.integers(0, 3, size=ids[::7].shape).astype(np.uint32)  # ties
    knob = rng.integers(1, P + 1, size=R).astype(np.int32)
    ans = ctx.sc_aggregate(torch.from_numpy(ids.view(np.int32)).cuda(), torch.from_numpy(knob).cuda())
    ctx.sync()
    assert np.array_equal(ans.cpu().numpy().view(np.uint32), O.sc_aggregate(ids, knob))


@pytest.mark.gpu
@pytest.mark.parametrize("G,T,W", [(1, 1, 1), (4096, 16, 64), (300, 7, 40), (65, 3, 200)])
def test_reward_aggregate_gpu(ctx, G, T, W):
    import torch
    rng = np.random.default_rng(G + W)
    rw, ids = O.gen_reward(O.gen_params(seed=G, conv_hi=T), G, T, W)
    rw[::5] = np.float32(0.5)  # exact weight ties -> earliest-seen cluster
    agg = (np.arange(G) % 2).astype(np.uint8)
    ex = rng.integers(0, T, size=G).astype(np.int32)
    ans, inexact = ctx.reward_aggregate(torch.from_numpy(rw).cuda(), torch.from_numpy(ids.view(np.int32)).cuda(),
                                        torch.from_numpy(agg).cuda(), torch.from_numpy(ex).cuda())
    ctx.sync()
    assert int(inexact) == 0
    assert np.array_equal(ans.cpu().numpy().view(np.uint32), O.reward_aggregate(rw, ids, agg, ex))


@pytest.mark.gpu
@pytest.mark.parametrize("dtype", [np.float32, np.float64])
def test_reward_aggregate_off_grid_exact(ctx, dtype):
    """Off-grid rewards with near-tied Rebase weights: the device exp is the host libm's, so
    the vote equals the oracle's (host std::exp) for f32 and f64 rewards alike."""
    import torch
    rng = np.random.default_rng(7)
    G, T, W = 20000, 3, 24
    rw = rng.random((G, T, W)).astype(dtype)
    rw[::4] = (np.round(rw[::4] * 8) / 8 + rng.integers(-3, 4, size=rw[::4].shape) *
               np.finfo(dtype).eps).astype(dtype)  # weight sums that differ in the last bits
    rw[11, :, 3] = np.nan
    rw[13] = np.nan  # all-NaN layer: no winner (the reference's empty string)
    ids = rng.integers(0, 3, size=(G, T, W)).astype(np.uint32)
    agg = (np.arange(G) % 2).astype(np.uint8)
    ex = rng.integers(0, T, size=G).astype(np.int32)
    ans, inexact = ctx.reward_aggregate(torch.from_numpy(rw).cuda(), torch.from_numpy(ids.view(np.int32)).cuda(),
                                        torch.from_numpy(agg).cuda(), torch.from_numpy(ex).cuda())
    ctx.sync()
    assert int(inexact) == 0
    want = O.reward_aggregate(rw, ids, agg, ex)
    assert want[13] == 0xFFFFFFFF
    assert np.array_equal(ans.cpu().numpy().view(np.uint32), want)


@pytest.mark.gpu
def test_device_exp_is_host_libm_exp(ctx):
    """cdx_libm_exp vs this box's own std::exp (numpy's exp is not libm's: use math.exp,
    which is the C library's) on rewards in [0,1], the whole finite range and specials."""
    import math
    import struct

    import torch
    rng = np.random.default_rng(3)
    xs = np.concatenate([rng.random(1 << 20), rng.uniform(-760, 720, 1 << 20),
                         rng.integers(0, 1 << 63, 1 << 18, dtype=np.int64).view(np.float64),
                         np.array([0.0, -0.0, 1.0, -1.0, np.inf, -np.inf, np.nan, 709.78, 709.79, -745.13, -745.2,
                                   -708.4, 2.0 ** -54, 2.0 ** -55, 512.0, -512.0, 1024.0, -1024.0, 5e-324])])
    got = ctx.libm_exp(torch.from_numpy(xs).cuda()).cpu().numpy()

    def host(x):
        try:
            return math.exp(x)
        except OverflowError:
            return math.inf
    want = np.array([host(float(x)) for x in xs])
    same = (got.view(np.uint64) == want.view(np.uint64)) | (np.isnan(got) & np.isnan(want))
    bad = np.flatnonzero(~same)
    assert bad.size == 0, [(struct.pack("<d", xs[i]).hex(), got[i], want[i]) for i in bad[:5]]
