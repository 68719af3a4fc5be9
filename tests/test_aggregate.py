"""Aggregation per archetype (ProgramDriver::aggregate_prefix, runtime.cpp:316-403).

CPU: the C restatement (oracle/cdx_oracle.c) is pinned against the reference's own
aggregate_prefix, called through oracle/_ref on injected SC / MCTS / Rebase paths, plus the
SPEC examples.  GPU: cdx_sc_aggregate / cdx_reward_aggregate must equal the restatement
bit-for-bit (answer ids) at the BASELINE shapes; the Rebase exp() weights must be the host
libm's (no off-grid rewards on the synthetic traces: the inexact counter stays 0).
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
def test_reward_aggregate_off_grid_is_counted(ctx):
    import torch
    rw = np.full((2, 1, 4), 0.1, np.float32)  # 0.1f is not a multiple of 2^-24
    ids = np.array([[[0, 1, 1, 0]], [[2, 2, 3, 3]]], np.uint32)
    agg = np.array([1, 1], np.uint8)
    ex = np.zeros(2, np.int32)
    ans, inexact = ctx.reward_aggregate(torch.from_numpy(rw).cuda(), torch.from_numpy(ids.view(np.int32)).cuda(),
                                        torch.from_numpy(agg).cuda(), torch.from_numpy(ex).cuda())
    ctx.sync()
    assert int(inexact) == 8
    assert ans.cpu().numpy().tolist() == [0, 2]  # equal weights: earliest-seen cluster
