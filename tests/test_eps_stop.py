"""Epsilon-accuracy stop test (probe::stationary_by_epsilon_test, probe.cpp:104-120, over
theory::epsilon_stop_test, theory.cpp:100-146) at every prefix of every CoT trace.

CPU: the C restatement is pinned against the reference itself (oracle/_ref, the reference's
own probe.cpp/theory.cpp) on random traces and exhaustively on short ones.  GPU:
cdx_cot_eps_stop must reproduce the restatement's per-prefix states and first-true step.
"""
import itertools

import numpy as np
import pytest

from oracle import oracle as O

VOC = O.vocab(4)
CASES = [(1, 0.5), (2, 0.3), (3, 0.9), (3, 1.0 / 3.0), (4, 0.05), (5, 2.0)]


def _traces(R, P, groups, hes_p, seed):
    rng = np.random.default_rng(seed)
    ids = rng.integers(0, groups, size=(R, P)).astype(np.uint32)
    ids[::4, P // 2:] = 0  # converging tails
    hb = rng.random((R, P)) < hes_p
    hes = np.zeros((R, (P + 63) // 64), np.uint64)
    for p in range(P):
        hes[:, p // 64] |= hb[:, p].astype(np.uint64) << np.uint64(p % 64)
    return ids, hes


def _ref_or_skip():
    if not O.ref_available():
        pytest.skip("oracle/_ref not built")


@pytest.mark.parametrize("k,eps", CASES)
def test_oracle_pinned_to_reference_random(k, eps):
    _ref_or_skip()
    ids, hes = _traces(60, 24, 3, 0.15, k)
    step, state = O.cot_eps_stop(ids, hes, k, eps)
    ref = O.ref_eps_prefixes(ids, hes, k, eps, VOC)
    assert np.array_equal(state, ref)
    first = np.array([np.flatnonzero(r == 2)[0] if (r == 2).any() else -1 for r in ref], np.int32)
    assert np.array_equal(step, first)


def test_oracle_pinned_to_reference_exhaustive():
    """Every trace of length 6 over 3 answers with 0/1/2 hesitant probes, k in {1,2,3}."""
    _ref_or_skip()
    P = 6
    seqs = np.array(list(itertools.product(range(3), repeat=P)), np.uint32)
    masks = [0] + [1 << i for i in range(P)] + [(1 << i) | (1 << j) for i in range(P) for j in range(i + 1, P)]
    for k, eps in ((1, 0.5), (2, 0.4), (3, 0.7)):
        for mk in masks[:: 3]:
            hes = np.full((len(seqs), 1), mk, np.uint64)
            _, st = O.cot_eps_stop(seqs, hes, k, eps)
            assert np.array_equal(st, O.ref_eps_prefixes(seqs, hes, k, eps, VOC)), (k, eps, mk)


def test_reference_error_texts():
    _ref_or_skip()
    ids, hes = _traces(2, 4, 2, 0.0, 0)
    with pytest.raises(O.RefError, match="k must be >= 1"):
        O.ref_eps_prefixes(ids, hes, 0, 0.5, VOC)
    with pytest.raises(O.RefError, match="epsilon must be > 0"):
        O.ref_eps_prefixes(ids, hes, 2, 0.0, VOC)


@pytest.mark.gpu
@pytest.mark.parametrize("k,eps", CASES)
@pytest.mark.parametrize("R,P", [(1, 1), (3000, 64), (777, 37)])
def test_eps_stop_gpu(ctx, R, P, k, eps):
    import torch
    ids, hes = _traces(R, P, 4, 0.1, R + k)
    step, state = ctx.cot_eps_stop(torch.from_numpy(ids.view(np.int32)).cuda(),
                                   torch.from_numpy(hes.view(np.int64)).cuda(), k, eps, want_state=True)
    ctx.sync()
    ostep, ostate = O.cot_eps_stop(ids, hes, k, eps)
    assert np.array_equal(state.cpu().numpy(), ostate)
    assert np.array_equal(step.cpu().numpy(), ostep)
    step2, _ = ctx.cot_eps_stop(torch.from_numpy(ids.view(np.int32)).cuda(),
                                torch.from_numpy(hes.view(np.int64)).cuda(), k, eps)
    ctx.sync()
    assert np.array_equal(step2.cpu().numpy(), ostep)


@pytest.mark.gpu
def test_eps_stop_gpu_synthetic_trace(ctx):
    """The device generator's CoT trace (config B distribution, reduced R)."""
    from paper_2412_20993_b200 import GenParams
    ids, hes = ctx.gen_cot(GenParams(seed=5, conv_hi=64, hesitation_prob=0.05), 20000, 64)
    step, _ = ctx.cot_eps_stop(ids, hes, 3, 0.5)
    ctx.sync()
    ostep, _ = O.cot_eps_stop(ids.cpu().numpy().view(np.uint32), hes.cpu().numpy().view(np.uint64), 3, 0.5)
    assert np.array_equal(step.cpu().numpy(), ostep)


@pytest.mark.gpu
def test_eps_stop_gpu_errors(ctx):
    import torch
    from paper_2412_20993_b200 import CdxInvalidArgument
    ids = torch.zeros((2, 4), dtype=torch.int32, device="cuda")
    hes = torch.zeros((2, 1), dtype=torch.int64, device="cuda")
    with pytest.raises(CdxInvalidArgument, match="k must be >= 1"):
        ctx.cot_eps_stop(ids, hes, 0, 0.5)
    with pytest.raises(CdxInvalidArgument, match="epsilon must be > 0"):
        ctx.cot_eps_stop(ids, hes, 2, -1.0)
