"""GPU parity: K3 cot_exit vs the oracle's literal prefix replay of probe::should_exit /
consistency / final_answer (probe.cpp:48-102), bit-exact on every output."""
import itertools

import numpy as np
import pytest

from oracle import oracle as O

pytestmark = pytest.mark.gpu


def _run(ctx, ids_np, hes_np, cfg, offsets=None, want_ck=True):
    import torch
    from paper_2412_20993_b200 import ProbeConfig
    ids = torch.from_numpy(np.ascontiguousarray(ids_np).view(np.int32)).cuda()
    hes = torch.from_numpy(np.ascontiguousarray(hes_np).view(np.int64)).cuda()
    off = None if offsets is None else torch.from_numpy(np.ascontiguousarray(offsets, dtype=np.int64)).cuda()
    out = ctx.cot_exit(ids, hes, ProbeConfig(cfg.interval_tokens, cfg.window, cfg.threshold, cfg.max_tokens),
                       offsets=off, want_ck=want_ck)
    ctx.sync()
    return {k: (v.cpu().numpy() if v is not None else None) for k, v in out.items()}


def _check(got, ref, want_ck=True):
    assert np.array_equal(got["exit_step"], ref["exit_step"])
    assert np.array_equal(got["reason"], ref["reason"])
    assert np.array_equal(got["final_id"].view(np.uint32), ref["final_id"])
    assert np.array_equal(got["low_conf"], ref["low_conf"])
    if want_ck:
        assert np.array_equal(got["ck"].view(np.uint32), ref["ck"].view(np.uint32))


@pytest.mark.parametrize("R,P", [(1, 1), (5, 7), (127, 64), (128, 64), (129, 64), (1000, 64), (300, 32), (77, 100),
                                 (64, 256), (40, 6)])
@pytest.mark.parametrize("w,tau,max_tokens", [(3, 0.9, 4096), (1, 1.0, 1 << 20), (2, 0.5, 640), (5, 0.6, 2000),
                                              (8, 0.75, 4096), (11, 0.7, 1 << 20), (3, 0.6667, 128)])
def test_cot_parity(ctx, R, P, w, tau, max_tokens):
    g = O.gen_params(seed=R * 31 + P + w, conv_hi=max(1, P), hesitation_prob=0.1)
    ids, hes = O.gen_cot(g, R, P)
    cfg = O.probe_cfg(64, w, tau, max_tokens)
    ref = O.cot_exit(ids, hes, cfg, replay=True, want_ck=True)
    got = _run(ctx, ids, hes, cfg)
    _check(got, ref)
    got2 = _run(ctx, ids, hes, cfg, want_ck=False)
    _check(got2, ref, want_ck=False)


def test_cot_device_generator(ctx):
    from paper_2412_20993_b200 import GenParams
    R, P = 4099, 64
    ids, hes = ctx.gen_cot(GenParams(seed=99, conv_hi=64, hesitation_prob=0.05), R, P)
    oi, oh = O.gen_cot(O.gen_params(seed=99, conv_hi=64, hesitation_prob=0.05), R, P)
    assert np.array_equal(ids.cpu().numpy().view(np.uint32), oi)
    assert np.array_equal(hes.cpu().numpy().view(np.uint64), oh)


def test_cot_explicit_offsets(ctx):
    rng = np.random.default_rng(3)
    R, P = 500, 64
    g = O.gen_params(seed=5, conv_hi=64, hesitation_prob=0.2)
    ids, hes = O.gen_cot(g, R, P)
    offsets = np.cumsum(rng.integers(1, 200, size=(R, P)), axis=1).astype(np.int64)
    cfg = O.probe_cfg(64, 3, 0.9, 3000)
    ref = O.cot_exit(ids, hes, cfg, offsets=offsets, replay=True, want_ck=True)
    got = _run(ctx, ids, hes, cfg, offsets=offsets)
    _check(got, ref)


def test_cot_exhaustive_small(ctx):
    """All traces of length 6 over 3 answers x all hesitation masks, several windows/taus
    and budgets (a GPU-sized slice of SURVEY §4's 120.9M-case exhaustive set)."""
    P = 6
    seqs = np.array(list(itertools.product(range(3), repeat=P)), np.uint32)  # 729
    masks = np.arange(1 << P, dtype=np.uint64)  # 64
    ids = np.repeat(seqs, len(masks), axis=0)
    hes = np.tile(masks, len(seqs)).reshape(-1, 1)
    for w, tau, mt in [(1, 1.0, 10 ** 6), (2, 1.0, 256), (2, 0.5, 10 ** 6), (3, 0.9, 384), (3, 0.6, 10 ** 6),
                       (4, 0.75, 320), (4, 0.5, 64)]:
        cfg = O.probe_cfg(64, w, tau, mt)
        ref = O.cot_exit(ids, hes, cfg, replay=True, want_ck=True)
        got = _run(ctx, ids, hes, cfg)
        _check(got, ref)


def test_cot_errors(ctx):
    import torch
    from paper_2412_20993_b200 import CdxInvalidArgument, ProbeConfig
    ids = torch.zeros((2, 4), dtype=torch.int32, device="cuda")
    hes = torch.zeros((2, 1), dtype=torch.int64, device="cuda")
    with pytest.raises(CdxInvalidArgument, match=r"threshold must be in \(0,1\]"):
        ctx.cot_exit(ids, hes, ProbeConfig(64, 3, 0.0, 100))
    with pytest.raises(CdxInvalidArgument, match="window must be >= 1"):
        ctx.cot_exit(ids, hes, ProbeConfig(64, 0, 0.5, 100))
    with pytest.raises(CdxInvalidArgument, match="interval_tokens must be >= 1"):
        ctx.cot_exit(ids, hes, ProbeConfig(0, 3, 0.5, 100))
    with pytest.raises(CdxInvalidArgument, match="max_tokens must be >= 1"):
        ctx.cot_exit(ids, hes, ProbeConfig(64, 3, 0.5, 0))


@pytest.mark.parametrize("w", [1, 2, 3, 4])
def test_cot_exhaustive_len8(ctx, w):
    """SURVEY §4 plan item 2 at full length: all 6,561 traces of length 8 over 3 answers x all
    256 hesitation masks (1,679,616 traces), against the literal prefix replay of
    should_exit, for 5 thresholds x 3 budgets per window."""
    P = 8
    seqs = np.array(list(itertools.product(range(3), repeat=P)), np.uint32)
    masks = np.arange(1 << P, dtype=np.uint64)
    ids = np.repeat(seqs, len(masks), axis=0)
    hes = np.tile(masks, len(seqs)).reshape(-1, 1)
    for tau in (0.5, 0.6, 0.75, 0.9, 1.0):
        for mt in (10 ** 6, 64 * 5, 64 * 8):
            cfg = O.probe_cfg(64, w, tau, mt)
            ref = O.cot_exit(ids, hes, cfg, replay=True, want_ck=True)
            got = _run(ctx, ids, hes, cfg)
            _check(got, ref)


@pytest.mark.parametrize("R,P", [(1000, 32), (129, 32), (1000, 64), (3, 64), (500, 96), (700, 128), (65, 128)])
@pytest.mark.parametrize("w,tau,max_tokens", [(3, 0.9, 4096), (1, 1.0, 640), (5, 1.0, 10 ** 6), (2, 0.5, 64)])
def test_cot_run_kernel_parity_no_ck(ctx, R, P, w, tau, max_tokens):
    """The branch-free run kernel (P = 32 or 64, a_min == w, no C_k output), implicit offsets."""
    g = O.gen_params(seed=R + P + w, conv_hi=max(1, P), hesitation_prob=0.15)
    ids, hes = O.gen_cot(g, R, P)
    cfg = O.probe_cfg(64, w, tau, max_tokens)
    ref = O.cot_exit(ids, hes, cfg)
    _check(_run(ctx, ids, hes, cfg, want_ck=False), ref, want_ck=False)


@pytest.mark.parametrize("R,P", [(1000, 64), (257, 64), (500, 40), (300, 128), (33, 7), (700, 32)])
@pytest.mark.parametrize("w,tau", [(3, 0.9), (4, 0.7), (1, 1.0)])
def test_cot_explicit_offsets_parity(ctx, R, P, w, tau):
    """Explicit token offsets without ck: the per-request budget steps come from the coalesced
    pre-pass and feed every kernel (run64 included); offsets not monotone, some rows never
    reach the budget, some reach it at probe 0."""
    rng = np.random.default_rng(R + P + w)
    g = O.gen_params(seed=R * 7 + P, conv_hi=max(1, P), hesitation_prob=0.1)
    ids, hes = O.gen_cot(g, R, P)
    offsets = rng.integers(0, 5000, size=(R, P)).astype(np.int64)
    offsets[::5] = np.cumsum(rng.integers(1, 40, size=(len(offsets[::5]), P)), axis=1)
    offsets[1::7, 0] = 10 ** 6
    cfg = O.probe_cfg(64, w, tau, 4000)
    ref = O.cot_exit(ids, hes, cfg, offsets=offsets)
    got = _run(ctx, ids, hes, cfg, offsets=offsets, want_ck=False)
    _check(got, ref, want_ck=False)
