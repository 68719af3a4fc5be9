"""GPU parity of the mixed-archetype decision step (cdx_mixed_allocate, cdx_cot_meets) and
its composition with the gang order (K6): every threshold bit, decision, grant, cap, budget
offset and the resulting program order equal the restatement (oracle/cdx_oracle.c, pinned
in tests/test_mixed.py)."""
import numpy as np
import pytest

from oracle import oracle as O
from paper_2412_20993_b200 import synth

pytestmark = pytest.mark.gpu
SC, REB, MCT, COT = 0, 1, 2, 3
EVEN, STATIC, KSTEP = 0, 2, 4
TH = {SC: [(0, 0.7, 0)], MCT: [(0, 0.99, 0), (1, 0.4, 0)], REB: [(0, 0.85, 0), (1, 0.99, 0)], COT: [(0, 0.9, 0)]}


def _dev(a, dt=None):
    import torch
    a = np.ascontiguousarray(a)
    if a.dtype == np.uint32:
        a = a.view(np.int32)
    if a.dtype == np.uint64:
        a = a.view(np.int64)
    return torch.from_numpy(a).cuda()


@pytest.mark.parametrize("R,P,w,hp", [(1, 1, 1, 0.0), (1000, 64, 3, 0.05), (777, 40, 5, 0.3), (300, 13, 2, 0.5),
                                      (513, 100, 12, 0.1), (64, 64, 8, 0.0), (2000, 96, 1, 0.2), (100, 70, 62, 0.1)])
def test_cot_meets_parity(ctx, R, P, w, hp):
    from paper_2412_20993_b200 import Threshold
    ids, hes = O.gen_cot(O.gen_params(seed=R + P, conv_hi=P, hesitation_prob=hp), R, P)
    for ths in ([(0, 0.9, 0)], [(0, 2 / 3, 0)], [(0, 0.5, 1)], [(0, 0.0, 0)], [(0, float("nan"), 0)], []):
        got = ctx.cot_meets(_dev(ids), _dev(hes), w, [Threshold(*t) for t in ths])
        ctx.sync()
        assert np.array_equal(got.cpu().numpy().view(np.uint32), O.cot_meets(ids, hes, w, ths)), ths


def _trace(N, seed, sc_shape=(32, 16), cot_P=64, rw_shape=(16, 16), w=3, with_rw_ids=True, mix=(0.4, 0.4, 0.1, 0.1)):
    arch, slot, sizes = synth.mixed_layout(N, seed, mix)
    P, S = sc_shape
    T, W = rw_shape
    sc = O.gen_sc(O.gen_params(seed=seed + 1, conv_hi=P), sizes[0], P, S)
    cid, ches = O.gen_cot(O.gen_params(seed=seed + 2, conv_hi=cot_P, hesitation_prob=0.05), sizes[1], cot_P)
    rw, rid = O.gen_reward(O.gen_params(seed=seed + 3, conv_hi=T), sizes[2], T, W)
    host = dict(sc_ids=sc, cot_ids=cid, cot_hes=ches, cot_window=w, rw=rw, rw_ids=rid if with_rw_ids else None)
    return arch, slot, host


def _run(ctx, arch, slot, knob, host, pols_o):
    from paper_2412_20993_b200 import AllocPolicy, Threshold
    dev = {k: (_dev(v) if isinstance(v, np.ndarray) else v) for k, v in host.items() if v is not None}
    pols = []
    for a in range(4):
        p = pols_o[a]
        ths = [Threshold(p.th[i].signal, p.th[i].cutoff, p.th[i].dir) for i in range(p.n_th)]
        q = p.alloc
        pols.append((ths, AllocPolicy(kind=q.kind, detect_at=q.detect_at, resource_cap=q.resource_cap,
                                      recheck_every=q.recheck_every, tokens_per_unit=q.tokens_per_unit)))
    out = ctx.mixed_allocate(dev, _dev(arch), _dev(slot), _dev(knob), pols)
    ctx.sync()
    return {k: v.cpu().numpy() for k, v in out.items()}


@pytest.mark.parametrize("N,seed,kinds", [(1, 0, (STATIC,) * 4), (5000, 1, (STATIC,) * 4),
                                          (20000, 2, (KSTEP, STATIC, KSTEP, KSTEP)),
                                          (9000, 3, (EVEN, KSTEP, STATIC, EVEN))])
def test_mixed_allocate_parity(ctx, N, seed, kinds):
    caps = (32, 16, 16, 64)
    pols = [O.arch_policy(TH[a], kinds[a], (5, 3, 3, 4)[a], caps[a], (2, 1, 3, 1)[a], 64 * (a + 1)) for a in range(4)]
    arch, slot, host = _trace(N, seed)
    knob = synth.mixed_knobs(arch, caps, seed)
    got = _run(ctx, arch, slot, knob, host, pols)
    want = O.mixed_allocate(host, arch, slot, knob, pols)
    for k in ("decision", "grant", "cap", "offsets"):
        assert np.array_equal(got[k], want[k]), k
    assert int(got["total"][0]) == want["total"]


def test_mixed_shapes_and_groups(ctx):
    """Odd shapes (S = 5, P = 7, W = 48, window 4), an empty group, no reward ids (reward
    thresholds only)."""
    pols = [O.arch_policy([(0, 0.6, 0)], STATIC, 2, 7, 1, 10), O.arch_policy([(1, 0.5, 0)], KSTEP, 1, 5, 2, 3),
            O.arch_policy([(1, 0.35, 0)], STATIC, 2, 5, 1, 7), O.arch_policy([(0, 0.75, 0)], KSTEP, 4, 30, 3, 5)]
    arch, slot, host = _trace(4000, 9, sc_shape=(7, 5), cot_P=30, rw_shape=(5, 48), w=4, with_rw_ids=False)
    knob = synth.mixed_knobs(arch, (7, 5, 5, 30), 9)
    got = _run(ctx, arch, slot, knob, host, pols)
    want = O.mixed_allocate(host, arch, slot, knob, pols)
    for k in ("decision", "grant", "cap", "offsets"):
        assert np.array_equal(got[k], want[k]), k
    # no SC programs at all
    arch2, slot2, host2 = _trace(3000, 10, mix=(0.0, 0.5, 0.25, 0.25))
    host2["sc_ids"] = None
    pols2 = [O.arch_policy(TH[a], STATIC, 3, (32, 16, 16, 64)[a]) for a in range(4)]
    knob2 = synth.mixed_knobs(arch2, (32, 16, 16, 64), 10)
    got = _run(ctx, arch2, slot2, knob2, host2, pols2)
    want = O.mixed_allocate(host2, arch2, slot2, knob2, pols2)
    assert np.array_equal(got["decision"], want["decision"]) and np.array_equal(got["offsets"], want["offsets"])


def test_mixed_bad_program_raises(ctx):
    from paper_2412_20993_b200 import CdxInvalidArgument
    pols = [O.arch_policy(TH[a], STATIC, 3, (32, 16, 16, 64)[a]) for a in range(4)]
    arch, slot, host = _trace(500, 4)
    knob = synth.mixed_knobs(arch, (32, 16, 16, 64), 4)
    knob[7] = 999
    with pytest.raises(CdxInvalidArgument, match="knob out of range"):
        _run(ctx, arch, slot, knob, host, pols)
    knob[7] = 0
    arch[3] = 9
    with pytest.raises(CdxInvalidArgument, match="archetype"):
        _run(ctx, arch, slot, knob, host, pols)


def test_mixed_then_gang_order(ctx):
    """The scheduling round: decisions of the mixed step are the `terminated` flags and caps
    of the gang order; the order equals the restatement's."""
    import torch
    from paper_2412_20993_b200 import InterPolicy
    N = 60000
    caps = (32, 16, 16, 64)
    pols = [O.arch_policy(TH[a], STATIC, (5, 3, 3, 4)[a], caps[a]) for a in range(4)]
    arch, slot, host = _trace(N, 21)
    knob = synth.mixed_knobs(arch, caps, 21)
    got = _run(ctx, arch, slot, knob, host, pols)
    want = O.mixed_allocate(host, arch, slot, knob, pols)
    assert np.array_equal(got["decision"], want["decision"])
    state, now = synth.gang_state(N, 22, 0.5, knob=knob, cap=want["cap"])
    soa = dict(state, terminated=want["decision"])
    dev = {k: _dev(v) for k, v in soa.items()}
    order, _, _ = ctx.gang_priority(dev, InterPolicy(order=1, starvation_limit=0.5, prior_tokens=128.0), now)
    ctx.sync()
    ref, _ = O.gang_order(soa, 1, 0.5, 128.0, now)
    assert np.array_equal(order.cpu().numpy().view(np.uint32), ref)
    assert len(ref) == int((want["decision"] == 0).sum())
    del torch


@pytest.mark.parametrize("serial", ["0", "1"])
def test_mixed_concurrent_engines_and_graph(ctx, monkeypatch, serial):
    """The archetype engines forked onto side streams (SC and reward rows present) and the
    serial form (CDX_MIXED_SERIAL=1) give the oracle's decisions; the forked step captured as
    a CUDA graph replays bit-identically (the fork / join are stream events)."""
    import torch
    from paper_2412_20993_b200 import AllocPolicy, Threshold
    monkeypatch.setenv("CDX_MIXED_SERIAL", serial)
    caps = (32, 16, 16, 64)
    pols_o = [O.arch_policy(TH[a], (STATIC, KSTEP, STATIC, KSTEP)[a], (5, 3, 3, 4)[a], caps[a], (2, 1, 3, 1)[a],
                            64 * (a + 1)) for a in range(4)]
    arch, slot, host = _trace(30000, 21)
    knob = synth.mixed_knobs(arch, caps, 21)
    want = O.mixed_allocate(host, arch, slot, knob, pols_o)
    got = _run(ctx, arch, slot, knob, host, pols_o)
    for k in ("decision", "grant", "cap", "offsets"):
        assert np.array_equal(got[k], want[k]), k
    dev = {k: (_dev(v) if isinstance(v, np.ndarray) else v) for k, v in host.items() if v is not None}
    pols = []
    for a in range(4):
        p = pols_o[a]
        q = p.alloc
        pols.append(([Threshold(p.th[i].signal, p.th[i].cutoff, p.th[i].dir) for i in range(p.n_th)],
                     AllocPolicy(kind=q.kind, detect_at=q.detect_at, resource_cap=q.resource_cap,
                                 recheck_every=q.recheck_every, tokens_per_unit=q.tokens_per_unit)))
    a_d, s_d, k_d = _dev(arch), _dev(slot), _dev(knob)
    n = arch.shape[0]
    out = {k: torch.empty((n,), dtype=dt, device="cuda") for k, dt in
           (("decision", torch.uint8), ("grant", torch.int32), ("cap", torch.int32), ("offsets", torch.int64))}
    out["total"] = torch.empty((1,), dtype=torch.int64, device="cuda")
    ctx.mixed_allocate(dev, a_d, s_d, k_d, pols, out=out)  # warm (tables, occupancy caches)
    ctx.sync()
    graph = ctx.graph_capture(lambda: ctx.mixed_allocate(dev, a_d, s_d, k_d, pols, out=out))
    for _ in range(2):
        for v in out.values():
            v.fill_(-1) if v.dtype != torch.uint8 else v.fill_(255)
        graph()
        ctx.sync()
        for k in ("decision", "grant", "cap", "offsets"):
            assert np.array_equal(out[k].cpu().numpy(), want[k]), k
        assert int(out["total"][0]) == want["total"]
