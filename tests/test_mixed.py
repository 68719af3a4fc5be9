"""Mixed-archetype decision step (cdx_mixed_allocate): ProgramDriver::update_certaindex's
dispatch (runtime.cpp:264-313) + scheduler.allocate at each program's current knob
(SPEC.md:404-412), then the gang order (K6) over the resulting live programs.

CPU: the restated CoT signal (cdxo_cot_meets) is pinned to the reference's own
probe::consistency as update_certaindex calls it (oracle/_ref ref_cot_signal); the restated
decision (cdxo_mixed_decide) is pinned to the SPEC allocate examples and to the K5
restatement's exit knobs.  GPU: the device step equals the restatement bit for bit."""
import numpy as np
import pytest

from oracle import oracle as O
from paper_2412_20993_b200 import synth

SC, REB, MCT, COT = 0, 1, 2, 3
EVEN, STATIC, KSTEP = 0, 2, 4


def _ref_or_skip():
    if not O.ref_available():
        pytest.skip("oracle/_ref not built")


@pytest.mark.parametrize("seed,w", [(0, 3), (1, 1), (2, 5), (3, 12)])
def test_cot_signal_restatement_pinned_to_reference(seed, w):
    _ref_or_skip()
    g = O.gen_params(seed=seed, conv_hi=40, hesitation_prob=0.2 if seed % 2 else 0.05)
    ids, hes = O.gen_cot(g, 300, 40)
    ck = O.ref_cot_signal(ids, hes, w)
    for ths in ([(0, 0.9, 0)], [(0, 2 / 3, 0)], [(0, 0.5, 1)], [(0, 0.0, 0), (0, 1.0, 1)], [(0, float("nan"), 0)], []):
        want = np.zeros((300, 2), np.uint32)
        ok = np.ones_like(ck, bool)
        for _, cut, d in ths:
            ok &= (ck >= cut) if d == 0 else (ck <= cut)
        for p in range(40):
            want[:, p // 32] |= ok[:, p].astype(np.uint32) << np.uint32(p % 32)
        assert np.array_equal(O.cot_meets(ids, hes, w, ths), want), ths


def _policies(caps=(32, 16, 16, 64), kinds=(STATIC, STATIC, STATIC, STATIC), detect=(5, 3, 3, 4), recheck=(1, 1, 1, 1)):
    ths = {SC: [(0, 0.7, 0)], MCT: [(0, 0.99, 0), (1, 0.4, 0)], REB: [(0, 0.85, 0), (1, 0.99, 0)], COT: [(0, 0.9, 0)]}
    return [O.arch_policy(ths[a], kinds[a], detect[a], caps[a], recheck[a], 64 * (a + 1)) for a in range(4)]


def _py_allocate(row_bits, k, kind, detect, cap, recheck):
    """scheduler.hpp allocate restated in Python."""
    if k >= cap:
        return 2, 0
    tests = []
    if kind == STATIC and detect <= k:
        tests = [detect]
    if kind == KSTEP:
        tests = list(range(detect, k + 1, recheck))
    if any((row_bits >> (t - 1)) & 1 for t in tests):
        return 1, 0
    nxt = cap
    if kind == STATIC and k < detect:
        nxt = detect
    if kind == KSTEP:
        nxt = detect
        while nxt <= k:
            nxt += recheck
        nxt = min(nxt, cap)
    return 0, nxt - k


def test_spec_allocate_examples_through_mixed_decide():
    """SC detect@5, H~ = 0.72 >= 0.7 -> terminate; 0.3 -> grant to cap 20;
    knob == cap -> terminate."""
    pol = [O.arch_policy([(0, 0.7, 0)], STATIC, 5, 20) for _ in range(4)]
    sc = np.zeros((3, 20, 1), np.uint32)  # placeholders: meets come from H~ below
    h = {0: 0.72, 1: 0.3}
    meets = np.zeros((3, 1), np.uint32)
    for r, v in h.items():
        meets[r, 0] = (1 << 4) if v >= 0.7 else 0
    import ctypes as C
    arch = np.zeros(3, np.uint8)
    slot = np.arange(3, dtype=np.uint32)
    knob = np.array([5, 5, 20], np.int32)
    dec, grant, cap, off = (np.empty(3, np.uint8), np.empty(3, np.int32), np.empty(3, np.int32), np.empty(3, np.int64))
    tot = C.c_int64(0)
    z = np.zeros((1, 1), np.uint32)
    mp = (C.c_void_p * 3)(meets.ctypes.data, z.ctypes.data, z.ctypes.data)
    st = O.lib().cdxo_mixed_decide(O._p(arch), O._p(slot), O._p(knob), 3, C.cast(mp, C.c_void_p),
                                   C.cast((C.c_uint32 * 3)(1, 1, 1), C.c_void_p),
                                   C.cast((C.c_uint64 * 3)(3, 0, 0), C.c_void_p),
                                   C.cast((O.ArchPolicy * 4)(*pol), C.c_void_p), O._p(dec), O._p(grant), O._p(cap),
                                   O._p(off), C.byref(tot))
    assert st == 0
    assert dec.tolist() == [1, 0, 2] and grant.tolist() == [0, 15, 0]
    del sc


@pytest.mark.parametrize("seed", range(4))
def test_mixed_decide_matches_python_allocate_and_k5(seed):
    rng = np.random.default_rng(seed)
    N = 3000
    arch, slot, sizes = synth.mixed_layout(N, seed)
    kinds = [(STATIC, KSTEP, EVEN, STATIC), (KSTEP, KSTEP, KSTEP, KSTEP), (EVEN, STATIC, KSTEP, STATIC),
             (STATIC, STATIC, STATIC, KSTEP)][seed]
    caps = (30, 12, 12, 40)
    pols = _policies(caps=caps, kinds=kinds, detect=(4, 2, 3, 5), recheck=(3, 2, 1, 4))
    units = (32, 16, 16, 40)  # SC probes, reward steps, CoT probes
    knob = synth.mixed_knobs(arch, caps, seed)
    meets = [rng.integers(0, 1 << 32, size=(sizes[0], 1), dtype=np.uint64).astype(np.uint32),
             rng.integers(0, 1 << 32, size=(sizes[1], 2), dtype=np.uint64).astype(np.uint32) & np.uint32(
                 0xAAAAAAAA if seed % 2 else 0x00010001),
             rng.integers(0, 1 << 16, size=(sizes[2], 1)).astype(np.uint32)]
    import ctypes as C
    dec, grant, cap, off = (np.empty(N, np.uint8), np.empty(N, np.int32), np.empty(N, np.int32), np.empty(N, np.int64))
    tot = C.c_int64(0)
    mp = (C.c_void_p * 3)(*[m.ctypes.data for m in meets])
    st = O.lib().cdxo_mixed_decide(O._p(arch), O._p(slot), O._p(knob), N, C.cast(mp, C.c_void_p),
                                   C.cast((C.c_uint32 * 3)(1, 2, 1), C.c_void_p),
                                   C.cast((C.c_uint64 * 3)(*sizes), C.c_void_p),
                                   C.cast((O.ArchPolicy * 4)(*pols), C.c_void_p), O._p(dec), O._p(grant),
                                   O._p(cap), O._p(off), C.byref(tot))
    assert st == 0
    g_of = {SC: 0, COT: 1, MCT: 2, REB: 2}
    run = 0
    for i in range(N):
        a = int(arch[i])
        m = meets[g_of[a]][slot[i]]
        bits = int(m[0]) | (int(m[1]) << 32 if m.shape[0] > 1 else 0)
        p = pols[a].alloc
        d, gu = _py_allocate(bits, int(knob[i]), p.kind, p.detect_at, p.resource_cap, p.recheck_every)
        assert (dec[i], grant[i], cap[i], off[i]) == (d, gu, p.resource_cap, run), i
        run += gu * p.tokens_per_unit
        # K5 restatement (pinned by SPEC): terminated certain <=> first met test point <= knob
        if p.resource_cap <= units[a] and d != 2:
            r = O.allocate_scan(m[None, :], 1, units[a], p.kind, p.detect_at, p.resource_cap, p.recheck_every)
            certain = r["reason"][0] == 1 and r["exit_knob"][0] <= knob[i]
            assert certain == (d == 1), i
    assert tot.value == run
