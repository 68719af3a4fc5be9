"""CPU: pin the oracle (the C restatement, oracle/cdx_oracle.c) against the reference.

Two anchors: tests/golden/reference_golden.json (produced by the reference's own C++
sources compiled here, tests/golden/make_golden.py) and — when oracle/_ref is built — the
reference library itself on randomized and exhaustive cases.
"""
import ctypes as C
import itertools
import json
import os

import numpy as np
import pytest

from oracle import oracle as O

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "reference_golden.json")))
need_ref = pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref not built")


def test_rng_matches_reference_fixture():
    for x, y in GOLD["spec"]["mix64"]:
        assert O.lib().cdxo_mix64(x) == y
    for a, b, c, y in GOLD["spec"]["derive_seed"]:
        assert O.lib().cdxo_derive_seed(a, b, c) == y


def _entropy(sizes):
    arr = (C.c_int * len(sizes))(*sizes)
    n = sum(sizes)
    L = O.lib()
    L.cdxo_semantic_entropy.argtypes = [C.c_void_p, C.c_int, C.c_int]
    L.cdxo_certaindex_entropy.argtypes = [C.c_void_p, C.c_int, C.c_int]
    return L.cdxo_semantic_entropy(arr, len(sizes), n), L.cdxo_certaindex_entropy(arr, len(sizes), n)


def test_entropy_suite_bit_exact():
    """Every clustering shape and order for n <= 12 (SPEC.md:641 acceptance, tol 0 here)."""
    for sizes, H, Hc in GOLD["entropy_suite"]:
        h, hc = _entropy(sizes)
        if sum(sizes) > 1:
            assert h.hex() == H, sizes
        assert hc.hex() == Hc, sizes


def test_spec_entropy_examples():
    for e in GOLD["spec"]["entropy"]:
        h, hc = _entropy(e["sizes"])
        assert hc == e["Hc"]
    assert _entropy([2, 2])[1] == 0.5
    assert _entropy([1, 1, 1, 1])[1] == 0.0


def test_spec_cluster_exact_examples():
    for e in GOLD["spec"]["cluster_exact"]:
        ids, _, _ = O.canon_intern(e["in"], markers=())
        sizes = (C.c_int * len(ids))()
        leaders = (C.c_int * len(ids))()
        m = O.lib().cdxo_cluster_exact_ids(ids.ctypes.data_as(C.c_void_p), len(ids), sizes, leaders)
        got = [(e["in"][leaders[k]].strip(" \t\n\r\f\v"), sizes[k]) for k in range(m)]
        assert got == [tuple(x) for x in e["out"]]


def test_spec_reward_examples():
    L = O.lib()
    L.cdxo_certaindex_reward.argtypes = [C.c_void_p, C.c_size_t, C.c_int, C.c_void_p]
    for e in GOLD["spec"]["reward"]:
        arr = np.array(e["r"], np.float64)
        out = C.c_double()
        assert L.cdxo_certaindex_reward(arr.ctypes.data_as(C.c_void_p), len(arr), e["agg_max"], C.byref(out)) == 0
        assert out.value == e["out"]  # incl. 0.4000000000000001 for the left fold
    for e in GOLD["spec"]["reward_errors"]:
        arr = np.array(e["r"] or [0.0], np.float64)
        out = C.c_double()
        st = L.cdxo_certaindex_reward(arr.ctypes.data_as(C.c_void_p), len(e["r"]), 0, C.byref(out))
        assert st == (2 if not e["r"] else 1)


def test_spec_meets_examples():
    L = O.lib()
    for e in GOLD["spec"]["meets"]:
        sig = (C.c_double * 4)()
        pres = (C.c_int * 4)()
        for k, v in e["signals"].items():
            sig[int(k)] = v
            pres[int(k)] = 1
        arr, n = O.thresholds([tuple(t) for t in e["th"]])
        assert bool(L.cdxo_meets_thresholds(sig, pres, arr, n)) == e["out"]
    assert GOLD["spec"]["meets_absent_error"] == "combined_meets_thresholds: signal 'certaindex_reward' absent"


def test_spec_hesitation_examples():
    for e in GOLD["spec"]["hesitation"]:
        mk = "".join(e["m"]).encode()
        moff = np.zeros(len(e["m"]) + 1, np.uint32)
        moff[1:] = np.cumsum([len(m) for m in e["m"]])
        a = e["a"].encode()
        assert bool(O.lib().cdxo_flag_hesitation(a, len(a), mk, moff.ctypes.data_as(C.c_void_p), len(e["m"]))) \
            == e["out"]


def _trace_arrays(recs):
    names = sorted({r[2].strip() for r in recs})
    ids = np.array([[names.index(r[2].strip()) for r in recs]], np.uint32)
    hes = np.zeros((1, (len(recs) + 63) // 64), np.uint64)
    for i, r in enumerate(recs):
        if r[3]:
            hes[0, i // 64] |= np.uint64(1) << np.uint64(i % 64)
    return ids, hes, names


def test_spec_should_exit_examples():
    for e in GOLD["spec"]["should_exit"]:
        ids, hes, _ = _trace_arrays(e["recs"])
        cfg = O.probe_cfg(64, e["w"], e["tau"], e["max_tokens"])
        r = O.cot_exit(ids, hes, cfg, replay=True, want_ck=True)
        n = len(e["recs"])
        # should_exit on the whole trace = the per-prefix decision at the latest record
        c = float(r["ck"][0, n - 1])
        got = 1 if (c > 0 and c >= e["tau"]) else (2 if n * 64 >= e["max_tokens"] else 0)
        assert got == e["out"]


def test_spec_final_answer_examples():
    for e in GOLD["spec"]["final_answer"]:
        ids, hes, names = _trace_arrays(e["recs"])
        n = len(e["recs"])
        cfg = O.probe_cfg(64, 1000, 1.0, (n) * 64)  # window never fills: budget exit at the last probe
        r = O.cot_exit(ids, hes, cfg, replay=True)
        if e["reason"] == 1:  # budget termination
            assert names[r["final_id"][0]] == e["out"][0] and bool(r["low_conf"][0]) == e["out"][1]


def test_sc_rows_fixture():
    f = GOLD["sc"]
    ids = O.gen_sc(O.gen_params(seed=f["seed"], conv_hi=f["conv_hi"]), f["R"], f["P"], f["S"])
    import hashlib
    assert hashlib.sha256(ids.tobytes()).hexdigest() == f["ids_sha"]
    h64, h32, meets = O.sc_certaindex(ids, [(0, f["tau"], 0)])
    assert [float(x).hex() for x in h64.ravel()] == f["hcert"]
    assert meets.ravel().tolist() == f["meets"]


def test_cot_rows_fixture():
    f = GOLD["cot"]
    ids, hes = O.gen_cot(O.gen_params(seed=f["seed"], conv_hi=64, hesitation_prob=f["hes_prob"]), f["R"], f["P"])
    cfg = O.probe_cfg(64, f["w"], f["tau"], f["max_tokens"])
    for replay in (True, False):
        r = O.cot_exit(ids, hes, cfg, replay=replay, want_ck=True)
        for k in ("exit_step", "reason", "final_id", "low_conf"):
            assert r[k].ravel().tolist() == f[k], (k, replay)
        assert [float(x).hex() for x in r["ck"].ravel()] == f["ck"]


def test_reward_rows_fixture():
    f = GOLD["reward"]
    rw, ids = O.gen_reward(O.gen_params(seed=f["seed"], conv_hi=f["conv_hi"]), f["G"], f["T"], f["W"])
    agg = (np.arange(f["G"]) % 2).astype(np.uint8)
    R64, R32, H = O.reward_certaindex(rw, ids, agg)
    assert [float(x).hex() for x in R64.ravel()] == f["R"]
    assert [float(np.float32(float.fromhex(x))).hex() for x in f["H"]] == [float(x).hex() for x in H.ravel()]


def test_generator_is_on_the_reward_grid():
    rw, _ = O.gen_reward(O.gen_params(seed=3), 50, 4, 8)
    k = rw.astype(np.float64) * 2 ** 24
    assert np.all(k == np.round(k)) and rw.min() >= 0 and rw.max() <= 1


@need_ref
@pytest.mark.parametrize("seed,R,P,S", [(1, 64, 32, 16), (2, 40, 64, 32), (3, 33, 20, 7), (4, 16, 5, 1)])
def test_sc_oracle_vs_reference(seed, R, P, S):
    ids = O.gen_sc(O.gen_params(seed=seed, conv_hi=P), R, P, S)
    for tau in (0.4, 0.7, 0.99):
        h64, _, meets = O.sc_certaindex(ids, [(0, tau, 0)])
        rh, rm = O.ref_sc_batch(ids, 5, [(0, tau, 0)], nthreads=2)
        assert np.array_equal(h64.view(np.uint64), rh.view(np.uint64))
        assert np.array_equal(meets, rm)


@need_ref
def test_sc_all_partitions_n16_vs_reference():
    rows = []
    def parts(n, mx):
        if n == 0:
            yield []
            return
        for k in range(min(n, mx), 0, -1):
            for rest in parts(n - k, k):
                yield [k] + rest
    rng = np.random.default_rng(0)
    for part in parts(16, 16):
        lab = np.concatenate([np.full(c, i, np.uint32) for i, c in enumerate(part)])
        rows += [lab, rng.permutation(lab)]
    ids = np.stack(rows)[:, None, :].astype(np.uint32)  # (rows, P=1, S=16)
    h64, _, _ = O.sc_certaindex(ids, [])
    rh, _ = O.ref_sc_batch(ids, 16, [], nthreads=4)  # vocab covers ids < 2*16
    assert np.array_equal(h64.view(np.uint64), rh.view(np.uint64))


@need_ref
@pytest.mark.parametrize("w,tau,mt", [(3, 0.9, 4096), (1, 1.0, 10 ** 6), (4, 0.5, 2000), (5, 0.6, 640)])
def test_cot_oracle_vs_reference(w, tau, mt):
    ids, hes = O.gen_cot(O.gen_params(seed=w * 13, conv_hi=64, hesitation_prob=0.15), 300, 64)
    cfg = O.probe_cfg(64, w, tau, mt)
    r = O.ref_cot_batch(ids, hes, 5, 64, w, tau, mt, nthreads=2)
    for replay in (True, False):
        o = O.cot_exit(ids, hes, cfg, replay=replay, want_ck=True)
        for k in ("exit_step", "reason", "final_id", "low_conf"):
            assert np.array_equal(o[k], r[k]), (k, replay)
        assert np.array_equal(o["ck"].view(np.uint32), r["ck"].view(np.uint32))


def test_cot_batched_equals_replay_exhaustive():
    """All traces of length 7 over 3 answers x all hesitation masks, several (w, tau,
    budget): the single-pass batched rule == the literal prefix replay."""
    P = 7
    seqs = np.array(list(itertools.product(range(3), repeat=P)), np.uint32)
    masks = np.arange(1 << P, dtype=np.uint64)
    ids = np.repeat(seqs, len(masks), axis=0)
    hes = np.tile(masks, len(seqs)).reshape(-1, 1)
    for w, tau, mt in [(1, 1.0, 10 ** 6), (2, 1.0, 320), (2, 0.5, 10 ** 6), (3, 0.9, 448), (3, 0.6, 10 ** 6),
                       (4, 0.75, 256)]:
        cfg = O.probe_cfg(64, w, tau, mt)
        a = O.cot_exit(ids, hes, cfg, replay=True, want_ck=True)
        b = O.cot_exit(ids, hes, cfg, replay=False, want_ck=True)
        for k in a:
            assert np.array_equal(a[k], b[k]), (k, w, tau, mt)


@need_ref
def test_reward_oracle_vs_reference():
    rw, ids = O.gen_reward(O.gen_params(seed=21, conv_hi=16), 200, 16, 64)
    agg = (np.arange(200) % 2).astype(np.uint8)
    R64, R32, H = O.reward_certaindex(rw, ids, agg)
    RR, RH = O.ref_reward_batch(rw, ids, agg, nthreads=4)
    assert np.array_equal(R64.view(np.uint64), RR.view(np.uint64))
    assert np.array_equal(H.view(np.uint32), RH.astype(np.float32).view(np.uint32))


def test_allocate_spec_examples():
    """SC static_threshold detect@5 (Table 3 tau 0.7): H~=0.72 -> terminate
    at 5; H~=0.3 -> grant to cap 20; knob == cap -> terminate."""
    P = 20
    meets = np.zeros((2, 1), np.uint32)
    meets[0, 0] = 1 << 4  # probe index 4 (knob 5) meets the threshold (0.72 >= 0.7)
    r = O.allocate_scan(meets, 2, P, 2, 5, 20, 1, 64)
    assert r["exit_knob"].tolist() == [5, 20]
    assert r["reason"].tolist() == [1, 2]
    assert r["offsets"].tolist() == [0, 5 * 64]
    assert r["kept"].tolist() == [1] and r["tokens_saved"] == 15 * 64
    r = O.allocate_scan(np.zeros((1, 1), np.uint32), 1, P, 2, 20, 20, 1, 64)  # detect at the cap
    assert r["exit_knob"].tolist() == [20] and r["reason"].tolist() == [2]


def test_gang_spec_examples():
    """estimate_iteration_tokens and inclusive FIFO escalation."""
    L = O.lib()
    assert L.cdxo_estimate_iteration_tokens(300, 2, 128.0) == 150.0
    assert L.cdxo_estimate_iteration_tokens(0, 0, 128.0) == 128.0
    assert L.cdxo_estimate_iteration_tokens(64, 1, 128.0) == 64.0
    soa = dict(arrival=np.array([0.0, 1.0, 2.0, 3.0]), last_service=np.array([10.0, 5.0, 9.0, 0.0]),
               iter_tok_sum=np.array([100, 100, 100, 0]), iter_count=np.array([1, 1, 1, 0]),
               knob=np.array([1, 1, 1, 0]), cap=np.array([10, 2, 5, 4]), terminated=np.array([0, 0, 0, 0]))
    order, esc = O.gang_order(soa, 1, 5.0, 128.0, now=10.0)
    # wait = now - last_service = [0, 5, 1, 10]; limit 5 -> programs 1 (boundary) and 3 escalate
    assert esc.tolist() == [0, 1, 0, 1]
    # escalated FIFO by arrival (1 then 3), then SJF: est*remaining = [900, -, 400] -> 2, 0
    assert order.tolist() == [1, 3, 2, 0]
