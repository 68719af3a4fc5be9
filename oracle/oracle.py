"""oracle.py — numpy/ctypes access to the CHECKERS (test infrastructure only).

  Oracle   : liboracle.so, the C restatement of the hot path (cdx_oracle.c)
  Ref      : _ref/libcdxref.so, the reference's own C++ sources + ref_harness.cpp

Only tests/, __graft_entry__.smoke() and bench.py's CPU legs import this module.  The
product (libcdx.so / paper_2412_20993_b200) never does.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.environ.get("CDX_ORACLE_SO", os.path.join(HERE, "liboracle.so"))  # override: sanitizer builds
REF_SO = os.path.join(HERE, "_ref", "libcdxref.so")

P = C.c_void_p


class Threshold(C.Structure):
    _fields_ = [("signal", C.c_uint8), ("dir", C.c_uint8), ("_pad", C.c_uint8 * 6), ("cutoff", C.c_double)]


class AllocPolicy(C.Structure):
    _fields_ = [("kind", C.c_uint8), ("_pad", C.c_uint8 * 3), ("detect_at", C.c_int32),
                ("recheck_every", C.c_int32), ("resource_cap", C.c_int32), ("tokens_per_unit", C.c_int64)]


class ProbeCfg(C.Structure):
    _fields_ = [("interval_tokens", C.c_int32), ("window", C.c_int32), ("threshold", C.c_double),
                ("max_tokens", C.c_int64)]


class InterPolicy(C.Structure):
    _fields_ = [("gang", C.c_uint8), ("order", C.c_uint8), ("_pad", C.c_uint8 * 6),
                ("starvation_limit", C.c_double), ("prior_tokens", C.c_double)]


class ProgSoA(C.Structure):
    _fields_ = [("arrival", P), ("last_service", P), ("iter_tok_sum", P), ("iter_count", P), ("knob", P),
                ("cap", P), ("terminated", P), ("program_id", P), ("id_base", C.c_uint32), ("_pad", C.c_uint32)]


class ArchPolicy(C.Structure):
    _fields_ = [("th", Threshold * 4), ("n_th", C.c_uint32), ("_pad", C.c_uint32), ("alloc", AllocPolicy)]


class GenParams(C.Structure):
    _fields_ = [("seed", C.c_uint64), ("groups", C.c_uint32), ("conv_lo", C.c_uint32), ("conv_hi", C.c_uint32),
                ("_pad", C.c_uint32), ("noise_level", C.c_double), ("residual_noise", C.c_double),
                ("solvable_fraction", C.c_double), ("hesitation_prob", C.c_double),
                ("reward_start_k", C.c_uint32), ("reward_final_k", C.c_uint32),
                ("reward_unsolvable_k", C.c_uint32), ("reward_jitter_k", C.c_uint32)]


def build():
    """Build the checkers (the reference part only where /root/reference exists)."""
    subprocess.run(["make", "-s", "-C", HERE], check=True)


def _load(path):
    if not os.path.exists(path):
        build()
    return C.CDLL(path)


_O = None
_R = None


def lib():
    global _O
    if _O is None:
        _O = _load(ORACLE_SO)
        _O.cdxo_mix64.restype = C.c_uint64
        _O.cdxo_mix64.argtypes = [C.c_uint64]
        _O.cdxo_derive_seed.restype = C.c_uint64
        _O.cdxo_derive_seed.argtypes = [C.c_uint64] * 3
        _O.cdxo_semantic_entropy.restype = C.c_double
        _O.cdxo_certaindex_entropy.restype = C.c_double
        _O.cdxo_estimate_iteration_tokens.restype = C.c_double
        _O.cdxo_estimate_iteration_tokens.argtypes = [C.c_int64, C.c_uint32, C.c_double]
        _O.cdxo_answer.restype = C.c_uint32
        _O.cdxo_answer.argtypes = [P, C.c_uint64, C.c_uint64, C.c_uint32]
        _O.cdxo_cot_amin.argtypes = [C.c_int, C.c_double]
        _O.cdxo_trim.restype = C.c_size_t
        _O.cdxo_trim.argtypes = [C.c_char_p, C.c_size_t, C.POINTER(C.c_size_t)]
        for name in ("cdxo_gen_sc", "cdxo_gen_cot", "cdxo_gen_reward"):
            getattr(_O, name).restype = None
    return _O


def ref_available() -> bool:
    if os.path.exists(REF_SO):
        return True
    if os.path.isdir("/root/reference/proj/src"):
        build()
    return os.path.exists(REF_SO)


def ref():
    global _R
    if _R is None:
        if not ref_available():
            raise RuntimeError("oracle/_ref/libcdxref.so unavailable (reference not built)")
        _R = C.CDLL(REF_SO)
        _R.ref_last_error.restype = C.c_char_p
        _R.ref_mix64.restype = C.c_uint64
        _R.ref_mix64.argtypes = [C.c_uint64]
        _R.ref_derive_seed.restype = C.c_uint64
        _R.ref_derive_seed.argtypes = [C.c_uint64] * 3
    return _R


def _p(a):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


def gen_params(seed=20993, groups=5, conv_lo=1, conv_hi=64, noise_level=0.5, residual_noise=0.0,
               solvable_fraction=0.9, hesitation_prob=0.0, reward_start_k=5033165, reward_final_k=15099494,
               reward_unsolvable_k=4194304, reward_jitter_k=1677722) -> GenParams:
    g = GenParams()
    g.seed, g.groups, g.conv_lo, g.conv_hi = seed, groups, conv_lo, conv_hi
    g.noise_level, g.residual_noise, g.solvable_fraction = noise_level, residual_noise, solvable_fraction
    g.hesitation_prob = hesitation_prob
    g.reward_start_k, g.reward_final_k = reward_start_k, reward_final_k
    g.reward_unsolvable_k, g.reward_jitter_k = reward_unsolvable_k, reward_jitter_k
    return g


def vocab(groups):
    names = ["S"] + [f"D{i}" for i in range(1, groups)]
    return names + ["wait, " + n for n in names]


def _vocab_c(v):
    arr = (C.c_char_p * len(v))(*[s.encode() for s in v])
    return arr, len(v)


def thresholds(ths):
    """ths: list of (signal, cutoff, dir)."""
    arr = (Threshold * max(1, len(ths)))()
    for i, (sig, cut, d) in enumerate(ths):
        arr[i].signal, arr[i].cutoff, arr[i].dir = sig, cut, d
    return arr, len(ths)


# ---------------------------------------------------------------- generators (restated)
def gen_sc(g, R, P_, S, r0=0):
    ids = np.empty((R, P_, S), np.uint32)
    lib().cdxo_gen_sc(C.byref(g), C.c_uint64(r0), C.c_uint64(R), C.c_uint32(P_), C.c_uint32(S), _p(ids))
    return ids


def gen_cot(g, R, P_, r0=0):
    ids = np.empty((R, P_), np.uint32)
    hes = np.empty((R, (P_ + 63) // 64), np.uint64)
    lib().cdxo_gen_cot(C.byref(g), C.c_uint64(r0), C.c_uint64(R), C.c_uint32(P_), _p(ids), _p(hes))
    return ids, hes


def gen_reward(g, G, T, W, g0=0):
    rw = np.empty((G, T, W), np.float32)
    ids = np.empty((G, T, W), np.uint32)
    lib().cdxo_gen_reward(C.byref(g), C.c_uint64(g0), C.c_uint64(G), C.c_uint32(T), C.c_uint32(W), _p(rw), _p(ids))
    return rw, ids


# ---------------------------------------------------------------- restated hot path
def sc_certaindex(ids, ths):
    R, P_, S = ids.shape
    h64 = np.empty((R, P_), np.float64)
    h32 = np.empty((R, P_), np.float32)
    meets = np.empty((R, (P_ + 31) // 32), np.uint32)
    arr, n = thresholds(ths)
    st = lib().cdxo_sc_certaindex(_p(np.ascontiguousarray(ids)), C.c_uint64(R), C.c_uint32(P_), C.c_uint32(S), arr,
                                  C.c_uint32(n), _p(h64), _p(h32), _p(meets))
    if st:
        raise ValueError(f"oracle sc_certaindex status {st}")
    return h64, h32, meets


def sc_certaindex_ex(ids, ths):
    """K2 restated with the majority fraction: (h64, h32, maj64, maj32, meets)."""
    R, P_, S = ids.shape
    h64 = np.empty((R, P_), np.float64)
    h32 = np.empty((R, P_), np.float32)
    m64 = np.empty((R, P_), np.float64)
    m32 = np.empty((R, P_), np.float32)
    meets = np.empty((R, (P_ + 31) // 32), np.uint32)
    arr, n = thresholds(ths)
    st = lib().cdxo_sc_certaindex_ex(_p(np.ascontiguousarray(ids)), C.c_uint64(R), C.c_uint32(P_), C.c_uint32(S),
                                     arr, C.c_uint32(n), _p(h64), _p(h32), _p(m64), _p(m32), _p(meets))
    if st:
        raise ValueError(f"oracle sc_certaindex_ex status {st}")
    return h64, h32, m64, m32, meets


def majority_fraction(sizes):
    a = (C.c_int * len(sizes))(*[int(x) for x in sizes])
    f = lib().cdxo_majority_fraction
    f.restype = C.c_double
    f.argtypes = [P, C.c_int, C.c_int]
    return f(C.cast(a, P), len(sizes), int(sum(sizes)))


def allocate_scan(meets, R, P_, kind, detect_at, cap, recheck_every=1, tokens_per_unit=64, base_offset=0):
    pol = AllocPolicy()
    pol.kind, pol.detect_at, pol.resource_cap = kind, detect_at, cap
    pol.recheck_every, pol.tokens_per_unit = recheck_every, tokens_per_unit
    ek = np.empty(R, np.int32)
    why = np.empty(R, np.uint8)
    gr = np.empty(R, np.int32)
    off = np.empty(R, np.int64)
    kept = np.empty(max(R, 1), np.uint32)
    nk = C.c_uint64(0)
    saved = C.c_int64(0)
    mb = np.ascontiguousarray(meets, dtype=np.uint32) if meets is not None else np.zeros((R, (P_ + 31) // 32),
                                                                                          np.uint32)
    st = lib().cdxo_allocate_scan(_p(mb), C.c_uint64(R), C.c_uint32(P_), C.byref(pol), C.c_int64(base_offset),
                                  _p(ek), _p(why), _p(gr), _p(off), _p(kept), C.byref(nk), C.byref(saved))
    if st:
        raise ValueError(f"oracle allocate status {st}")
    return dict(exit_knob=ek, reason=why, granted=gr, offsets=off, kept=kept[:nk.value], n_kept=nk.value,
                tokens_saved=saved.value)


def probe_cfg(interval_tokens=64, window=3, threshold=0.9, max_tokens=1 << 20):
    c = ProbeCfg()
    c.interval_tokens, c.window, c.threshold, c.max_tokens = interval_tokens, window, threshold, max_tokens
    return c


def cot_exit(ids, hes, cfg, offsets=None, replay=False, want_ck=False):
    R, P_ = ids.shape
    ex = np.empty(R, np.int32)
    why = np.empty(R, np.uint8)
    fid = np.empty(R, np.uint32)
    low = np.empty(R, np.uint8)
    ck = np.empty((R, P_), np.float32) if want_ck else None
    fn = lib().cdxo_cot_exit_replay if replay else lib().cdxo_cot_exit_batched
    st = fn(_p(np.ascontiguousarray(ids)), _p(np.ascontiguousarray(hes)),
            _p(None if offsets is None else np.ascontiguousarray(offsets, dtype=np.int64)), C.c_uint64(R),
            C.c_uint32(P_), C.byref(cfg), _p(ex), _p(why), _p(fid), _p(low), _p(ck))
    if st:
        raise ValueError(f"oracle cot status {st}")
    return dict(exit_step=ex, reason=why, final_id=fid, low_conf=low, ck=ck)


def reward_certaindex(rw, ids, agg, want_h64=False):
    """(R64, R32, H32) — plus H64 (the FP64 certaindex the thresholds see) with want_h64."""
    G, T, W = rw.shape
    R64 = np.empty((G, T), np.float64)
    R32 = np.empty((G, T), np.float32)
    H = np.empty((G, T), np.float32) if ids is not None else None
    H64 = np.empty((G, T), np.float64) if (ids is not None and want_h64) else None
    f = lib().cdxo_reward_certaindex_f64 if rw.dtype == np.float64 else lib().cdxo_reward_certaindex2
    st = f(_p(np.ascontiguousarray(rw)),
                                       _p(None if ids is None else np.ascontiguousarray(ids)),
                                       _p(np.ascontiguousarray(agg, dtype=np.uint8)), C.c_uint64(G), C.c_uint32(T),
                                       C.c_uint32(W), _p(R64), _p(R32), _p(H), _p(H64))
    if st:
        raise ValueError(f"oracle reward status {st}")
    return (R64, R32, H, H64) if want_h64 else (R64, R32, H)


def gang_order_mt(soa, order_kind, starvation_limit, prior, now, nthreads):
    """cdxo_gang_order_mt: the same order from per-thread qsorts + parallel merges."""
    N = soa["arrival"].shape[0]
    s = ProgSoA()
    keep = {}
    for k, dt in (("arrival", np.float64), ("last_service", np.float64), ("iter_tok_sum", np.int64),
                  ("iter_count", np.uint32), ("knob", np.int32), ("cap", np.int32), ("terminated", np.uint8)):
        keep[k] = np.ascontiguousarray(soa[k], dtype=dt)
        setattr(s, k, keep[k].ctypes.data)
    pol = InterPolicy()
    pol.gang, pol.order, pol.starvation_limit, pol.prior_tokens = 1, order_kind, starvation_limit, prior
    order = np.empty(max(N, 1), np.uint32)
    n = C.c_uint64(0)
    lib().cdxo_gang_order_mt.argtypes = [P, C.c_uint64, P, C.c_double, P, P, C.c_int]
    st = lib().cdxo_gang_order_mt(C.byref(s), C.c_uint64(N), C.byref(pol), C.c_double(now), _p(order), C.byref(n),
                                  C.c_int(nthreads))
    if st:
        raise ValueError(f"oracle gang status {st}")
    return order[:n.value]


def gang_order(soa, order_kind, starvation_limit, prior, now, id_base=0):
    N = soa["arrival"].shape[0]
    s = ProgSoA()
    keep = {}
    for k, dt in (("arrival", np.float64), ("last_service", np.float64), ("iter_tok_sum", np.int64),
                  ("iter_count", np.uint32), ("knob", np.int32), ("cap", np.int32), ("terminated", np.uint8)):
        keep[k] = np.ascontiguousarray(soa[k], dtype=dt)
        setattr(s, k, keep[k].ctypes.data)
    if soa.get("program_id") is not None:
        keep["program_id"] = np.ascontiguousarray(soa["program_id"], dtype=np.uint32)
        s.program_id = keep["program_id"].ctypes.data
    s.id_base = id_base
    pol = InterPolicy()
    pol.gang, pol.order, pol.starvation_limit, pol.prior_tokens = 1, order_kind, starvation_limit, prior
    order = np.empty(max(N, 1), np.uint32)
    esc = np.empty(max(N, 1), np.uint8)
    n = C.c_uint64(0)
    lib().cdxo_gang_order.argtypes = [P, C.c_uint64, P, C.c_double, P, P, P]
    st = lib().cdxo_gang_order(C.byref(s), C.c_uint64(N), C.byref(pol), C.c_double(now), _p(order), C.byref(n),
                               _p(esc))
    if st:
        raise ValueError(f"oracle gang status {st}")
    return order[:n.value], esc[:N]


def canon_intern(strings, markers=("wait", "hmm")):
    bs = [s.encode() if isinstance(s, str) else s for s in strings]
    arena = b"".join(bs)
    offs = np.zeros(len(bs) + 1, np.uint64)
    np.cumsum([len(b) for b in bs], out=offs[1:]) if bs else None
    mk = b"".join(m.encode() for m in markers)
    moff = np.zeros(len(markers) + 1, np.uint32)
    if markers:
        np.cumsum([len(m.encode()) for m in markers], out=moff[1:])
    ids = np.empty(max(len(bs), 1), np.uint32)
    hes = np.empty(max(len(bs), 1), np.uint8)
    nu = C.c_uint64(0)
    ab = C.create_string_buffer(arena, len(arena) + 1)
    mb = C.create_string_buffer(mk, len(mk) + 1)
    st = lib().cdxo_canon_intern(ab, _p(offs), C.c_uint64(len(bs)), mb, _p(moff), C.c_uint32(len(markers)), _p(ids),
                                 _p(hes), C.byref(nu))
    if st:
        raise ValueError("oracle intern failed")
    return ids[:len(bs)], hes[:len(bs)], nu.value


def canon_intern_arena(arena, offs, markers=("wait", "hmm")):
    """canon_intern over a byte arena u8[] + offsets u64[n+1] (no Python strings)."""
    arena = np.ascontiguousarray(arena, np.uint8)
    offs = np.ascontiguousarray(offs, np.uint64)
    n = len(offs) - 1
    mk = b"".join(m.encode() for m in markers)
    moff = np.zeros(len(markers) + 1, np.uint32)
    if markers:
        np.cumsum([len(m.encode()) for m in markers], out=moff[1:])
    ids = np.empty(max(n, 1), np.uint32)
    hes = np.empty(max(n, 1), np.uint8)
    nu = C.c_uint64(0)
    ab = np.concatenate([arena, np.zeros(1, np.uint8)])
    mb = C.create_string_buffer(mk, len(mk) + 1)
    st = lib().cdxo_canon_intern(ab.ctypes.data_as(C.c_char_p), _p(offs), C.c_uint64(n), mb, _p(moff),
                                 C.c_uint32(len(markers)), _p(ids), _p(hes), C.byref(nu))
    if st:
        raise ValueError("oracle intern failed")
    return ids[:n], hes[:n], nu.value


# ---------------------------------------------------------------- the reference itself
class RefError(Exception):
    pass


def _ref_err():
    return ref().ref_last_error().decode(errors="replace")


def ref_cluster_exact(answers):
    n = len(answers)
    arr = (C.c_char_p * max(n, 1))(*[a.encode() if isinstance(a, str) else a for a in answers])
    sizes = (C.c_int32 * max(n, 1))()
    labels = C.create_string_buffer(64 * max(n, 1))
    m = ref().ref_cluster_exact(arr, C.c_uint32(n), sizes, labels, C.c_uint32(64))
    if m < 0:
        raise RefError(_ref_err())
    return [(labels.raw[k * 64:(k + 1) * 64].split(b"\0")[0].decode(), sizes[k]) for k in range(m)]


def ref_entropy(sizes):
    arr = (C.c_int32 * max(1, len(sizes)))(*sizes)
    H, Hc = C.c_double(), C.c_double()
    if ref().ref_entropy(arr, C.c_uint32(len(sizes)), C.c_int32(sum(sizes)), C.byref(H), C.byref(Hc)) < 0:
        raise RefError(_ref_err())
    return H.value, Hc.value


def ref_certaindex_reward(values, agg_max):
    arr = (C.c_double * max(1, len(values)))(*values)
    out = C.c_double()
    if ref().ref_certaindex_reward(arr, C.c_uint32(len(values)), C.c_int(agg_max), C.byref(out)) < 0:
        raise RefError(_ref_err())
    return out.value


def ref_meets(signals: dict, ths):
    sig = (C.c_double * 4)()
    pres = (C.c_int32 * 4)()
    for k, v in signals.items():
        sig[k] = v
        pres[k] = 1
    arr, n = thresholds(ths)
    r = ref().ref_meets(sig, pres, arr, C.c_uint32(n))
    if r < 0:
        raise RefError(_ref_err())
    return bool(r)


def ref_flag_hesitation(answer, markers):
    arr = (C.c_char_p * max(1, len(markers)))(*[m.encode() for m in markers])
    return bool(ref().ref_flag_hesitation(answer.encode() if isinstance(answer, str) else answer, arr,
                                          C.c_uint32(len(markers))))


def _records(records):
    n = len(records)
    step = (C.c_int32 * max(n, 1))(*[r[0] for r in records])
    off = (C.c_int64 * max(n, 1))(*[r[1] for r in records])
    ans = (C.c_char_p * max(n, 1))(*[r[2].encode() for r in records])
    hes = (C.c_uint8 * max(n, 1))(*[1 if r[3] else 0 for r in records])
    return step, off, ans, hes, n


def ref_should_exit(records, interval_tokens=64, window=3, threshold=0.9, max_tokens=1 << 20):
    """records: list of (step_index, token_offset, answer, hesitant)."""
    step, off, ans, hes, n = _records(records)
    cfg = probe_cfg(interval_tokens, window, threshold, max_tokens)
    r = ref().ref_should_exit(step, off, ans, hes, C.c_uint32(n), C.byref(cfg))
    if r < 0:
        raise RefError(_ref_err())
    return r


def ref_consistency(records, k, w):
    step, off, ans, hes, n = _records(records)
    out = C.c_double()
    r = ref().ref_consistency(step, ans, hes, C.c_uint32(n), C.c_int32(k), C.c_int32(w), C.byref(out))
    if r < 0:
        raise RefError(_ref_err())
    return out.value if r == 1 else None


def ref_final_answer(records, terminated_at=None, reason=1):
    step, off, ans, hes, n = _records(records)
    buf = C.create_string_buffer(256)
    low = C.c_uint8()
    r = ref().ref_final_answer(step, ans, hes, C.c_uint32(n), C.c_int32(-1 if terminated_at is None else terminated_at),
                               C.c_int32(reason), buf, C.c_uint32(256), C.byref(low))
    if r < 0:
        raise RefError(_ref_err())
    return buf.value.decode(), bool(low.value)


def ref_read_trace_jsonl(text):
    r = ref().ref_read_trace_jsonl(text.encode() if isinstance(text, str) else text)
    if r < 0:
        raise RefError(_ref_err())
    return r


def ref_read_trace_jsonl_mt(text, nthreads):
    """The reference's read_trace_jsonl on line-aligned chunks, one per host thread, plus the
    cross-chunk order checks (oracle/ref_harness.cpp)."""
    r = ref().ref_read_trace_jsonl_mt(text.encode() if isinstance(text, str) else text, C.c_int(nthreads))
    if r < 0:
        raise RefError(_ref_err())
    return r


def ref_driver_signals(archetype, seed, cap, conv, solvable, units):
    ent = (C.c_double * units)()
    rew = (C.c_double * units)()
    ln = (C.c_double * units)()
    r = ref().ref_driver_signals(archetype, C.c_uint64(seed), cap, conv, solvable, units, ent, rew, ln)
    if r < 0:
        raise RefError(_ref_err())
    return list(ent), list(rew), list(ln)


def ref_sc_batch(ids, groups, ths, nthreads=1, mode=0, want=True):
    R, P_, S = ids.shape
    v, nv = _vocab_c(vocab(groups))
    h = np.empty((R, P_), np.float64) if want else None
    meets = np.empty((R, (P_ + 31) // 32), np.uint32) if want else None
    arr, n = thresholds(ths)
    r = ref().ref_sc_batch(_p(np.ascontiguousarray(ids)), C.c_uint64(R), C.c_uint32(P_), C.c_uint32(S), v,
                           C.c_uint32(nv), arr, C.c_uint32(n), _p(h), _p(meets), C.c_int(nthreads), C.c_int(mode))
    if r < 0:
        raise RefError(_ref_err())
    return h, meets


def ref_intern_batch(arena, offsets, S, markers=("wait", "hmm"), nthreads=1, want=True):
    """The reference's cluster_exact over rows of S answers + flag_hesitation per answer."""
    n = len(offsets) - 1
    rows = (n + S - 1) // S
    ncl = np.empty(max(rows, 1), np.uint32) if want else None
    hes = np.empty(max(n, 1), np.uint8) if want else None
    mk = (C.c_char_p * max(1, len(markers)))(*[m.encode() for m in markers])
    f = ref().ref_intern_batch
    f.argtypes = [P, P, C.c_uint64, C.c_uint32, P, C.c_uint32, P, P, C.c_int]
    a = np.ascontiguousarray(arena, dtype=np.uint8)
    o = np.ascontiguousarray(offsets, dtype=np.uint64)
    if f(_p(a), _p(o), n, S, C.cast(mk, P), len(markers), _p(ncl), _p(hes), nthreads) < 0:
        raise RefError(_ref_err())
    return (ncl[:rows], hes[:n]) if want else (None, None)


def ref_cot_batch(ids, hes, groups, interval_tokens=64, window=3, threshold=0.9, max_tokens=1 << 20, nthreads=1,
                  want_ck=True):
    R, P_ = ids.shape
    v, nv = _vocab_c(vocab(groups))
    cfg = probe_cfg(interval_tokens, window, threshold, max_tokens)
    ex = np.empty(R, np.int32)
    why = np.empty(R, np.uint8)
    fid = np.empty(R, np.uint32)
    low = np.empty(R, np.uint8)
    ck = np.empty((R, P_), np.float32) if want_ck else None
    r = ref().ref_cot_batch(_p(np.ascontiguousarray(ids)), _p(np.ascontiguousarray(hes)), C.c_uint64(R),
                            C.c_uint32(P_), v, C.c_uint32(nv), C.byref(cfg), _p(ex), _p(why), _p(fid), _p(low), _p(ck),
                            C.c_int(nthreads))
    if r < 0:
        raise RefError(_ref_err())
    return dict(exit_step=ex, reason=why, final_id=fid, low_conf=low, ck=ck)


def ref_reward_batch(rw, ids, agg, groups=5, nthreads=1):
    G, T, W = rw.shape
    v, nv = _vocab_c(vocab(groups))
    R = np.empty((G, T), np.float64)
    H = np.empty((G, T), np.float64) if ids is not None else None
    r = ref().ref_reward_batch(_p(np.ascontiguousarray(rw)), _p(None if ids is None else np.ascontiguousarray(ids)),
                               _p(np.ascontiguousarray(agg, dtype=np.uint8)), C.c_uint64(G), C.c_uint32(T),
                               C.c_uint32(W), v, C.c_uint32(nv), _p(R), _p(H), C.c_int(nthreads))
    if r < 0:
        raise RefError(_ref_err())
    return R, H


def hardware_threads():
    try:
        return int(ref().ref_hardware_threads())
    except Exception:
        return os.cpu_count() or 1


# ---------------------------------------------------------------- aggregation (runtime.cpp:316-403)
def sc_aggregate(ids, exit_knob):
    R, P_, S = ids.shape
    out = np.empty(max(R, 1), np.uint32)
    lib().cdxo_sc_aggregate.argtypes = [P, C.c_uint64, C.c_uint32, C.c_uint32, P, P]
    st = lib().cdxo_sc_aggregate(_p(np.ascontiguousarray(ids)), R, P_, S,
                                 _p(np.ascontiguousarray(exit_knob, dtype=np.int32)), _p(out))
    if st:
        raise ValueError(f"oracle sc_aggregate status {st}")
    return out[:R]


def reward_aggregate(rw, ids, agg, exit_step):
    """f32 or f64 rewards (the latter: PathSample::reward / RewardSet doubles)."""
    G, T, W = rw.shape
    out = np.empty(max(G, 1), np.uint32)
    f64 = rw.dtype == np.float64
    f = lib().cdxo_reward_aggregate_f64 if f64 else lib().cdxo_reward_aggregate
    f.argtypes = [P, P, P, C.c_uint64, C.c_uint32, C.c_uint32, P, P]
    st = f(_p(np.ascontiguousarray(rw)), _p(np.ascontiguousarray(ids)),
           _p(np.ascontiguousarray(agg, dtype=np.uint8)), G, T, W,
           _p(np.ascontiguousarray(exit_step, dtype=np.int32)), _p(out))
    if st:
        raise ValueError(f"oracle reward_aggregate status {st}")
    return out[:G]


def ref_aggregate(archetype, ids, rewards, layer_widths, units, vocab_list):
    """The reference's own ProgramDriver::aggregate_prefix on injected paths -> vocab index."""
    n = len(ids)
    a_ids = (C.c_uint32 * max(n, 1))(*[int(x) for x in ids])
    a_rw = None if rewards is None else (C.c_double * max(n, 1))(*[float(x) for x in rewards])
    a_lw = (C.c_int * max(1, len(layer_widths)))(*layer_widths)
    v, nv = _vocab_c(vocab_list)
    out = C.c_uint32(0)
    f = ref().ref_aggregate
    f.argtypes = [C.c_int, P, P, C.c_int, P, C.c_int, C.c_int, P, C.c_uint32, P]
    if f(archetype, C.cast(a_ids, P), None if a_rw is None else C.cast(a_rw, P), n, C.cast(a_lw, P),
         len(layer_widths), units, C.cast(v, P), nv, C.byref(out)) < 0:
        raise RefError(_ref_err())
    return out.value


# ---------------------------------------------------------------- epsilon stop test (probe.cpp:104-120)
def cot_eps_stop(ids, hes, k, epsilon):
    R, P_ = ids.shape
    step = np.empty(max(R, 1), np.int32)
    state = np.empty((R, P_), np.uint8)
    lib().cdxo_cot_eps_stop.argtypes = [P, P, C.c_uint64, C.c_uint32, C.c_int, C.c_double, P, P]
    st = lib().cdxo_cot_eps_stop(_p(np.ascontiguousarray(ids)), _p(np.ascontiguousarray(hes)), R, P_, k,
                                 float(epsilon), _p(step), _p(state))
    if st:
        raise ValueError(f"oracle cot_eps_stop status {st}")
    return step[:R], state


def ref_eps_prefixes(ids, hes, k, epsilon, vocab_list):
    """The reference's stationary_by_epsilon_test at every prefix -> state u8[R][P]."""
    R, P_ = ids.shape
    state = np.empty((R, P_), np.uint8)
    v, nv = _vocab_c(vocab_list)
    f = ref().ref_eps_prefixes
    f.argtypes = [P, P, C.c_uint64, C.c_uint32, C.c_int, C.c_double, P, C.c_uint32, P]
    if f(_p(np.ascontiguousarray(ids)), _p(np.ascontiguousarray(hes)), R, P_, k, float(epsilon), C.cast(v, P), nv,
         _p(state)) < 0:
        raise RefError(_ref_err())
    return state


def ref_parse_jsonl(text: bytes):
    """The reference's read_trace_jsonl with every field: list of (program_id bytes,
    step_index, token_offset, answer bytes, hesitant), or RefError with its message."""
    n = len(text)
    cap = text.count(b"\n") + 1
    step = np.empty(cap, np.int32)
    tok = np.empty(cap, np.int64)
    hes = np.empty(cap, np.uint8)
    pid = C.create_string_buffer(max(n, 1))
    ans = C.create_string_buffer(max(n, 1))
    po = np.empty(cap + 1, np.uint64)
    ao = np.empty(cap + 1, np.uint64)
    f = ref().ref_parse_jsonl
    f.argtypes = [C.c_char_p, C.c_uint64, C.c_uint64, P, P, P, P, P, P, P]
    r = f(text, n, cap, _p(step), _p(tok), _p(hes), pid, _p(po), ans, _p(ao))
    if r < 0:
        raise RefError(_ref_err())
    praw, araw = pid.raw, ans.raw
    return [(praw[po[i]:po[i + 1]], int(step[i]), int(tok[i]), araw[ao[i]:ao[i + 1]], bool(hes[i]))
            for i in range(r)]


# ---------------------------------------------------------------- mixed-archetype step
def cot_meets(ids, hes, window, ths, nthreads=None):
    """CoT signal (runtime.cpp:293-299) as threshold bits per probe (cdxo_cot_meets), run
    over request chunks on host threads (the restatement is O(P^2) per request)."""
    from concurrent.futures import ThreadPoolExecutor
    R, P_ = ids.shape
    words = (P_ + 31) // 32
    out = np.zeros((R, words), np.uint32)
    if R == 0:
        return out
    ids = np.ascontiguousarray(ids, dtype=np.uint32)
    hes = np.ascontiguousarray(hes).view(np.uint64)
    arr, n = thresholds(ths)
    f = lib().cdxo_cot_meets
    f.argtypes = [P, P, C.c_uint64, C.c_uint32, C.c_int, P, C.c_uint32, P]
    nth = nthreads or hardware_threads()
    chunk = max(1, -(-R // (4 * nth)))

    def run(b):
        e = min(R, b + chunk)
        st = f(_p(ids[b:e]), _p(hes[b:e]), e - b, P_, window, C.cast(arr, P), n, _p(out[b:e]))
        if st:
            raise ValueError(f"oracle cot_meets status {st}")
    with ThreadPoolExecutor(nth) as ex:
        list(ex.map(run, range(0, R, chunk)))
    return out


def ref_cot_signal(ids, hes, window, groups=5, nthreads=1):
    """The reference's own consistency(records, latest, w).value_or(0.0) after every probe
    (runtime.cpp:293-299 through oracle/_ref), f64[R][P]."""
    R, P_ = ids.shape
    v, nv = _vocab_c(vocab(groups))
    ck = np.empty((R, P_), np.float64)
    r = ref().ref_cot_signal(_p(np.ascontiguousarray(ids)), _p(np.ascontiguousarray(hes)), C.c_uint64(R),
                             C.c_uint32(P_), v, C.c_uint32(nv), C.c_int(window), _p(ck), C.c_int(nthreads))
    if r < 0:
        raise RefError(_ref_err())
    return ck


def arch_policy(ths, kind, detect_at, cap, recheck_every=1, tokens_per_unit=64):
    a = ArchPolicy()
    for i, (sig, cut, d) in enumerate(ths):
        a.th[i].signal, a.th[i].cutoff, a.th[i].dir = sig, cut, d
    a.n_th = len(ths)
    a.alloc.kind, a.alloc.detect_at, a.alloc.resource_cap = kind, detect_at, cap
    a.alloc.recheck_every, a.alloc.tokens_per_unit = recheck_every, tokens_per_unit
    return a


def mixed_allocate(trace, arch, slot, knob, policies, nthreads=None):
    """The mixed step restated: per-archetype threshold bits from the restated signals (SC:
    cdxo_sc_certaindex rows; CoT: cdxo_cot_meets; MCTS/Rebase: cdxo reward certaindex with
    the FP64 values against each archetype's thresholds), then cdxo_mixed_decide.
    trace: dict sc_ids[n][P][S], cot_ids[n][P], cot_hes, cot_window, rw[n][T][W], rw_ids.
    policies: list of 4 ArchPolicy (by CDX_ARCH_*: SC, Rebase, MCTS, CoT)."""
    SC_, REB, MCT, COT = 0, 1, 2, 3

    def ths_of(a):
        pa = policies[a]
        return [(pa.th[i].signal, pa.th[i].cutoff, pa.th[i].dir) for i in range(pa.n_th)]

    sc = trace.get("sc_ids")
    cot = trace.get("cot_ids")
    rw = trace.get("rw")
    meets, words, ns = [], [], []
    if sc is not None and len(sc):
        _, _, m = sc_certaindex(sc, ths_of(SC_))
    else:
        m = np.zeros((0, 1), np.uint32)
    meets.append(np.ascontiguousarray(m))
    if cot is not None and len(cot):
        m = cot_meets(cot, trace["cot_hes"], trace["cot_window"], ths_of(COT), nthreads)
    else:
        m = np.zeros((0, 1), np.uint32)
    meets.append(m)
    if rw is not None and len(rw):
        G, T, W = rw.shape
        agg = np.zeros(G, np.uint8)
        a = np.asarray(arch)
        sl = np.asarray(slot)
        sel = (a == REB) | (a == MCT)
        agg[sl[sel]] = (a[sel] == REB).astype(np.uint8)
        R64, _, _, H64 = reward_certaindex(rw, trace.get("rw_ids"), agg, want_h64=True) if trace.get("rw_ids") \
            is not None else (*reward_certaindex(rw, None, agg), None)
        # combined_meets_thresholds on the FP64 signals, per archetype (an AND of compares)
        ok = np.ones((G, T), bool)
        for a_, rows in ((REB, agg == 1), (MCT, agg == 0)):
            for sig, cut, d in ths_of(a_):
                if sig == 0 and H64 is None or sig > 1:
                    raise ValueError("absent signal")
                v = (R64 if sig == 1 else H64)[rows]
                ok[rows] &= (v >= cut) if d == 0 else (v <= cut)
        m = np.zeros((G, (T + 31) // 32), np.uint32)
        for t in range(T):
            m[:, t // 32] |= ok[:, t].astype(np.uint32) << np.uint32(t % 32)
    else:
        m = np.zeros((0, 1), np.uint32)
    meets.append(m)
    for mm in meets:
        words.append(mm.shape[1] if mm.ndim == 2 else 1)
        ns.append(mm.shape[0])
    N = len(arch)
    dec = np.empty(N, np.uint8)
    grant = np.empty(N, np.int32)
    cap = np.empty(N, np.int32)
    off = np.empty(N, np.int64)
    tot = C.c_int64(0)
    mp = (P * 3)(*[_p(mm) for mm in meets])
    wa = (C.c_uint32 * 3)(*words)
    na = (C.c_uint64 * 3)(*ns)
    pa = (ArchPolicy * 4)(*policies)
    f = lib().cdxo_mixed_decide
    f.argtypes = [P, P, P, C.c_uint64, P, P, P, P, P, P, P, P, P]
    st = f(_p(np.ascontiguousarray(arch, dtype=np.uint8)), _p(np.ascontiguousarray(slot, dtype=np.uint32)),
           _p(np.ascontiguousarray(knob, dtype=np.int32)), N, C.cast(mp, P), C.cast(wa, P), C.cast(na, P),
           C.cast(pa, P), _p(dec), _p(grant), _p(cap), _p(off), C.byref(tot))
    if st:
        raise ValueError(f"oracle mixed_decide status {st}")
    return dict(decision=dec, grant=grant, cap=cap, offsets=off, total=tot.value, meets=meets)
