"""paper_2412_20993_b200 — B200-native Certaindex (Dynasor, arXiv 2412.20993) hot path.

The product is libcdx.so: hand-written sm_100a kernels behind the C-ABI declared in
include/cdx_c.h, with the reference's C++ API (include/cdx/*.hpp) layered above it.  This
Python module is plumbing for tests and the bench: it binds the C-ABI with ctypes and
moves torch CUDA tensors (device memory + the current stream) in and out.  It never
computes a certaindex itself and has no CPU fallback.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass
from typing import Optional, Sequence

from . import _abi
from ._abi import (AGG_MAX, AGG_MEAN, ARCH_COT, ARCH_MCTS, ARCH_REBASE, ARCH_SC, DIR_GE, DIR_LE,  # noqa: F401
                   EXIT_BUDGET, EXIT_CERTAIN, EXIT_CONTINUE, ORDER_FIFO, ORDER_SJF, POL_EVEN,
                   POL_K_STEP_THRESHOLD, POL_STATIC_THRESHOLD, SIG_ENTROPY, SIG_LOGPROB, SIG_MEAN_LEN,
                   SIG_REWARD)

__all__ = ["Context", "CdxError", "Threshold", "AllocPolicy", "ProbeConfig", "InterPolicy", "GenParams",
           "load_library"]


class CdxError(Exception):
    code = -1


class CdxInvalidArgument(CdxError, ValueError):
    """std::invalid_argument in the reference."""
    code = _abi.CDX_EINVAL


class CdxRuntimeError(CdxError, RuntimeError):
    """std::runtime_error in the reference."""
    code = _abi.CDX_ERUNTIME


class CdxOutOfRange(CdxError, IndexError):
    code = _abi.CDX_ERANGE


class CdxLogicError(CdxError):
    code = _abi.CDX_ELOGIC


class CdxCudaError(CdxError, RuntimeError):
    code = _abi.CDX_ECUDA


class CdxNcclError(CdxError, RuntimeError):
    code = _abi.CDX_ENCCL


_ERR = {c.code: c for c in (CdxInvalidArgument, CdxRuntimeError, CdxOutOfRange, CdxLogicError, CdxCudaError,
                             CdxNcclError)}


def load_library():
    return _abi.load()


@dataclass
class Threshold:
    """metrics.hpp:107-112 SignalThreshold."""
    signal: int = SIG_ENTROPY
    cutoff: float = 0.0
    dir: int = DIR_GE


@dataclass
class AllocPolicy:
    """SPEC.md:390-393 AllocationPolicy (batched subset)."""
    kind: int = POL_STATIC_THRESHOLD
    detect_at: int = 5
    resource_cap: int = 64
    recheck_every: int = 1
    tokens_per_unit: int = 64


@dataclass
class ProbeConfig:
    """probe.hpp:25-33 ProbeConfig."""
    interval_tokens: int = 64
    window: int = 3
    threshold: float = 0.9
    max_tokens: int = 1 << 20


@dataclass
class InterPolicy:
    """SPEC.md:394-397 InterSchedPolicy."""
    order: int = ORDER_SJF
    starvation_limit: float = 1.0
    prior_tokens: float = 128.0
    gang: bool = True


@dataclass
class GenParams:
    """Synthetic trace parameters (runtime.hpp:45-69 restated counter-based)."""
    seed: int = 20993
    groups: int = 5
    conv_lo: int = 1
    conv_hi: int = 64
    noise_level: float = 0.5
    residual_noise: float = 0.0
    solvable_fraction: float = 0.9
    hesitation_prob: float = 0.0
    reward_start_k: int = 5033165      # 0.3 * 2^24
    reward_final_k: int = 15099494     # 0.9 * 2^24
    reward_unsolvable_k: int = 4194304  # 0.25 * 2^24
    reward_jitter_k: int = 1677722     # 0.1 * 2^24

    def c(self) -> _abi.GenParams:
        g = _abi.GenParams()
        for k in ("seed", "groups", "conv_lo", "conv_hi", "noise_level", "residual_noise", "solvable_fraction",
                  "hesitation_prob", "reward_start_k", "reward_final_k", "reward_unsolvable_k", "reward_jitter_k"):
            setattr(g, k, getattr(self, k))
        return g


def vocab(groups: int) -> list:
    """Answer strings behind the synthetic ids (cdx_c.h cdx_gen_params)."""
    names = ["S"] + [f"D{i}" for i in range(1, groups)]
    return names + ["wait, " + n for n in names]


def c_thresholds(ths: Sequence[Threshold]):
    arr = (_abi.Threshold * max(1, len(ths)))()
    for i, t in enumerate(ths):
        arr[i].signal, arr[i].dir, arr[i].cutoff = t.signal, t.dir, float(t.cutoff)
    return arr, len(ths)


def c_policy(p: AllocPolicy) -> _abi.AllocPolicy:
    a = _abi.AllocPolicy()
    a.kind, a.detect_at, a.recheck_every = p.kind, p.detect_at, p.recheck_every
    a.resource_cap, a.tokens_per_unit = p.resource_cap, p.tokens_per_unit
    return a


def c_probe(c: ProbeConfig) -> _abi.ProbeCfg:
    a = _abi.ProbeCfg()
    a.interval_tokens, a.window, a.threshold, a.max_tokens = c.interval_tokens, c.window, float(c.threshold), \
        c.max_tokens
    return a


def c_inter(p: InterPolicy) -> _abi.InterPolicy:
    a = _abi.InterPolicy()
    a.gang, a.order, a.starvation_limit, a.prior_tokens = int(p.gang), p.order, float(p.starvation_limit), \
        float(p.prior_tokens)
    return a


def _ptr(t) -> Optional[int]:
    return None if t is None else t.data_ptr()


def nccl_unique_id() -> bytes:
    """128-byte NCCL unique id for Context.with_nccl (host only)."""
    buf = (C.c_uint8 * 128)()
    st = _abi.load().cdx_nccl_unique_id(C.cast(buf, C.c_void_p))
    if st != _abi.CDX_OK:
        raise CdxNcclError("cdx_nccl_unique_id failed (libnccl.so.2 not loadable)")
    return bytes(buf)


def shard_splitters(samples, counts, world: int, s: int):
    """Host-only planning step of the sharded gang order (cdx_shard_splitters): samples
    u64[world][s][3], counts u64[world] (numpy) -> splitters u64[world-1][3]."""
    import numpy as np
    smp = np.ascontiguousarray(samples, dtype=np.uint64).reshape(world, s, 3)
    cnt = np.ascontiguousarray(counts, dtype=np.uint64).reshape(world)
    out = np.zeros((max(world - 1, 1), 3), np.uint64)
    st = _abi.load().cdx_shard_splitters(smp.ctypes.data, cnt.ctypes.data, world, s, out.ctypes.data)
    if st != _abi.CDX_OK:
        raise CdxInvalidArgument("shard_splitters: bad arguments")
    return out[: world - 1]


class Context:
    """One cdx_ctx bound to a CUDA device; calls run on torch's current stream."""

    def __init__(self, device: int = 0, comm: Optional["_abi.Comm"] = None):
        import torch
        self.torch = torch
        self.lib = _abi.load()
        self.device = device
        h = C.c_void_p()
        self._comm = comm  # keeps the callbacks / id buffer alive as long as the context
        if comm is None:
            st = self.lib.cdx_ctx_create(device, C.byref(h))
        else:
            st = self.lib.cdx_ctx_create_comm(device, C.byref(comm), C.byref(h))
        if st != _abi.CDX_OK:
            raise _ERR.get(st, CdxError)(f"cdx_ctx_create(device={device}) failed with status {st}"
                                         " (a B200 / sm_100 device is required; there is no CPU fallback)")
        self.h = h
        self.dev = torch.device("cuda", device)
        self.rank = comm.rank if comm is not None else 0
        self.world = comm.world if comm is not None else 1

    @classmethod
    def with_nccl(cls, device: int, rank: int, world: int, nccl_id: bytes) -> "Context":
        """A context owning an NCCL communicator (collective: every rank calls it with the
        same 128-byte id from nccl_unique_id())."""
        buf = (C.c_uint8 * 128).from_buffer_copy(nccl_id)
        comm = _abi.Comm(rank=rank, world=world, nccl_id=C.cast(buf, C.c_void_p))
        comm._id_buf = buf
        return cls(device, comm)

    @classmethod
    def for_process_group(cls, device: int, group=None) -> "Context":
        """A context whose NCCL communicator spans torch.distributed's `group` (rank 0 makes
        the id, torch broadcasts it; torch's own communicator is not used by the kernels)."""
        import torch.distributed as dist
        rank, world = dist.get_rank(group), dist.get_world_size(group)
        obj = [nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=dist.get_global_rank(group, 0) if group is not None else 0, group=group)
        return cls.with_nccl(device, rank, world, obj[0])

    def close(self):
        if getattr(self, "h", None):
            self.lib.cdx_ctx_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # -- plumbing --
    def _bind_stream(self):
        s = self.torch.cuda.current_stream(self.dev).cuda_stream
        if s != self.__dict__.get("_bound_stream"):  # only this method sets the context's stream
            self.lib.cdx_ctx_set_stream(self.h, C.c_void_p(s))
            self._bound_stream = s

    def _check(self, st: int):
        if st != _abi.CDX_OK:
            msg = self.lib.cdx_last_error(self.h).decode()
            raise _ERR.get(st, CdxError)(msg)

    def sync(self):
        self._check(self.lib.cdx_sync(self.h))

    @property
    def launches(self) -> int:
        return int(self.lib.cdx_launch_count(self.h))

    def empty(self, shape, dtype):
        return self.torch.empty(shape, dtype=dtype, device=self.dev)

    # -- synthetic traces --
    def gen_sc(self, g: GenParams, R: int, P: int, S: int, r0: int = 0, out=None):
        t = self.torch
        ids = out if out is not None else self.empty((R, P, S), t.int32)
        self._bind_stream()
        gp = g.c()
        self._check(self.lib.cdx_gen_sc(self.h, C.byref(gp), r0, R, P, S, _ptr(ids)))
        return ids

    def gen_cot(self, g: GenParams, R: int, P: int, r0: int = 0):
        t = self.torch
        ids = self.empty((R, P), t.int32)
        hes = self.empty((R, (P + 63) // 64), t.int64)
        self._bind_stream()
        gp = g.c()
        self._check(self.lib.cdx_gen_cot(self.h, C.byref(gp), r0, R, P, _ptr(ids), _ptr(hes)))
        return ids, hes

    def gen_reward(self, g: GenParams, G: int, T: int, W: int, g0: int = 0, with_ids: bool = True):
        t = self.torch
        rw = self.empty((G, T, W), t.float32)
        ids = self.empty((G, T, W), t.int32) if with_ids else None
        self._bind_stream()
        gp = g.c()
        self._check(self.lib.cdx_gen_reward(self.h, C.byref(gp), g0, G, T, W, _ptr(rw), _ptr(ids)))
        return rw, ids

    # -- K2 --
    def sc_certaindex(self, ids, thresholds: Sequence[Threshold] = (), want_hcert: bool = True,
                      hcert=None, meets=None):
        t = self.torch
        R, P, S = ids.shape
        if want_hcert and hcert is None:
            hcert = self.empty((R, P), t.float32)
        if meets is None:
            meets = self.empty((R, (P + 31) // 32), t.int32)
        arr, n = c_thresholds(thresholds)
        self._bind_stream()
        self._check(self.lib.cdx_sc_certaindex(self.h, _ptr(ids), R, P, S, arr, n,
                                               _ptr(hcert) if want_hcert else None, _ptr(meets)))
        return hcert, meets

    def sc_certaindex_ex(self, ids, thresholds: Sequence[Threshold] = (), want_hcert: bool = True,
                         want_majority: bool = True):
        """K2 with the majority-fraction certaindex (largest cluster / S, SIG_MAJORITY)."""
        t = self.torch
        R, P, S = ids.shape
        hcert = self.empty((R, P), t.float32) if want_hcert else None
        maj = self.empty((R, P), t.float32) if want_majority else None
        meets = self.empty((R, (P + 31) // 32), t.int32)
        arr, n = c_thresholds(thresholds)
        self._bind_stream()
        self._check(self.lib.cdx_sc_certaindex_ex(self.h, _ptr(ids), R, P, S, arr, n, _ptr(hcert), _ptr(maj),
                                                  _ptr(meets)))
        return hcert, maj, meets

    def cluster_rows(self, ids2d):
        t = self.torch
        rows, S = ids2d.shape
        ncl = self.empty((rows,), t.int32)
        leader = self.torch.zeros((rows, S), dtype=t.int32, device=self.dev)
        size = self.torch.zeros((rows, S), dtype=t.int32, device=self.dev)
        self._bind_stream()
        self._check(self.lib.cdx_cluster_rows(self.h, _ptr(ids2d), rows, S, _ptr(ncl), _ptr(leader), _ptr(size)))
        return ncl, leader, size

    def entropy_from_sizes(self, sizes, m, max_n: int, totals=None):
        t = self.torch
        rows, max_m = sizes.shape
        H = self.empty((rows,), t.float64)
        Hc = self.empty((rows,), t.float64)
        self._bind_stream()
        self._check(self.lib.cdx_entropy_from_sizes(self.h, _ptr(sizes), _ptr(m), _ptr(totals), rows, max_m, max_n, _ptr(H),
                                                    _ptr(Hc)))
        return H, Hc

    # -- K5 --
    def allocate_scan(self, meets, R: int, P: int, policy: AllocPolicy, base_offset: int = 0, kept_base: int = 0,
                      out=None):
        t = self.torch
        o = out or {}
        # defaults allocated only when missing (a dict.get default would be evaluated, and a
        # torch.zeros default launched, on every call)
        exit_knob = o["exit_knob"] if "exit_knob" in o else self.empty((R,), t.int32)
        reason = o["reason"] if "reason" in o else self.empty((R,), t.uint8)
        granted = o["granted"] if "granted" in o else self.empty((R,), t.int32)
        offsets = o["offsets"] if "offsets" in o else self.empty((R,), t.int64)
        kept = o["kept"] if "kept" in o else self.empty((max(R, 1),), t.int32)
        scal = o["scalars"] if "scalars" in o else self.empty((3,), t.int64)  # written by the kernel
        pol = c_policy(policy)
        self._bind_stream()
        self._check(self.lib.cdx_allocate_scan(self.h, _ptr(meets), R, P, C.byref(pol), base_offset, kept_base,
                                               _ptr(exit_knob), _ptr(reason), _ptr(granted), _ptr(offsets),
                                               _ptr(kept), scal.data_ptr(), scal.data_ptr() + 8,
                                               scal.data_ptr() + 16))
        return dict(exit_knob=exit_knob, reason=reason, granted=granted, offsets=offsets, kept=kept,
                    scalars=scal)

    def sc_decide(self, ids, thresholds: Sequence[Threshold], policy: AllocPolicy, hcert=None, meets=None,
                  base_offset: int = 0, kept_base: int = 0, out=None):
        """K2 + K5 in one call (cdx_sc_decide: one launch on the fast path).  Returns
        (hcert or None, meets, the allocate_scan output dict)."""
        t = self.torch
        R, P, S = ids.shape
        if meets is None:
            meets = self.empty((R, (P + 31) // 32), t.int32)
        o = out or {}
        exit_knob = o["exit_knob"] if "exit_knob" in o else self.empty((R,), t.int32)
        reason = o["reason"] if "reason" in o else self.empty((R,), t.uint8)
        granted = o["granted"] if "granted" in o else self.empty((R,), t.int32)
        offsets = o["offsets"] if "offsets" in o else self.empty((R,), t.int64)
        kept = o["kept"] if "kept" in o else self.empty((max(R, 1),), t.int32)
        scal = o["scalars"] if "scalars" in o else self.empty((3,), t.int64)
        arr, n = c_thresholds(thresholds)
        pol = c_policy(policy)
        self._bind_stream()
        self._check(self.lib.cdx_sc_decide(self.h, _ptr(ids), R, P, S, arr, n, _ptr(hcert), _ptr(meets),
                                           C.byref(pol), base_offset, kept_base, _ptr(exit_knob), _ptr(reason),
                                           _ptr(granted), _ptr(offsets), _ptr(kept), scal.data_ptr(),
                                           scal.data_ptr() + 8, scal.data_ptr() + 16))
        return hcert, meets, dict(exit_knob=exit_knob, reason=reason, granted=granted, offsets=offsets, kept=kept,
                                  scalars=scal)

    # -- mixed-archetype step (update_certaindex dispatch + allocate at the current knob) --
    def cot_meets(self, ids, hes, window: int, thresholds: Sequence[Threshold]):
        t = self.torch
        R, P = ids.shape
        meets = self.empty((R, (P + 31) // 32), t.int32)
        arr, n = c_thresholds(thresholds)
        self._bind_stream()
        self._check(self.lib.cdx_cot_meets(self.h, _ptr(ids), _ptr(hes), R, P, window, arr, n, _ptr(meets)))
        return meets

    def mixed_allocate(self, trace: dict, archetype, slot, knob, policies, out=None):
        """trace: sc_ids [n][P][S], cot_ids [n][P] + cot_hes + cot_window, rw [n][T][W] (+ rw_ids);
        archetype u8[N], slot i32[N], knob i32[N]; policies: 4 (thresholds, AllocPolicy) pairs
        indexed by CDX_ARCH_* (SC, Rebase, MCTS, CoT).  Returns decision / grant / cap /
        offsets tensors and the device total budget."""
        t = self.torch
        N = archetype.shape[0]
        tr = _abi.MixedTrace()
        sc, cot, rw = trace.get("sc_ids"), trace.get("cot_ids"), trace.get("rw")
        if sc is not None:
            tr.sc_ids, (tr.sc_n, tr.sc_P, tr.sc_S) = sc.data_ptr(), sc.shape
        if cot is not None:
            tr.cot_ids, tr.cot_hes = cot.data_ptr(), trace["cot_hes"].data_ptr()
            tr.cot_n, tr.cot_P = cot.shape
            tr.cot_window = int(trace["cot_window"])
        if rw is not None:
            tr.rw_rewards, (tr.rw_n, tr.rw_T, tr.rw_W) = rw.data_ptr(), rw.shape
            tr.rw_ids = _ptr(trace.get("rw_ids"))
        pols = (_abi.ArchPolicy * 4)()
        for a, (ths, pol) in enumerate(policies):
            for i, th in enumerate(ths):
                pols[a].th[i].signal, pols[a].th[i].dir, pols[a].th[i].cutoff = th.signal, th.dir, float(th.cutoff)
            pols[a].n_th = len(ths)
            pols[a].alloc = c_policy(pol)
        o = out or {}
        dec = o["decision"] if "decision" in o else self.empty((max(N, 1),), t.uint8)
        grant = o["grant"] if "grant" in o else self.empty((max(N, 1),), t.int32)
        cap = o["cap"] if "cap" in o else self.empty((max(N, 1),), t.int32)
        offs = o["offsets"] if "offsets" in o else self.empty((max(N, 1),), t.int64)
        total = o["total"] if "total" in o else self.empty((1,), t.int64)
        self._bind_stream()
        self._check(self.lib.cdx_mixed_allocate(self.h, C.byref(tr), _ptr(archetype), _ptr(slot), _ptr(knob), N,
                                                pols, _ptr(dec), _ptr(grant), _ptr(cap), _ptr(offs), _ptr(total)))
        return dict(decision=dec[:N], grant=grant[:N], cap=cap[:N], offsets=offs[:N], total=total)

    # -- end-to-end entries from HOST buffers (chunked H2D / kernels / D2H, double buffered) --
    @staticmethod
    def _host(a):
        """(pointer, keep-alive) of a host array: numpy array or CPU torch tensor."""
        if a is None:
            return None, None
        if hasattr(a, "data_ptr"):
            assert not a.is_cuda, "host entry points take host buffers"
            return a.data_ptr(), a
        import numpy as np
        a = np.ascontiguousarray(a)
        return a.ctypes.data, a

    def sc_decide_host(self, ids, thresholds, policy: AllocPolicy, want_hcert: bool = False):
        import numpy as np
        R, P, S = ids.shape
        out = dict(exit_knob=np.empty(R, np.int32), reason=np.empty(R, np.uint8), offsets=np.empty(R, np.int64),
                   hcert=np.empty((R, P), np.float32) if want_hcert else None)
        p_ids, keep = self._host(ids)
        arr, n = c_thresholds(thresholds)
        pol = c_policy(policy)
        saved = C.c_int64(0)
        self._check(self.lib.cdx_sc_decide_host(self.h, p_ids, R, P, S, arr, n, C.byref(pol),
                                                out["exit_knob"].ctypes.data, out["reason"].ctypes.data,
                                                out["offsets"].ctypes.data,
                                                out["hcert"].ctypes.data if want_hcert else None, C.byref(saved)))
        out["tokens_saved"] = saved.value
        del keep
        return out

    def cot_decide_host(self, ids, hes, cfg: ProbeConfig, offsets=None, out=None):
        import numpy as np
        R, P = ids.shape
        o = out or {}
        res = {k: o[k] if k in o else np.empty(R, dt) for k, dt in (("exit_step", np.int32), ("reason", np.uint8),
                                                                     ("final_id", np.uint32), ("low_conf", np.uint8))}
        p_ids, k1 = self._host(ids)
        p_hes, k2 = self._host(hes)
        p_off, k3 = self._host(offsets)
        c = c_probe(cfg)
        ptr = lambda a: a.ctypes.data if hasattr(a, "ctypes") else a.data_ptr()  # noqa: E731
        self._check(self.lib.cdx_cot_decide_host(self.h, p_ids, p_hes, p_off, R, P, C.byref(c),
                                                 *[ptr(res[k]) for k in ("exit_step", "reason", "final_id",
                                                                         "low_conf")]))
        del k1, k2, k3
        return res

    def reward_decide_host(self, rewards, ids, agg, th_mean, th_max, policy: AllocPolicy, want_R: bool = False,
                           out=None):
        import numpy as np
        G, T, W = rewards.shape
        o = out or {}
        res = {k: o[k] if k in o else np.empty(G, dt) for k, dt in (("exit_knob", np.int32), ("reason", np.uint8),
                                                                     ("offsets", np.int64))}
        res["R"] = o.get("R") if "R" in o else (np.empty((G, T), np.float32) if want_R else None)
        p_rw, k1 = self._host(rewards)
        p_ids, k2 = self._host(ids)
        p_agg, k3 = self._host(agg)
        a1, n1 = c_thresholds(th_mean)
        a2, n2 = c_thresholds(th_max)
        pol = c_policy(policy)
        saved = C.c_int64(0)
        ptr = lambda a: None if a is None else (a.ctypes.data if hasattr(a, "ctypes") else a.data_ptr())  # noqa
        self._check(self.lib.cdx_reward_decide_host(self.h, p_rw, p_ids, p_agg, G, T, W, a1, n1, a2, n2, C.byref(pol),
                                                    ptr(res["exit_knob"]), ptr(res["reason"]), ptr(res["offsets"]),
                                                    ptr(res["R"]), C.byref(saved)))
        res["tokens_saved"] = saved.value
        del k1, k2, k3
        return res

    # -- K3 --
    def cot_exit(self, ids, hes, cfg: ProbeConfig, offsets=None, want_ck: bool = False, out=None):
        t = self.torch
        R, P = ids.shape
        o = out or {}
        ex = o["exit_step"] if "exit_step" in o else self.empty((R,), t.int32)
        reason = o["reason"] if "reason" in o else self.empty((R,), t.uint8)
        fid = o["final_id"] if "final_id" in o else self.empty((R,), t.int32)
        low = o["low_conf"] if "low_conf" in o else self.empty((R,), t.uint8)
        ck = self.empty((R, P), t.float32) if want_ck else None
        c = c_probe(cfg)
        self._bind_stream()
        self._check(self.lib.cdx_cot_exit(self.h, _ptr(ids), _ptr(hes), _ptr(offsets), R, P, C.byref(c), _ptr(ex),
                                          _ptr(reason), _ptr(fid), _ptr(low), _ptr(ck)))
        return dict(exit_step=ex, reason=reason, final_id=fid, low_conf=low, ck=ck)

    # -- K4 --
    def reward_certaindex(self, rewards, ids, agg, th_mean: Sequence[Threshold] = (),
                          th_max: Sequence[Threshold] = (), want_H: bool = True, want_meets: bool = True):
        t = self.torch
        G, T, W = rewards.shape
        R = self.empty((G, T), t.float32)
        H = self.empty((G, T), t.float32) if (want_H and ids is not None) else None
        meets = self.empty((G, (T + 31) // 32), t.int32) if want_meets else None
        a1, n1 = c_thresholds(th_mean)
        a2, n2 = c_thresholds(th_max)
        self._bind_stream()
        f = self.lib.cdx_reward_certaindex_f64 if rewards.dtype == t.float64 else self.lib.cdx_reward_certaindex
        self._check(f(self.h, _ptr(rewards), _ptr(ids), _ptr(agg), G, T, W, a1, n1, a2, n2, _ptr(R), _ptr(H),
                      _ptr(meets)))
        return R, H, meets

    def reward_sets(self, values, row_off, agg):
        t = self.torch
        rows = agg.shape[0]
        out = self.empty((rows,), t.float64)
        self._bind_stream()
        self._check(self.lib.cdx_reward_sets(self.h, _ptr(values), _ptr(row_off), _ptr(agg), rows, _ptr(out)))
        return out

    # -- K1 --
    def canon_intern(self, arena, offsets, markers: Sequence[str] = ("wait", "hmm"), want_hes: bool = True):
        t = self.torch
        n = offsets.shape[0] - 1
        ids = self.empty((max(n, 1),), t.int32)
        hes = self.empty((max(n, 1),), t.uint8) if want_hes else None
        first = self.empty((max(n, 1),), t.int64)
        mk = (C.c_char_p * max(1, len(markers)))(*[m.encode() for m in markers])
        nu = C.c_uint64(0)
        self._bind_stream()
        self._check(self.lib.cdx_canon_intern(self.h, _ptr(arena), _ptr(offsets), n, mk, len(markers), _ptr(ids),
                                              _ptr(hes), _ptr(first), C.byref(nu)))
        return ids[:n], (hes[:n] if hes is not None else None), first[:nu.value], nu.value

    # -- K6 --
    _SOA_FIELDS = ("arrival", "last_service", "iter_tok_sum", "iter_count", "knob", "cap", "terminated")

    def _prog_soa(self, soa: dict, id_base: int):
        """cdx_prog_soa for these tensors; the ctypes struct is reused while the same storage
        is passed again (a scheduling loop calls the order on the same state every round)."""
        pid = soa.get("program_id")
        key = tuple(soa[k].data_ptr() for k in self._SOA_FIELDS) + (pid.data_ptr() if pid is not None else 0,
                                                                     id_base)
        cache = self.__dict__.setdefault("_soa_cache", {})
        s = cache.get(key)
        if s is None:
            s = _abi.ProgSoA()
            for k, p in zip(self._SOA_FIELDS, key):
                setattr(s, k, p)
            if pid is not None:  # explicit ids (u32 stored in an int32 tensor)
                s.program_id = key[7]
            s.id_base = id_base
            if len(cache) > 64:
                cache.clear()
            cache[key] = s
        return s

    def gang_priority(self, soa: dict, policy: InterPolicy, now: float, id_base: int = 0, want_keys: bool = False,
                      want_escalated: bool = False, out=None):
        """Program order of the live programs (cdx_gang_priority).  `out` (int32[>= N], device)
        receives the order instead of a fresh tensor."""
        t = self.torch
        N = soa["arrival"].shape[0]
        s = self._prog_soa(soa, id_base)
        order = out if out is not None else self.empty((max(N, 1),), t.int32)
        esc = self.empty((max(N, 1),), t.uint8) if want_escalated else None
        keys = self.empty((max(N, 1), 3), t.int64) if want_keys else None
        n_out = C.c_uint64(0)
        pol = c_inter(policy)
        self._bind_stream()
        self._check(self.lib.cdx_gang_priority(self.h, C.byref(s), N, C.byref(pol), float(now), order.data_ptr(),
                                               C.byref(n_out), _ptr(esc), _ptr(keys)))
        n = n_out.value
        return order[:n], (esc[:N] if esc is not None else None), (keys[:n] if keys is not None else None)

    def gang_merge(self, keys, run_len, stride: int, total=None):
        """keys i64[runs*stride][3] (padded runs), run_len i64[runs] on the device."""
        t = self.torch
        runs = run_len.shape[0]
        out = self.empty((max(runs * stride, 1),), t.int32)
        self._bind_stream()
        self._check(self.lib.cdx_gang_merge(self.h, _ptr(keys), _ptr(run_len), runs, stride, _ptr(out),
                                            _ptr(total)))
        return out

    # -- multi-GPU: the context's communicator (shard.cu) --
    def allocate_scan_sharded(self, meets, R: int, P: int, policy: AllocPolicy, out=None):
        """K5 over this rank's requests with global offsets / kept indices / totals."""
        t = self.torch
        o = out or {}
        exit_knob = o["exit_knob"] if "exit_knob" in o else self.empty((max(R, 1),), t.int32)
        reason = o["reason"] if "reason" in o else self.empty((max(R, 1),), t.uint8)
        granted = o["granted"] if "granted" in o else self.empty((max(R, 1),), t.int32)
        offsets = o["offsets"] if "offsets" in o else self.empty((max(R, 1),), t.int64)
        kept = o["kept"] if "kept" in o else self.empty((max(R, 1),), t.int32)
        scal = o["scalars"] if "scalars" in o else self.empty((3,), t.int64)
        info = o["shard_info"] if "shard_info" in o else self.empty((self.world, 4), t.int64)
        pol = c_policy(policy)
        self._bind_stream()
        self._check(self.lib.cdx_allocate_scan_sharded(self.h, _ptr(meets), R, P, C.byref(pol), _ptr(exit_knob),
                                                       _ptr(reason), _ptr(granted), _ptr(offsets), _ptr(kept),
                                                       scal.data_ptr(), scal.data_ptr() + 8, scal.data_ptr() + 16,
                                                       _ptr(info)))
        return dict(exit_knob=exit_knob[:R], reason=reason[:R], granted=granted[:R], offsets=offsets[:R],
                    kept=kept, scalars=scal, shard_info=info)

    def gang_priority_sharded(self, soa: dict, policy: InterPolicy, now: float, id_base: int = 0,
                              capacity: Optional[int] = None, out=None):
        """The global gang order on every rank (distributed sample sort); `capacity` bounds
        the global live count (default: world x this rank's programs)."""
        t = self.torch
        N = soa["arrival"].shape[0]
        s = _abi.ProgSoA()
        for k in ("arrival", "last_service", "iter_tok_sum", "iter_count", "knob", "cap", "terminated"):
            setattr(s, k, soa[k].data_ptr())
        if soa.get("program_id") is not None:
            s.program_id = soa["program_id"].data_ptr()
        s.id_base = id_base
        cap = capacity if capacity is not None else self.world * max(N, 1)
        order = out if out is not None else self.empty((max(cap, 1),), t.int32)
        n_out = C.c_uint64(0)
        pol = c_inter(policy)
        self._bind_stream()
        self._check(self.lib.cdx_gang_priority_sharded(self.h, C.byref(s), N, C.byref(pol), float(now), _ptr(order),
                                                       C.byref(n_out)))
        return order[: n_out.value]

    def shard_samples(self, keys, s: int):
        out = self.empty((s, 3), self.torch.int64)
        self._bind_stream()
        self._check(self.lib.cdx_shard_samples(self.h, _ptr(keys), keys.shape[0], s, _ptr(out)))
        return out

    def shard_bounds(self, keys, splitters, world: int):
        out = self.empty((world + 1,), self.torch.int64)
        self._bind_stream()
        self._check(self.lib.cdx_shard_bounds(self.h, _ptr(keys), keys.shape[0], _ptr(splitters), world, _ptr(out)))
        return out

    def gang_merge_runs(self, keys, run_off):
        """keys i64[n][3] holding sorted runs at run_off (device i64[runs+1]) -> program ids."""
        n = keys.shape[0]
        out = self.empty((max(n, 1),), self.torch.int32)
        self._bind_stream()
        self._check(self.lib.cdx_gang_merge_runs(self.h, _ptr(keys), _ptr(run_off), run_off.shape[0] - 1, _ptr(out)))
        return out[:n]

    def offsets_rebase(self, offsets, shard_totals, rank: int):
        self._bind_stream()
        self._check(self.lib.cdx_offsets_rebase(self.h, _ptr(offsets), offsets.shape[0], _ptr(shard_totals), rank))

    # -- aggregation (runtime.cpp:318-403) --
    def sc_aggregate(self, ids, exit_knob):
        t = self.torch
        R, P, S = ids.shape
        ans = self.empty((max(R, 1),), t.int32)
        self._bind_stream()
        self._check(self.lib.cdx_sc_aggregate(self.h, _ptr(ids), R, P, S, _ptr(exit_knob), _ptr(ans)))
        return ans[:R]

    def reward_aggregate(self, rewards, ids, agg, exit_step):
        """f32 or f64 rewards; answer CDX_NO_ANSWER (0xffffffff) where the reference's vote
        has no winner.  Returns (answer, inexact) — inexact stays 0 (ABI v2 counter)."""
        t = self.torch
        G, T, W = rewards.shape
        ans = self.empty((max(G, 1),), t.int32)
        inexact = self.torch.zeros((1,), dtype=t.int64, device=self.dev)
        self._bind_stream()
        if rewards.dtype == t.float64:
            self._check(self.lib.cdx_reward_aggregate_f64(self.h, _ptr(rewards), _ptr(ids), _ptr(agg), G, T, W,
                                                          _ptr(exit_step), _ptr(ans)))
        else:
            self._check(self.lib.cdx_reward_aggregate(self.h, _ptr(rewards), _ptr(ids), _ptr(agg), G, T, W,
                                                      _ptr(exit_step), _ptr(ans), _ptr(inexact)))
        return ans[:G], inexact

    def libm_exp(self, x):
        """std::exp with the host libm's bits, on the device (f64 tensor in, f64 out)."""
        y = self.torch.empty_like(x)
        self._bind_stream()
        self._check(self.lib.cdx_libm_exp(self.h, _ptr(x), x.numel(), _ptr(y)))
        return y

    # -- epsilon-accuracy stop test (probe.cpp:104-120, theory.cpp:117-146) --
    def cot_eps_stop(self, ids, hes, k: int, epsilon: float, want_state: bool = False):
        t = self.torch
        R, P = ids.shape
        step = self.empty((max(R, 1),), t.int32)
        state = self.empty((R, P), t.uint8) if want_state else None
        self._bind_stream()
        self._check(self.lib.cdx_cot_eps_stop(self.h, _ptr(ids), _ptr(hes), R, P, k, float(epsilon), _ptr(step),
                                              _ptr(state)))
        return step[:R], state

    # -- JSONL trace ingestion (probe.cpp:126-165) --
    def jsonl_parse(self, text_dev, cap_records: int):
        """text_dev: uint8 device tensor with the JSON-lines bytes.  Returns a dict of device
        tensors (records in line order) and the record / program counts."""
        t = self.torch
        nbytes = text_dev.numel()
        cap = max(cap_records, 1)
        out = dict(program=self.empty((cap,), t.int32), step_index=self.empty((cap,), t.int32),
                   token_offset=self.empty((cap,), t.int64), hesitant=self.empty((cap,), t.uint8),
                   answer_off=self.empty((cap + 1,), t.int64), answer_arena=self.empty((max(nbytes, 1),), t.uint8),
                   program_off=self.empty((cap + 1,), t.int64), program_arena=self.empty((max(nbytes, 1),), t.uint8),
                   program_first=self.empty((cap,), t.int64))
        nr, npg = C.c_uint64(0), C.c_uint64(0)
        self._bind_stream()
        self._check(self.lib.cdx_jsonl_parse(self.h, _ptr(text_dev), nbytes, cap_records, *[_ptr(out[k]) for k in (
            "program", "step_index", "token_offset", "hesitant", "answer_off", "answer_arena", "program_off",
            "program_arena", "program_first")], C.byref(nr), C.byref(npg)))
        out["n_records"], out["n_programs"] = nr.value, npg.value
        return out

    # -- CUDA graphs of call sequences (launch-bound small batches) --
    def graph_capture(self, fn):
        """Capture fn() (a sequence of Context calls) on a side stream into a replayable
        graph; returns a callable that replays it on torch's current stream."""
        t = self.torch
        side = t.cuda.Stream(device=self.dev)
        side.wait_stream(t.cuda.current_stream(self.dev))
        with t.cuda.stream(side):
            fn()  # warm: allocations and table builds happen outside the capture
            self.sync()
            self._bind_stream()
            self._check(self.lib.cdx_graph_begin(self.h))
            try:
                fn()
            finally:
                g = C.c_void_p()
                st = self.lib.cdx_graph_end(self.h, C.byref(g))
            self._check(st)
        t.cuda.current_stream(self.dev).wait_stream(side)
        ctx = self

        class _Graph:
            def __call__(self):
                ctx._bind_stream()
                ctx._check(ctx.lib.cdx_graph_launch(ctx.h, g))

            def __del__(self):
                ctx.lib.cdx_graph_destroy(g)

        return _Graph()
