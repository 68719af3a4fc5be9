"""ctypes mirror of include/cdx_c.h (the C-ABI of libcdx.so).

Plumbing only: the compute lives in the sm_100a kernels behind the C-ABI.  Loading fails
loudly when the library has not been built; every compute call fails loudly (CDX_ECUDA)
when no B200 is present — there is no CPU fallback anywhere in the product path.
"""
from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "lib", "libcdx.so")

CDX_OK, CDX_EINVAL, CDX_ERUNTIME, CDX_ERANGE, CDX_ELOGIC, CDX_ECUDA, CDX_ENCCL = range(7)
SIG_ENTROPY, SIG_REWARD, SIG_MEAN_LEN, SIG_LOGPROB = range(4)
DIR_GE, DIR_LE = 0, 1
AGG_MEAN, AGG_MAX = 0, 1
EXIT_CONTINUE, EXIT_CERTAIN, EXIT_BUDGET = 0, 1, 2
ARCH_SC, ARCH_REBASE, ARCH_MCTS, ARCH_COT = range(4)
POL_EVEN, POL_LENGTH_PROXY, POL_STATIC_THRESHOLD, POL_INITIAL_CURVE_FIT, POL_K_STEP_THRESHOLD, \
    POL_DYNAMIC_CURVE_FIT = range(6)
ORDER_FIFO, ORDER_SJF, ORDER_LPM = range(3)


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
    _fields_ = [("arrival", C.c_void_p), ("last_service", C.c_void_p), ("iter_tok_sum", C.c_void_p),
                ("iter_count", C.c_void_p), ("knob", C.c_void_p), ("cap", C.c_void_p),
                ("terminated", C.c_void_p), ("program_id", C.c_void_p), ("id_base", C.c_uint32),
                ("_pad", C.c_uint32)]


class GenParams(C.Structure):
    _fields_ = [("seed", C.c_uint64), ("groups", C.c_uint32), ("conv_lo", C.c_uint32), ("conv_hi", C.c_uint32),
                ("_pad", C.c_uint32), ("noise_level", C.c_double), ("residual_noise", C.c_double),
                ("solvable_fraction", C.c_double), ("hesitation_prob", C.c_double),
                ("reward_start_k", C.c_uint32), ("reward_final_k", C.c_uint32),
                ("reward_unsolvable_k", C.c_uint32), ("reward_jitter_k", C.c_uint32)]


P = C.c_void_p
U64, U32, I64, I32 = C.c_uint64, C.c_uint32, C.c_int64, C.c_int32


class MixedTrace(C.Structure):
    _fields_ = [("sc_ids", P), ("sc_n", U64), ("sc_P", U32), ("sc_S", U32),
                ("cot_ids", P), ("cot_hes", P), ("cot_n", U64), ("cot_P", U32), ("cot_window", U32),
                ("rw_rewards", P), ("rw_ids", P), ("rw_n", U64), ("rw_T", U32), ("rw_W", U32)]


class ArchPolicy(C.Structure):
    _fields_ = [("th", Threshold * 4), ("n_th", U32), ("_pad", U32), ("alloc", AllocPolicy)]

ALLGATHER_FN = C.CFUNCTYPE(C.c_int, P, P, P, U64, P)
ALLTOALLV_FN = C.CFUNCTYPE(C.c_int, P, P, C.POINTER(U64), C.POINTER(U64), P, C.POINTER(U64), C.POINTER(U64), P)


class Comm(C.Structure):
    _fields_ = [("rank", U32), ("world", U32), ("nccl_id", P), ("user", P), ("allgather", ALLGATHER_FN),
                ("alltoallv", ALLTOALLV_FN)]


SIG_MAJORITY = 4

# name -> (restype, argtypes); this table is also the export list tests check against cdx_c.h
SIGNATURES = {
    "cdx_abi_version": (C.c_int, []),
    "cdx_ctx_create": (C.c_int, [C.c_int, C.POINTER(P)]),
    "cdx_ctx_destroy": (C.c_int, [P]),
    "cdx_ctx_set_stream": (C.c_int, [P, P]),
    "cdx_ctx_use_own_stream": (C.c_int, [P]),
    "cdx_ctx_stream": (P, [P]),
    "cdx_sync": (C.c_int, [P]),
    "cdx_last_error": (C.c_char_p, [P]),
    "cdx_launch_count": (U64, [P]),
    "cdx_graph_begin": (C.c_int, [P]),
    "cdx_graph_end": (C.c_int, [P, C.POINTER(P)]),
    "cdx_graph_launch": (C.c_int, [P, P]),
    "cdx_graph_destroy": (C.c_int, [P]),
    "cdx_gen_sc": (C.c_int, [P, C.POINTER(GenParams), U64, U64, U32, U32, P]),
    "cdx_gen_cot": (C.c_int, [P, C.POINTER(GenParams), U64, U64, U32, P, P]),
    "cdx_gen_reward": (C.c_int, [P, C.POINTER(GenParams), U64, U64, U32, U32, P, P]),
    "cdx_sc_certaindex": (C.c_int, [P, P, U64, U32, U32, C.POINTER(Threshold), U32, P, P]),
    "cdx_sc_certaindex_ex": (C.c_int, [P, P, U64, U32, U32, C.POINTER(Threshold), U32, P, P, P]),
    "cdx_cluster_rows": (C.c_int, [P, P, U64, U32, P, P, P]),
    "cdx_entropy_from_sizes": (C.c_int, [P, P, P, P, U64, U32, U32, P, P]),
    "cdx_probe_consistency": (C.c_int, [P, P, P, P, P, P, U64, I32, P, P]),
    "cdx_probe_should_exit": (C.c_int, [P, P, P, P, P, P, U64, C.POINTER(ProbeCfg), P]),
    "cdx_probe_final_answer": (C.c_int, [P, P, P, P, P, P, U64, P, P]),
    "cdx_meets_thresholds_rows": (C.c_int, [P, P, P, U64, C.POINTER(Threshold), U32, P]),
    "cdx_id_histogram": (C.c_int, [P, P, U64, U32, P]),
    "cdx_entropy_one": (C.c_int, [P, P, U32, U32, P, P]),
    "cdx_cluster_host": (C.c_int, [P, P, P, U32, P, U32, P, P, P, P, P]),
    "cdx_consistency_host": (C.c_int, [P, P, P, U32, P, P, C.c_int32, C.c_int32, P, P]),
    "cdx_should_exit_host": (C.c_int, [P, P, P, U32, P, P, P, P, P]),
    "cdx_final_answer_host": (C.c_int, [P, P, P, U32, C.c_int32, C.c_uint8, P, P]),
    "cdx_entropy_host": (C.c_int, [P, P, U32, C.c_int32, P, P]),
    "cdx_reward_host": (C.c_int, [P, P, U64, C.c_uint8, P]),
    "cdx_meets_host": (C.c_int, [P, P, C.c_uint8, P, U32, P]),
    "cdx_entropy_sizes_host": (C.c_int, [P, P, U32, C.c_int32, P, P]),
    "cdx_iteration_tokens_rows": (C.c_int, [P, P, P, U64, C.c_double, P]),
    "cdx_alloc": (C.c_int, [P, U64, C.POINTER(P)]),
    "cdx_free": (C.c_int, [P, P]),
    "cdx_memcpy": (C.c_int, [P, P, P, U64]),
    "cdx_memset": (C.c_int, [P, P, C.c_int, U64]),
    "cdx_allocate_scan": (C.c_int, [P, P, U64, U32, C.POINTER(AllocPolicy), I64, U32, P, P, P, P, P, P, P, P]),
    "cdx_sc_decide": (C.c_int, [P, P, U64, U32, U32, C.POINTER(Threshold), U32, P, P, C.POINTER(AllocPolicy), I64,
                                U32, P, P, P, P, P, P, P, P]),
    "cdx_cot_exit": (C.c_int, [P, P, P, P, U64, U32, C.POINTER(ProbeCfg), P, P, P, P, P]),
    "cdx_cot_meets": (C.c_int, [P, P, P, U64, U32, I32, C.POINTER(Threshold), U32, P]),
    "cdx_mixed_allocate": (C.c_int, [P, C.POINTER(MixedTrace), P, P, P, U64, C.POINTER(ArchPolicy), P, P, P, P, P]),
    "cdx_reward_certaindex": (C.c_int, [P, P, P, P, U64, U32, U32, C.POINTER(Threshold), U32,
                                        C.POINTER(Threshold), U32, P, P, P]),
    "cdx_reward_certaindex_f64": (C.c_int, [P, P, P, P, U64, U32, U32, C.POINTER(Threshold), U32,
                                        C.POINTER(Threshold), U32, P, P, P]),
    "cdx_reward_sets": (C.c_int, [P, P, P, P, U64, P]),
    "cdx_canon_intern": (C.c_int, [P, P, P, U64, C.POINTER(C.c_char_p), U32, P, P, P, C.POINTER(U64)]),
    "cdx_gang_priority": (C.c_int, [P, C.POINTER(ProgSoA), U64, C.POINTER(InterPolicy), C.c_double, P,
                                    C.POINTER(U64), P, P]),
    "cdx_gang_merge": (C.c_int, [P, P, P, U32, U64, P, P]),
    "cdx_offsets_rebase": (C.c_int, [P, P, U64, P, U32]),
    "cdx_nccl_unique_id": (C.c_int, [P]),
    "cdx_ctx_create_comm": (C.c_int, [C.c_int, C.POINTER(Comm), C.POINTER(P)]),
    "cdx_ctx_comm_info": (C.c_int, [P, C.POINTER(U32), C.POINTER(U32)]),
    "cdx_allgather": (C.c_int, [P, P, P, U64]),
    "cdx_allocate_scan_sharded": (C.c_int, [P, P, U64, U32, C.POINTER(AllocPolicy), P, P, P, P, P, P, P, P, P]),
    "cdx_gang_priority_sharded": (C.c_int, [P, C.POINTER(ProgSoA), U64, C.POINTER(InterPolicy), C.c_double, P,
                                            C.POINTER(U64)]),
    "cdx_shard_samples": (C.c_int, [P, P, U64, U32, P]),
    "cdx_shard_splitters": (C.c_int, [P, P, U32, U32, P]),
    "cdx_shard_bounds": (C.c_int, [P, P, U64, P, U32, P]),
    "cdx_gang_merge_runs": (C.c_int, [P, P, P, U32, P]),
    "cdx_jsonl_parse": (C.c_int, [P, P, U64, U64, P, P, P, P, P, P, P, P, P, C.POINTER(U64), C.POINTER(U64)]),
    "cdx_cot_eps_stop": (C.c_int, [P, P, P, U64, U32, I32, C.c_double, P, P]),
    "cdx_probe_eps_stop_rows": (C.c_int, [P, P, P, P, U64, I32, C.c_double, P]),
    "cdx_sc_aggregate": (C.c_int, [P, P, U64, U32, U32, P, P]),
    "cdx_reward_aggregate": (C.c_int, [P, P, P, P, U64, U32, U32, P, P, P]),
    "cdx_reward_aggregate_f64": (C.c_int, [P, P, P, P, U64, U32, U32, P, P]),
    "cdx_libm_exp": (C.c_int, [P, P, U64, P]),
    "cdx_sc_decide_host": (C.c_int, [P, P, U64, U32, U32, C.POINTER(Threshold), U32, C.POINTER(AllocPolicy),
                                     P, P, P, P, P]),
    "cdx_cot_decide_host": (C.c_int, [P, P, P, P, U64, U32, C.POINTER(ProbeCfg), P, P, P, P]),
    "cdx_reward_decide_host": (C.c_int, [P, P, P, P, U64, U32, U32, C.POINTER(Threshold), U32, C.POINTER(Threshold),
                                         U32, C.POINTER(AllocPolicy), P, P, P, P, P]),
}

_lib = None


def load(path: str = LIB_PATH, require_all: bool = False) -> C.CDLL:
    """Load libcdx.so (in-tree build).  Raises if it is missing: no fallback."""
    global _lib
    if _lib is not None and path == LIB_PATH:
        return _lib
    if not os.path.exists(path):
        raise RuntimeError(f"libcdx.so not built at {path}; run `make lib` (or __graft_entry__.build())")
    lib = C.CDLL(path)
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name, None)
        if fn is None:
            if require_all:
                raise RuntimeError(f"libcdx.so does not export {name}")
            continue
        fn.restype = res
        fn.argtypes = args
    if path == LIB_PATH:
        _lib = lib
    return lib
