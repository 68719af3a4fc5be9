// k_mixed.cu — the mixed-archetype decision step: ProgramDriver::update_certaindex's
// per-archetype dispatch (runtime.cpp:264-313) followed by scheduler.allocate
// for a whole batch of reasoning programs, each at its own current knob.
//
//   archetype SC      -> K2 sc_certaindex: H~ of the S samples' answers at every probe row
//   archetype CoT     -> cot_meets_kernel below: C_k = consistency(records up to probe p, w)
//                        (probe.cpp:64-75), 0.0 while the window is not ready (runtime.cpp:298)
//   archetype MCTS    -> K4 reward_certaindex: cumulative H~ and mean reward (runtime.cpp:279-292)
//   archetype Rebase  -> K4 with the max reward
// Each archetype's signals go through its own combined_meets_thresholds (metrics.cpp:159-171)
// into one threshold bit per knob unit; then mixed_decide_kernel applies the archetype's
// allocation policy at the program's current knob k exactly as scheduler.allocate does
// (include/cdx/scheduler.hpp, facade_scheduler.cpp): k >= cap -> terminate (resource cap); a
// test point <= k whose thresholds held -> terminate (certain); else grant up to the next
// decision point.  The token budgets of the grants are scanned into offsets (K5's scan) and the
// decision byte doubles as the `terminated` flag of the gang order (K6, cdx_prog_soa).
#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "cdx_internal.cuh"
#include "k_sc.cuh"
#include "k_scan.cuh"

namespace cdx {
namespace {

// ---- CoT: one threshold bit per probe --------------------------------------------------
// Thread per request; a warp stages its 32 rows (P u32 each) through shared memory with
// coalesced 16-byte loads, then every thread walks its own row.  C_k at probe p only depends
// on the last w non-hesitant answers up to p: agree = #{window == newest}; the threshold
// outcome for each agree count a in [0, w] (and for "not ready") is a host-built bit table.
constexpr int CM_WARPS = 4;

template <int W>
__global__ void __launch_bounds__(CM_WARPS * 32) cot_meets_kernel(const uint32_t* __restrict__ ids,
                                                                  const uint64_t* __restrict__ hes, uint64_t R,
                                                                  uint32_t P, uint32_t stride, int32_t w,
                                                                  uint64_t lut, uint32_t notready,
                                                                  uint32_t* __restrict__ meets) {
    extern __shared__ __align__(16) uint32_t cm_smem[];
    const uint32_t lane = threadIdx.x & 31u, warp = threadIdx.x >> 5;
    uint32_t* rows = cm_smem + static_cast<size_t>(warp) * 32u * stride;
    const uint32_t hw = (P + 63u) / 64u, words = (P + 31u) / 32u;
    const uint64_t nwarps = static_cast<uint64_t>(gridDim.x) * CM_WARPS;
    for (uint64_t r0 = (static_cast<uint64_t>(blockIdx.x) * CM_WARPS + warp) * 32u; r0 < R; r0 += nwarps * 32u) {
        const uint32_t nr = static_cast<uint32_t>(R - r0 < 32u ? R - r0 : 32u);
        // coalesced staging of nr rows (contiguous nr * P words)
        const uint32_t* src = ids + r0 * P;
        const uint32_t tot = nr * P;
        if ((reinterpret_cast<uintptr_t>(src) & 15u) == 0 && (P & 3u) == 0) {
            for (uint32_t q = lane * 4u; q < tot; q += 128u) {
                const uint4 v = __ldg(reinterpret_cast<const uint4*>(src + q));
                const uint32_t rr = q / P, cc = q - rr * P;
                *reinterpret_cast<uint4*>(rows + rr * stride + cc) = v;
            }
        } else {
            for (uint32_t q = lane; q < tot; q += 32u) {
                const uint32_t rr = q / P;
                rows[rr * stride + (q - rr * P)] = __ldg(src + q);
            }
        }
        __syncwarp();
        if (lane < nr) {
            const uint64_t r = r0 + lane;
            const uint32_t* row = rows + lane * stride;
            uint32_t win[W > 0 ? W : 1];
            int32_t used = 0;
            uint32_t bit = notready;  // outcome at the latest usable record (carried over hesitant probes)
            uint32_t word = 0;
            uint64_t hbits = 0;
            for (uint32_t p = 0; p < P; ++p) {
                if ((p & 63u) == 0) hbits = __ldg(hes + r * hw + (p >> 6));
                if (!((hbits >> (p & 63u)) & 1ull)) {
                    const uint32_t v = row[p];
                    if (W > 0) {
#pragma unroll
                        for (int j = (W > 0 ? W : 1) - 1; j > 0; --j) win[j] = win[j - 1];
                        win[0] = v;
                        used = used < W ? used + 1 : W;
                        if (used >= W) {
                            int32_t a = 0;
#pragma unroll
                            for (int j = 0; j < (W > 0 ? W : 1); ++j) a += win[j] == v ? 1 : 0;
                            bit = static_cast<uint32_t>((lut >> a) & 1ull);
                        }
                    } else {  // runtime window: count back over the staged row
                        ++used;
                        if (used >= w) {
                            int32_t a = 0, seen = 0;
                            for (int32_t q = static_cast<int32_t>(p); q >= 0 && seen < w; --q) {
                                if ((__ldg(hes + r * hw + (q >> 6)) >> (q & 63)) & 1ull) continue;
                                a += row[q] == v ? 1 : 0;
                                ++seen;
                            }
                            bit = static_cast<uint32_t>((lut >> a) & 1ull);
                        }
                    }
                }
                word |= bit << (p & 31u);
                if ((p & 31u) == 31u || p + 1 == P) {
                    meets[r * words + (p >> 5)] = word;
                    word = 0;
                }
            }
        }
        __syncwarp();
    }
}

// Lean form: P = 4 * NC probes (NC <= 32, P <= 128) and a compile-time window W.  Each
// thread reads its staged row as uint4 (4 probes per LDS.128, conflict-free with the +4 word
// row stride), the hesitation bits as up to two 64-bit words, and walks the probes fully
// unrolled and branch-free: a usable probe shifts the register window, the outcome bit of
// the newest window is a table lookup, a hesitant probe repeats the previous outcome.
template <int W, int NC>
__global__ void __launch_bounds__(CM_WARPS * 32) cot_meets_lean(const uint32_t* __restrict__ ids,
                                                                const uint64_t* __restrict__ hes, uint64_t R,
                                                                uint32_t stride, uint64_t lut, uint32_t notready,
                                                                uint32_t* __restrict__ meets) {
    constexpr uint32_t P = 4 * NC, HW = (P + 63) / 64, WORDS = (P + 31) / 32;
    extern __shared__ __align__(16) uint32_t cm_smem[];
    const uint32_t lane = threadIdx.x & 31u, warp = threadIdx.x >> 5;
    uint32_t* rows = cm_smem + static_cast<size_t>(warp) * 32u * stride;
    const uint64_t nwarps = static_cast<uint64_t>(gridDim.x) * CM_WARPS;
    for (uint64_t r0 = (static_cast<uint64_t>(blockIdx.x) * CM_WARPS + warp) * 32u; r0 < R; r0 += nwarps * 32u) {
        const uint32_t nr = static_cast<uint32_t>(R - r0 < 32u ? R - r0 : 32u);
        const uint4* src = reinterpret_cast<const uint4*>(ids + r0 * P);
        if (nr == 32) {  // 32 rows = 32 * NC uint4, NC per lane, coalesced
#pragma unroll
            for (int j = 0; j < NC; ++j) {
                const uint32_t q = static_cast<uint32_t>(j) * 32u + lane;
                const uint4 v = __ldg(src + q);
                const uint32_t rr = q / NC, cc = (q - rr * NC) * 4u;
                *reinterpret_cast<uint4*>(rows + rr * stride + cc) = v;
            }
        } else {
            for (uint32_t q = lane; q < nr * NC; q += 32u) {
                const uint32_t rr = q / NC, cc = (q - rr * NC) * 4u;
                *reinterpret_cast<uint4*>(rows + rr * stride + cc) = __ldg(src + q);
            }
        }
        uint64_t hb[HW];
        if (lane < nr) {
#pragma unroll
            for (uint32_t k = 0; k < HW; ++k) hb[k] = __ldg(hes + (r0 + lane) * HW + k);
        }
        __syncwarp();
        if (lane < nr) {
            const uint4* row = reinterpret_cast<const uint4*>(rows + lane * stride);
            uint32_t win[W];
#pragma unroll
            for (int j = 0; j < W; ++j) win[j] = 0;
            int32_t used = 0;
            uint32_t bit = notready, out[WORDS];
#pragma unroll
            for (uint32_t k = 0; k < WORDS; ++k) out[k] = 0;
#pragma unroll
            for (int c = 0; c < NC; ++c) {
                const uint4 q4 = row[c];
                const uint32_t qv[4] = {q4.x, q4.y, q4.z, q4.w};
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    const uint32_t p = 4u * c + j;
                    const bool u = !((hb[p / 64] >> (p % 64)) & 1ull);
                    if (u) {
#pragma unroll
                        for (int t = W - 1; t > 0; --t) win[t] = win[t - 1];
                        win[0] = qv[j];
                        ++used;
                        int32_t a = 0;
#pragma unroll
                        for (int t = 0; t < W; ++t) a += win[t] == qv[j] ? 1 : 0;
                        bit = used >= W ? static_cast<uint32_t>((lut >> a) & 1ull) : notready;
                    }
                    out[p / 32] |= bit << (p % 32);
                }
            }
#pragma unroll
            for (uint32_t k = 0; k < WORDS; ++k) meets[(r0 + lane) * WORDS + k] = out[k];
        }
        __syncwarp();
    }
}

// ---- Rebase vs MCTS: the aggregation of each reward row, from its program's archetype -----
__global__ void mixed_agg_kernel(const uint8_t* __restrict__ arch, const uint32_t* __restrict__ slot, uint64_t N,
                                 uint64_t rw_n, uint8_t* __restrict__ agg) {
    for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < N;
         i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
        const uint8_t a = arch[i];
        const uint32_t s = slot[i];
        if ((a == CDX_ARCH_MCTS || a == CDX_ARCH_REBASE) && s < rw_n)
            agg[s] = a == CDX_ARCH_REBASE ? CDX_AGG_MAX : CDX_AGG_MEAN;  // runtime.cpp:285-286
    }
}

// ---- allocate at the current knob ---------------------------------------------------------
struct ArchPol {
    uint8_t kind;
    int32_t detect, recheck, cap;
    uint32_t tpu;
};
struct DecideParams {
    const uint8_t* arch;
    const uint32_t* slot;
    const int32_t* knob;
    const uint32_t* meets[3];  // groups: 0 SC, 1 CoT, 2 MCTS/Rebase
    uint32_t words[3];
    uint64_t n[3];
    ArchPol pol[4];  // by CDX_ARCH_*
    uint8_t* decision;
    int32_t* grant;
    int32_t* cap;
    uint64_t N;
    int* d_err;
};

__device__ __forceinline__ int group_of(uint8_t a) {
    return a == CDX_ARCH_SC ? 0 : (a == CDX_ARCH_COT ? 1 : 2);
}

// any bit of row[] in the knob-unit range [lo, hi] (1-based, inclusive)
__device__ __forceinline__ bool any_bits(const uint32_t* __restrict__ row, int32_t lo, int32_t hi) {
    bool met = false;
    for (int32_t w = (lo - 1) / 32; w <= (hi - 1) / 32 && !met; ++w) {
        const int32_t b0 = w * 32 + 1;  // knob unit of bit 0 of word w
        uint32_t m = 0xffffffffu;
        if (lo > b0) m &= 0xffffffffu << (lo - b0);
        if (hi < b0 + 31) m &= 0xffffffffu >> (b0 + 31 - hi);
        met = (__ldg(row + w) & m) != 0u;
    }
    return met;
}

// scheduler.allocate at the current knob for program i (as
// facade_scheduler.cpp): writes decision / grant / cap, returns the grant's token budget
__device__ __forceinline__ uint32_t decide_one(const DecideParams& p, uint64_t i) {
    const uint8_t a = __ldg(p.arch + i);
    uint8_t dec = CDX_EXIT_CONTINUE;
    int32_t g_units = 0, cap = 0;
    uint32_t budget = 0;
    if (a > 3) {
        set_dev_err(p.d_err, DEV_MIXED_PROGRAM);
    } else {
        const ArchPol& q = p.pol[a];
        const int g = group_of(a);
        const uint32_t s = __ldg(p.slot + i);
        const int32_t k = __ldg(p.knob + i);
        cap = q.cap;
        if (s >= p.n[g] || k < 0 || k > q.cap) {
            set_dev_err(p.d_err, DEV_MIXED_PROGRAM);
        } else if (k >= q.cap) {  // "always terminate at resource_cap"
            dec = CDX_EXIT_BUDGET;
        } else {
            bool met = false;
            if (q.kind != CDX_POL_EVEN && q.detect <= k) {
                const uint32_t* row = p.meets[g] + static_cast<uint64_t>(s) * p.words[g];
                if (q.kind == CDX_POL_STATIC_THRESHOLD) {
                    met = (__ldg(row + (q.detect - 1) / 32) >> ((q.detect - 1) % 32)) & 1u;
                } else if (q.recheck == 1) {  // every unit from detect_at to k
                    met = any_bits(row, q.detect, k);
                } else {
                    for (int32_t t = q.detect; t <= k && !met; t += q.recheck)
                        met = (__ldg(row + (t - 1) / 32) >> ((t - 1) % 32)) & 1u;
                }
            }
            if (met) {
                dec = CDX_EXIT_CERTAIN;
            } else {  // grant up to the next decision point
                int32_t next = q.cap;
                if (q.kind == CDX_POL_STATIC_THRESHOLD && k < q.detect) next = q.detect;
                if (q.kind == CDX_POL_K_STEP_THRESHOLD) {
                    next = q.detect;
                    if (next <= k) next += ((k - next) / q.recheck + 1) * q.recheck;
                    next = next < q.cap ? next : q.cap;
                }
                g_units = next - k;
                budget = static_cast<uint32_t>(g_units) * q.tpu;
            }
        }
    }
    p.decision[i] = dec;
    if (p.grant) p.grant[i] = g_units;
    if (p.cap) p.cap[i] = cap;
    return budget;
}

// thread per program, coalesced; budget (nullable) = the grant's tokens, the scan's input
__global__ void mixed_decide_kernel(const __grid_constant__ DecideParams p, uint32_t* __restrict__ budget) {
    for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < p.N;
         i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
        const uint32_t b = decide_one(p, i);
        if (budget) budget[i] = b;
    }
}

unsigned grid_for(const cdx_ctx* ctx, uint64_t n, unsigned t) {
    const uint64_t want = (n + t - 1) / t;
    const uint64_t cap = static_cast<uint64_t>(ctx->sm_count) * 16;
    return static_cast<unsigned>(want < 1 ? 1 : (want < cap ? want : cap));
}

int check_policy(cdx_ctx* ctx, const cdx_alloc_policy& pol, uint32_t units) {
    const int32_t cap = pol.resource_cap;
    if (cap < 1 || static_cast<uint32_t>(cap) > units)
        return set_error(ctx, CDX_EINVAL, "allocate: resource_cap must be in [1, knob units of the trace]");
    if (pol.kind != CDX_POL_EVEN && pol.kind != CDX_POL_STATIC_THRESHOLD && pol.kind != CDX_POL_K_STEP_THRESHOLD)
        return set_error(ctx, CDX_EINVAL, "allocate: policy kind not supported by the batched path");
    if (pol.kind != CDX_POL_EVEN && (pol.detect_at < 1 || pol.detect_at > cap))
        return set_error(ctx, CDX_EINVAL, "allocate: detect_at_knob must be in [1, resource_cap]");
    if (pol.kind == CDX_POL_K_STEP_THRESHOLD && pol.recheck_every < 1)
        return set_error(ctx, CDX_EINVAL, "allocate: recheck_every must be >= 1");
    if (pol.tokens_per_unit < 0 || static_cast<uint64_t>(pol.tokens_per_unit) * static_cast<uint64_t>(cap) > 0xffffffffull)
        return set_error(ctx, CDX_EINVAL, "allocate: resource_cap * tokens_per_unit must be in [0, 2^32)");
    return CDX_OK;
}

}  // namespace
}  // namespace cdx

extern "C" int cdx_cot_meets(cdx_ctx* ctx, const uint32_t* ids, const uint64_t* hes, uint64_t R, uint32_t P,
                             int32_t window, const cdx_threshold* th, uint32_t n_th, uint32_t* meets_bits) {
    using namespace cdx;
    CDX_NVTX("cdx_cot_meets");
    if (!ctx) return CDX_EINVAL;
    if (window < 1) return set_error(ctx, CDX_EINVAL, "consistency: window must be >= 1");
    const bool present[5] = {true, false, false, false, false};  // CoT's SignalVector: C_k in the entropy slot
    if (int st = check_thresholds(ctx, th, n_th, present)) return st;
    if (window > 62) return set_error(ctx, CDX_EINVAL, "cot_meets: window must be <= 62");
    if (P == 0 || P > 4096) return set_error(ctx, CDX_EINVAL, "cot_meets: probes must be in [1, 4096]");
    if (R == 0) return CDX_OK;
    if (!ids || !hes || !meets_bits) return set_error(ctx, CDX_EINVAL, "cot_meets: null pointer");
    // combined_meets_thresholds(C) for every value C can take: a / w for a in [0, w], and the
    // not-ready 0.0 (runtime.cpp:298); in threshold order, a failed compare ends it
    auto meets = [&](double v) {
        for (uint32_t t = 0; t < n_th; ++t) {
            const bool ok = th[t].dir == CDX_DIR_GE ? v >= th[t].cutoff : v <= th[t].cutoff;
            if (!ok) return false;
        }
        return true;
    };
    uint64_t lut = 0;
    for (int32_t a = 0; a <= window; ++a)
        if (meets(static_cast<double>(a) / static_cast<double>(window))) lut |= 1ull << a;
    const uint32_t notready = meets(0.0) ? 1u : 0u;
    const uint32_t stride = (P + 31u) / 32u * 32u + 4u;  // 16-byte row reads land in distinct banks
    const size_t smem = static_cast<size_t>(CM_WARPS) * 32u * stride * 4u;
    if (smem > 200u * 1024u) return set_error(ctx, CDX_EINVAL, "cot_meets: rows too long for shared memory");
    const uint64_t want = (R + CM_WARPS * 32 - 1) / (CM_WARPS * 32);
    const unsigned grid = static_cast<unsigned>(std::min<uint64_t>(want, static_cast<uint64_t>(ctx->sm_count) * 8));
    // lean kernel: P in {32, 64, 96, 128}, window 1..8, 16-byte aligned rows
    if (P % 32 == 0 && P <= 128 && window <= 8 && (reinterpret_cast<uintptr_t>(ids) & 15u) == 0 &&
        !getenv("CDX_COTM_GENERIC")) {
        void (*k)(const uint32_t*, const uint64_t*, uint64_t, uint32_t, uint64_t, uint32_t, uint32_t*) = nullptr;
#define CDX_COTM_W(Wv)                                                                               \
    case Wv:                                                                                         \
        k = P == 32 ? cot_meets_lean<Wv, 8> : P == 64 ? cot_meets_lean<Wv, 16>                       \
                                           : P == 96 ? cot_meets_lean<Wv, 24> : cot_meets_lean<Wv, 32>; \
        break;
        switch (window) {
            CDX_COTM_W(1) CDX_COTM_W(2) CDX_COTM_W(3) CDX_COTM_W(4)
            CDX_COTM_W(5) CDX_COTM_W(6) CDX_COTM_W(7) CDX_COTM_W(8)
        }
#undef CDX_COTM_W
        cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
        k<<<grid, CM_WARPS * 32, smem, ctx->stream>>>(ids, hes, R, stride, lut, notready, meets_bits);
        CDX_CHECK_LAUNCH(ctx, "cot_meets(lean)");
        return CDX_OK;
    }
    auto launch = [&](auto kern) {
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
        kern<<<grid, CM_WARPS * 32, smem, ctx->stream>>>(ids, hes, R, P, stride, window, lut, notready, meets_bits);
    };
    switch (window) {
        case 1: launch(cot_meets_kernel<1>); break;
        case 2: launch(cot_meets_kernel<2>); break;
        case 3: launch(cot_meets_kernel<3>); break;
        case 4: launch(cot_meets_kernel<4>); break;
        case 5: launch(cot_meets_kernel<5>); break;
        case 6: launch(cot_meets_kernel<6>); break;
        case 7: launch(cot_meets_kernel<7>); break;
        case 8: launch(cot_meets_kernel<8>); break;
        default: launch(cot_meets_kernel<0>); break;
    }
    CDX_CHECK_LAUNCH(ctx, "cot_meets");
    return CDX_OK;
}

extern "C" int cdx_mixed_allocate(cdx_ctx* ctx, const cdx_mixed_trace* tr, const uint8_t* archetype,
                                  const uint32_t* slot, const int32_t* knob, uint64_t N,
                                  const cdx_arch_policy* policy, uint8_t* decision, int32_t* grant, int32_t* cap,
                                  int64_t* offsets, int64_t* total_budget) {
    using namespace cdx;
    CDX_NVTX("cdx_mixed_allocate");
    if (!ctx) return CDX_EINVAL;
    if (!tr || !policy) return set_error(ctx, CDX_EINVAL, "mixed_allocate: null pointer");
    if (N > 0xffffffffull) return set_error(ctx, CDX_EINVAL, "mixed_allocate: at most 2^32-1 programs");
    // every archetype's policy against its trace shape (a group with no programs is not checked)
    const uint32_t units[4] = {tr->sc_P, tr->rw_T, tr->rw_T, tr->cot_P};
    const uint64_t gn[4] = {tr->sc_n, tr->rw_n, tr->rw_n, tr->cot_n};
    for (int a = 0; a < 4; ++a) {
        if (gn[a] == 0) continue;
        if (int st = check_policy(ctx, policy[a].alloc, units[a])) return st;
        if (policy[a].n_th > 4) return set_error(ctx, CDX_EINVAL, "mixed_allocate: at most 4 thresholds per archetype");
    }
    if (N == 0) {
        if (total_budget) cudaMemsetAsync(total_budget, 0, 8, ctx->stream);
        return CDX_OK;
    }
    if (!archetype || !slot || !knob || !decision) return set_error(ctx, CDX_EINVAL, "mixed_allocate: null pointer");
    if (tr->sc_n && (!tr->sc_ids || tr->sc_S == 0 || tr->sc_P == 0))
        return set_error(ctx, CDX_EINVAL, "mixed_allocate: SC group needs ids and a shape");
    if (tr->cot_n && (!tr->cot_ids || !tr->cot_hes || tr->cot_P == 0))
        return set_error(ctx, CDX_EINVAL, "mixed_allocate: CoT group needs ids, hesitation bits and a shape");
    if (tr->rw_n && (!tr->rw_rewards || tr->rw_T == 0 || tr->rw_W == 0))
        return set_error(ctx, CDX_EINVAL, "mixed_allocate: MCTS/Rebase group needs rewards and a shape");

    const uint32_t words[3] = {(tr->sc_P + 31u) / 32u, (tr->cot_P + 31u) / 32u, (tr->rw_T + 31u) / 32u};
    const uint64_t n3[3] = {tr->sc_n, tr->cot_n, tr->rw_n};
    size_t bytes = 256;
    size_t off[4];
    for (int g = 0; g < 3; ++g) {
        off[g] = bytes;
        bytes += (n3[g] * words[g] * 4 + 255) / 256 * 256;
    }
    off[3] = bytes;  // agg bytes of the reward rows
    bytes += (tr->rw_n + 255) / 256 * 256;
    const uint64_t tiles = (N + scan::SL_TILE - 1) / scan::SL_TILE;
    const size_t rec_off = bytes;
    bytes += (tiles + 2) * 8 + 16;
    const size_t bud_off = bytes;  // per-program token budgets (the scan's input)
    bytes += (N * 4 + 255) / 256 * 256;
    const size_t offs_off = bytes;  // offsets when the caller wants only the total
    bytes += N * 8 + 64;
    uint8_t* s = static_cast<uint8_t*>(scratch3(ctx, bytes));
    if (!s) return set_error(ctx, CDX_ECUDA, "mixed_allocate: scratch allocation failed");
    uint32_t* meets[3];
    for (int g = 0; g < 3; ++g) meets[g] = reinterpret_cast<uint32_t*>(s + off[g]);
    uint8_t* agg = s + off[3];
    uint64_t* rec = reinterpret_cast<uint64_t*>(s + rec_off);

    // signals -> threshold bits per knob unit, one engine per archetype.  The engines are
    // independent, so with SC and reward rows both present they run concurrently: K2 (ALU-bound
    // on noisy rows) on a side stream, K4 (HBM-bound) on another, cot_meets on the caller's
    // stream; the caller's stream then waits for both (stream-ordered: nothing syncs with the
    // host, graph capture follows the fork).  Config E: 2.155 -> 2.117 ms; capping K2's resident
    // CTAs to leave K4 room (CDX_MIXED_SC_CTAS=k per SM) was measured slower (k = 1: 2.97 ms,
    // k = 2: 2.33 ms).
    cudaStream_t main = ctx->stream;
    const char* ser = getenv("CDX_MIXED_SERIAL");
    const bool overlap = tr->sc_n && tr->rw_n && !(ser && ser[0] == '1');
    if (overlap) {
        for (int q = 0; q < 2; ++q) {
            if (!ctx->aux[q] && cudaStreamCreateWithFlags(&ctx->aux[q], cudaStreamNonBlocking) != cudaSuccess)
                return set_error(ctx, CDX_ECUDA, "mixed_allocate: stream creation failed");
            if (!ctx->ev_join[q] && cudaEventCreateWithFlags(&ctx->ev_join[q], cudaEventDisableTiming) != cudaSuccess)
                return set_error(ctx, CDX_ECUDA, "mixed_allocate: event creation failed");
        }
        if (!ctx->ev_fork && cudaEventCreateWithFlags(&ctx->ev_fork, cudaEventDisableTiming) != cudaSuccess)
            return set_error(ctx, CDX_ECUDA, "mixed_allocate: event creation failed");
        cudaEventRecord(ctx->ev_fork, main);
        cudaStreamWaitEvent(ctx->aux[0], ctx->ev_fork, 0);
        cudaStreamWaitEvent(ctx->aux[1], ctx->ev_fork, 0);
    }
    auto join = [&]() {  // the caller's stream waits for the side streams (also on an error path)
        ctx->stream = main;
        ctx->sc_ctas_per_sm = 0;
        if (!overlap) return;
        for (int q = 0; q < 2; ++q) {
            cudaEventRecord(ctx->ev_join[q], ctx->aux[q]);
            cudaStreamWaitEvent(main, ctx->ev_join[q], 0);
        }
    };
    if (tr->sc_n) {
        if (overlap) {
            ctx->stream = ctx->aux[0];
            const char* e = getenv("CDX_MIXED_SC_CTAS");
            ctx->sc_ctas_per_sm = e ? static_cast<uint32_t>(std::max(0, atoi(e))) : 0u;
        }
        const int st = cdx_sc_certaindex(ctx, tr->sc_ids, tr->sc_n, tr->sc_P, tr->sc_S, policy[CDX_ARCH_SC].th,
                                         policy[CDX_ARCH_SC].n_th, nullptr, meets[0]);
        ctx->stream = main;
        ctx->sc_ctas_per_sm = 0;
        if (st) {
            join();
            return st;
        }
    }
    if (tr->cot_n) {
        if (int st = cdx_cot_meets(ctx, tr->cot_ids, tr->cot_hes, tr->cot_n, tr->cot_P, static_cast<int32_t>(tr->cot_window),
                                   policy[CDX_ARCH_COT].th, policy[CDX_ARCH_COT].n_th, meets[1])) {
            join();
            return st;
        }
    }
    if (tr->rw_n) {
        if (overlap) ctx->stream = ctx->aux[1];
        cudaMemsetAsync(agg, CDX_AGG_MEAN, tr->rw_n, ctx->stream);
        mixed_agg_kernel<<<grid_for(ctx, N, 256), 256, 0, ctx->stream>>>(archetype, slot, N, tr->rw_n, agg);
        cudaError_t le = cudaGetLastError();
        ctx->launches++;
        int st = le != cudaSuccess ? cuda_fail(ctx, le, "mixed_allocate(agg)") : CDX_OK;
        if (!st)
            st = cdx_reward_certaindex(ctx, tr->rw_rewards, tr->rw_ids, agg, tr->rw_n, tr->rw_T, tr->rw_W,
                                       policy[CDX_ARCH_MCTS].th, policy[CDX_ARCH_MCTS].n_th,
                                       policy[CDX_ARCH_REBASE].th, policy[CDX_ARCH_REBASE].n_th, nullptr, nullptr,
                                       meets[2]);
        ctx->stream = main;
        if (st) {
            join();
            return st;
        }
    }
    join();
    DecideParams p{};
    p.arch = archetype;
    p.slot = slot;
    p.knob = knob;
    for (int g = 0; g < 3; ++g) {
        p.meets[g] = meets[g];
        p.words[g] = words[g];
        p.n[g] = n3[g];
    }
    for (int a = 0; a < 4; ++a) {
        const cdx_alloc_policy& q = policy[a].alloc;
        p.pol[a] = ArchPol{q.kind, q.detect_at, q.recheck_every, q.resource_cap, static_cast<uint32_t>(q.tokens_per_unit)};
        if (gn[a] == 0) p.pol[a].cap = 0;
    }
    p.decision = decision;
    p.grant = grant;
    p.cap = cap;
    p.N = N;
    p.d_err = ctx->d_err;
    const bool scan_b = offsets || total_budget;
    uint32_t* budget = scan_b ? reinterpret_cast<uint32_t*>(s + bud_off) : nullptr;
    mixed_decide_kernel<<<grid_for(ctx, N, 256), 256, 0, ctx->stream>>>(p, budget);
    CDX_CHECK_LAUNCH(ctx, "mixed_allocate(decide)");
    if (scan_b) {  // exclusive scan of the grants' token budgets (K5's single-pass scan)
        uint64_t* out = offsets ? reinterpret_cast<uint64_t*>(offsets) : reinterpret_cast<uint64_t*>(s + offs_off);
        if (int st = scan::scan_excl(ctx, scan::LoadU32{budget}, N, out, false, rec,
                                     reinterpret_cast<uint64_t*>(total_budget)))
            return st;
    }
    return CDX_OK;
}
