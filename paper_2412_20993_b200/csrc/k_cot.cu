// k_cot.cu — K3: chain-of-thought probe-window early exit.
//
// Replaces, for every prefix of every request's probe trace (the reference evaluates the
// decision once per probe as the trace grows):
//   probe::consistency  (probe.cpp:64-75, usable_up_to :53-60)
//   probe::should_exit  (probe.cpp:77-85; certainty wins ties)
//   probe::final_answer (probe.cpp:87-102) after ProgramDriver::terminate (runtime.cpp:405-411)
// The reference rebuilds the usable list from record 0 at every step (O(P^2) per trace).
// Here one thread owns one request and slides a register window of the last w usable
// answers over the probes once: certain_step = first non-hesitant probe whose full window
// has agree >= a_min(w,tau) (a_min = min{a : (double)a/w >= tau}, computed on the host, so
// the device decision is an integer compare); budget_step = first probe whose token offset
// reaches max_tokens.  Equivalence to the prefix replay is property-tested (tests/).
//
// Data path: ids u32[R][P] are staged by TMA (2-D tensor map, 128-byte swizzle, multi-stage
// mbarrier ring) so that each thread reads its own 256-byte row as 16-byte chunks without
// shared-memory bank conflicts (chunk c of row r sits at chunk c ^ (r & 7)).
#include <algorithm>
#include <cstdlib>

#include "cdx_internal.cuh"

namespace cdx {

constexpr int COT_MAX_STAGES = 3;

struct CotParams {
    CUtensorMap tmap;  // 64-byte aligned first member
    const uint32_t* ids;
    const uint64_t* hes;
    const int64_t* offsets;
    int32_t* exit_step;
    uint8_t* reason;
    uint32_t* final_id;
    uint8_t* low_conf;
    float* ck;
    uint64_t R;
    uint64_t ntiles;
    uint32_t P, hw, boxes, rows;
    uint32_t stage_bytes, stages;
    int32_t w, amin;
    int32_t bstep_implicit;  // first probe index whose implicit offset >= max_tokens, or -1
    const int32_t* bsteps;   // explicit offsets: per-request budget step (cot_budget_steps), or null
    int32_t _pad;
    int64_t max_tokens;
};

// Per-request state of the sliding window (W = compile-time window, 0 = runtime window).
template <int W>
struct CotWin {
    uint32_t win[W > 0 ? W : 1];
    int32_t usable = 0, last_agree = -1;
    uint32_t last_nh = 0;
    bool has_nh = false;
};

template <int W, bool TMA>
__device__ __forceinline__ uint32_t cot_id(const CotParams& p, const uint8_t* tsm, uint32_t tid, uint64_t r,
                                           uint32_t q) {
    if (TMA) {
        const uint32_t bb = q >> 5, cc = (q & 31u) >> 2, ee = q & 3u;
        return *reinterpret_cast<const uint32_t*>(tsm + bb * p.rows * 128u + swz128(tid, cc) + ee * 4u);
    }
    return __ldg(p.ids + r * p.P + q);
}

// CK = also emit the consistency value C at every probe (runtime.cpp:298 value_or(0.0)).
template <int W, bool TMA, bool CK>
__global__ void __launch_bounds__(128) cot_exit_kernel(const __grid_constant__ CotParams p) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    // 128B-swizzled TMA destinations must be 1024-byte aligned
    uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
    uint64_t* bar = reinterpret_cast<uint64_t*>(smem + p.stages * p.stage_bytes);
    const uint32_t tid = threadIdx.x;

    if (TMA) {
        if (tid == 0) {
            tma_prefetch_desc(&p.tmap);
            for (uint32_t s = 0; s < p.stages; ++s) mbar_init(&bar[s], 1);
            fence_mbar_init();
        }
        __syncthreads();
    }
    const uint64_t policy = policy_evict_first();
    const uint64_t stride = gridDim.x;
    auto issue = [&](uint64_t tile, uint32_t stage) {
        uint8_t* dst = smem + stage * p.stage_bytes;
        mbar_expect_tx(&bar[stage], p.stage_bytes);
        for (uint32_t b = 0; b < p.boxes; ++b)
            tma_load_2d(dst + b * p.rows * 128u, &p.tmap, static_cast<int32_t>(b * 32),
                        static_cast<int32_t>(tile * p.rows), &bar[stage], policy);
    };
    if (TMA && tid == 0) {
        for (uint32_t s = 0; s < p.stages; ++s) {
            const uint64_t t = blockIdx.x + s * stride;
            if (t < p.ntiles) issue(t, s);
        }
    }

    uint32_t stage = 0, parity = 0;
    for (uint64_t tile = blockIdx.x; tile < p.ntiles; tile += stride) {
        if (TMA) mbar_wait(&bar[stage], parity);
        const uint8_t* tsm = smem + stage * p.stage_bytes;
        const uint64_t r = tile * p.rows + tid;

        if (r < p.R) {
            const uint32_t P = p.P;
            const int32_t bstep = p.bsteps ? __ldg(p.bsteps + r) : p.bstep_implicit;
            // without ck only probes up to the budget step can decide the exit
            const uint32_t L = CK ? P : (bstep >= 0 ? static_cast<uint32_t>(bstep) + 1 : P);
            CotWin<W> st;
#pragma unroll
            for (int i = 0; i < (W > 0 ? W : 1); ++i) st.win[i] = 0;
            bool done = false;
            int32_t cstep = -1;
            uint32_t cid = 0;
            // snapshot of the window state at the budget step (CK mode runs past it)
            uint32_t b_nh = 0;
            bool b_has = false;
            uint32_t hw32 = 0;
            uint64_t hw64 = 0;

            for (uint32_t b = 0; b * 32u < L; ++b) {
                if (!CK && done) break;
                if ((b & 1u) == 0) {  // one u64 hesitation word covers two 32-probe boxes
                    hw64 = __ldg(p.hes + r * p.hw + (b >> 1));
                    hw32 = static_cast<uint32_t>(hw64);
                } else {
                    hw32 = static_cast<uint32_t>(hw64 >> 32);
                }
#pragma unroll
                for (uint32_t c = 0; c < 8; ++c) {
                    const uint32_t col = b * 32u + c * 4u;
                    if (col >= L) break;
                    if (!CK && done) break;
                    uint4 v4;
                    if (TMA) {
                        v4 = *reinterpret_cast<const uint4*>(tsm + b * p.rows * 128u + swz128(tid, c));
                    } else {
                        const uint32_t* src = p.ids + r * P + col;
                        v4.x = __ldg(src);
                        v4.y = col + 1 < P ? __ldg(src + 1) : 0u;
                        v4.z = col + 2 < P ? __ldg(src + 2) : 0u;
                        v4.w = col + 3 < P ? __ldg(src + 3) : 0u;
                    }
                    const uint32_t vv[4] = {v4.x, v4.y, v4.z, v4.w};
#pragma unroll
                    for (uint32_t e = 0; e < 4; ++e) {
                        const uint32_t q = col + e;
                        if (q >= L) break;
                        const uint32_t v = vv[e];
                        const bool hz = (hw32 >> (c * 4u + e)) & 1u;
                        if (!hz) {
                            ++st.usable;
                            st.last_nh = v;
                            st.has_nh = true;
                            int32_t agree = -1;
                            if (W > 0) {
#pragma unroll
                                for (int i = 0; i < W - 1; ++i) st.win[i] = st.win[i + 1];
                                st.win[W > 0 ? W - 1 : 0] = v;
                                if (st.usable >= W) {
                                    agree = 0;
#pragma unroll
                                    for (int i = 0; i < W; ++i) agree += st.win[i] == v ? 1 : 0;
                                }
                            } else if (st.usable >= p.w) {
                                // runtime window: scan back over the last w usable probes
                                agree = 0;
                                int32_t seen = 0;
                                for (int32_t qq = static_cast<int32_t>(q); qq >= 0 && seen < p.w; --qq) {
                                    const uint64_t h2 = __ldg(p.hes + r * p.hw + (qq >> 6));
                                    if ((h2 >> (qq & 63)) & 1ull) continue;
                                    ++seen;
                                    agree += cot_id<W, TMA>(p, tsm, tid, r, static_cast<uint32_t>(qq)) == v ? 1 : 0;
                                }
                            }
                            if (agree >= 0) {
                                st.last_agree = agree;
                                if (!done && agree >= p.amin) {  // C >= tau: exit certain
                                    done = true;
                                    cstep = static_cast<int32_t>(q);
                                    cid = v;  // the terminating record's answer
                                }
                            }
                        }
                        if (CK) {
                            const double cv = st.last_agree < 0
                                                  ? 0.0
                                                  : __ddiv_rn(static_cast<double>(st.last_agree),
                                                              static_cast<double>(p.w));
                            p.ck[r * P + q] = static_cast<float>(cv);
                            if (static_cast<int32_t>(q) == bstep) {
                                b_nh = st.last_nh;
                                b_has = st.has_nh;
                            }
                        }
                    }
                }
            }
            if (!CK) {
                b_nh = st.last_nh;
                b_has = st.has_nh;
            }
            int32_t ex = -1;
            uint8_t why = CDX_EXIT_CONTINUE;
            uint32_t fid;
            uint8_t low = 0;
            if (cstep >= 0 && (bstep < 0 || cstep <= bstep)) {
                ex = cstep;
                why = CDX_EXIT_CERTAIN;
                fid = cid;
            } else if (bstep >= 0) {  // token budget exhausted at bstep
                ex = bstep;
                why = CDX_EXIT_BUDGET;
                // latest non-hesitant answer up to bstep, else the latest answer
                fid = b_has ? b_nh : cot_id<W, TMA>(p, tsm, tid, r, static_cast<uint32_t>(bstep));
                low = b_has ? 0 : 1;
            } else {  // never exited: final answer of the full trace (criteria_external)
                fid = st.has_nh ? st.last_nh : cot_id<W, TMA>(p, tsm, tid, r, P - 1);
                low = st.has_nh ? 0 : 1;
            }
            p.exit_step[r] = ex;
            p.reason[r] = why;
            if (p.final_id) p.final_id[r] = fid;
            if (p.low_conf) p.low_conf[r] = low;
        }
        if (TMA) {
            __syncthreads();
            if (tid == 0) {
                const uint64_t nt = tile + static_cast<uint64_t>(p.stages) * stride;
                if (nt < p.ntiles) issue(nt, stage);
            }
            if (++stage == p.stages) {
                stage = 0;
                parity ^= 1u;
            }
        }
    }
}

// Lean variant for the common threshold regime a_min == w (tau > (w-1)/w, e.g. the paper's
// w=3, tau=0.9): the window agrees fully iff the last w usable answers are all equal, i.e.
// iff the run of equal consecutive usable answers ending here is >= w.  One compare and a
// counter per probe instead of a w-wide window; runtime w; no per-probe consistency output.
template <bool TMA>
__global__ void __launch_bounds__(128) cot_run_kernel(const __grid_constant__ CotParams p) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
    uint64_t* bar = reinterpret_cast<uint64_t*>(smem + p.stages * p.stage_bytes);
    const uint32_t tid = threadIdx.x;
    if (TMA) {
        if (tid == 0) {
            tma_prefetch_desc(&p.tmap);
            for (uint32_t s = 0; s < p.stages; ++s) mbar_init(&bar[s], 1);
            fence_mbar_init();
        }
        __syncthreads();
    }
    const uint64_t policy = policy_evict_first();
    const uint64_t stride = gridDim.x;
    auto issue = [&](uint64_t tile, uint32_t stage) {
        uint8_t* dst = smem + stage * p.stage_bytes;
        mbar_expect_tx(&bar[stage], p.stage_bytes);
        for (uint32_t b = 0; b < p.boxes; ++b)
            tma_load_2d(dst + b * p.rows * 128u, &p.tmap, static_cast<int32_t>(b * 32),
                        static_cast<int32_t>(tile * p.rows), &bar[stage], policy);
    };
    if (TMA && tid == 0)
        for (uint32_t s = 0; s < p.stages; ++s) {
            const uint64_t t = blockIdx.x + s * stride;
            if (t < p.ntiles) issue(t, s);
        }
    const int32_t w = p.w;
    uint32_t stage = 0, parity = 0;
    for (uint64_t tile = blockIdx.x; tile < p.ntiles; tile += stride) {
        const uint64_t r = tile * p.rows + tid;
        const bool live = r < p.R;
        // the first hesitation word is independent of the tile data: load it before the wait
        uint64_t hw64 = live ? __ldg(p.hes + r * p.hw) : 0ull;
        const int32_t bstep = (live && p.bsteps) ? __ldg(p.bsteps + r) : p.bstep_implicit;
        if (TMA) mbar_wait(&bar[stage], parity);
        const uint8_t* tsm = smem + stage * p.stage_bytes;
        if (live) {
            const uint32_t P = p.P;
            const uint32_t L = bstep >= 0 ? static_cast<uint32_t>(bstep) + 1 : P;
            int32_t run = 0, cstep = -1;
            uint32_t last = 0, cid = 0;
            bool has = false;
            for (uint32_t b = 0; b * 32u < L && cstep < 0; ++b) {
                if (b > 0 && (b & 1u) == 0) hw64 = __ldg(p.hes + r * p.hw + (b >> 1));
                const uint32_t hw32 = (b & 1u) ? static_cast<uint32_t>(hw64 >> 32) : static_cast<uint32_t>(hw64);
#pragma unroll
                for (uint32_t c = 0; c < 8; ++c) {
                    const uint32_t col = b * 32u + c * 4u;
                    if (col >= L || cstep >= 0) break;
                    uint4 v4;
                    if (TMA) {
                        v4 = *reinterpret_cast<const uint4*>(tsm + b * p.rows * 128u + swz128(tid, c));
                    } else {
                        const uint32_t* src = p.ids + r * P + col;
                        v4.x = __ldg(src);
                        v4.y = col + 1 < P ? __ldg(src + 1) : 0u;
                        v4.z = col + 2 < P ? __ldg(src + 2) : 0u;
                        v4.w = col + 3 < P ? __ldg(src + 3) : 0u;
                    }
                    const uint32_t vv[4] = {v4.x, v4.y, v4.z, v4.w};
#pragma unroll
                    for (uint32_t e = 0; e < 4; ++e) {
                        const uint32_t q = col + e;
                        const bool use = q < L && cstep < 0 && !((hw32 >> (c * 4u + e)) & 1u);
                        if (use) {
                            run = (has && vv[e] == last) ? run + 1 : 1;
                            last = vv[e];
                            has = true;
                            if (run >= w) {  // last w usable answers equal: C = 1 >= tau
                                cstep = static_cast<int32_t>(q);
                                cid = vv[e];
                            }
                        }
                    }
                }
            }
            int32_t ex = -1;
            uint8_t why = CDX_EXIT_CONTINUE;
            uint32_t fid;
            uint8_t low = 0;
            if (cstep >= 0) {  // certainty wins ties with the budget
                ex = cstep;
                why = CDX_EXIT_CERTAIN;
                fid = cid;
            } else if (bstep >= 0) {
                ex = bstep;
                why = CDX_EXIT_BUDGET;
                fid = has ? last : cot_id<1, TMA>(p, tsm, tid, r, static_cast<uint32_t>(bstep));
                low = has ? 0 : 1;
            } else {
                fid = has ? last : cot_id<1, TMA>(p, tsm, tid, r, P - 1);
                low = has ? 0 : 1;
            }
            p.exit_step[r] = ex;
            p.reason[r] = why;
            if (p.final_id) p.final_id[r] = fid;
            if (p.low_conf) p.low_conf[r] = low;
        }
        if (TMA) {
            __syncthreads();
            if (tid == 0) {
                const uint64_t nt = tile + static_cast<uint64_t>(p.stages) * stride;
                if (nt < p.ntiles) issue(nt, stage);
            }
            if (++stage == p.stages) {
                stage = 0;
                parity ^= 1u;
            }
        }
    }
}

// Branch-free variant of the run-length rule for P = 32 * NB probes (NB = 1..4; config B is
// P = 64): the budget step (implicit, or per request from cot_budget_steps) and the
// hesitation bits fold into a usable mask of P bits up front; the probes are then walked
// fully unrolled with selects only (no early exit, no data-dependent branches) and every
// probe whose run reaches w sets a bit in a P-bit hit mask, so the certain step is the
// mask's lowest bit.  Same decisions as cot_run_kernel (and therefore as the reference's
// prefix replay).
template <int NB>
__global__ void __launch_bounds__(128) cot_run64_kernel(const __grid_constant__ CotParams p) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
    uint64_t* bar = reinterpret_cast<uint64_t*>(smem + p.stages * p.stage_bytes);
    const uint32_t tid = threadIdx.x;
    if (tid == 0) {
        tma_prefetch_desc(&p.tmap);
        for (uint32_t s = 0; s < p.stages; ++s) mbar_init(&bar[s], 1);
        fence_mbar_init();
    }
    __syncthreads();
    const uint64_t policy = policy_evict_first();
    const uint64_t stride = gridDim.x;
    auto issue = [&](uint64_t tile, uint32_t stage) {
        uint8_t* dst = smem + stage * p.stage_bytes;
        mbar_expect_tx(&bar[stage], p.stage_bytes);
#pragma unroll
        for (uint32_t b = 0; b < NB; ++b)
            tma_load_2d(dst + b * p.rows * 128u, &p.tmap, static_cast<int32_t>(b * 32),
                        static_cast<int32_t>(tile * p.rows), &bar[stage], policy);
    };
    if (tid == 0)
        for (uint32_t s = 0; s < p.stages; ++s) {
            const uint64_t t = blockIdx.x + s * stride;
            if (t < p.ntiles) issue(t, s);
        }
    const int32_t w = p.w;
    const int32_t bstep_u = p.bstep_implicit;  // -1: the budget never fires within the trace
    uint32_t stage = 0, parity = 0;
    for (uint64_t tile = blockIdx.x; tile < p.ntiles; tile += stride) {
        const uint64_t r = tile * p.rows + tid;
        const bool live = r < p.R;
        const int32_t bstep = (live && p.bsteps) ? __ldg(p.bsteps + r) : bstep_u;
        // usable probes (not hesitant, <= the budget step) as NB 32-bit words
        uint32_t uw[NB];
        bool any_usable = false;
#pragma unroll
        for (int k = 0; k < NB; ++k) {
            const uint64_t hw = live ? __ldg(p.hes + r * p.hw + (k >> 1)) : ~0ull;
            const uint32_t nh = ~static_cast<uint32_t>(hw >> (32 * (k & 1)));
            const int32_t rel = bstep - 32 * k;  // budget step relative to this word
            const uint32_t lim = (bstep < 0 || rel >= 31) ? 0xffffffffu : (rel < 0 ? 0u : ((2u << rel) - 1u));
            uw[k] = live ? (nh & lim) : 0u;
            any_usable = any_usable || uw[k] != 0u;
        }
        mbar_wait(&bar[stage], parity);
        const uint8_t* tsm = smem + stage * p.stage_bytes;
        if (live) {
            int32_t run = 0;
            uint32_t last = 0;
            uint32_t hw[NB];
#pragma unroll
            for (int k = 0; k < NB; ++k) hw[k] = 0u;
#pragma unroll
            for (uint32_t c = 0; c < 8 * NB; ++c) {  // 16-byte chunks: box c/8, chunk c%8
                const uint4 v4 = *reinterpret_cast<const uint4*>(tsm + (c >> 3) * p.rows * 128u + swz128(tid, c & 7u));
                const uint32_t vv[4] = {v4.x, v4.y, v4.z, v4.w};
#pragma unroll
                for (uint32_t e = 0; e < 4; ++e) {
                    const uint32_t q = c * 4 + e;
                    const uint32_t bit = 1u << (q & 31u);  // compile-time mask: one LOP3 test
                    if (uw[q >> 5] & bit) {
                        run = vv[e] == last ? run + 1 : 1;  // first usable: run 0 -> 1
                        last = vv[e];
                        if (run >= w) hw[q >> 5] |= bit;
                    }
                }
            }
            int32_t cs = -1;  // first certain probe
#pragma unroll
            for (int k = NB - 1; k >= 0; --k)
                if (hw[k]) cs = 32 * k + __ffs(hw[k]) - 1;
            int32_t ex = -1;
            uint8_t why = CDX_EXIT_CONTINUE;
            uint32_t fid;
            uint8_t low = 0;
            if (cs >= 0) {  // certainty wins ties with the budget
                ex = cs;
                why = CDX_EXIT_CERTAIN;
                fid = *reinterpret_cast<const uint32_t*>(tsm + (cs >> 5) * p.rows * 128u + swz128(tid, (cs & 31u) >> 2) +
                                                         (cs & 3u) * 4u);
            } else {
                const uint32_t end = bstep >= 0 ? static_cast<uint32_t>(bstep) : 32u * NB - 1u;  // last probe seen
                if (bstep >= 0) {
                    ex = bstep;
                    why = CDX_EXIT_BUDGET;
                }
                low = any_usable ? 0 : 1;  // every probe up to the end hesitated
                fid = any_usable ? last
                                 : *reinterpret_cast<const uint32_t*>(tsm + (end >> 5) * p.rows * 128u +
                                                                      swz128(tid, (end & 31u) >> 2) + (end & 3u) * 4u);
            }
            p.exit_step[r] = ex;
            p.reason[r] = why;
            if (p.final_id) p.final_id[r] = fid;
            if (p.low_conf) p.low_conf[r] = low;
        }
        __syncthreads();
        if (tid == 0) {
            const uint64_t nt = tile + static_cast<uint64_t>(p.stages) * stride;
            if (nt < p.ntiles) issue(nt, stage);
        }
        if (++stage == p.stages) {
            stage = 0;
            parity ^= 1u;
        }
    }
}

// Explicit token offsets: the budget step of every request (first probe whose offset is
// >= max_tokens, hesitant or not, probe.cpp:77-85) in one coalesced pass, a warp
// per request and a ballot per 32 probes, instead of a serial offset scan in every lane.
__global__ void cot_budget_steps(const int64_t* __restrict__ off, uint64_t R, uint32_t P, int64_t max_tokens,
                                 int32_t* __restrict__ bsteps) {
    const uint32_t lane = threadIdx.x & 31u;
    const uint64_t nw = (static_cast<uint64_t>(gridDim.x) * blockDim.x) >> 5;
    for (uint64_t r = (blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x) >> 5; r < R; r += nw) {
        int32_t b = -1;
        for (uint32_t q0 = 0; q0 < P; q0 += 32) {
            const uint32_t q = q0 + lane;
            const uint32_t hit = __ballot_sync(0xffffffffu, q < P && __ldg(off + r * P + q) >= max_tokens);
            if (hit) {
                b = static_cast<int32_t>(q0 + __ffs(hit) - 1);
                break;
            }
        }
        if (lane == 0) bsteps[r] = b;
    }
}

template <bool TMA>
static void launch_cot_run(cdx_ctx* ctx, const CotParams& p, size_t smem) {
    auto k = cot_run_kernel<TMA>;
    if (TMA) cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k, p.rows, TMA ? smem : 0);
    if (per_sm < 1) per_sm = 1;
    const uint64_t grid = std::min<uint64_t>(p.ntiles, static_cast<uint64_t>(ctx->sm_count) * per_sm);
    k<<<static_cast<unsigned>(grid), p.rows, TMA ? smem : 0, ctx->stream>>>(p);
}

template <int W, bool TMA, bool CK>
static void launch_cot_k(cdx_ctx* ctx, const CotParams& p, size_t smem) {
    auto k = cot_exit_kernel<W, TMA, CK>;
    if (TMA) cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k, p.rows, TMA ? smem : 0);
    if (per_sm < 1) per_sm = 1;
    const uint64_t grid = std::min<uint64_t>(p.ntiles, static_cast<uint64_t>(ctx->sm_count) * per_sm);
    k<<<static_cast<unsigned>(grid), p.rows, TMA ? smem : 0, ctx->stream>>>(p);
}

template <int W>
static void launch_cot(cdx_ctx* ctx, const CotParams& p, bool tma, bool ck, size_t smem) {
    if (tma) {
        if (ck) launch_cot_k<W, true, true>(ctx, p, smem);
        else launch_cot_k<W, true, false>(ctx, p, smem);
    } else {
        if (ck) launch_cot_k<W, false, true>(ctx, p, smem);
        else launch_cot_k<W, false, false>(ctx, p, smem);
    }
}

}  // namespace cdx

extern "C" int cdx_cot_exit(cdx_ctx* ctx, const uint32_t* ids, const uint64_t* hes, const int64_t* offsets,
                            uint64_t R, uint32_t P, const cdx_probe_cfg* cfg, int32_t* exit_step,
                            uint8_t* reason, uint32_t* final_id, uint8_t* low_conf, float* ck) {
    using namespace cdx;
    CDX_NVTX("cdx_cot_exit");
    if (!ctx) return CDX_EINVAL;
    if (!cfg) return set_error(ctx, CDX_EINVAL, "probe: null config");
    // ProbeConfig::validate, probe.cpp:19-25
    if (cfg->interval_tokens < 1) return set_error(ctx, CDX_EINVAL, "probe: interval_tokens must be >= 1");
    if (cfg->window < 1) return set_error(ctx, CDX_EINVAL, "probe: window must be >= 1");
    if (cfg->threshold <= 0.0 || cfg->threshold > 1.0)
        return set_error(ctx, CDX_EINVAL, "probe: threshold must be in (0,1]");
    if (cfg->max_tokens < 1) return set_error(ctx, CDX_EINVAL, "probe: max_tokens must be >= 1");
    if (P == 0) return set_error(ctx, CDX_EINVAL, "final_answer: empty trace");
    if (!ids || !hes || !exit_step || !reason) return set_error(ctx, CDX_EINVAL, "cot_exit: null pointer");
    if (R == 0) return CDX_OK;

    CotParams p{};
    p.ids = ids;
    p.hes = hes;
    p.offsets = offsets;
    p.exit_step = exit_step;
    p.reason = reason;
    p.final_id = final_id;
    p.low_conf = low_conf;
    p.ck = ck;
    p.R = R;
    p.P = P;
    p.hw = (P + 63) / 64;
    p.boxes = (P + 31) / 32;
    p.w = cfg->window;
    int amin = cfg->window + 1;
    for (int a = 0; a <= cfg->window; ++a)
        if (static_cast<double>(a) / static_cast<double>(cfg->window) >= cfg->threshold) {
            amin = a;
            break;
        }
    p.amin = amin;
    p.max_tokens = cfg->max_tokens;
    // implicit offsets (p+1)*interval: first probe with offset >= max_tokens
    {
        const int64_t I = cfg->interval_tokens;
        const int64_t k = (cfg->max_tokens + I - 1) / I;  // smallest p+1 with (p+1)*I >= max
        p.bstep_implicit = (k - 1 < static_cast<int64_t>(P)) ? static_cast<int32_t>(k - 1) : -1;
    }
    p.bsteps = nullptr;
    if (offsets) {  // per-request budget steps in one coalesced pass
        auto* bs = static_cast<int32_t*>(scratch(ctx, R * 4 + 256));
        if (!bs) return set_error(ctx, CDX_ECUDA, "cot_exit: scratch allocation failed");
        const uint64_t want = (R + 7) / 8;  // 8 warps (requests) per 256-thread block
        cot_budget_steps<<<static_cast<unsigned>(std::min<uint64_t>(want, static_cast<uint64_t>(ctx->sm_count) * 16)),
                           256, 0, ctx->stream>>>(offsets, R, P, cfg->max_tokens, bs);
        CDX_CHECK_LAUNCH(ctx, "cot_exit(budget steps)");
        p.bsteps = bs;
    }
    bool tma = (P % 4 == 0) && (reinterpret_cast<uintptr_t>(ids) % 16 == 0) && P <= 512 && R <= 0x7fffffffull;
    // rows (= threads) per CTA and ring depth: small single-stage CTAs keep ~28 warps
    // per SM resident; other CTAs on the SM overlap each one's TMA wait (tuned on B200)
    // run path (P a multiple of 32 up to 128, a_min == w, no ck): 128-request CTAs with a 2-deep ring
    // measured best on B200 (51 us on config B vs 55 us for 64 x 1)
    const bool run64 = P % 32 == 0 && P <= 128 && !ck && amin == cfg->window;
    uint32_t rows = run64 ? 128 : 64, stages = run64 ? 2 : 1;
    if (const char* e = getenv("CDX_COT_ROWS")) rows = static_cast<uint32_t>(atoi(e));
    if (const char* e = getenv("CDX_COT_STAGES")) stages = static_cast<uint32_t>(atoi(e));
    rows = std::max<uint32_t>(32, std::min<uint32_t>(128, rows / 32 * 32));
    stages = std::max<uint32_t>(1, std::min<uint32_t>(COT_MAX_STAGES, stages));
    if (tma) {
        while (rows > 32 && static_cast<uint64_t>(rows) * p.boxes * 128u * stages > 96u * 1024u) rows -= 32;
        while (stages > 1 && static_cast<uint64_t>(rows) * p.boxes * 128u * stages > 200u * 1024u) --stages;
        p.rows = rows;
        p.stage_bytes = rows * p.boxes * 128u;
        p.stages = stages;
        // the descriptor depends only on (ids, R, P, rows): re-encode only when they change
        // (a repeated batch then costs one launch of host work; config B's kernel is ~47 us)
        struct TmapCache {
            const void* ids = nullptr;
            uint64_t R = 0;
            uint32_t P = 0, rows = 0;
            CUtensorMap map;
        };
        static thread_local TmapCache tc;
        if (tc.ids == ids && tc.R == R && tc.P == P && tc.rows == rows) {
            p.tmap = tc.map;
        } else {
            tma = encode_tmap_2d(&p.tmap, ids, P, R, static_cast<uint64_t>(P) * 4u, 32, rows,
                                 CU_TENSOR_MAP_DATA_TYPE_UINT32, CU_TENSOR_MAP_SWIZZLE_128B);
            if (tma) tc = TmapCache{ids, R, P, rows, p.tmap};
        }
    }
    if (!tma) {
        p.rows = 128;
        p.stages = 1;
        p.stage_bytes = 0;
    }
    p.ntiles = (R + p.rows - 1) / p.rows;
    const size_t smem = tma ? static_cast<size_t>(p.stages) * p.stage_bytes + 1024 + 8 * COT_MAX_STAGES : 0;
    const bool want_ck = ck != nullptr;
    const char* impl = getenv("CDX_COT_IMPL");
    if (!want_ck && amin == cfg->window && !(impl && impl[0] == 'w')) {
        if (tma && P % 32 == 0 && P <= 128 && !(impl && impl[0] == 'r')) {
            auto k = P == 64 ? cot_run64_kernel<2>
                             : (P == 32 ? cot_run64_kernel<1> : (P == 96 ? cot_run64_kernel<3> : cot_run64_kernel<4>));
            // attribute + occupancy per (kernel, device, shape), not per call
            struct OccCache {
                const void* k = nullptr;
                int dev = -1;
                uint32_t rows = 0;
                size_t smem = 0;
                int per_sm = 0;
            };
            static thread_local OccCache oc;
            int per_sm = 0;
            if (oc.k == reinterpret_cast<const void*>(k) && oc.dev == ctx->device && oc.rows == p.rows && oc.smem == smem) {
                per_sm = oc.per_sm;
            } else {
                cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
                cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k, p.rows, smem);
                oc = OccCache{reinterpret_cast<const void*>(k), ctx->device, p.rows, smem, per_sm};
            }
            const uint64_t grid = std::min<uint64_t>(p.ntiles, static_cast<uint64_t>(ctx->sm_count) * std::max(per_sm, 1));
            k<<<static_cast<unsigned>(grid), p.rows, smem, ctx->stream>>>(p);
            CDX_CHECK_LAUNCH(ctx, "cot_exit(run64)");
            return CDX_OK;
        }
        if (tma) launch_cot_run<true>(ctx, p, smem);
        else launch_cot_run<false>(ctx, p, smem);
        CDX_CHECK_LAUNCH(ctx, "cot_exit(run)");
        return CDX_OK;
    }
    switch (cfg->window) {
        case 1: launch_cot<1>(ctx, p, tma, want_ck, smem); break;
        case 2: launch_cot<2>(ctx, p, tma, want_ck, smem); break;
        case 3: launch_cot<3>(ctx, p, tma, want_ck, smem); break;
        case 4: launch_cot<4>(ctx, p, tma, want_ck, smem); break;
        case 5: launch_cot<5>(ctx, p, tma, want_ck, smem); break;
        case 6: launch_cot<6>(ctx, p, tma, want_ck, smem); break;
        case 7: launch_cot<7>(ctx, p, tma, want_ck, smem); break;
        case 8: launch_cot<8>(ctx, p, tma, want_ck, smem); break;
        default: launch_cot<0>(ctx, p, tma, want_ck, smem); break;
    }
    CDX_CHECK_LAUNCH(ctx, "cot_exit");
    return CDX_OK;
}
