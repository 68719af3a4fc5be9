// k_sc.cu — K2: Self-Consistency certaindex over (request, probe) rows of S answers.
//
// Replaces, per row, metrics::certaindex_entropy(metrics::cluster_exact(row)) and
// metrics::combined_meets_thresholds (metrics.cpp:21-37, 107-125, 159-171) — the SC branch
// of ProgramDriver::update_certaindex (runtime.cpp:266-271) evaluated at every probe step.
//
// Data path (HBM-bound; no tensor cores: nothing here is a contraction):
//   ids u32[R][P][S] is cut into GROUPS of 32 consecutive probe rows of one request
//   (<= 4 KB, contiguous).  Every warp streams its own groups through a private ring of
//   shared-memory stages filled by 1-D bulk copies (cp.async.bulk, evict-first, one
//   mbarrier per stage): no CTA-wide barrier, so warps never wait for each other.
//   Per group: __match_any_sync over each row's S lanes = exact-match clusters; the lowest
//   lane of a match set is the cluster's first-seen answer (cluster order of metrics.cpp:
//   29-31) and popc(match) its size.  The owner lane of each row then folds the entropy in
//   FP64 in first-seen order: h -= term[size], with term[c] = (c/S)*log(c/S) built on the
//   host with the reference's libm, so the device only does IEEE subtract/divide and
//   reproduces the reference bits; clamp; thresholds on the FP64 value; fp32 store and one
//   meets word per group.
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <vector>

#include "k_alloc.cuh"
#include "k_sc.cuh"

namespace cdx {

// ALU peel engine for a runtime S (SB = S rounded up to a multiple of 8): lane = row, the
// row's S ids in registers, clusters peeled in first-seen order with S compares each
// (ISETP + predicated OR).  Rows with more than RT_PEEL_MAX clusters report *more and the
// warp redoes the group with the match engine below.  The same fold as every engine: the
// composition table for S <= 16, else h -= term[size] in first-seen order in FP64.
constexpr uint32_t RT_PEEL_MAX = 8;

__device__ __forceinline__ void or_if_eq_rt(uint32_t& a, uint32_t x, uint32_t v, uint32_t bit) {
    asm("{\n\t.reg .pred p;\n\tsetp.eq.u32 p, %1, %2;\n\t@p or.b32 %0, %0, %3;\n\t}"
        : "+r"(a)
        : "r"(x), "r"(v), "r"(bit));
}
template <int SB>
__device__ __forceinline__ uint32_t eq_mask_rt(const uint32_t (&x)[SB], uint32_t v) {
    uint32_t a0 = 0, a1 = 0, a2 = 0, a3 = 0;
#pragma unroll
    for (uint32_t e = 0; e < SB; e += 4) {
        or_if_eq_rt(a0, x[e], v, 1u << e);
        or_if_eq_rt(a1, x[e + 1], v, 2u << e);
        or_if_eq_rt(a2, x[e + 2], v, 4u << e);
        or_if_eq_rt(a3, x[e + 3], v, 8u << e);
    }
    return (a0 | a1) | (a2 | a3);
}

template <int SB>
__device__ __forceinline__ double alu_row_rt(const uint32_t* __restrict__ row, uint32_t S,
                                             const double* __restrict__ term, double logn,
                                             const double* __restrict__ comp, bool* more, uint32_t& maxc) {
    uint32_t x[SB];
    if ((S & 3u) == 0) {  // 16-byte rows: vector loads (rows of a group are 16B-aligned)
#pragma unroll
        for (uint32_t j = 0; j < SB / 4; ++j) {
            const uint4 v = j * 4 < S ? reinterpret_cast<const uint4*>(row)[j] : make_uint4(0, 0, 0, 0);
            x[4 * j] = v.x;
            x[4 * j + 1] = v.y;
            x[4 * j + 2] = v.z;
            x[4 * j + 3] = v.w;
        }
    } else {  // odd strides are bank-conflict free for scalar loads
#pragma unroll
        for (uint32_t e = 0; e < SB; ++e) x[e] = e < S ? row[e] : 0u;
    }
    const uint32_t valid = S >= 32 ? 0xffffffffu : ((1u << S) - 1u);
    uint32_t eq = eq_mask_rt<SB>(x, x[0]) & valid;
    uint32_t un = valid & ~eq;
    maxc = __popc(eq);  // largest cluster so far (majority fraction = maxc / S)
    if (un == 0) return 1.0;  // one cluster holds every answer: H~ = 1 exactly
    uint32_t peeled = 1;
    if (comp) {  // S <= 16: composition code -> table
        uint32_t cum = maxc, code = 1u << (cum - 1);
        while (un) {
            if (peeled == RT_PEEL_MAX) {
                *more = true;
                return 0.0;
            }
            ++peeled;
            eq = eq_mask_rt<SB>(x, row[__ffs(un) - 1]) & valid;
            un &= ~eq;
            const uint32_t c = __popc(eq);
            maxc = max(maxc, c);
            cum += c;
            code |= 1u << (cum - 1);
        }
        return __ldg(comp + (code & ((1u << (S - 1)) - 1u)));
    }
    double h = __dsub_rn(0.0, term[maxc]);
    while (un) {
        if (peeled == RT_PEEL_MAX) {
            *more = true;
            return 0.0;
        }
        ++peeled;
        eq = eq_mask_rt<SB>(x, row[__ffs(un) - 1]) & valid;
        un &= ~eq;
        const uint32_t c = __popc(eq);
        maxc = max(maxc, c);
        h = __dsub_rn(h, term[c]);  // h -= p*log(p), first-seen order
    }
    h = (0.0 < h) ? h : 0.0;
    const double v = __ddiv_rn(__dsub_rn(logn, h), logn);
    return v < 0.0 ? 0.0 : (1.0 < v ? 1.0 : v);
}

// One warp, one group of up to 32 rows of one request: cluster every row with a warp
// match, then fold each row's entropy on its owner lane (lane == row within the group).
// SCT = compile-time S (a divisor of 32: 1,2,4,8,16,32), or 0 for a runtime S <= 32.
//
// Cluster sizes travel through shared memory as one byte per (row, sample): the cluster's
// size at its first-seen sample, 0 elsewhere ([row][32] bytes per warp).  The owner lane
// then walks its row's nonzero bytes in sample order = first-seen cluster order.  The
// byte stores of one row land in one 32-byte segment (no bank conflicts).
template <int SCT>
__device__ __forceinline__ void sc_group(const ScParams& p, const uint32_t* __restrict__ base, uint32_t rows,
                                         uint8_t* __restrict__ cntw, const double* __restrict__ term, uint32_t lane,
                                         uint64_t req, uint32_t row0, uint32_t g) {
    const uint32_t S = SCT ? static_cast<uint32_t>(SCT) : p.S;
    const uint32_t rpi = 32u / S;  // rows per match iteration
    const uint32_t smask = S >= 32 ? 0xffffffffu : ((1u << S) - 1u);
    const uint32_t sub = lane / S, s = lane - sub * S;
    const bool lane_ok = sub < rpi;
    const uint32_t subm = lane_ok ? (smask << (sub * S)) : 0u;
    const uint32_t ltm = (1u << lane) - 1u;  // lanes below me
    uint8_t* my_cnt = cntw + sub * 32u + s;  // byte (row = it*rpi + sub, sample s)
    if (SCT == 0) {  // runtime S: the ALU engine first, the match engine only for its overflow
        bool more = false;
        double hc = 1.0;
        uint32_t maxc = S;
        if (lane < rows) {
            const uint32_t* rowp = base + lane * S;
            if (S <= 8) hc = alu_row_rt<8>(rowp, S, term, p.logn, p.comp, &more, maxc);
            else if (S <= 16) hc = alu_row_rt<16>(rowp, S, term, p.logn, p.comp, &more, maxc);
            else if (S <= 24) hc = alu_row_rt<24>(rowp, S, term, p.logn, p.comp, &more, maxc);
            else hc = alu_row_rt<32>(rowp, S, term, p.logn, p.comp, &more, maxc);
        }
        if (!__any_sync(0xffffffffu, more)) {
            bool meets = false;
            if (lane < rows) {
                meets = sc_meets(p, hc, maxc);
                if (p.hcert) p.hcert[req * p.P + row0 + lane] = static_cast<float>(hc);
                if (p.maj) p.maj[req * p.P + row0 + lane] = p.maj_tab[maxc];
            }
            const uint32_t mw = __ballot_sync(0xffffffffu, meets);
            if (lane == 0 && p.meets) p.meets[req * p.words + g] = mw;
            __syncwarp();
            return;
        }
    }
    if (SCT != 0 && rows == 32) {
        // full group, S | 32: row (it*rpi + sub) element s sits at word it*32 + lane
#pragma unroll 8
        for (uint32_t it = 0; it < static_cast<uint32_t>(SCT ? SCT : 1); ++it) {
            const uint32_t m = __match_any_sync(0xffffffffu, base[it * 32u + lane]) & subm;
            const bool leader = (m & ltm) == 0u;  // first-seen answer of its cluster
            my_cnt[it * rpi * 32u] = leader ? static_cast<uint8_t>(__popc(m)) : uint8_t(0);
        }
    } else {
        const uint32_t iters = (rows + rpi - 1) / rpi;
        for (uint32_t it = 0; it < iters; ++it) {
            const uint32_t rloc = it * rpi + sub;
            const bool act = lane_ok && rloc < rows;
            const uint32_t v = act ? base[rloc * S + s] : 0xffffffffu;
            const uint32_t m = __match_any_sync(0xffffffffu, v) & subm;
            const bool leader = (m & ltm) == 0u;
            if (act) my_cnt[it * rpi * 32u] = leader ? static_cast<uint8_t>(__popc(m)) : uint8_t(0);
        }
    }
    __syncwarp();
    bool meets = false;
    if (lane < rows) {
        double hc = 1.0;  // metrics.cpp:121: a single path is fully certain
        uint32_t maxc = S;
        const uint4* rowp = reinterpret_cast<const uint4*>(cntw + lane * 32u);
        const uint4 a = rowp[0];
        // one cluster holding every answer: H = -(1*log 1) = 0 exactly, so H~ = 1 exactly
        if (S > 1 && (a.x & 0xffu) != S) {
            const uint4 b = S > 16 ? rowp[1] : make_uint4(0, 0, 0, 0);
            const uint32_t wv[8] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w};
            maxc = 0;  // largest size byte among the row's S slots (the rest are stale)
#pragma unroll
            for (uint32_t k = 0; k < 8; ++k) {
                if (k * 4u >= S) break;
                const uint32_t keep = S >= k * 4u + 4u ? 0xffffffffu : ((1u << ((S - k * 4u) * 8u)) - 1u);
                maxc = __vmaxu4(maxc, wv[k] & keep);
            }
            maxc = __vmaxu4(maxc, maxc >> 16);
            maxc = __vmaxu4(maxc, maxc >> 8) & 0xffu;
            double h = 0.0;
            if (SCT != 0) {
                // Branch-free fold over every sample slot in order: term[0] = +0.0 and h >= 0,
                // so a non-leader slot subtracts +0.0, which leaves h bit-identical.  (Data-
                // dependent loops here cost divergence-unit cycles that the match needs.)
#pragma unroll
                for (uint32_t k = 0; k < 8; ++k) {
                    if (k * 4u >= S) break;
#pragma unroll
                    for (uint32_t j = 0; j < 4; ++j) {
                        if (k * 4u + j >= S) break;
                        h = __dsub_rn(h, term[__byte_perm(wv[k], 0, 0x4440 + j)]);  // h -= p*log(p)
                    }
                }
            } else {
#pragma unroll
                for (uint32_t k = 0; k < 8; ++k) {
                    if (k * 4u >= S) break;
                    // keep only the bytes of samples < S (the rest of the 32-byte row is stale)
                    const uint32_t keep = S >= k * 4u + 4u ? 0xffffffffu : ((1u << ((S - k * 4u) * 8u)) - 1u);
                    uint32_t x = wv[k] & keep;
                    while (x) {  // nonzero bytes in sample order = first-seen cluster order
                        const uint32_t sh = static_cast<uint32_t>(__ffs(x) - 1) & ~7u;
                        const uint32_t c = (x >> sh) & 0xffu;
                        x &= ~(0xffu << sh);
                        h = __dsub_rn(h, term[c]);  // h -= p*log(p), metrics.cpp:113-116
                    }
                }
            }
            h = (0.0 < h) ? h : 0.0;  // std::max(0.0, h)
            const double v = __ddiv_rn(__dsub_rn(p.logn, h), p.logn);
            hc = v < 0.0 ? 0.0 : (1.0 < v ? 1.0 : v);  // std::clamp
        }
        meets = sc_meets(p, hc, maxc);
        if (p.hcert) p.hcert[req * p.P + row0 + lane] = static_cast<float>(hc);
        if (p.maj) p.maj[req * p.P + row0 + lane] = p.maj_tab[maxc];
    }
    const uint32_t mw = __ballot_sync(0xffffffffu, meets);
    if (lane == 0 && p.meets) p.meets[req * p.words + g] = mw;
    __syncwarp();
}

// Warp-autonomous streaming: warp w of the grid owns groups w, w + nwarps, ...; each warp
// keeps `stages` groups in flight in its private ring.
template <int SCT>
__global__ void __launch_bounds__(SC_MAX_WARPS * 32) sc_certaindex_kernel(const __grid_constant__ ScParams p) {
    extern __shared__ __align__(128) uint8_t smem[];
    const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const uint32_t nw_cta = blockDim.x >> 5;
    const uint32_t S = SCT ? static_cast<uint32_t>(SCT) : p.S;
    // per-warp layout: [stages][4 KB ring] [1 KB counts]; CTA tail: term table, mbarriers
    uint8_t* wbase = smem + warp * (p.stages * SC_GROUP_BYTES + 1024u);
    uint8_t* cntw = wbase + p.stages * SC_GROUP_BYTES;
    double* term = reinterpret_cast<double*>(smem + nw_cta * (p.stages * SC_GROUP_BYTES + 1024u));
    uint64_t* bar = reinterpret_cast<uint64_t*>(term + 34) + warp * SC_MAX_STAGES;

    if (threadIdx.x < 33) term[threadIdx.x] = p.term[threadIdx.x];
    if (lane == 0) {
        for (uint32_t s = 0; s < p.stages; ++s) mbar_init(&bar[s], 1);
        fence_mbar_init();
    }
    __syncthreads();  // the only CTA-wide barrier: term table + barrier init

    const uint64_t policy = policy_evict_first();
    const uint64_t gw = static_cast<uint64_t>(blockIdx.x) * nw_cta + warp;
    const uint64_t nwarps = static_cast<uint64_t>(gridDim.x) * nw_cta;
    // group G = (request, g) with G = request * words + g; walk it incrementally (no 64-bit
    // divisions in the loop): one step = nwarps groups = (dq requests, dr groups)
    const uint64_t dq = nwarps / p.words;
    const uint32_t dr = static_cast<uint32_t>(nwarps - dq * p.words);
    struct Cursor {
        uint64_t req;
        uint32_t g;
    };
    auto advance = [&](Cursor& c, uint32_t times) {
        for (uint32_t i = 0; i < times; ++i) {
            c.req += dq;
            c.g += dr;
            if (c.g >= p.words) {
                c.g -= p.words;
                ++c.req;
            }
        }
    };
    // a group goes by bulk copy when its bytes start 16B-aligned and fill whole 16-byte
    // units (every group when S % 4 == 0; full groups of any S when P % 4 == 0)
    auto bulkable = [&](const Cursor& c) {
        const uint32_t rows = min(32u, p.P - c.g * 32u);
        return p.bulk_ok && (((c.req * p.P + c.g * 32u) * S) & 3u) == 0 && ((rows * S) & 3u) == 0;
    };
    auto issue = [&](const Cursor& c, uint32_t stage) {  // lane 0 only
        const uint32_t rows = min(32u, p.P - c.g * 32u);
        mbar_expect_tx(&bar[stage], rows * S * 4u);
        bulk_g2s(wbase + stage * SC_GROUP_BYTES, p.ids + (c.req * p.P + c.g * 32u) * S, rows * S * 4u, &bar[stage],
                 policy);
    };
    Cursor cur{gw / p.words, static_cast<uint32_t>(gw % p.words)};
    Cursor pre = cur;  // prefetch cursor, stages groups ahead
    if (lane == 0)
        for (uint32_t s = 0; s < p.stages; ++s) {
            if (pre.req < p.R && bulkable(pre)) issue(pre, s);
            advance(pre, 1);
        }

    uint32_t stage = 0, parity = 0;
    while (cur.req < p.R) {
        const uint32_t rows = min(32u, p.P - cur.g * 32u);
        uint32_t* buf = reinterpret_cast<uint32_t*>(wbase + stage * SC_GROUP_BYTES);
        if (bulkable(cur)) {
            mbar_wait(&bar[stage], parity);
        } else {  // misaligned base or a group of odd size: plain coalesced loads
            const uint32_t* src = p.ids + (cur.req * p.P + cur.g * 32u) * S;
            for (uint32_t i = lane; i < rows * S; i += 32) buf[i] = __ldg(src + i);
            __syncwarp();
        }
        sc_group<SCT>(p, buf, rows, cntw, term, lane, cur.req, cur.g * 32u, cur.g);
        // sc_group ends with __syncwarp: every lane is done with this stage's data
        if (lane == 0) {
            if (pre.req < p.R && bulkable(pre)) issue(pre, stage);
            advance(pre, 1);
        }
        advance(cur, 1);
        if (++stage == p.stages) {
            stage = 0;
            parity ^= 1u;
        }
    }
}

// Full clusterings per row (façade path of metrics::cluster_exact): one warp per 32/S rows.
__global__ void cluster_rows_kernel(const uint32_t* __restrict__ ids, uint64_t rows, uint32_t S,
                                    uint32_t* __restrict__ ncl, uint32_t* __restrict__ leader,
                                    uint32_t* __restrict__ size) {
    const uint32_t lane = threadIdx.x & 31;
    const uint32_t rpi = 32u / S;
    const uint32_t smask = S == 32 ? 0xffffffffu : ((1u << S) - 1u);
    const uint32_t sub = lane / S, s = lane - sub * S;
    const bool lane_ok = sub < rpi;
    const uint32_t subm = lane_ok ? (smask << (sub * S)) : 0u;
    const uint64_t warps = (static_cast<uint64_t>(gridDim.x) * blockDim.x) >> 5;
    for (uint64_t wr = (blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x) >> 5; wr * rpi < rows;
         wr += warps) {
        const uint64_t row = wr * rpi + sub;
        const bool act = lane_ok && row < rows;
        const uint32_t v = act ? ids[row * S + s] : 0xffffffffu;
        const uint32_t m = __match_any_sync(0xffffffffu, v) & subm;
        const bool lead = act && (static_cast<uint32_t>(__ffs(m) - 1) == lane);
        const uint32_t lm = __ballot_sync(0xffffffffu, lead) & subm;
        if (lead) {
            const uint32_t k = __popc(lm & ((1u << lane) - 1u));
            leader[row * S + k] = s;
            size[row * S + k] = __popc(m);
        }
        if (act && s == 0) ncl[row] = __popc(lm);
    }
}

// Entropy of explicit clusterings from a triangular term table T[n][c] (n <= max_n).
// totals (nullable): Clustering::total per row; absent -> the sum of the sizes (what
// cluster_exact produces).  Validation in the reference's order (metrics.cpp:107-112):
// total < 1 or no clusters -> "invalid clustering"; a cluster of size < 1 -> "empty
// cluster".  A cluster larger than its total (p > 1) is rejected as an invalid clustering:
// the host term table only holds c <= n (documented deviation).
__global__ void entropy_sizes_kernel(const uint32_t* __restrict__ sizes, const uint32_t* __restrict__ m,
                                     const uint32_t* __restrict__ totals, uint64_t rows, uint32_t max_m,
                                     const double* __restrict__ tri, const double* __restrict__ logs, uint32_t max_n,
                                     double* H, double* Hc, int* bad) {
    for (uint64_t r = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; r < rows;
         r += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
        const uint32_t mm = m[r];
        uint64_t n = 0;
        if (mm < 1 || mm > max_m || (totals && totals[r] < 1)) {
            set_dev_err(bad, DEV_BAD_CLUSTERING);
            continue;
        }
        bool empty = false, big = false;
        for (uint32_t k = 0; k < mm; ++k) {
            const uint32_t c = sizes[r * max_m + k];
            empty |= c < 1;
            n += c;
        }
        if (empty) {
            set_dev_err(bad, DEV_EMPTY_CLUSTER);
            continue;
        }
        if (totals) {
            for (uint32_t k = 0; k < mm; ++k) big |= sizes[r * max_m + k] > totals[r];
            n = totals[r];
        }
        if (big || n > max_n) {
            set_dev_err(bad, DEV_BAD_CLUSTERING);
            continue;
        }
        const double* T = tri + (n * (n + 1)) / 2;  // row n holds c = 0..n
        double h = 0.0;
        for (uint32_t k = 0; k < mm; ++k) h = __dsub_rn(h, T[sizes[r * max_m + k]]);
        h = (0.0 < h) ? h : 0.0;
        if (H) H[r] = h;
        if (Hc) {
            double hc = 1.0;
            if (n != 1) {
                const double v = __ddiv_rn(__dsub_rn(logs[n], h), logs[n]);
                hc = v < 0.0 ? 0.0 : (1.0 < v ? 1.0 : v);
            }
            Hc[r] = hc;
        }
    }
}

int check_thresholds(cdx_ctx* ctx, const cdx_threshold* th, uint32_t n_th, const bool present[5]) {
    static const char* names[5] = {"certaindex_entropy", "certaindex_reward", "mean_output_length",
                                   "mean_norm_logprob", "majority_fraction"};
    if (n_th > MAX_TH) return set_error(ctx, CDX_EINVAL, "thresholds: at most 8 per call");
    if (n_th && !th) return set_error(ctx, CDX_EINVAL, "thresholds: null array");
    for (uint32_t i = 0; i < n_th; ++i) {
        if (th[i].signal > CDX_SIG_MAJORITY || th[i].dir > 1) return set_error(ctx, CDX_EINVAL, "thresholds: bad enum");
        if (!present[th[i].signal])
            return set_error(ctx, CDX_EINVAL,
                             std::string("combined_meets_thresholds: signal '") + names[th[i].signal] +
                                 "' absent");
    }
    return CDX_OK;
}

void majority_interval(const cdx_threshold* th, uint32_t n_th, uint32_t S, uint32_t* lo, uint32_t* hi) {
    *lo = S + 1;
    *hi = 0;
    for (uint32_t c = 0; c <= S; ++c) {
        const double v = static_cast<double>(c) / static_cast<double>(S);
        bool ok = true;
        for (uint32_t i = 0; i < n_th; ++i)
            if (th[i].signal == CDX_SIG_MAJORITY)
                ok = ok && (th[i].dir == CDX_DIR_GE ? v >= th[i].cutoff : v <= th[i].cutoff);
        if (ok) {  // v is monotone in c and each compare is a half-line: the set is an interval
            *lo = std::min(*lo, c);
            *hi = c;
        }
    }
}

template <int SCT>
void launch_sc(cdx_ctx* ctx, const ScParams& p, uint32_t warps_per_cta) {
    const size_t smem = static_cast<size_t>(warps_per_cta) * (p.stages * SC_GROUP_BYTES + 1024u) + 34 * 8 +
                        SC_MAX_WARPS * SC_MAX_STAGES * 8;
    cudaFuncSetAttribute(sc_certaindex_kernel<SCT>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, sc_certaindex_kernel<SCT>, warps_per_cta * 32, smem);
    if (per_sm < 1) per_sm = 1;
    const uint64_t want = (p.ngroups + warps_per_cta - 1) / warps_per_cta;
    const uint64_t grid = std::min<uint64_t>(want, static_cast<uint64_t>(ctx->sm_count) * per_sm);
    sc_certaindex_kernel<SCT><<<static_cast<unsigned>(grid), warps_per_cta * 32, smem, ctx->stream>>>(p);
}

// ---- wide rows (32 < S <= SC_WIDE_MAX): a warp per row ----------------------------------
// The row streams through the warp 32 answers at a time.  Per round, equal values find
// each other with MATCH; the round's first occurrence of each value looks it up in the
// warp's shared-memory hash (value -> first-seen ordinal); values not seen before take
// ordinals in lane order = first-seen order, one insertion at a time.  The owner (lane 0)
// folds h -= T_S[count] over ordinals 0..m-1 in FP64 (term row T_S from the host libm),
// clamps, applies the thresholds and ORs the row's meets bit into its word.
constexpr uint32_t SC_WIDE_MAX = 4096;
constexpr uint32_t SC_WIDE_WARPS = 4;

struct WideParams {
    const uint32_t* ids;
    float* hcert;
    float* maj;         // majority fraction f32 (nullable)
    uint32_t maj_lo, maj_hi;
    int maj_th;
    uint32_t* meets;
    const double* tab;  // T_S[0..S]
    double logn;
    uint64_t rows;      // R * P
    uint32_t P, S, words, cap_log2;
    int n_th;
    uint8_t th_sig[MAX_TH];
    uint8_t th_dir[MAX_TH];
    double th_cut[MAX_TH];
};

// One row of S answers clustered by the warp: ordinal k (first-seen order) gets its count in
// cnt[k] and, when `first` is given, the sample index of its first answer.  Returns m.
__device__ uint32_t wide_cluster(const uint32_t* __restrict__ src, uint32_t S, uint32_t cap_log2,
                                 uint32_t* __restrict__ hkey, uint32_t* __restrict__ hord,
                                 uint32_t* __restrict__ cnt, uint32_t* __restrict__ first, uint32_t lane) {
    const uint32_t cap = 1u << cap_log2;
    for (uint32_t i = lane; i < cap; i += 32) hord[i] = 0xffffffffu;  // empty
    __syncwarp();
    uint32_t m = 0;
    for (uint32_t c0 = 0; c0 < S; c0 += 32) {
        const uint32_t e = c0 + lane;
        const bool act = e < S;
        const uint32_t v = act ? __ldg(src + e) : 0u;
        const uint32_t mm = __match_any_sync(0xffffffffu, v) & __ballot_sync(0xffffffffu, act);
        const bool lead = act && (mm & ((1u << lane) - 1u)) == 0u;
        uint32_t slot = (v * 0x9E3779B1u) >> (32 - cap_log2);
        bool fresh = false;
        if (lead) {
            while (true) {
                if (hord[slot] == 0xffffffffu) {
                    fresh = true;
                    break;
                }
                if (hkey[slot] == v) break;
                slot = (slot + 1) & (cap - 1);
            }
        }
        const uint32_t fb = __ballot_sync(0xffffffffu, fresh);
        for (uint32_t bits = fb; bits; bits &= bits - 1) {  // new values in lane order
            const uint32_t l = __ffs(bits) - 1;
            if (lane == l) {
                uint32_t s2 = slot;
                while (hord[s2] != 0xffffffffu) s2 = (s2 + 1) & (cap - 1);
                hkey[s2] = v;
                hord[s2] = m;
                cnt[m] = 0;
                if (first) first[m] = e;
                slot = s2;
            }
            ++m;
            __syncwarp();
        }
        if (lead) cnt[hord[slot]] += __popc(mm);
        __syncwarp();
    }
    return m;
}

__global__ void __launch_bounds__(SC_WIDE_WARPS * 32) sc_wide_kernel(const __grid_constant__ WideParams p) {
    extern __shared__ __align__(16) uint8_t smem[];
    const uint32_t lane = threadIdx.x & 31u, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    const uint32_t cap = 1u << p.cap_log2;
    uint32_t* hkey = reinterpret_cast<uint32_t*>(smem) + warp * (2 * cap + p.S);
    uint32_t* hord = hkey + cap;
    uint32_t* cnt = hord + cap;
    const uint64_t gw = static_cast<uint64_t>(blockIdx.x) * nw + warp, nwarps = static_cast<uint64_t>(gridDim.x) * nw;
    for (uint64_t row = gw; row < p.rows; row += nwarps) {
        const uint32_t m = wide_cluster(p.ids + row * p.S, p.S, p.cap_log2, hkey, hord, cnt, nullptr, lane);
        if (lane == 0) {
            double hc = 1.0;  // one cluster holds every answer: H~ = 1 exactly
            uint32_t maxc = p.S;
            if (m > 1) {
                double h = 0.0;
                maxc = 0;
                for (uint32_t k = 0; k < m; ++k) {
                    h = __dsub_rn(h, __ldg(p.tab + cnt[k]));  // first-seen order
                    maxc = max(maxc, cnt[k]);
                }
                h = (0.0 < h) ? h : 0.0;
                const double v = __ddiv_rn(__dsub_rn(p.logn, h), p.logn);
                hc = v < 0.0 ? 0.0 : (1.0 < v ? 1.0 : v);
            }
            bool meets = true;
            for (int t = 0; t < p.n_th; ++t) {
                if (p.th_sig[t] == CDX_SIG_MAJORITY) continue;  // the integer interval below
                const bool ok = p.th_dir[t] == CDX_DIR_GE ? hc >= p.th_cut[t] : hc <= p.th_cut[t];
                meets = meets && ok;
            }
            if (p.maj_th) meets = meets && maxc >= p.maj_lo && maxc <= p.maj_hi;
            if (p.hcert) p.hcert[row] = static_cast<float>(hc);
            if (p.maj) p.maj[row] = static_cast<float>(__ddiv_rn(static_cast<double>(maxc), static_cast<double>(p.S)));
            if (p.meets && meets) {
                const uint64_t r = row / p.P;
                const uint32_t pp = static_cast<uint32_t>(row - r * p.P);
                atomicOr(p.meets + r * p.words + (pp >> 5), 1u << (pp & 31u));
            }
        }
        __syncwarp();
    }
}

// cluster_rows for S > 32: the same warp clustering, leaders and sizes in first-seen order
__global__ void __launch_bounds__(SC_WIDE_WARPS * 32) cluster_rows_wide_kernel(
    const uint32_t* __restrict__ ids, uint64_t rows, uint32_t S, uint32_t cap_log2, uint32_t* __restrict__ ncl,
    uint32_t* __restrict__ leader, uint32_t* __restrict__ size) {
    extern __shared__ __align__(16) uint8_t smem[];
    const uint32_t lane = threadIdx.x & 31u, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    const uint32_t cap = 1u << cap_log2;
    uint32_t* hkey = reinterpret_cast<uint32_t*>(smem) + warp * (2 * cap + 2 * S);
    uint32_t* hord = hkey + cap;
    uint32_t* cnt = hord + cap;
    uint32_t* first = cnt + S;
    const uint64_t gw = static_cast<uint64_t>(blockIdx.x) * nw + warp, nwarps = static_cast<uint64_t>(gridDim.x) * nw;
    for (uint64_t row = gw; row < rows; row += nwarps) {
        const uint32_t m = wide_cluster(ids + row * S, S, cap_log2, hkey, hord, cnt, first, lane);
        for (uint32_t k = lane; k < m; k += 32) {
            leader[row * S + k] = first[k];
            size[row * S + k] = cnt[k];
        }
        if (lane == 0) ncl[row] = m;
        __syncwarp();
    }
}

// H~ of a row depends only on its cluster sizes in first-seen order, a composition of S.
// For S <= 16 there are 2^(S-1) of them (cut bit c-1 set for every cumulative size c < S),
// so the host evaluates every one once per context with exactly the device's IEEE
// sequence (h = 0 - T[s1] - T[s2] - ..., max(0, h), (log S - h) / log S, clamp: only
// subtractions and one division, nothing to contract) and the peel engine replaces its
// FP64 fold and division by one table load.  The result is the same double bit for bit.
int comp_table(cdx_ctx* ctx, const ScParams& p) {
    const uint32_t S = p.S;
    if (ctx->comp_tab[S]) return CDX_OK;  // term[] and log S depend on S only
    const uint32_t n = 1u << (S - 1);
    std::vector<double> tab(n);
    for (uint32_t code = 0; code < n; ++code) {
        if (code == 0) {  // one cluster holds every answer
            tab[code] = 1.0;
            continue;
        }
        double h = 0.0;
        uint32_t prev = 0;
        bool first = true;
        for (uint32_t c = 1; c <= S; ++c) {
            if (c < S && !((code >> (c - 1)) & 1u)) continue;
            const uint32_t size = c - prev;
            prev = c;
            h = first ? 0.0 - p.term[size] : h - p.term[size];
            first = false;
        }
        h = (0.0 < h) ? h : 0.0;
        const double v = (p.logn - h) / p.logn;
        tab[code] = v < 0.0 ? 0.0 : (1.0 < v ? 1.0 : v);
    }
    double* d = nullptr;
    if (cudaMalloc(&d, n * sizeof(double)) != cudaSuccess) return set_error(ctx, CDX_ECUDA, "sc_certaindex: table");
    const cudaError_t e = cudaMemcpyAsync(d, tab.data(), n * sizeof(double), cudaMemcpyHostToDevice, ctx->stream);
    if (e == cudaSuccess) cudaStreamSynchronize(ctx->stream);  // tab is a host temporary
    if (e != cudaSuccess) {
        cudaFree(d);
        return cuda_fail(ctx, e, "sc_certaindex: table");
    }
    ctx->comp_tab[S] = d;
    return CDX_OK;
}

}  // namespace cdx

extern "C" {

int cdx_sc_certaindex(cdx_ctx* ctx, const uint32_t* ids, uint64_t R, uint32_t P, uint32_t S,
                      const cdx_threshold* th, uint32_t n_th, float* hcert, uint32_t* meets_bits) {
    return cdx_sc_certaindex_ex(ctx, ids, R, P, S, th, n_th, hcert, nullptr, meets_bits);
}

}  // extern "C"

namespace cdx {
namespace {
// cdx_sc_certaindex_ex's body
int sc_impl(cdx_ctx* ctx, const uint32_t* ids, uint64_t R, uint32_t P, uint32_t S, const cdx_threshold* th,
            uint32_t n_th, float* hcert, float* majority, uint32_t* meets_bits, const al::AllocParams* tail = nullptr,
            bool* tail_done = nullptr) {
    if (S == 0) return set_error(ctx, CDX_EINVAL, "cluster_exact: empty answer set");
    if (S > SC_WIDE_MAX) return set_error(ctx, CDX_EINVAL, "sc_certaindex: at most 4096 samples per row");
    if (P == 0) return set_error(ctx, CDX_EINVAL, "sc_certaindex: probes must be >= 1");
    if (!ids) return set_error(ctx, CDX_EINVAL, "sc_certaindex: null ids");
    const bool present[5] = {true, false, false, false, true};
    if (int st = check_thresholds(ctx, th, n_th, present)) return st;
    if (R == 0) return CDX_OK;
    uint32_t maj_lo = 0, maj_hi = 0;
    int maj_th = 0;
    for (uint32_t i = 0; i < n_th; ++i) maj_th |= th[i].signal == CDX_SIG_MAJORITY;
    if (maj_th) majority_interval(th, n_th, S, &maj_lo, &maj_hi);
    if (S > 32) {  // wide rows: a warp per row, shared-memory hash of first-seen ordinals
        WideParams w{};
        w.ids = ids;
        w.hcert = hcert;
        w.maj = majority;
        w.maj_th = maj_th;
        w.maj_lo = maj_lo;
        w.maj_hi = maj_hi;
        w.meets = meets_bits;
        w.rows = R * P;
        w.P = P;
        w.S = S;
        w.words = (P + 31) / 32;
        w.cap_log2 = 1;
        while ((1u << w.cap_log2) < 2u * S) ++w.cap_log2;
        w.n_th = static_cast<int>(n_th);
        for (uint32_t i = 0; i < n_th; ++i) {
            w.th_sig[i] = th[i].signal;
            w.th_dir[i] = th[i].dir;
            w.th_cut[i] = th[i].cutoff;
        }
        TermTables tt;
        const uint32_t ns[1] = {S};
        if (int st = build_term_tables(ctx, ns, 1, &tt)) return st;
        w.tab = tt.tab;
        w.logn = std::log(static_cast<double>(S));
        if (meets_bits) cudaMemsetAsync(meets_bits, 0, R * w.words * 4, ctx->stream);  // bits are OR-ed in
        const size_t per_warp = ((2u << w.cap_log2) + S) * 4u;
        const uint32_t wpc = static_cast<uint32_t>(std::max<size_t>(1, std::min<size_t>(SC_WIDE_WARPS, (200u << 10) / per_warp)));
        const size_t smem = wpc * per_warp;
        cudaFuncSetAttribute(sc_wide_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
        int per_sm = 0;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, sc_wide_kernel, wpc * 32, smem);
        const uint64_t want = (w.rows + wpc - 1) / wpc;
        const uint64_t grid = std::min<uint64_t>(want, static_cast<uint64_t>(ctx->sm_count) * std::max(per_sm, 1));
        sc_wide_kernel<<<static_cast<unsigned>(grid), wpc * 32, smem, ctx->stream>>>(w);
        CDX_CHECK_LAUNCH(ctx, "sc_certaindex(wide)");
        return CDX_OK;
    }

    ScParams p{};
    p.ids = ids;
    p.hcert = hcert;
    p.maj = majority;
    p.maj_th = maj_th;
    p.maj_lo = maj_lo;
    p.maj_hi = maj_hi;
    for (uint32_t c = 0; c <= S; ++c)
        p.maj_tab[c] = static_cast<float>(static_cast<double>(c) / static_cast<double>(S));
    p.meets = meets_bits;
    p.R = R;
    p.P = P;
    p.S = S;
    p.words = (P + 31) / 32;
    p.ngroups = R * p.words;
    p.bulk_ok = reinterpret_cast<uintptr_t>(ids) % 16 == 0;  // per group: see bulkable()
    // per-warp ring depth and warps per CTA (tuned on B200: see profiles/)
    uint32_t stages = 1, wpc = 4;
    if (const char* e = getenv("CDX_SC_STAGES")) stages = static_cast<uint32_t>(atoi(e));
    if (const char* e = getenv("CDX_SC_WARPS")) wpc = static_cast<uint32_t>(atoi(e));
    p.stages = std::max<uint32_t>(1, std::min<uint32_t>(SC_MAX_STAGES, stages));
    wpc = std::max<uint32_t>(1, std::min<uint32_t>(SC_MAX_WARPS, wpc));
    p.n_th = static_cast<int>(n_th);
    p.box_lo = -HUGE_VAL;
    p.box_hi = HUGE_VAL;
    p.box_never = 0;
    for (uint32_t i = 0; i < n_th; ++i) {
        p.th_dir[i] = th[i].dir;
        p.th_cut[i] = th[i].cutoff;
        if (th[i].signal == CDX_SIG_MAJORITY) continue;  // the integer interval [maj_lo, maj_hi]
        if (std::isnan(th[i].cutoff)) p.box_never = 1;
        else if (th[i].dir == CDX_DIR_GE) p.box_lo = std::max(p.box_lo, th[i].cutoff);
        else p.box_hi = std::min(p.box_hi, th[i].cutoff);
    }
    p.term[0] = 0.0;
    for (uint32_t c = 1; c <= S; ++c) p.term[c] = host_term(c, S);
    p.logn = std::log(static_cast<double>(S));

    p.comp = nullptr;
    if (S >= 2 && S <= 16) {
        if (int st = comp_table(ctx, p)) return st;
        p.comp = ctx->comp_tab[S];
    }
    // fast path: TMA-staged groups, warp-match + ALU-peel engines side by side (k_sc_fast.cu)
    if (launch_sc_fast(ctx, p, tail, tail_done)) {
        CDX_CHECK_LAUNCH(ctx, "sc_certaindex(fast)");
        return CDX_OK;
    }
    switch (S) {
        case 32: launch_sc<32>(ctx, p, wpc); break;
        case 16: launch_sc<16>(ctx, p, wpc); break;
        case 8: launch_sc<8>(ctx, p, wpc); break;
        case 4: launch_sc<4>(ctx, p, wpc); break;
        case 2: launch_sc<2>(ctx, p, wpc); break;
        case 1: launch_sc<1>(ctx, p, wpc); break;
        default: launch_sc<0>(ctx, p, wpc); break;
    }
    CDX_CHECK_LAUNCH(ctx, "sc_certaindex");
    return CDX_OK;
}
}  // namespace
}  // namespace cdx

extern "C" {

int cdx_sc_certaindex_ex(cdx_ctx* ctx, const uint32_t* ids, uint64_t R, uint32_t P, uint32_t S,
                         const cdx_threshold* th, uint32_t n_th, float* hcert, float* majority,
                         uint32_t* meets_bits) {
    using namespace cdx;
    CDX_NVTX("cdx_sc_certaindex");
    if (!ctx) return CDX_EINVAL;
    return sc_impl(ctx, ids, R, P, S, th, n_th, hcert, majority, meets_bits);
}

int cdx_sc_decide(cdx_ctx* ctx, const uint32_t* ids, uint64_t R, uint32_t P, uint32_t S, const cdx_threshold* th,
                  uint32_t n_th, float* hcert, uint32_t* meets_bits, const cdx_alloc_policy* pol, int64_t base_offset,
                  uint32_t kept_base, int32_t* exit_knob, uint8_t* reason, int32_t* granted, int64_t* offsets,
                  uint32_t* kept, uint64_t* n_kept, int64_t* tokens_saved, int64_t* total_budget) {
    using namespace cdx;
    CDX_NVTX("cdx_sc_decide");
    if (!ctx) return CDX_EINVAL;
    if (!meets_bits) return set_error(ctx, CDX_EINVAL, "sc_decide: null meets bits");
    // the policy is validated before anything is launched (the two calls' errors, in order)
    al::AllocParams ap;
    bool empty = false;
    if (int st = alloc_prepare(ctx, meets_bits, R, P, pol, base_offset, kept_base, exit_knob, reason, granted, offsets,
                               kept, n_kept, tokens_saved, total_budget, &ap, &empty))
        return st;
    // a batch of one K5 tile runs K5 in K2's last CTA (one launch); larger ones launch K5
    bool tail_done = false;
    if (int st = sc_impl(ctx, ids, R, P, S, th, n_th, hcert, nullptr, meets_bits, empty ? nullptr : &ap, &tail_done))
        return st;
    if (empty || tail_done) return CDX_OK;
    return cdx_allocate_scan(ctx, meets_bits, R, P, pol, base_offset, kept_base, exit_knob, reason, granted, offsets,
                             kept, n_kept, tokens_saved, total_budget);
}

int cdx_cluster_rows(cdx_ctx* ctx, const uint32_t* ids, uint64_t rows, uint32_t S, uint32_t* n_clusters,
                     uint32_t* leader, uint32_t* size) {
    using namespace cdx;
    CDX_NVTX("cdx_cluster_rows");
    if (!ctx) return CDX_EINVAL;
    if (S == 0) return set_error(ctx, CDX_EINVAL, "cluster_exact: empty answer set");
    if (S > SC_WIDE_MAX) return set_error(ctx, CDX_EINVAL, "cluster_rows: at most 4096 answers per row");
    if (!ids || !n_clusters || !leader || !size) return set_error(ctx, CDX_EINVAL, "cluster_rows: null pointer");
    if (rows == 0) return CDX_OK;
    if (S > 32) {  // a warp per row, shared-memory hash of first-seen ordinals
        uint32_t cap_log2 = 1;
        while ((1u << cap_log2) < 2u * S) ++cap_log2;
        const size_t per_warp = ((2u << cap_log2) + 2u * S) * 4u;
        const uint32_t wpc = static_cast<uint32_t>(std::max<size_t>(1, std::min<size_t>(SC_WIDE_WARPS, (200u << 10) / per_warp)));
        const size_t smem = wpc * per_warp;
        cudaFuncSetAttribute(cluster_rows_wide_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             static_cast<int>(smem));
        const uint64_t grid = std::min<uint64_t>((rows + wpc - 1) / wpc, static_cast<uint64_t>(ctx->sm_count) * 8);
        cluster_rows_wide_kernel<<<static_cast<unsigned>(grid), wpc * 32, smem, ctx->stream>>>(
            ids, rows, S, cap_log2, n_clusters, leader, size);
        CDX_CHECK_LAUNCH(ctx, "cluster_rows(wide)");
        return CDX_OK;
    }
    const uint64_t warps = (rows + (32 / S) - 1) / (32 / S);
    const uint64_t blocks = std::min<uint64_t>((warps + 7) / 8, static_cast<uint64_t>(ctx->sm_count) * 16);
    cluster_rows_kernel<<<static_cast<unsigned>(blocks), 256, 0, ctx->stream>>>(ids, rows, S, n_clusters, leader, size);
    CDX_CHECK_LAUNCH(ctx, "cluster_rows");
    return CDX_OK;
}

int cdx_entropy_from_sizes(cdx_ctx* ctx, const uint32_t* sizes, const uint32_t* m, const uint32_t* totals,
                           uint64_t rows,
                           uint32_t max_m, uint32_t max_n, double* H, double* Hcert) {
    using namespace cdx;
    CDX_NVTX("cdx_entropy_from_sizes");
    if (!ctx) return CDX_EINVAL;
    if (!sizes || !m || max_m == 0) return set_error(ctx, CDX_EINVAL, "semantic_entropy: invalid clustering");
    if (max_n == 0 || max_n > 2048) return set_error(ctx, CDX_EINVAL, "entropy_from_sizes: max_n must be 1..2048 (use cdx_entropy_one above)");
    if (rows == 0) return CDX_OK;
    std::vector<uint32_t> ns(max_n + 1);
    for (uint32_t i = 0; i <= max_n; ++i) ns[i] = i;
    TermTables tt;
    if (int st = build_term_tables(ctx, ns.data(), max_n + 1, &tt)) return st;
    const uint64_t blocks = std::min<uint64_t>((rows + 255) / 256, static_cast<uint64_t>(ctx->sm_count) * 8);
    entropy_sizes_kernel<<<static_cast<unsigned>(blocks), 256, 0, ctx->stream>>>(sizes, m, totals, rows, max_m, tt.tab, tt.logs,
                                                                               max_n, H, Hcert, ctx->d_err);
    CDX_CHECK_LAUNCH(ctx, "entropy_from_sizes");
    return CDX_OK;
}

}  // extern "C"

