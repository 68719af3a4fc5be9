// k_sc.cu — K2: Self-Consistency certaindex over (request, probe) rows of S answers.
//
// Replaces, per row, metrics::certaindex_entropy(metrics::cluster_exact(row)) and
// metrics::combined_meets_thresholds (metrics.cpp:21-37, 107-125, 159-171) — the SC branch
// of ProgramDriver::update_certaindex (runtime.cpp:266-271) evaluated at every probe step.
//
// Data path (HBM-bound; no tensor cores: nothing here is a contraction):
//   ids u32[R][P][S] --(cp.async.bulk, 3-stage mbarrier ring, evict-first)--> smem tile of
//   whole requests --> one warp per group of 32 rows:
//     __match_any_sync over the row's S lanes = exact-match clusters; the lowest lane of a
//     match set is the cluster's first-seen answer (cluster order of metrics.cpp:29-31);
//     ballot of leaders + popc(match) = cluster sizes;
//   --> per-row ordered FP64 fold h -= term[size] in first-seen order (term[c] =
//     (c/S)*log(c/S) built on the host with the reference's libm, so the device performs
//     only IEEE subtract/divide and reproduces the reference bits), clamp, thresholds on the
//     FP64 value, fp32 store + one meets word per 32 rows.
#include <algorithm>
#include <cmath>
#include <vector>

#include "cdx_internal.cuh"

namespace cdx {

constexpr int SC_THREADS = 256;
constexpr int SC_WARPS = SC_THREADS / 32;
constexpr int SC_MAX_STAGES = 3;
constexpr int MAX_TH = 8;

struct ScParams {
    const uint32_t* ids;
    float* hcert;
    uint32_t* meets;
    uint64_t R;
    uint64_t ntiles;
    uint32_t P, S, words, q;  // words = ceil(P/32); q = requests per tile
    uint32_t tile_stride;     // bytes between smem stages
    uint32_t stages;
    int bulk_ok;
    int n_th;
    uint8_t th_dir[MAX_TH];
    double th_cut[MAX_TH];
    double term[33];
    double logn;
};

__device__ __forceinline__ bool sc_tile_bulk(const ScParams& p, uint32_t nreq) {
    return p.bulk_ok && ((static_cast<uint64_t>(nreq) * p.P * p.S * 4u) % 16u == 0);
}

__global__ void __launch_bounds__(SC_THREADS, 2) sc_certaindex_kernel(const __grid_constant__ ScParams p) {
    extern __shared__ __align__(128) uint8_t smem[];
    uint8_t* cnt_all = smem + p.stages * p.tile_stride;          // [warp][leader s][row] u8
    double* term = reinterpret_cast<double*>(cnt_all + SC_WARPS * 1024);
    uint64_t* bar = reinterpret_cast<uint64_t*>(term + 34);

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    if (tid < 33) term[tid] = p.term[tid];
    if (tid == 0) {
        for (uint32_t s = 0; s < p.stages; ++s) mbar_init(&bar[s], 1);
        fence_mbar_init();
    }
    __syncthreads();

    const uint64_t policy = policy_evict_first();
    const uint64_t stride = gridDim.x;
    auto issue = [&](uint64_t tile, uint32_t stage) {
        const uint64_t r0 = tile * p.q;
        const uint32_t nreq = static_cast<uint32_t>((p.R - r0 < p.q ? p.R - r0 : static_cast<uint64_t>(p.q)));
        if (!sc_tile_bulk(p, nreq)) return;
        const uint32_t bytes = nreq * p.P * p.S * 4u;
        mbar_expect_tx(&bar[stage], bytes);
        bulk_g2s(smem + stage * p.tile_stride, p.ids + r0 * p.P * p.S, bytes, &bar[stage], policy);
    };
    if (tid == 0) {
        for (uint32_t s = 0; s < p.stages; ++s) {
            const uint64_t t = blockIdx.x + s * stride;
            if (t < p.ntiles) issue(t, s);
        }
    }

    const uint32_t S = p.S;
    const uint32_t rpi = 32u / S;  // rows per match iteration
    const uint32_t smask = S == 32 ? 0xffffffffu : ((1u << S) - 1u);
    const uint32_t sub = lane / S, s = lane - sub * S;
    const bool lane_ok = sub < rpi;
    const uint32_t subm = lane_ok ? (smask << (sub * S)) : 0u;
    uint8_t* cntw = cnt_all + warp * 1024;

    uint32_t it_count = 0;
    for (uint64_t tile = blockIdx.x; tile < p.ntiles; tile += stride, ++it_count) {
        const uint32_t stage = it_count % p.stages;
        const uint32_t parity = (it_count / p.stages) & 1u;
        const uint64_t r0 = tile * p.q;
        const uint32_t nreq = static_cast<uint32_t>((p.R - r0 < p.q ? p.R - r0 : static_cast<uint64_t>(p.q)));
        const uint32_t* tids = reinterpret_cast<const uint32_t*>(smem + stage * p.tile_stride);
        if (sc_tile_bulk(p, nreq)) {
            mbar_wait(&bar[stage], parity);
        } else {
            // unaligned / ragged tail tile: cooperative coalesced loads
            uint32_t* dst = reinterpret_cast<uint32_t*>(smem + stage * p.tile_stride);
            const uint32_t n = nreq * p.P * S;
            const uint32_t* src = p.ids + r0 * p.P * S;
            for (uint32_t i = tid; i < n; i += SC_THREADS) dst[i] = __ldg(src + i);
            __syncthreads();
        }

        const uint32_t groups = nreq * p.words;
        for (uint32_t gi = warp; gi < groups; gi += SC_WARPS) {
            const uint32_t req = gi / p.words;
            const uint32_t g = gi - req * p.words;
            const uint32_t row0 = g * 32u;
            const uint32_t rows = min(32u, p.P - row0);
            const uint32_t* base = tids + (req * p.P + row0) * S;
            const uint32_t iters = (rows + rpi - 1) / rpi;
            uint32_t my_lm = 0;
#pragma unroll 4
            for (uint32_t it = 0; it < iters; ++it) {
                const uint32_t rloc = it * rpi + sub;
                const bool act = lane_ok && rloc < rows;
                const uint32_t v = act ? base[rloc * S + s] : 0xffffffffu;
                const uint32_t m = __match_any_sync(0xffffffffu, v) & subm;
                const bool leader = act && (static_cast<uint32_t>(__ffs(m) - 1) == static_cast<uint32_t>(lane));
                const uint32_t lm = __ballot_sync(0xffffffffu, leader);
                if (leader) cntw[s * 32 + rloc] = static_cast<uint8_t>(__popc(m));
                if (it == static_cast<uint32_t>(lane) / rpi)
                    my_lm = (lm >> ((static_cast<uint32_t>(lane) % rpi) * S)) & smask;
            }
            __syncwarp();
            bool meets = false;
            if (static_cast<uint32_t>(lane) < rows) {
                double hc = 1.0;  // metrics.cpp:121: a single path is fully certain
                if (S > 1) {
                    double h = 0.0;
                    uint32_t bits = my_lm;
                    while (bits) {
                        const uint32_t l = __ffs(bits) - 1;
                        bits &= bits - 1;
                        h = __dsub_rn(h, term[cntw[l * 32 + lane]]);  // h -= p*log(p)
                    }
                    h = (0.0 < h) ? h : 0.0;  // std::max(0.0, h)
                    const double v = __ddiv_rn(__dsub_rn(p.logn, h), p.logn);
                    hc = v < 0.0 ? 0.0 : (1.0 < v ? 1.0 : v);  // std::clamp
                }
                meets = true;
                for (int t = 0; t < p.n_th; ++t) {
                    const bool ok = p.th_dir[t] == CDX_DIR_GE ? hc >= p.th_cut[t] : hc <= p.th_cut[t];
                    meets = meets && ok;
                }
                if (p.hcert) p.hcert[(r0 + req) * p.P + row0 + lane] = static_cast<float>(hc);
            }
            const uint32_t mw = __ballot_sync(0xffffffffu, meets);
            if (lane == 0 && p.meets) p.meets[(r0 + req) * p.words + g] = mw;
            __syncwarp();
        }
        __syncthreads();
        if (tid == 0) {
            const uint64_t nt = tile + static_cast<uint64_t>(p.stages) * stride;
            if (nt < p.ntiles) issue(nt, stage);
        }
    }
}

// ---------------------------------------------------------------------------------------
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
__global__ void entropy_sizes_kernel(const uint32_t* __restrict__ sizes, const uint32_t* __restrict__ m,
                                     uint64_t rows, uint32_t max_m, const double* __restrict__ tri,
                                     const double* __restrict__ logs, uint32_t max_n, double* H,
                                     double* Hc, int* bad) {
    for (uint64_t r = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; r < rows;
         r += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
        const uint32_t mm = m[r];
        uint64_t n = 0;
        bool ok = mm >= 1 && mm <= max_m;
        for (uint32_t k = 0; ok && k < mm; ++k) {
            const uint32_t c = sizes[r * max_m + k];
            ok = c >= 1;
            n += c;
        }
        if (!ok || n > max_n) {
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

int check_thresholds(cdx_ctx* ctx, const cdx_threshold* th, uint32_t n_th, const bool present[4]) {
    static const char* names[4] = {"certaindex_entropy", "certaindex_reward", "mean_output_length",
                                   "mean_norm_logprob"};
    if (n_th > MAX_TH) return set_error(ctx, CDX_EINVAL, "thresholds: at most 8 per call");
    if (n_th && !th) return set_error(ctx, CDX_EINVAL, "thresholds: null array");
    for (uint32_t i = 0; i < n_th; ++i) {
        if (th[i].signal > 3 || th[i].dir > 1) return set_error(ctx, CDX_EINVAL, "thresholds: bad enum");
        if (!present[th[i].signal])
            return set_error(ctx, CDX_EINVAL,
                             std::string("combined_meets_thresholds: signal '") + names[th[i].signal] +
                                 "' absent");
    }
    return CDX_OK;
}

}  // namespace cdx

extern "C" {

int cdx_sc_certaindex(cdx_ctx* ctx, const uint32_t* ids, uint64_t R, uint32_t P, uint32_t S,
                      const cdx_threshold* th, uint32_t n_th, float* hcert, uint32_t* meets_bits) {
    using namespace cdx;
    if (!ctx) return CDX_EINVAL;
    if (S == 0) return set_error(ctx, CDX_EINVAL, "cluster_exact: empty answer set");
    if (S > 32) return set_error(ctx, CDX_EINVAL, "sc_certaindex: at most 32 samples per row");
    if (P == 0 || P > 4096) return set_error(ctx, CDX_EINVAL, "sc_certaindex: probes must be 1..4096");
    if (!ids) return set_error(ctx, CDX_EINVAL, "sc_certaindex: null ids");
    const bool present[4] = {true, false, false, false};
    if (int st = check_thresholds(ctx, th, n_th, present)) return st;
    if (R == 0) return CDX_OK;

    ScParams p{};
    p.ids = ids;
    p.hcert = hcert;
    p.meets = meets_bits;
    p.R = R;
    p.P = P;
    p.S = S;
    p.words = (P + 31) / 32;
    const uint64_t req_bytes = static_cast<uint64_t>(P) * S * 4u;
    if (req_bytes > 200u * 1024u)
        return set_error(ctx, CDX_EINVAL, "sc_certaindex: one request (P*S*4 bytes) exceeds 200 KiB");
    uint32_t q = static_cast<uint32_t>(32768u / req_bytes);
    if (q < 1) q = 1;
    // keep every full tile a multiple of 16 bytes so it can be bulk-copied
    while ((static_cast<uint64_t>(q) * P * S) % 4u) ++q;
    if (q * req_bytes > 200u * 1024u) q = 1;
    p.q = q;
    p.ntiles = (R + q - 1) / q;
    const uint64_t tile_bytes = q * req_bytes;
    p.tile_stride = static_cast<uint32_t>((tile_bytes + 127) / 128 * 128);
    p.stages = static_cast<uint32_t>(std::min<uint64_t>(SC_MAX_STAGES, (200u * 1024u) / p.tile_stride));
    if (p.stages < 1) p.stages = 1;
    p.bulk_ok = (reinterpret_cast<uintptr_t>(ids) % 16 == 0) && ((static_cast<uint64_t>(q) * P * S) % 4 == 0);
    p.n_th = static_cast<int>(n_th);
    for (uint32_t i = 0; i < n_th; ++i) {
        p.th_dir[i] = th[i].dir;
        p.th_cut[i] = th[i].cutoff;
    }
    p.term[0] = 0.0;
    for (uint32_t c = 1; c <= S; ++c) p.term[c] = host_term(c, S);
    p.logn = std::log(static_cast<double>(S));

    const size_t smem = static_cast<size_t>(p.stages) * p.tile_stride + SC_WARPS * 1024 + 34 * 8 + 8 * SC_MAX_STAGES;
    cudaFuncSetAttribute(sc_certaindex_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, sc_certaindex_kernel, SC_THREADS, smem);
    if (per_sm < 1) per_sm = 1;
    const uint64_t grid = std::min<uint64_t>(p.ntiles, static_cast<uint64_t>(ctx->sm_count) * per_sm);
    sc_certaindex_kernel<<<static_cast<unsigned>(grid), SC_THREADS, smem, ctx->stream>>>(p);
    CDX_CHECK_LAUNCH(ctx, "sc_certaindex");
    return CDX_OK;
}

int cdx_cluster_rows(cdx_ctx* ctx, const uint32_t* ids, uint64_t rows, uint32_t S, uint32_t* n_clusters,
                     uint32_t* leader, uint32_t* size) {
    using namespace cdx;
    if (!ctx) return CDX_EINVAL;
    if (S == 0) return set_error(ctx, CDX_EINVAL, "cluster_exact: empty answer set");
    if (S > 32) return set_error(ctx, CDX_EINVAL, "cluster_rows: at most 32 answers per row");
    if (!ids || !n_clusters || !leader || !size) return set_error(ctx, CDX_EINVAL, "cluster_rows: null pointer");
    if (rows == 0) return CDX_OK;
    const uint64_t warps = (rows + (32 / S) - 1) / (32 / S);
    const uint64_t blocks = std::min<uint64_t>((warps + 7) / 8, static_cast<uint64_t>(ctx->sm_count) * 16);
    cluster_rows_kernel<<<static_cast<unsigned>(blocks), 256, 0, ctx->stream>>>(ids, rows, S, n_clusters, leader, size);
    CDX_CHECK_LAUNCH(ctx, "cluster_rows");
    return CDX_OK;
}

int cdx_entropy_from_sizes(cdx_ctx* ctx, const uint32_t* sizes, const uint32_t* m, uint64_t rows,
                           uint32_t max_m, uint32_t max_n, double* H, double* Hcert) {
    using namespace cdx;
    if (!ctx) return CDX_EINVAL;
    if (!sizes || !m || max_m == 0) return set_error(ctx, CDX_EINVAL, "semantic_entropy: invalid clustering");
    if (max_n == 0 || max_n > (1u << 16)) return set_error(ctx, CDX_EINVAL, "entropy_from_sizes: max_n must be 1..65536");
    if (rows == 0) return CDX_OK;
    std::vector<uint32_t> ns(max_n + 1);
    for (uint32_t i = 0; i <= max_n; ++i) ns[i] = i;
    TermTables tt;
    if (int st = build_term_tables(ctx, ns.data(), max_n + 1, &tt)) return st;
    const uint64_t blocks = std::min<uint64_t>((rows + 255) / 256, static_cast<uint64_t>(ctx->sm_count) * 8);
    entropy_sizes_kernel<<<static_cast<unsigned>(blocks), 256, 0, ctx->stream>>>(sizes, m, rows, max_m, tt.tab, tt.logs,
                                                                               max_n, H, Hcert, ctx->d_err);
    CDX_CHECK_LAUNCH(ctx, "entropy_from_sizes");
    return CDX_OK;
}

}  // extern "C"
