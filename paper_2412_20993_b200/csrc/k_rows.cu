// k_rows.cu — variable-length row kernels behind the scalar C++ API (include/cdx/*.hpp).
//
// The batched kernels (K2-K4) take fixed-shape tensors.  The reference's own functions take
// arbitrary spans: a probe trace of any length with any step_index sequence, a SignalVector
// with any subset of signals present, a clustering of any size.  These kernels evaluate
// such ragged rows (concatenated, row_off[rows+1]) with one thread per row, so the façade
// (csrc/host/facade.cpp) routes every reference call through the device — there is no
// host-side certaindex arithmetic anywhere in the product.
//
//   probe_consistency_kernel  probe::consistency   probe.cpp:64-75 (usable_up_to :53-60)
//   probe_should_exit_kernel  probe::should_exit   probe.cpp:77-85
//   probe_final_answer_kernel probe::final_answer  probe.cpp:87-102
//   meets_rows_kernel         metrics::combined_meets_thresholds  metrics.cpp:159-171
//   id_histogram_kernel       cluster sizes of dense first-seen ids (cluster_exact :21-37)
//
// Answers arrive interned (K1): equal id <=> equal trimmed bytes, which is exactly the
// reference's same_answer (probe.cpp:48-50).  FP64 results use IEEE-rounded ops only.

#include <climits>
#include <cmath>
#include <vector>

#include "cdx_internal.cuh"

namespace cdx {
namespace {

// usable_up_to(records, k): records are scanned from the start and the scan stops at the
// first step_index > k; hesitant records are skipped.  Returns the end of the scanned
// prefix and the usable count.
__device__ __forceinline__ void usable_prefix(const uint8_t* __restrict__ hes, const int32_t* __restrict__ step,
                                              uint64_t b, uint64_t e, int64_t k, uint64_t* end, uint64_t* usable) {
    uint64_t u = 0, i = b;
    for (; i < e; ++i) {
        if (static_cast<int64_t>(step[i]) > k) break;
        u += hes[i] ? 0u : 1u;
    }
    *end = i;
    *usable = u;
}

// agree count over the last w usable records of [b, end) against the last usable one
__device__ __forceinline__ uint64_t window_agree(const uint32_t* __restrict__ ids, const uint8_t* __restrict__ hes,
                                                 uint64_t b, uint64_t end, uint64_t w) {
    uint64_t i = end, seen = 0, agree = 0;
    uint32_t last = 0;
    while (i > b && seen < w) {
        --i;
        if (hes[i]) continue;
        if (seen == 0) last = ids[i];
        agree += ids[i] == last ? 1u : 0u;
        ++seen;
    }
    return agree;
}

__global__ void probe_consistency_kernel(const uint32_t* __restrict__ ids, const uint8_t* __restrict__ hes,
                                         const int32_t* __restrict__ step, const uint64_t* __restrict__ row_off,
                                         const int32_t* __restrict__ k, uint64_t rows, int32_t w,
                                         double* __restrict__ C, uint8_t* __restrict__ ready) {
    for (uint64_t r = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; r < rows;
         r += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
        const uint64_t b = row_off[r], e = row_off[r + 1];
        uint64_t end, u;
        usable_prefix(hes, step, b, e, k[r], &end, &u);
        if (u < static_cast<uint64_t>(w)) {  // "window not ready" -> nullopt
            ready[r] = 0;
            C[r] = 0.0;
            continue;
        }
        const uint64_t agree = window_agree(ids, hes, b, end, static_cast<uint64_t>(w));
        ready[r] = 1;
        C[r] = __ddiv_rn(static_cast<double>(agree), static_cast<double>(w));
    }
}

__global__ void probe_should_exit_kernel(const uint32_t* __restrict__ ids, const uint8_t* __restrict__ hes,
                                         const int32_t* __restrict__ step, const int64_t* __restrict__ tok,
                                         const uint64_t* __restrict__ row_off, uint64_t rows, int32_t w,
                                         double tau, int64_t max_tokens, uint8_t* __restrict__ decision) {
    for (uint64_t r = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; r < rows;
         r += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
        const uint64_t b = row_off[r], e = row_off[r + 1];
        if (b == e) {  // empty trace -> Continue
            decision[r] = CDX_EXIT_CONTINUE;
            continue;
        }
        uint64_t end, u;
        usable_prefix(hes, step, b, e, step[e - 1], &end, &u);
        uint8_t d = CDX_EXIT_CONTINUE;
        if (u >= static_cast<uint64_t>(w)) {
            const uint64_t agree = window_agree(ids, hes, b, end, static_cast<uint64_t>(w));
            if (__ddiv_rn(static_cast<double>(agree), static_cast<double>(w)) >= tau) d = CDX_EXIT_CERTAIN;
        }
        if (d == CDX_EXIT_CONTINUE && tok[e - 1] >= max_tokens) d = CDX_EXIT_BUDGET;
        decision[r] = d;
    }
}

// terminated_at: INT32_MIN = nullopt; reason: probe.hpp:42 TerminationReason ordinal
__global__ void probe_final_answer_kernel(const uint8_t* __restrict__ hes, const int32_t* __restrict__ step,
                                          const uint64_t* __restrict__ row_off, const int32_t* __restrict__ term_at,
                                          const uint8_t* __restrict__ term_reason, uint64_t rows,
                                          uint64_t* __restrict__ pos, uint8_t* __restrict__ low) {
    for (uint64_t r = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; r < rows;
         r += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
        const uint64_t b = row_off[r], e = row_off[r + 1];
        uint64_t found = e;
        uint8_t lc = 0;
        if (term_at && term_at[r] != INT_MIN && term_reason && term_reason[r] == 0 /* Certain */) {
            for (uint64_t i = e; i > b;) {
                --i;
                if (step[i] == term_at[r]) {
                    found = i;
                    break;
                }
            }
        }
        if (found == e) {
            for (uint64_t i = e; i > b;) {
                --i;
                if (!hes[i]) {
                    found = i;
                    break;
                }
            }
        }
        if (found == e) {  // every probe hesitated: the last one, marked
            found = e - 1;
            lc = 1;
        }
        pos[r] = found - b;
        low[r] = lc;
    }
}

struct RowThresholds {
    cdx_threshold th[8];
    uint32_t n;
};

// signals f64[rows][4] (SignalKind order), present u8[rows] bit k = signal k present.
// In threshold order: an absent signal raises (the reference throws there), a failed
// threshold returns false before any later threshold is looked at (metrics.cpp:161-169).
__global__ void meets_rows_kernel(const double* __restrict__ sig, const uint8_t* __restrict__ present,
                                  uint64_t rows, RowThresholds t, uint8_t* __restrict__ out, int* err) {
    for (uint64_t r = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; r < rows;
         r += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
        uint8_t ok = 1;
        for (uint32_t i = 0; i < t.n; ++i) {
            const uint32_t s = t.th[i].signal;
            if (!((present[r] >> s) & 1u)) {
                set_dev_err(err, DEV_ABSENT_SIGNAL + static_cast<int>(s));
                ok = 0;
                break;
            }
            const double v = sig[r * 4 + s];
            const bool pass = t.th[i].dir == CDX_DIR_GE ? (v >= t.th[i].cutoff) : (v <= t.th[i].cutoff);
            if (!pass) {
                ok = 0;
                break;
            }
        }
        out[r] = ok;
    }
}

__global__ void id_histogram_kernel(const uint32_t* __restrict__ ids, uint64_t n, uint32_t n_unique,
                                    uint32_t* __restrict__ counts, int* err) {
    for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
        const uint32_t id = ids[i];
        if (id >= n_unique) {
            set_dev_err(err, DEV_BAD_CLUSTERING);
            continue;
        }
        atomicAdd(counts + id, 1u);
    }
}

// one clustering with a host-known total n: T_n[c] from the host libm, fold on the device
__global__ void entropy_one_kernel(const uint32_t* __restrict__ sizes, uint32_t m, uint32_t n,
                                   const double* __restrict__ T, double log_n, double* H, double* Hc, int* err) {
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    double h = 0.0;
    for (uint32_t k = 0; k < m; ++k) {
        const uint32_t c = sizes[k];
        if (c < 1) {
            set_dev_err(err, DEV_EMPTY_CLUSTER);
            return;
        }
        if (c > n) {
            set_dev_err(err, DEV_BAD_CLUSTERING);
            return;
        }
        h = __dsub_rn(h, T[c]);
    }
    h = (0.0 < h) ? h : 0.0;
    if (H) *H = h;
    if (Hc) {
        double hc = 1.0;
        if (n != 1) {
            const double v = __ddiv_rn(__dsub_rn(log_n, h), log_n);
            hc = v < 0.0 ? 0.0 : (1.0 < v ? 1.0 : v);
        }
        *Hc = hc;
    }
}

// one clustering with host-built per-cluster terms (any sizes, any total): fold in order
__global__ void entropy_terms_kernel(const double* __restrict__ terms, uint32_t m, double log_n, int n_is_one,
                                     double* H, double* Hc) {
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    double h = 0.0;
    for (uint32_t k = 0; k < m; ++k) h = __dsub_rn(h, terms[k]);
    h = (0.0 < h) ? h : 0.0;
    if (H) *H = h;
    if (Hc) {
        double hc = 1.0;
        if (!n_is_one) {
            const double v = __ddiv_rn(__dsub_rn(log_n, h), log_n);
            hc = v < 0.0 ? 0.0 : (1.0 < v ? 1.0 : v);
        }
        *Hc = hc;
    }
}

// SPEC.md:431-439 estimate_iteration_tokens over ragged histories: exact i64 sum, one
// IEEE division (the same arithmetic as K6's in-kernel estimate)
__global__ void iteration_tokens_kernel(const int64_t* __restrict__ v, const uint64_t* __restrict__ row_off,
                                        uint64_t rows, double prior, double* __restrict__ out) {
    for (uint64_t r = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; r < rows;
         r += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
        const uint64_t b = row_off[r], e = row_off[r + 1];
        int64_t s = 0;
        for (uint64_t i = b; i < e; ++i) s += v[i];
        out[r] = e > b ? __ddiv_rn(static_cast<double>(s), static_cast<double>(e - b)) : prior;
    }
}

unsigned grid_for(const cdx_ctx* ctx, uint64_t n) {
    const uint64_t want = (n + 255) / 256;
    const uint64_t cap = static_cast<uint64_t>(ctx->sm_count) * 8;
    return static_cast<unsigned>(want < 1 ? 1 : (want < cap ? want : cap));
}

int check_probe_cfg(cdx_ctx* ctx, const cdx_probe_cfg* cfg) {
    // probe.cpp:19-25 ProbeConfig::validate, same messages
    if (cfg->interval_tokens < 1) return set_error(ctx, CDX_EINVAL, "probe: interval_tokens must be >= 1");
    if (cfg->window < 1) return set_error(ctx, CDX_EINVAL, "probe: window must be >= 1");
    if (cfg->threshold <= 0.0 || cfg->threshold > 1.0)  // probe.cpp:22 (NaN passes)
        return set_error(ctx, CDX_EINVAL, "probe: threshold must be in (0,1]");
    if (cfg->max_tokens < 1) return set_error(ctx, CDX_EINVAL, "probe: max_tokens must be >= 1");
    return CDX_OK;
}

}  // namespace

int check_probe_cfg_c(cdx_ctx* ctx, const cdx_probe_cfg* cfg) { return check_probe_cfg(ctx, cfg); }

int entropy_terms_launch(cdx_ctx* ctx, const double* terms, uint32_t m, double log_n, bool n_is_one, double* H,
                         double* Hc) {
    entropy_terms_kernel<<<1, 32, 0, ctx->stream>>>(terms, m, log_n, n_is_one ? 1 : 0, H, Hc);
    CDX_CHECK_LAUNCH(ctx, "entropy_terms");
    return CDX_OK;
}

}  // namespace cdx

extern "C" {

int cdx_probe_consistency(cdx_ctx* ctx, const uint32_t* ids, const uint8_t* hes, const int32_t* step_index,
                          const uint64_t* row_off, const int32_t* k, uint64_t rows, int32_t window, double* C,
                          uint8_t* ready) {
    using namespace cdx;
    if (!ctx) return CDX_EINVAL;
    if (window < 1) return set_error(ctx, CDX_EINVAL, "consistency: window must be >= 1");
    if (rows == 0) return CDX_OK;
    if (!ids || !hes || !step_index || !row_off || !k || !C || !ready)
        return set_error(ctx, CDX_EINVAL, "consistency: null pointer");
    probe_consistency_kernel<<<grid_for(ctx, rows), 256, 0, ctx->stream>>>(ids, hes, step_index, row_off, k, rows,
                                                                          window, C, ready);
    CDX_CHECK_LAUNCH(ctx, "probe_consistency");
    return CDX_OK;
}

int cdx_probe_should_exit(cdx_ctx* ctx, const uint32_t* ids, const uint8_t* hes, const int32_t* step_index,
                          const int64_t* token_offset, const uint64_t* row_off, uint64_t rows,
                          const cdx_probe_cfg* cfg, uint8_t* decision) {
    using namespace cdx;
    if (!ctx) return CDX_EINVAL;
    if (!cfg) return set_error(ctx, CDX_EINVAL, "should_exit: null config");
    if (int st = check_probe_cfg(ctx, cfg)) return st;
    if (rows == 0) return CDX_OK;
    if (!ids || !hes || !step_index || !token_offset || !row_off || !decision)
        return set_error(ctx, CDX_EINVAL, "should_exit: null pointer");
    probe_should_exit_kernel<<<grid_for(ctx, rows), 256, 0, ctx->stream>>>(
        ids, hes, step_index, token_offset, row_off, rows, cfg->window, cfg->threshold, cfg->max_tokens, decision);
    CDX_CHECK_LAUNCH(ctx, "probe_should_exit");
    return CDX_OK;
}

int cdx_probe_final_answer(cdx_ctx* ctx, const uint8_t* hes, const int32_t* step_index, const uint64_t* row_off,
                           const int32_t* terminated_at, const uint8_t* termination_reason, uint64_t rows,
                           uint64_t* pos, uint8_t* low_conf) {
    using namespace cdx;
    if (!ctx) return CDX_EINVAL;
    if (rows == 0) return CDX_OK;
    if (!hes || !step_index || !row_off || !pos || !low_conf)
        return set_error(ctx, CDX_EINVAL, "final_answer: null pointer");
    probe_final_answer_kernel<<<grid_for(ctx, rows), 256, 0, ctx->stream>>>(hes, step_index, row_off, terminated_at,
                                                                           termination_reason, rows, pos, low_conf);
    CDX_CHECK_LAUNCH(ctx, "probe_final_answer");
    return CDX_OK;
}

int cdx_meets_thresholds_rows(cdx_ctx* ctx, const double* signals, const uint8_t* present, uint64_t rows,
                              const cdx_threshold* th, uint32_t n_th, uint8_t* meets) {
    using namespace cdx;
    if (!ctx) return CDX_EINVAL;
    if (n_th > 8) return set_error(ctx, CDX_EINVAL, "thresholds: at most 8 per call");
    if (n_th && !th) return set_error(ctx, CDX_EINVAL, "thresholds: null array");
    RowThresholds t{};
    t.n = n_th;
    for (uint32_t i = 0; i < n_th; ++i) {
        if (th[i].signal > 3 || th[i].dir > 1) return set_error(ctx, CDX_EINVAL, "thresholds: bad enum");
        t.th[i] = th[i];
    }
    if (rows == 0) return CDX_OK;
    if (!signals || !present || !meets) return set_error(ctx, CDX_EINVAL, "meets_thresholds: null pointer");
    meets_rows_kernel<<<grid_for(ctx, rows), 256, 0, ctx->stream>>>(signals, present, rows, t, meets, ctx->d_err);
    CDX_CHECK_LAUNCH(ctx, "meets_thresholds_rows");
    return CDX_OK;
}

int cdx_id_histogram(cdx_ctx* ctx, const uint32_t* ids, uint64_t n, uint32_t n_unique, uint32_t* counts) {
    using namespace cdx;
    if (!ctx) return CDX_EINVAL;
    if (n_unique == 0) return CDX_OK;
    if (!ids || !counts) return set_error(ctx, CDX_EINVAL, "id_histogram: null pointer");
    cudaError_t e = cudaMemsetAsync(counts, 0, static_cast<size_t>(n_unique) * 4, ctx->stream);
    if (e != cudaSuccess) return cuda_fail(ctx, e, "id_histogram");
    if (n == 0) return CDX_OK;
    id_histogram_kernel<<<grid_for(ctx, n), 256, 0, ctx->stream>>>(ids, n, n_unique, counts, ctx->d_err);
    CDX_CHECK_LAUNCH(ctx, "id_histogram");
    return CDX_OK;
}

int cdx_entropy_one(cdx_ctx* ctx, const uint32_t* sizes, uint32_t m, uint32_t total, double* H, double* Hcert) {
    using namespace cdx;
    if (!ctx) return CDX_EINVAL;
    // metrics.cpp:108-109 (validation order of semantic_entropy)
    if (total < 1 || m == 0) return set_error(ctx, CDX_EINVAL, "semantic_entropy: invalid clustering");
    if (!sizes) return set_error(ctx, CDX_EINVAL, "entropy_one: null pointer");
    if (total > (1u << 26)) return set_error(ctx, CDX_EINVAL, "entropy_one: total above 2^26");
    const uint32_t ns[1] = {total};
    TermTables tt;
    if (int st = build_term_tables(ctx, ns, 1, &tt)) return st;
    entropy_one_kernel<<<1, 32, 0, ctx->stream>>>(sizes, m, total, tt.tab, std::log(static_cast<double>(total)), H,
                                                  Hcert, ctx->d_err);
    CDX_CHECK_LAUNCH(ctx, "entropy_one");
    return CDX_OK;
}

int cdx_entropy_sizes_host(cdx_ctx* ctx, const int32_t* sizes, uint32_t m, int32_t total, double* H,
                           double* Hcert) {
    using namespace cdx;
    if (!ctx) return CDX_EINVAL;
    // metrics.cpp:108-112, in the reference's order: the clustering, then each cluster
    if (total < 1 || m == 0) return set_error(ctx, CDX_EINVAL, "semantic_entropy: invalid clustering");
    if (!sizes) return set_error(ctx, CDX_EINVAL, "entropy_sizes_host: null pointer");
    std::vector<double> terms(m);
    for (uint32_t k = 0; k < m; ++k) {
        if (sizes[k] < 1) return set_error(ctx, CDX_EINVAL, "semantic_entropy: empty cluster");
        terms[k] = host_term(static_cast<uint32_t>(sizes[k]), static_cast<uint32_t>(total));
    }
    double* d = static_cast<double*>(scratch2(ctx, static_cast<size_t>(m) * 8));
    if (!d) return set_error(ctx, CDX_ECUDA, "entropy_sizes_host: scratch allocation failed");
    cudaError_t e = cudaMemcpyAsync(d, terms.data(), static_cast<size_t>(m) * 8, cudaMemcpyHostToDevice, ctx->stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize(ctx->stream);  // `terms` is pageable and local
    if (e != cudaSuccess) return cuda_fail(ctx, e, "entropy_sizes_host");
    entropy_terms_kernel<<<1, 32, 0, ctx->stream>>>(d, m, std::log(static_cast<double>(total)), total == 1 ? 1 : 0, H,
                                                    Hcert);
    CDX_CHECK_LAUNCH(ctx, "entropy_sizes_host");
    return CDX_OK;
}

int cdx_iteration_tokens_rows(cdx_ctx* ctx, const int64_t* tokens, const uint64_t* row_off, uint64_t rows,
                              double prior, double* est) {
    using namespace cdx;
    if (!ctx) return CDX_EINVAL;
    if (rows == 0) return CDX_OK;
    if (!row_off || !est) return set_error(ctx, CDX_EINVAL, "iteration_tokens: null pointer");
    iteration_tokens_kernel<<<grid_for(ctx, rows), 256, 0, ctx->stream>>>(tokens, row_off, rows, prior, est);
    CDX_CHECK_LAUNCH(ctx, "iteration_tokens_rows");
    return CDX_OK;
}

// ---- device buffers on the context stream (for C/C++ hosts without cudart) ------------
int cdx_alloc(cdx_ctx* ctx, uint64_t bytes, void** out) {
    using namespace cdx;
    if (!ctx || !out) return CDX_EINVAL;
    *out = nullptr;
    cudaSetDevice(ctx->device);
    cudaError_t e = cudaMallocAsync(out, bytes ? bytes : 16, ctx->stream);
    if (e != cudaSuccess) return cuda_fail(ctx, e, "cdx_alloc");
    return CDX_OK;
}

int cdx_free(cdx_ctx* ctx, void* p) {
    using namespace cdx;
    if (!ctx) return CDX_EINVAL;
    if (!p) return CDX_OK;
    cudaError_t e = cudaFreeAsync(p, ctx->stream);
    if (e != cudaSuccess) return cuda_fail(ctx, e, "cdx_free");
    return CDX_OK;
}

int cdx_memcpy(cdx_ctx* ctx, void* dst, const void* src, uint64_t bytes) {
    using namespace cdx;
    if (!ctx) return CDX_EINVAL;
    if (bytes == 0) return CDX_OK;
    cudaError_t e = cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDefault, ctx->stream);
    if (e != cudaSuccess) return cuda_fail(ctx, e, "cdx_memcpy");
    return CDX_OK;
}

int cdx_memset(cdx_ctx* ctx, void* dst, int value, uint64_t bytes) {
    using namespace cdx;
    if (!ctx) return CDX_EINVAL;
    if (bytes == 0) return CDX_OK;
    cudaError_t e = cudaMemsetAsync(dst, value, bytes, ctx->stream);
    if (e != cudaSuccess) return cuda_fail(ctx, e, "cdx_memset");
    return CDX_OK;
}

}  // extern "C"
