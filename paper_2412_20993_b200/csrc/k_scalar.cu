// k_scalar.cu — one-round-trip entries behind the scalar C++ API (include/cdx/*.hpp).
//
// The reference's functions are called once per program with a handful of values (32
// answers, 16 rewards, a 64-record trace: runtime.cpp:264-313).  Every such call here is
// ONE pinned host->device copy of all its inputs, ONE kernel launch, ONE device->host copy
// of its outputs (plus the 4-byte device error word) and one stream synchronisation:
//
//   cdx_cluster_host        cluster_exact / flag_hesitation          metrics.cpp:21-37, probe.cpp:36-44
//   cdx_consistency_host    probe::consistency                       probe.cpp:64-75
//   cdx_should_exit_host    probe::should_exit                       probe.cpp:77-85
//   cdx_final_answer_host   probe::final_answer                      probe.cpp:87-102
//   cdx_entropy_host        semantic_entropy / certaindex_entropy    metrics.cpp:107-125
//   cdx_reward_host         certaindex_reward                        metrics.cpp:127-137
//   cdx_meets_host          combined_meets_thresholds                metrics.cpp:159-171
//
// Inputs and outputs are packed into a per-context staging pair (pinned host buffer, device
// buffer).  The clustering calls run one CTA: trim + 64-bit hash per answer, a shared-memory
// open-addressing table (atomicMin of the first index per hash), a byte verify against the
// first occurrence (a hash collision between distinct answers is reported, never merged),
// dense first-seen ids by a block scan, sizes by shared atomics.  The CoT decisions then
// follow in the same CTA on the interned ids (the same rules as k_rows.cu's row kernels).
// Larger calls (more than SC_MAX answers or SC_MAX_BYTES of text) use the batched kernels.
#include <cmath>
#include <cstring>
#include <vector>

#include "cdx_internal.cuh"

namespace cdx {
namespace {

constexpr uint32_t SC_MAX = 2048;              // answers per one-CTA call
constexpr uint64_t SC_MAX_BYTES = 1ull << 20;  // bytes of answer text per one-CTA call
constexpr uint32_t SC_TS = 2 * SC_MAX;         // hash table slots
constexpr uint32_t SC_THREADS = 512;
constexpr uint32_t EMPTY = 0xffffffffu;

// staging: inputs, then outputs, 16-byte aligned, in the context's pinned / device pair
struct Stage {
    cdx_ctx* ctx;
    size_t in = 0, out0 = 0, out = 0;
    bool ok = true, outs = false;
    static size_t up16(size_t x) { return (x + 15) & ~static_cast<size_t>(15); }
    explicit Stage(cdx_ctx* c, size_t bytes) : ctx(c) {
        if (bytes > ctx->sc_cap) {
            if (ctx->sc_h) cudaFreeHost(ctx->sc_h);
            if (ctx->sc_d) cudaFree(ctx->sc_d);
            ctx->sc_h = nullptr;
            ctx->sc_d = nullptr;
            ctx->sc_cap = 0;
            size_t cap = 1 << 16;
            while (cap < bytes) cap <<= 1;
            if (cudaHostAlloc(reinterpret_cast<void**>(&ctx->sc_h), cap, cudaHostAllocDefault) != cudaSuccess ||
                cudaMalloc(reinterpret_cast<void**>(&ctx->sc_d), cap) != cudaSuccess) {
                ok = false;
                return;
            }
            ctx->sc_cap = cap;
        }
    }
    template <class T>
    T* put(const T* src, size_t n) {  // an input: copied into the pinned buffer now
        const size_t off = in;
        if (n) std::memcpy(ctx->sc_h + off, src, n * sizeof(T));
        in = up16(in + n * sizeof(T));
        return reinterpret_cast<T*>(ctx->sc_d + off);
    }
    template <class T>
    T* put_zero(size_t n) {
        const size_t off = in;
        std::memset(ctx->sc_h + off, 0, n * sizeof(T));
        in = up16(in + n * sizeof(T));
        return reinterpret_cast<T*>(ctx->sc_d + off);
    }
    template <class T>
    T* outp(size_t n) {  // an output region (after every input)
        if (!outs) {
            out0 = out = in;
            outs = true;
        }
        const size_t off = out;
        out = up16(out + n * sizeof(T));
        return reinterpret_cast<T*>(ctx->sc_d + off);
    }
    template <class T>
    const T* host(const T* dev) const {  // an output's host copy after finish()
        return reinterpret_cast<const T*>(ctx->sc_h + (reinterpret_cast<const uint8_t*>(dev) - ctx->sc_d));
    }
    int upload() {
        const cudaError_t e = cudaMemcpyAsync(ctx->sc_d, ctx->sc_h, in, cudaMemcpyHostToDevice, ctx->stream);
        return e == cudaSuccess ? CDX_OK : cuda_fail(ctx, e, "scalar staging (upload)");
    }
    // outputs + the device error word back, one synchronisation, device errors surfaced
    int finish() {
        cudaError_t e = cudaSuccess;
        if (out > out0) e = cudaMemcpyAsync(ctx->sc_h + out0, ctx->sc_d + out0, out - out0, cudaMemcpyDeviceToHost, ctx->stream);
        if (e == cudaSuccess) e = cudaMemcpyAsync(ctx->h_err, ctx->d_err, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream);
        if (e == cudaSuccess) e = cudaStreamSynchronize(ctx->stream);
        if (e != cudaSuccess) return cuda_fail(ctx, e, "scalar staging (download)");
        return take_dev_err(ctx);
    }
};

// trimmed [b, b + len) of answer i: the six whitespace bytes of metrics::trim
__device__ __forceinline__ bool sc_space(uint8_t c) { return c == ' ' || (c >= '\t' && c <= '\r'); }

__device__ uint64_t sc_hash(const uint8_t* s, uint32_t len) {
    uint64_t h = 0xcbf29ce484222325ull ^ (static_cast<uint64_t>(len) * 0x9E3779B97F4A7C15ull);
    for (uint32_t i = 0; i < len; ++i) h = (h ^ s[i]) * 0x100000001b3ull;
    h ^= h >> 33;
    h *= 0xff51afd7ed558ccdull;
    h ^= h >> 33;
    return h ? h : 1;
}

// probe::flag_hesitation: ASCII-lowercased answer contains a non-empty marker (markers as given)
__device__ bool sc_hesitant(const uint8_t* s, uint32_t len, const uint8_t* mk, const uint32_t* moff, uint32_t nm) {
    for (uint32_t m = 0; m < nm; ++m) {
        const uint32_t mb = moff[m], ml = moff[m + 1] - mb;
        if (ml == 0 || ml > len) continue;
        for (uint32_t p = 0; p + ml <= len; ++p) {
            uint32_t j = 0;
            for (; j < ml; ++j) {
                uint8_t c = s[p + j];
                c = (c >= 'A' && c <= 'Z') ? c + 32 : c;
                if (c != mk[mb + j]) break;
            }
            if (j == ml) return true;
        }
    }
    return false;
}

struct ClusterIn {
    const uint8_t* bytes;
    const uint64_t* off;  // [n + 1]
    uint32_t n;
    const uint8_t* mk;    // markers (nullable)
    const uint32_t* moff;
    uint32_t nm;
};

// In shared memory after the call: id[i] (dense first-seen), and per cluster its first
// index and size; returns the cluster count.  Errors go to d_err.
__device__ uint32_t sc_cluster(const ClusterIn& a, uint8_t* hes_out, uint32_t* s_id, uint32_t* s_first, uint32_t* s_size,
                               uint64_t* s_key, uint32_t* s_min, uint32_t* s_tb, uint32_t* s_tl, uint64_t* s_h,
                               uint32_t* s_w, int* err) {
    const uint32_t tid = threadIdx.x, lane = tid & 31u, warp = tid >> 5;
    for (uint32_t s = tid; s < SC_TS; s += SC_THREADS) {
        s_key[s] = 0;
        s_min[s] = EMPTY;
    }
    for (uint32_t i = tid; i < a.n; i += SC_THREADS) {
        const uint64_t b = a.off[i], e = a.off[i + 1];
        const uint8_t* s = a.bytes + b;
        const uint32_t len = static_cast<uint32_t>(e - b);
        if (hes_out) hes_out[i] = sc_hesitant(s, len, a.mk, a.moff, a.nm) ? 1 : 0;
        uint32_t tb = 0, te = len;
        while (tb < te && sc_space(s[tb])) ++tb;
        while (te > tb && sc_space(s[te - 1])) --te;
        s_tb[i] = static_cast<uint32_t>(b) + tb;
        s_tl[i] = te - tb;
        s_h[i] = sc_hash(s + tb, te - tb);
    }
    __syncthreads();
    for (uint32_t i = tid; i < a.n; i += SC_THREADS) {  // insert: the smallest index per hash
        const uint64_t h = s_h[i];
        uint32_t slot = static_cast<uint32_t>(h) & (SC_TS - 1);
        for (;;) {
            const unsigned long long prev = atomicCAS(reinterpret_cast<unsigned long long*>(s_key + slot), 0ull, h);
            if (prev == 0ull || prev == h) break;
            slot = (slot + 1) & (SC_TS - 1);
        }
        atomicMin(s_min + slot, i);
        s_id[i] = slot;  // the slot for now
    }
    __syncthreads();
    for (uint32_t i = tid; i < a.n; i += SC_THREADS) {  // verify against the first occurrence
        const uint32_t f = s_min[s_id[i]];
        s_first[i] = f;
        if (f != i) {
            bool same = s_tl[i] == s_tl[f];
            for (uint32_t q = 0; same && q < s_tl[i]; ++q) same = a.bytes[s_tb[i] + q] == a.bytes[s_tb[f] + q];
            if (!same) set_dev_err(err, DEV_INTERN_COLLISION);
        }
    }
    __syncthreads();
    // dense ids: first occurrences numbered in index order (block scan in chunks); the hash
    // table's keys are no longer needed, their space holds each cluster's first index
    uint32_t* s_fidx = reinterpret_cast<uint32_t*>(s_key);
    uint32_t carry = 0;
    for (uint32_t c0 = 0; c0 < a.n; c0 += SC_THREADS) {
        const uint32_t i = c0 + tid;
        const uint32_t isf = i < a.n && s_first[i] == i ? 1u : 0u;
        const uint32_t bal = __ballot_sync(0xffffffffu, isf);
        if (lane == 0) s_w[warp] = __popc(bal);
        __syncthreads();
        uint32_t pre = carry, tot = 0;
        for (uint32_t w = 0; w < SC_THREADS / 32; ++w) {
            pre += w < warp ? s_w[w] : 0u;
            tot += s_w[w];
        }
        pre += __popc(bal & ((1u << lane) - 1u));
        if (isf) {
            s_min[s_id[i]] = pre;  // slot -> dense id
            s_size[pre] = 0;
            s_fidx[pre] = i;
        }
        carry += tot;
        __syncthreads();
    }
    for (uint32_t i = tid; i < a.n; i += SC_THREADS) s_id[i] = s_min[s_id[i]];
    __syncthreads();
    for (uint32_t i = tid; i < a.n; i += SC_THREADS) atomicAdd(s_size + s_id[i], 1u);
    __syncthreads();
    return carry;
}

constexpr size_t SC_SMEM = SC_TS * 8 + SC_TS * 4 + SC_MAX * (4 + 4 + 4 + 4 + 4 + 8) + 64 * 4;

struct ClusterOut {
    uint32_t* ids;      // [n] (nullable)
    uint8_t* hes;       // [n] (nullable)
    uint32_t* first;    // [n] first index per cluster (nullable)
    uint32_t* sizes;    // [n] (nullable)
    uint32_t* n_unique;
};

// op 0: clustering; 1: consistency(k, w); 2: should_exit; per-record arrays for ops 1-2
struct ProbeIn {
    int op;
    const uint8_t* rec_hes;
    const int32_t* step;
    const int64_t* tok;
    int32_t k, w;
    double tau;
    int64_t max_tokens;
    double* c_out;      // consistency value
    uint8_t* u8_out;    // ready flag / exit decision
};

__global__ void __launch_bounds__(SC_THREADS) scalar_cluster_kernel(ClusterIn a, ClusterOut o, ProbeIn pr, int* err) {
    extern __shared__ __align__(16) uint8_t sm[];
    uint64_t* s_key = reinterpret_cast<uint64_t*>(sm);
    uint64_t* s_h = s_key + SC_TS;
    uint32_t* s_min = reinterpret_cast<uint32_t*>(s_h + SC_MAX);
    uint32_t* s_id = s_min + SC_TS;
    uint32_t* s_first = s_id + SC_MAX;
    uint32_t* s_size = s_first + SC_MAX;
    uint32_t* s_tb = s_size + SC_MAX;
    uint32_t* s_tl = s_tb + SC_MAX;
    uint32_t* s_w = s_tl + SC_MAX;
    const uint32_t tid = threadIdx.x;
    const uint32_t nu = sc_cluster(a, o.hes, s_id, s_first, s_size, s_key, s_min, s_tb, s_tl, s_h, s_w, err);
    if (pr.op == 0) {
        const uint32_t* s_fidx = reinterpret_cast<const uint32_t*>(s_key);
        for (uint32_t i = tid; i < a.n; i += SC_THREADS)
            if (o.ids) o.ids[i] = s_id[i];
        for (uint32_t d = tid; d < nu; d += SC_THREADS) {
            if (o.sizes) o.sizes[d] = s_size[d];
            if (o.first) o.first[d] = s_fidx[d];
        }
        if (tid == 0 && o.n_unique) *o.n_unique = nu;
        return;
    }
    if (tid != 0) return;
    // the CoT decisions on the interned ids (k_rows.cu probe_consistency / should_exit rules)
    const uint32_t n = a.n;
    const int64_t kk = pr.op == 1 ? pr.k : static_cast<int64_t>(pr.step[n - 1]);
    uint32_t end = 0, usable = 0;
    for (; end < n; ++end) {
        if (static_cast<int64_t>(pr.step[end]) > kk) break;
        usable += pr.rec_hes[end] ? 0u : 1u;
    }
    uint32_t agree = 0;
    const bool ready = usable >= static_cast<uint32_t>(pr.w);
    if (ready) {
        uint32_t i = end, seen = 0, last = 0;
        while (i > 0 && seen < static_cast<uint32_t>(pr.w)) {
            --i;
            if (pr.rec_hes[i]) continue;
            if (seen == 0) last = s_id[i];
            agree += s_id[i] == last ? 1u : 0u;
            ++seen;
        }
    }
    const double c = ready ? __ddiv_rn(static_cast<double>(agree), static_cast<double>(pr.w)) : 0.0;
    if (pr.op == 1) {
        *pr.c_out = c;
        *pr.u8_out = ready ? 1 : 0;
    } else {
        uint8_t d = CDX_EXIT_CONTINUE;
        if (ready && c >= pr.tau) d = CDX_EXIT_CERTAIN;
        if (d == CDX_EXIT_CONTINUE && pr.tok[n - 1] >= pr.max_tokens) d = CDX_EXIT_BUDGET;
        *pr.u8_out = d;
    }
}

bool scalar_fits(uint64_t n, uint64_t bytes) { return n >= 1 && n <= SC_MAX && bytes <= SC_MAX_BYTES; }

int stage_answers(Stage& st, const char* bytes, const uint64_t* offsets, uint32_t n, const char* const* markers,
                  uint32_t n_markers, ClusterIn* a) {
    a->n = n;
    a->bytes = st.put(reinterpret_cast<const uint8_t*>(bytes), offsets[n] - offsets[0]);
    std::vector<uint64_t> off(n + 1);
    for (uint32_t i = 0; i <= n; ++i) off[i] = offsets[i] - offsets[0];
    a->off = st.put(off.data(), n + 1);
    std::vector<uint8_t> mk;
    std::vector<uint32_t> moff(1, 0);
    for (uint32_t m = 0; m < n_markers; ++m) {
        const size_t l = markers[m] ? std::strlen(markers[m]) : 0;
        mk.insert(mk.end(), markers[m], markers[m] + l);
        moff.push_back(static_cast<uint32_t>(mk.size()));
    }
    a->nm = n_markers;
    a->mk = st.put(mk.data(), mk.size());
    a->moff = st.put(moff.data(), moff.size());
    return CDX_OK;
}

size_t answers_bytes(const uint64_t* offsets, uint32_t n, const char* const* markers, uint32_t n_markers) {
    size_t b = (offsets[n] - offsets[0]) + (n + 1) * 8 + 64 + (n_markers + 1) * 4;
    for (uint32_t m = 0; m < n_markers; ++m) b += markers[m] ? std::strlen(markers[m]) : 0;
    return b;
}

int launch_cluster(cdx_ctx* ctx, const ClusterIn& a, const ClusterOut& o, const ProbeIn& pr) {
    static thread_local int dev = -1;
    if (dev != ctx->device) {
        cudaFuncSetAttribute(scalar_cluster_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(SC_SMEM));
        dev = ctx->device;
    }
    scalar_cluster_kernel<<<1, SC_THREADS, SC_SMEM, ctx->stream>>>(a, o, pr, ctx->d_err);
    CDX_CHECK_LAUNCH(ctx, "scalar_cluster");
    return CDX_OK;
}

}  // namespace
}  // namespace cdx

extern "C" {

int cdx_cluster_host(cdx_ctx* ctx, const char* bytes, const uint64_t* offsets, uint32_t n, const char* const* markers,
                     uint32_t n_markers, uint32_t* ids, uint8_t* hes, uint32_t* first_index, uint32_t* sizes,
                     uint32_t* n_unique) {
    using namespace cdx;
    CDX_NVTX("cdx_cluster_host");
    if (!ctx) return CDX_EINVAL;
    if (!offsets || !n_unique || (n && !bytes)) return set_error(ctx, CDX_EINVAL, "cluster_host: null pointer");
    if (!scalar_fits(n, offsets[n] - offsets[0]))
        return set_error(ctx, CDX_EINVAL, "cluster_host: 1..2048 answers of at most 1 MiB (use cdx_canon_intern)");
    if (n_markers > 16) return set_error(ctx, CDX_EINVAL, "cluster_host: at most 16 markers");
    Stage st(ctx, answers_bytes(offsets, n, markers, n_markers) + static_cast<size_t>(n) * 13 + 256);
    if (!st.ok) return set_error(ctx, CDX_ECUDA, "cluster_host: staging allocation failed");
    ClusterIn a{};
    stage_answers(st, bytes, offsets, n, markers, n_markers, &a);
    ClusterOut o{};
    o.ids = ids ? st.outp<uint32_t>(n) : nullptr;
    o.first = first_index ? st.outp<uint32_t>(n) : nullptr;
    o.sizes = sizes ? st.outp<uint32_t>(n) : nullptr;
    o.n_unique = st.outp<uint32_t>(1);
    o.hes = hes ? st.outp<uint8_t>(n) : nullptr;
    ProbeIn pr{};
    if (int s = st.upload()) return s;
    if (int s = launch_cluster(ctx, a, o, pr)) return s;
    if (int s = st.finish()) return s;
    const uint32_t nu = *st.host(o.n_unique);
    *n_unique = nu;
    if (ids) std::memcpy(ids, st.host(o.ids), n * 4);
    if (first_index) std::memcpy(first_index, st.host(o.first), nu * 4);
    if (sizes) std::memcpy(sizes, st.host(o.sizes), nu * 4);
    if (hes) std::memcpy(hes, st.host(o.hes), n);
    return CDX_OK;
}

static int probe_host(cdx_ctx* ctx, int op, const char* bytes, const uint64_t* offsets, uint32_t n, const uint8_t* hes,
                      const int32_t* step, const int64_t* tok, int32_t k, int32_t w, double tau, int64_t max_tokens,
                      double* c_out, uint8_t* u8_out) {
    using namespace cdx;
    if (!offsets || !hes || !step || !u8_out || (op == 2 && !tok) || (op == 1 && !c_out) || (n && !bytes))
        return set_error(ctx, CDX_EINVAL, "probe_host: null pointer");
    if (!scalar_fits(n, offsets[n] - offsets[0]))
        return set_error(ctx, CDX_EINVAL, "probe_host: 1..2048 records of at most 1 MiB (use the row kernels)");
    Stage st(ctx, answers_bytes(offsets, n, nullptr, 0) + static_cast<size_t>(n) * 13 + 256);
    if (!st.ok) return set_error(ctx, CDX_ECUDA, "probe_host: staging allocation failed");
    ClusterIn a{};
    stage_answers(st, bytes, offsets, n, nullptr, 0, &a);
    ProbeIn pr{};
    pr.op = op;
    pr.rec_hes = st.put(hes, n);
    pr.step = st.put(step, n);
    pr.tok = op == 2 ? st.put(tok, n) : nullptr;
    pr.k = k;
    pr.w = w;
    pr.tau = tau;
    pr.max_tokens = max_tokens;
    pr.c_out = st.outp<double>(1);
    pr.u8_out = st.outp<uint8_t>(1);
    ClusterOut o{};
    if (int s = st.upload()) return s;
    if (int s = launch_cluster(ctx, a, o, pr)) return s;
    if (int s = st.finish()) return s;
    if (c_out) *c_out = *st.host(pr.c_out);
    *u8_out = *st.host(pr.u8_out);
    return CDX_OK;
}

int cdx_consistency_host(cdx_ctx* ctx, const char* bytes, const uint64_t* offsets, uint32_t n, const uint8_t* hes,
                         const int32_t* step_index, int32_t k, int32_t w, double* C, uint8_t* ready) {
    using namespace cdx;
    CDX_NVTX("cdx_consistency_host");
    if (!ctx) return CDX_EINVAL;
    if (w < 1) return set_error(ctx, CDX_EINVAL, "consistency: window must be >= 1");
    return probe_host(ctx, 1, bytes, offsets, n, hes, step_index, nullptr, k, w, 0.0, 0, C, ready);
}

int cdx_should_exit_host(cdx_ctx* ctx, const char* bytes, const uint64_t* offsets, uint32_t n, const uint8_t* hes,
                         const int32_t* step_index, const int64_t* token_offset, const cdx_probe_cfg* cfg,
                         uint8_t* decision) {
    using namespace cdx;
    CDX_NVTX("cdx_should_exit_host");
    if (!ctx) return CDX_EINVAL;
    if (!cfg) return set_error(ctx, CDX_EINVAL, "should_exit_host: null config");
    if (int s = check_probe_cfg_c(ctx, cfg)) return s;
    return probe_host(ctx, 2, bytes, offsets, n, hes, step_index, token_offset, 0, cfg->window, cfg->threshold,
                      cfg->max_tokens, nullptr, decision);
}

int cdx_final_answer_host(cdx_ctx* ctx, const uint8_t* hes, const int32_t* step_index, uint32_t n,
                          int32_t terminated_at, uint8_t termination_reason, uint64_t* pos, uint8_t* low_conf) {
    using namespace cdx;
    CDX_NVTX("cdx_final_answer_host");
    if (!ctx) return CDX_EINVAL;
    if (!hes || !step_index || !pos || !low_conf) return set_error(ctx, CDX_EINVAL, "final_answer_host: null pointer");
    if (n == 0) return set_error(ctx, CDX_EINVAL, "final_answer: empty trace");
    Stage st(ctx, static_cast<size_t>(n) * 5 + 256);
    if (!st.ok) return set_error(ctx, CDX_ECUDA, "final_answer_host: staging allocation failed");
    const uint8_t* d_hes = st.put(hes, n);
    const int32_t* d_step = st.put(step_index, n);
    const uint64_t off[2] = {0, n};
    const uint64_t* d_off = st.put(off, 2);
    const int32_t* d_term = st.put(&terminated_at, 1);
    const uint8_t* d_why = st.put(&termination_reason, 1);
    uint64_t* d_pos = st.outp<uint64_t>(1);
    uint8_t* d_low = st.outp<uint8_t>(1);
    if (int s = st.upload()) return s;
    if (int s = cdx_probe_final_answer(ctx, d_hes, d_step, d_off, d_term, d_why, 1, d_pos, d_low)) return s;
    if (int s = st.finish()) return s;
    *pos = *st.host(d_pos);
    *low_conf = *st.host(d_low);
    return CDX_OK;
}

int cdx_entropy_host(cdx_ctx* ctx, const int32_t* sizes, uint32_t m, int32_t total, double* H, double* Hcert) {
    using namespace cdx;
    CDX_NVTX("cdx_entropy_host");
    if (!ctx) return CDX_EINVAL;
    // metrics.cpp:108-112, in the reference's order: the clustering, then each cluster
    if (total < 1 || m == 0) return set_error(ctx, CDX_EINVAL, "semantic_entropy: invalid clustering");
    if (!sizes || (!H && !Hcert)) return set_error(ctx, CDX_EINVAL, "entropy_host: null pointer");
    std::vector<double> terms(m);
    for (uint32_t k = 0; k < m; ++k) {
        if (sizes[k] < 1) return set_error(ctx, CDX_EINVAL, "semantic_entropy: empty cluster");
        terms[k] = host_term(static_cast<uint32_t>(sizes[k]), static_cast<uint32_t>(total));
    }
    Stage st(ctx, static_cast<size_t>(m) * 8 + 64);
    if (!st.ok) return set_error(ctx, CDX_ECUDA, "entropy_host: staging allocation failed");
    const double* d_terms = st.put(terms.data(), m);
    double* d_out = st.outp<double>(2);
    if (int s = st.upload()) return s;
    if (int s = entropy_terms_launch(ctx, d_terms, m, std::log(static_cast<double>(total)), total == 1, d_out, d_out + 1))
        return s;
    if (int s = st.finish()) return s;
    if (H) *H = st.host(d_out)[0];
    if (Hcert) *Hcert = st.host(d_out)[1];
    return CDX_OK;
}

int cdx_reward_host(cdx_ctx* ctx, const double* rewards, uint64_t n, uint8_t aggregation, double* out) {
    using namespace cdx;
    CDX_NVTX("cdx_reward_host");
    if (!ctx) return CDX_EINVAL;
    if (!out || (n && !rewards)) return set_error(ctx, CDX_EINVAL, "reward_host: null pointer");
    Stage st(ctx, static_cast<size_t>(n) * 8 + 96);
    if (!st.ok) return set_error(ctx, CDX_ECUDA, "reward_host: staging allocation failed");
    const double* d_v = st.put(rewards, n);
    const uint64_t off[2] = {0, n};
    const uint64_t* d_off = st.put(off, 2);
    const uint8_t* d_agg = st.put(&aggregation, 1);
    double* d_out = st.outp<double>(1);
    if (int s = st.upload()) return s;
    if (int s = cdx_reward_sets(ctx, d_v, d_off, d_agg, 1, d_out)) return s;
    if (int s = st.finish()) return s;
    *out = *st.host(d_out);
    return CDX_OK;
}

int cdx_meets_host(cdx_ctx* ctx, const double* signals4, uint8_t present, const cdx_threshold* th, uint32_t n_th,
                   uint8_t* meets) {
    using namespace cdx;
    CDX_NVTX("cdx_meets_host");
    if (!ctx) return CDX_EINVAL;
    if (!signals4 || !meets) return set_error(ctx, CDX_EINVAL, "meets_host: null pointer");
    Stage st(ctx, 128);
    if (!st.ok) return set_error(ctx, CDX_ECUDA, "meets_host: staging allocation failed");
    const double* d_sig = st.put(signals4, 4);
    const uint8_t* d_present = st.put(&present, 1);
    uint8_t* d_out = st.outp<uint8_t>(1);
    if (int s = st.upload()) return s;
    if (int s = cdx_meets_thresholds_rows(ctx, d_sig, d_present, 1, th, n_th, d_out)) return s;
    if (int s = st.finish()) return s;
    *meets = *st.host(d_out);
    return CDX_OK;
}

}  // extern "C"
