// k_gang.cu — K6: gang-scheduling program order (escalation + SJF/FIFO priority + total
// tie-break), as a hand-written LSD radix sort, plus the merge of per-rank sorted runs.
//
// Replaces scheduler.escalate / estimate_iteration_tokens / next_batch program order, which
// exist only in SPEC.md:422-448 (no reference code):
//   escalated  = (now - last_service) >= starvation_limit            (inclusive, :443,:472)
//   est tokens = mean of completed iteration tokens, else the prior     (:431-439)
//   key        = escalated: arrival (FIFO among escalated, :443)
//                else fifo: arrival | sjf: est * remaining knob          (:425,:469)
//   order      = (escalated first, key, arrival, program id)           (:470 total order)
//   terminated programs are dropped.
//
// Sort keys: every time is a finite non-negative double (validated), so its IEEE bits are
// order-preserving as u64 and bit 63 is free: hi = (escalated ? 0 : 1) << 63 | bits(key)
// (-0.0 canonicalised to +0.0 so bitwise order equals == order).  The (arrival, id)
// tie-break is applied first by a stable sort on bits(arrival) over the id-ordered input
// (skipped when arrivals are already non-decreasing), then a stable sort on hi; digits on
// which all keys agree are skipped.  One pass = upsweep histograms (all 8 digits in one
// read), an exclusive scan, and a stable scatter whose in-tile ranks come from warp
// match + popc (the ADU is idle in this kernel, so MATCH is the cheap ranker here).
#include <algorithm>
#include <cstring>
#include <vector>

#include "cdx_internal.cuh"

namespace cdx {
namespace {

constexpr int RS_THREADS = 256;
constexpr int RS_ITEMS = 16;
constexpr int RS_TILE = RS_THREADS * RS_ITEMS;  // keys per tile
constexpr int RS_WARPS = RS_THREADS / 32;

struct GangParams {
    const double* arrival;
    const double* last_service;
    const int64_t* iter_tok_sum;
    const uint32_t* iter_count;
    const uint16_t* knob;
    const uint16_t* cap;
    const uint8_t* terminated;
    uint8_t* escalated;
    uint64_t N;
    uint32_t id_base;
    int order;
    double now, limit, prior;
};

__device__ __forceinline__ uint64_t dbits(double x) {
    x = x == 0.0 ? 0.0 : x;  // -0.0 == +0.0 under the comparator
    return static_cast<uint64_t>(__double_as_longlong(x));
}

// per program: escalation flag, live flag, hi key, arrival bits; bad times flag an error
__global__ void gang_keys(const GangParams p, uint64_t* __restrict__ hi, uint64_t* __restrict__ arr,
                          uint32_t* __restrict__ live, int* bad) {
    for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < p.N;
         i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
        const double a = p.arrival[i], ls = p.last_service[i];
        if (!(a >= 0.0) || !(ls >= 0.0) || isinf(a) || isinf(ls)) atomicExch(bad, 1);
        const bool esc = (p.now - ls) >= p.limit;  // inclusive escalation
        if (p.escalated) p.escalated[i] = esc ? 1 : 0;
        double key;
        if (esc || p.order == CDX_ORDER_FIFO) {
            key = a;
        } else {
            const uint32_t c = p.iter_count[i];
            const double est = c ? __ddiv_rn(static_cast<double>(p.iter_tok_sum[i]), static_cast<double>(c)) : p.prior;
            const int rem = static_cast<int>(p.cap[i]) - static_cast<int>(p.knob[i]);
            key = __dmul_rn(est, static_cast<double>(rem > 0 ? rem : 0));
            if (!(key >= 0.0) || isinf(key)) atomicExch(bad, 1);
        }
        hi[i] = (esc ? 0ull : (1ull << 63)) | dbits(key);
        arr[i] = dbits(a);
        live[i] = p.terminated[i] ? 0u : 1u;
    }
}

// ---- generic u32 exclusive scan (3 phases) --------------------------------------------
constexpr int SCAN_T = 512;
__global__ void scan_blocks(const uint32_t* __restrict__ in, uint32_t* __restrict__ out, uint64_t n,
                            uint32_t* __restrict__ block_sums) {
    __shared__ uint32_t s[SCAN_T];
    const uint64_t i = blockIdx.x * static_cast<uint64_t>(SCAN_T) + threadIdx.x;
    const uint32_t x = i < n ? in[i] : 0u;
    s[threadIdx.x] = x;
    __syncthreads();
    for (int o = 1; o < SCAN_T; o <<= 1) {
        const uint32_t y = threadIdx.x >= static_cast<unsigned>(o) ? s[threadIdx.x - o] : 0u;
        __syncthreads();
        s[threadIdx.x] += y;
        __syncthreads();
    }
    if (i < n) out[i] = s[threadIdx.x] - x;
    if (threadIdx.x == SCAN_T - 1) block_sums[blockIdx.x] = s[threadIdx.x];
}
__global__ void scan_sums(uint32_t* __restrict__ sums, uint64_t nb, uint32_t* __restrict__ total) {
    __shared__ uint32_t s[1024];
    // chunked single-CTA exclusive scan of nb block sums
    uint32_t carry = 0;
    for (uint64_t base = 0; base < nb; base += 1024) {
        const uint64_t i = base + threadIdx.x;
        const uint32_t x = i < nb ? sums[i] : 0u;
        s[threadIdx.x] = x;
        __syncthreads();
        for (int o = 1; o < 1024; o <<= 1) {
            const uint32_t y = threadIdx.x >= static_cast<unsigned>(o) ? s[threadIdx.x - o] : 0u;
            __syncthreads();
            s[threadIdx.x] += y;
            __syncthreads();
        }
        if (i < nb) sums[i] = carry + s[threadIdx.x] - x;
        const uint32_t tot = s[1023];
        __syncthreads();
        carry += tot;
    }
    if (threadIdx.x == 0 && total) *total = carry;
}
__global__ void scan_add(uint32_t* __restrict__ v, uint64_t n, const uint32_t* __restrict__ sums) {
    const uint64_t i = blockIdx.x * static_cast<uint64_t>(SCAN_T) + threadIdx.x;
    if (i < n) v[i] += sums[blockIdx.x];
}

// compaction of live programs: position = excl[i]
__global__ void gang_compact(uint64_t N, const uint32_t* __restrict__ live, const uint32_t* __restrict__ pos,
                             const uint64_t* __restrict__ hi, const uint64_t* __restrict__ arr, uint32_t id_base,
                             uint64_t* __restrict__ khi, uint64_t* __restrict__ karr, uint32_t* __restrict__ kid) {
    for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < N;
         i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
        if (!live[i]) continue;
        const uint32_t j = pos[i];
        khi[j] = hi[i];
        karr[j] = arr[i];
        kid[j] = id_base + static_cast<uint32_t>(i);
    }
}

__global__ void count_unsorted(const uint64_t* __restrict__ k, uint64_t n, uint32_t* __restrict__ flag) {
    for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i + 1 < n;
         i += static_cast<uint64_t>(gridDim.x) * blockDim.x)
        if (k[i] > k[i + 1]) atomicExch(flag, 1u);
}

// ---- LSD radix sort of (u64 key, u32 value) --------------------------------------------
// all 8 digit histograms of one tile: hist[(d*256 + digit) * ntiles + tile]
__global__ void __launch_bounds__(RS_THREADS) rs_upsweep(const uint64_t* __restrict__ keys, uint64_t n,
                                                         uint32_t ntiles, uint32_t* __restrict__ hist) {
    __shared__ uint32_t h[8][256];
    for (int i = threadIdx.x; i < 8 * 256; i += RS_THREADS) (&h[0][0])[i] = 0;
    __syncthreads();
    const uint64_t base = static_cast<uint64_t>(blockIdx.x) * RS_TILE;
    for (int j = 0; j < RS_ITEMS; ++j) {
        const uint64_t i = base + j * RS_THREADS + threadIdx.x;
        if (i < n) {
            const uint64_t k = keys[i];
#pragma unroll
            for (int d = 0; d < 8; ++d) atomicAdd(&h[d][(k >> (8 * d)) & 0xff], 1u);
        }
    }
    __syncthreads();
    for (int i = threadIdx.x; i < 8 * 256; i += RS_THREADS) hist[static_cast<uint64_t>(i) * ntiles + blockIdx.x] = (&h[0][0])[i];
}

// stable scatter of one digit: warp w of a tile owns keys [base + w*32*ITEMS, +32*ITEMS),
// processed in order 32 at a time; peers with the same digit are ranked by match + popc
__global__ void __launch_bounds__(RS_THREADS) rs_scatter(const uint64_t* __restrict__ kin,
                                                         const uint32_t* __restrict__ vin, uint64_t* __restrict__ kout,
                                                         uint32_t* __restrict__ vout, uint64_t n, uint32_t ntiles,
                                                         const uint32_t* __restrict__ offs, int shift) {
    __shared__ uint32_t wcnt[RS_WARPS][256];
    const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (int i = threadIdx.x; i < RS_WARPS * 256; i += RS_THREADS) (&wcnt[0][0])[i] = 0;
    __syncthreads();
    const uint64_t base = static_cast<uint64_t>(blockIdx.x) * RS_TILE + static_cast<uint64_t>(warp) * 32 * RS_ITEMS;
    uint64_t k[RS_ITEMS];
    uint32_t v[RS_ITEMS], rank[RS_ITEMS], dig[RS_ITEMS];
    const uint32_t lt = (1u << lane) - 1u;
#pragma unroll
    for (int j = 0; j < RS_ITEMS; ++j) {
        const uint64_t i = base + j * 32 + lane;
        const bool ok = i < n;
        k[j] = ok ? kin[i] : 0;
        v[j] = ok ? vin[i] : 0;
        const uint32_t d = ok ? static_cast<uint32_t>((k[j] >> shift) & 0xff) : 256u + lane;  // unique dummy
        dig[j] = d;
        const uint32_t peers = __match_any_sync(0xffffffffu, d);
        uint32_t before = 0;
        if (ok) before = wcnt[warp][d];
        __syncwarp();
        rank[j] = before + __popc(peers & lt);
        if (ok && (peers & lt) == 0) wcnt[warp][d] = before + __popc(peers);
        __syncwarp();
    }
    __syncthreads();
    // exclusive prefix of each digit's count over the warps of this tile
    for (int d = threadIdx.x; d < 256; d += RS_THREADS) {
        uint32_t acc = 0;
        for (int w = 0; w < RS_WARPS; ++w) {
            const uint32_t c = wcnt[w][d];
            wcnt[w][d] = acc;
            acc += c;
        }
    }
    __syncthreads();
#pragma unroll
    for (int j = 0; j < RS_ITEMS; ++j) {
        const uint64_t i = base + j * 32 + lane;
        if (i < n) {
            const uint32_t d = dig[j];
            const uint64_t pos = static_cast<uint64_t>(offs[static_cast<uint64_t>(d) * ntiles + blockIdx.x]) +
                                 wcnt[warp][d] + rank[j];
            kout[pos] = k[j];
            vout[pos] = v[j];
        }
    }
}

// keys[i] = {hi, arrival bits, id} of the i-th program in priority order (merge input)
__global__ void pack_keys(const uint64_t* __restrict__ shi, const uint64_t* __restrict__ karr,
                          const uint32_t* __restrict__ kid, const uint32_t* __restrict__ fin, uint64_t* __restrict__ keys,
                          uint64_t n) {
    for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
        const uint32_t j = fin[i];
        keys[3 * i] = shi[i];
        keys[3 * i + 1] = karr[j];
        keys[3 * i + 2] = kid[j];
    }
}

__global__ void iota_u32(uint32_t* __restrict__ v, uint64_t n) {
    for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<uint64_t>(gridDim.x) * blockDim.x)
        v[i] = static_cast<uint32_t>(i);
}

template <typename T>
__global__ void gather(const T* __restrict__ src, const uint32_t* __restrict__ idx, T* __restrict__ dst, uint64_t n) {
    for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<uint64_t>(gridDim.x) * blockDim.x)
        dst[i] = src[idx[i]];
}

struct Launch {
    cdx_ctx* ctx;
    unsigned grid(uint64_t n, unsigned t = 256) const {
        return static_cast<unsigned>(std::max<uint64_t>(1, std::min<uint64_t>((n + t - 1) / t, ctx->sm_count * 16ull)));
    }
};

// exclusive scan of n u32 in place (out may alias in); returns total via device scalar
int scan_u32(cdx_ctx* ctx, const uint32_t* in, uint32_t* out, uint64_t n, uint32_t* sums, uint32_t* total) {
    const uint64_t nb = (n + SCAN_T - 1) / SCAN_T;
    scan_blocks<<<static_cast<unsigned>(nb), SCAN_T, 0, ctx->stream>>>(in, out, n, sums);
    CDX_CHECK_LAUNCH(ctx, "scan(blocks)");
    scan_sums<<<1, 1024, 0, ctx->stream>>>(sums, nb, total);
    CDX_CHECK_LAUNCH(ctx, "scan(sums)");
    scan_add<<<static_cast<unsigned>(nb), SCAN_T, 0, ctx->stream>>>(out, n, sums);
    CDX_CHECK_LAUNCH(ctx, "scan(add)");
    return CDX_OK;
}

// Stable LSD radix sort of (keys, vals) over 8-bit digits; digits where every key agrees
// are skipped (decided on the host from the upsweep histograms).  Returns which buffer
// holds the result (0: k0/v0, 1: k1/v1).
int radix_sort(cdx_ctx* ctx, uint64_t* k0, uint32_t* v0, uint64_t* k1, uint32_t* v1, uint64_t n, uint32_t* hist,
               uint32_t* sums, int* which) {
    *which = 0;
    if (n <= 1) return CDX_OK;
    const uint32_t ntiles = static_cast<uint32_t>((n + RS_TILE - 1) / RS_TILE);
    rs_upsweep<<<ntiles, RS_THREADS, 0, ctx->stream>>>(k0, n, ntiles, hist);
    CDX_CHECK_LAUNCH(ctx, "radix(upsweep)");
    // per-digit totals to decide which passes are needed
    std::vector<uint32_t> h(static_cast<size_t>(8) * 256 * ntiles);
    cudaError_t e = cudaMemcpyAsync(h.data(), hist, h.size() * 4, cudaMemcpyDeviceToHost, ctx->stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize(ctx->stream);
    if (e != cudaSuccess) return cuda_fail(ctx, e, "radix(histograms)");
    uint64_t* kin = k0;
    uint32_t* vin = v0;
    uint64_t* kout = k1;
    uint32_t* vout = v1;
    for (int d = 0; d < 8; ++d) {
        bool trivial = false;
        for (int b = 0; b < 256 && !trivial; ++b) {
            uint64_t tot = 0;
            const uint32_t* row = h.data() + (static_cast<size_t>(d) * 256 + b) * ntiles;
            for (uint32_t t = 0; t < ntiles; ++t) tot += row[t];
            if (tot == n) trivial = true;
            if (tot) break;  // first non-empty bucket decides
        }
        if (trivial) continue;
        uint32_t* dh = hist + static_cast<size_t>(d) * 256 * ntiles;
        // NOTE: digit histograms were taken on the ORIGINAL order; per-tile counts must
        // match the current order, so recompute this digit's histogram on kin.
        rs_upsweep<<<ntiles, RS_THREADS, 0, ctx->stream>>>(kin, n, ntiles, hist);
        CDX_CHECK_LAUNCH(ctx, "radix(upsweep)");
        if (int st = scan_u32(ctx, dh, dh, static_cast<uint64_t>(256) * ntiles, sums, nullptr)) return st;
        rs_scatter<<<ntiles, RS_THREADS, 0, ctx->stream>>>(kin, vin, kout, vout, n, ntiles, dh, 8 * d);
        CDX_CHECK_LAUNCH(ctx, "radix(scatter)");
        std::swap(kin, kout);
        std::swap(vin, vout);
    }
    *which = kin == k0 ? 0 : 1;
    return CDX_OK;
}

// ---- merge of sorted runs by ranking: pos = own index + #smaller keys in every other run
struct Key3 {
    uint64_t hi, arr;
    uint32_t id;
};
__device__ __forceinline__ bool key_less(const uint64_t* k, uint64_t i, uint64_t a0, uint64_t a1, uint64_t a2) {
    const uint64_t b0 = k[3 * i], b1 = k[3 * i + 1], b2 = k[3 * i + 2];
    if (b0 != a0) return b0 < a0;
    if (b1 != a1) return b1 < a1;
    return b2 < a2;
}
// Merge of per-rank sorted runs laid out with a fixed stride (the NCCL allgather receive
// buffer: run q occupies [q*stride, q*stride + run_len[q])).  Keys are unique (the id is the
// last key word), so an element's global position is its index in its own run plus, for
// every other run, the number of keys there that are smaller: a merge-path rank computed
// with one binary search per run, no global synchronisation.
__global__ void merge_rank(const uint64_t* __restrict__ keys, const uint64_t* __restrict__ run_len, uint32_t runs,
                           uint64_t stride, uint32_t* __restrict__ out, uint64_t* __restrict__ total) {
    const uint64_t slots = static_cast<uint64_t>(runs) * stride;
    for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < slots;
         i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
        const uint32_t r = static_cast<uint32_t>(i / stride);
        const uint64_t j = i - static_cast<uint64_t>(r) * stride;
        if (j >= run_len[r]) continue;
        const uint64_t a0 = keys[3 * i], a1 = keys[3 * i + 1], a2 = keys[3 * i + 2];
        uint64_t pos = j;
        for (uint32_t q = 0; q < runs; ++q) {
            if (q == r) continue;
            uint64_t lo = static_cast<uint64_t>(q) * stride, hi = lo + run_len[q];
            const uint64_t base = lo;
            while (lo < hi) {  // keys of run q that are < (a0,a1,a2)
                const uint64_t mid = (lo + hi) >> 1;
                if (key_less(keys, mid, a0, a1, a2)) lo = mid + 1;
                else hi = mid;
            }
            pos += lo - base;
        }
        out[pos] = static_cast<uint32_t>(a2);
    }
    if (total && blockIdx.x == 0 && threadIdx.x == 0) {
        uint64_t t = 0;
        for (uint32_t q = 0; q < runs; ++q) t += run_len[q];
        *total = t;
    }
}

}  // namespace
}  // namespace cdx

extern "C" int cdx_gang_priority(cdx_ctx* ctx, const cdx_prog_soa* progs, uint64_t N, const cdx_inter_policy* pol,
                                 double now, uint32_t* order, uint64_t* n_out, uint8_t* escalated, uint64_t* keys) {
    using namespace cdx;
    if (!ctx) return CDX_EINVAL;
    if (!progs || !pol || !order || !n_out) return set_error(ctx, CDX_EINVAL, "gang_priority: null pointer");
    if (!(pol->starvation_limit > 0.0))
        return set_error(ctx, CDX_EINVAL, "scheduler: starvation_limit must be > 0");
    if (pol->order != CDX_ORDER_FIFO && pol->order != CDX_ORDER_SJF)
        return set_error(ctx, CDX_EINVAL, "scheduler: order must be fifo or sjf_estimated");
    if (N >= 0xffffffffull) return set_error(ctx, CDX_EINVAL, "gang_priority: at most 2^32-2 programs");
    *n_out = 0;
    if (N == 0) return CDX_OK;
    GangParams p{progs->arrival, progs->last_service, progs->iter_tok_sum, progs->iter_count, progs->knob,
                 progs->cap, progs->terminated, escalated, N, progs->id_base, pol->order, now,
                 pol->starvation_limit, pol->prior_tokens};
    const uint32_t ntiles = static_cast<uint32_t>((N + RS_TILE - 1) / RS_TILE);
    const uint64_t nb = (N + SCAN_T - 1) / SCAN_T + 1;
    const uint64_t nh = static_cast<uint64_t>(8) * 256 * ntiles;
    // scratch layout
    const size_t bytes = N * 8 * 6 + N * 4 * 6 + nh * 4 + (nb + std::max<uint64_t>(nh / SCAN_T + 2, 1)) * 4 + 256;
    uint8_t* s = static_cast<uint8_t*>(scratch(ctx, bytes));
    if (!s) return set_error(ctx, CDX_ECUDA, "gang_priority: scratch allocation failed");
    uint64_t* hi = reinterpret_cast<uint64_t*>(s);
    uint64_t* arr = hi + N;
    uint64_t* khi = arr + N;
    uint64_t* karr = khi + N;
    uint64_t* t0 = karr + N;
    uint64_t* t1 = t0 + N;
    uint32_t* live = reinterpret_cast<uint32_t*>(t1 + N);
    uint32_t* pos = live + N;
    uint32_t* kid = pos + N;
    uint32_t* va = kid + N;
    uint32_t* vb = va + N;
    uint32_t* perm = vb + N;
    uint32_t* hist = perm + N;
    uint32_t* sums = hist + nh;
    uint32_t* misc = sums + std::max<uint64_t>(nb, nh / SCAN_T + 2);  // [0] total, [1] unsorted flag, [2] bad
    cudaMemsetAsync(misc, 0, 16, ctx->stream);
    Launch L{ctx};
    gang_keys<<<L.grid(N), 256, 0, ctx->stream>>>(p, hi, arr, live, reinterpret_cast<int*>(misc + 2));
    CDX_CHECK_LAUNCH(ctx, "gang_priority(keys)");
    if (int st = scan_u32(ctx, live, pos, N, sums, misc)) return st;
    gang_compact<<<L.grid(N), 256, 0, ctx->stream>>>(N, live, pos, hi, arr, progs->id_base, khi, karr, kid);
    CDX_CHECK_LAUNCH(ctx, "gang_priority(compact)");
    uint32_t hm[3];
    cudaError_t e = cudaMemcpyAsync(hm, misc, 12, cudaMemcpyDeviceToHost, ctx->stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize(ctx->stream);
    if (e != cudaSuccess) return cuda_fail(ctx, e, "gang_priority");
    if (hm[2]) return set_error(ctx, CDX_EINVAL, "gang_priority: times and keys must be finite and >= 0");
    const uint64_t n = hm[0];
    *n_out = n;
    if (n == 0) return CDX_OK;
    // 1) (arrival, id): programs are in id order; a stable sort on arrival bits yields the
    //    tie-break order.  Skip it when arrivals are already non-decreasing.
    count_unsorted<<<L.grid(n), 256, 0, ctx->stream>>>(karr, n, misc + 1);
    CDX_CHECK_LAUNCH(ctx, "gang_priority(sorted?)");
    e = cudaMemcpyAsync(hm, misc, 8, cudaMemcpyDeviceToHost, ctx->stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize(ctx->stream);
    if (e != cudaSuccess) return cuda_fail(ctx, e, "gang_priority");
    iota_u32<<<L.grid(n), 256, 0, ctx->stream>>>(va, n);
    CDX_CHECK_LAUNCH(ctx, "gang_priority(iota)");
    uint32_t* p1 = va;  // permutation: position -> compacted index
    if (hm[1]) {
        cudaMemcpyAsync(t0, karr, n * 8, cudaMemcpyDeviceToDevice, ctx->stream);
        int which = 0;
        if (int st = radix_sort(ctx, t0, va, t1, vb, n, hist, sums, &which)) return st;
        p1 = which ? vb : va;
    }
    // 2) stable sort on hi over the (arrival, id) order
    gather<uint64_t><<<L.grid(n), 256, 0, ctx->stream>>>(khi, p1, t0, n);
    CDX_CHECK_LAUNCH(ctx, "gang_priority(gather)");
    uint32_t* pa = p1 == va ? vb : va;  // free buffer pair for the second sort's values
    cudaMemcpyAsync(pa, p1, n * 4, cudaMemcpyDeviceToDevice, ctx->stream);
    uint32_t* pb = perm;
    int which = 0;
    if (int st = radix_sort(ctx, t0, pa, t1, pb, n, hist, sums, &which)) return st;
    uint32_t* fin = which ? pb : pa;  // position -> compacted index
    gather<uint32_t><<<L.grid(n), 256, 0, ctx->stream>>>(kid, fin, order, n);
    CDX_CHECK_LAUNCH(ctx, "gang_priority(order)");
    if (keys) {
        pack_keys<<<L.grid(n), 256, 0, ctx->stream>>>(which ? t1 : t0, karr, kid, fin, keys, n);
        CDX_CHECK_LAUNCH(ctx, "gang_priority(keys)");
    }
    return CDX_OK;
}

extern "C" int cdx_gang_merge(cdx_ctx* ctx, const uint64_t* keys, const uint64_t* run_len, uint32_t runs,
                              uint64_t stride, uint32_t* order_out, uint64_t* total) {
    using namespace cdx;
    if (!ctx) return CDX_EINVAL;
    if (!keys || !run_len || !order_out || runs == 0) return set_error(ctx, CDX_EINVAL, "gang_merge: bad args");
    if (stride == 0) return CDX_OK;
    Launch L{ctx};
    merge_rank<<<L.grid(static_cast<uint64_t>(runs) * stride), 256, 0, ctx->stream>>>(keys, run_len, runs, stride,
                                                                                      order_out, total);
    CDX_CHECK_LAUNCH(ctx, "gang_merge");
    return CDX_OK;
}
