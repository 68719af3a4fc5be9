// k_alloc.cu — K5: certaindex-driven allocation decision + exclusive scan of token budgets
// + stable compaction of continuing requests, in ONE single-pass kernel (decoupled
// look-back scan: each tile publishes its aggregate, then resolves its exclusive prefix
// from its predecessors' published state; tiles are claimed in order from an atomic
// counter so every predecessor is guaranteed to be resident or finished).
//
// Semantics restated from SPEC.md:404-412 (scheduler.allocate; no reference code exists):
//   even               -> grant to the cap
//   static_threshold   -> at detect_at, terminate iff the thresholds hold, else grant to cap
//   k_step_threshold   -> re-test every recheck_every units from detect_at on
//   always terminate at resource_cap.
// token budget = granted * tokens_per_unit; kept = requests granted past detect_at.
#include "cdx_internal.cuh"

namespace cdx {

constexpr int AL_THREADS = 256;
constexpr int AL_ITEMS = 4;
constexpr int AL_TILE = AL_THREADS * AL_ITEMS;
constexpr int AL_MAX_WORDS = 128;  // P <= 4096

struct AllocParams {
    const uint32_t* meets;
    int32_t* exit_knob;
    uint8_t* reason;
    int32_t* granted;
    int64_t* offsets;
    uint32_t* kept;
    uint64_t* n_kept;
    int64_t* tokens_saved;
    int64_t* total_budget;
    uint32_t* tile_counter;
    uint32_t* flags;     // [ntiles] 0 = none, 1 = aggregate, 2 = inclusive prefix
    int64_t* agg_b;      // [ntiles]
    int64_t* inc_b;
    uint32_t* agg_k;
    uint32_t* inc_k;
    uint64_t R;
    uint32_t ntiles;
    uint32_t words;
    int32_t cap, detect;
    int64_t tpu;
    int64_t base_offset;
    uint32_t kept_base;
    uint32_t chk[AL_MAX_WORDS];  // knob positions (bit p = knob p+1) at which to test
};

__device__ __forceinline__ uint32_t ld_acquire(const uint32_t* p) {
    uint32_t v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_release(uint32_t* p, uint32_t v) {
    asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

template <typename T>
__device__ __forceinline__ T warp_incl_scan(T v, int lane) {
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const T n = __shfl_up_sync(0xffffffffu, v, o);
        if (lane >= o) v += n;
    }
    return v;
}

__global__ void __launch_bounds__(AL_THREADS) allocate_scan_kernel(const __grid_constant__ AllocParams p) {
    __shared__ uint32_t s_tile;
    __shared__ int64_t s_wb[AL_THREADS / 32];
    __shared__ uint32_t s_wk[AL_THREADS / 32];
    __shared__ int64_t s_excl_b;
    __shared__ uint32_t s_excl_k;
    __shared__ int64_t s_saved[AL_THREADS / 32];

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    if (tid == 0) s_tile = atomicAdd(p.tile_counter, 1u);
    __syncthreads();
    const uint32_t tile = s_tile;
    const uint64_t base = static_cast<uint64_t>(tile) * AL_TILE;

    // --- per-request decision (thread owns AL_ITEMS consecutive requests) ---
    int32_t ek[AL_ITEMS];
    int64_t tb = 0;
    uint32_t tk = 0;
    int64_t saved = 0;
#pragma unroll
    for (int i = 0; i < AL_ITEMS; ++i) {
        const uint64_t r = base + static_cast<uint64_t>(tid) * AL_ITEMS + i;
        ek[i] = 0;
        if (r < p.R) {
            int32_t e = p.cap;
            uint8_t why = CDX_EXIT_BUDGET;
            const uint32_t* mw = p.meets + r * p.words;
            for (uint32_t w = 0; w < p.words; ++w) {
                const uint32_t x = __ldg(mw + w) & p.chk[w];
                if (x) {
                    e = static_cast<int32_t>(w * 32 + __ffs(x));  // knob = probe index + 1
                    why = CDX_EXIT_CERTAIN;
                    break;
                }
            }
            ek[i] = e;
            if (p.exit_knob) p.exit_knob[r] = e;
            if (p.reason) p.reason[r] = why;
            if (p.granted) p.granted[r] = e;
            tb += static_cast<int64_t>(e) * p.tpu;
            tk += e > p.detect ? 1u : 0u;
            saved += static_cast<int64_t>(p.cap - e) * p.tpu;
        }
    }

    // --- block scan of (budget, kept) thread totals ---
    int64_t ib = warp_incl_scan<int64_t>(tb, lane);
    uint32_t ik = warp_incl_scan<uint32_t>(tk, lane);
    int64_t sv = saved;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) sv += __shfl_down_sync(0xffffffffu, sv, o);
    if (lane == 31) {
        s_wb[warp] = ib;
        s_wk[warp] = ik;
    }
    if (lane == 0) s_saved[warp] = sv;
    __syncthreads();
    int64_t wpre_b = 0;
    uint32_t wpre_k = 0;
    int64_t tot_b = 0;
    uint32_t tot_k = 0;
    for (int w = 0; w < AL_THREADS / 32; ++w) {
        if (w < warp) {
            wpre_b += s_wb[w];
            wpre_k += s_wk[w];
        }
        tot_b += s_wb[w];
        tot_k += s_wk[w];
    }

    // --- decoupled look-back (one thread) ---
    if (tid == 0) {
        int64_t tsaved = 0;
        for (int w = 0; w < AL_THREADS / 32; ++w) tsaved += s_saved[w];
        if (p.tokens_saved) atomicAdd(reinterpret_cast<unsigned long long*>(p.tokens_saved),
                                      static_cast<unsigned long long>(tsaved));
        int64_t eb = 0;
        uint32_t ekk = 0;
        if (tile == 0) {
            p.inc_b[0] = tot_b;
            p.inc_k[0] = tot_k;
            __threadfence();
            st_release(&p.flags[0], 2u);
        } else {
            p.agg_b[tile] = tot_b;
            p.agg_k[tile] = tot_k;
            __threadfence();
            st_release(&p.flags[tile], 1u);
            int64_t j = static_cast<int64_t>(tile) - 1;
            while (j >= 0) {
                uint32_t f;
                do {
                    f = ld_acquire(&p.flags[j]);
                } while (f == 0);
                if (f == 2) {
                    eb += *reinterpret_cast<volatile int64_t*>(&p.inc_b[j]);
                    ekk += *reinterpret_cast<volatile uint32_t*>(&p.inc_k[j]);
                    break;
                }
                eb += *reinterpret_cast<volatile int64_t*>(&p.agg_b[j]);
                ekk += *reinterpret_cast<volatile uint32_t*>(&p.agg_k[j]);
                --j;
            }
            p.inc_b[tile] = eb + tot_b;
            p.inc_k[tile] = ekk + tot_k;
            __threadfence();
            st_release(&p.flags[tile], 2u);
        }
        s_excl_b = eb;
        s_excl_k = ekk;
        if (tile == p.ntiles - 1) {
            if (p.n_kept) *p.n_kept = static_cast<uint64_t>(ekk) + tot_k;
            if (p.total_budget) *p.total_budget = eb + tot_b;
        }
    }
    __syncthreads();

    // --- scatter offsets and the stable kept list ---
    int64_t ob = p.base_offset + s_excl_b + wpre_b + (ib - tb);
    uint32_t ok = s_excl_k + wpre_k + (ik - tk);
#pragma unroll
    for (int i = 0; i < AL_ITEMS; ++i) {
        const uint64_t r = base + static_cast<uint64_t>(tid) * AL_ITEMS + i;
        if (r < p.R) {
            if (p.offsets) p.offsets[r] = ob;
            ob += static_cast<int64_t>(ek[i]) * p.tpu;
            if (ek[i] > p.detect) {
                if (p.kept) p.kept[ok] = p.kept_base + static_cast<uint32_t>(r);
                ++ok;
            }
        }
    }
}

}  // namespace cdx

extern "C" int cdx_allocate_scan(cdx_ctx* ctx, const uint32_t* meets_bits, uint64_t R, uint32_t P,
                                 const cdx_alloc_policy* pol, int64_t base_offset, uint32_t kept_base,
                                 int32_t* exit_knob, uint8_t* reason, int32_t* granted, int64_t* offsets,
                                 uint32_t* kept, uint64_t* n_kept, int64_t* tokens_saved,
                                 int64_t* total_budget) {
    using namespace cdx;
    if (!ctx) return CDX_EINVAL;
    if (!pol) return set_error(ctx, CDX_EINVAL, "allocate: null policy");
    if (P == 0 || P > 32 * AL_MAX_WORDS) return set_error(ctx, CDX_EINVAL, "allocate: probes must be 1..4096");
    const int32_t cap = pol->resource_cap;
    if (cap < 1 || static_cast<uint32_t>(cap) > P)
        return set_error(ctx, CDX_EINVAL, "allocate: resource_cap must be in [1, probes]");
    if (pol->kind != CDX_POL_EVEN && pol->kind != CDX_POL_STATIC_THRESHOLD && pol->kind != CDX_POL_K_STEP_THRESHOLD)
        return set_error(ctx, CDX_EINVAL, "allocate: policy kind not supported by the batched path");
    if (pol->kind != CDX_POL_EVEN && (pol->detect_at < 1 || pol->detect_at > cap))
        return set_error(ctx, CDX_EINVAL, "allocate: detect_at_knob must be in [1, resource_cap]");
    if (pol->kind == CDX_POL_K_STEP_THRESHOLD && pol->recheck_every < 1)
        return set_error(ctx, CDX_EINVAL, "allocate: recheck_every must be >= 1");
    if (pol->tokens_per_unit < 0) return set_error(ctx, CDX_EINVAL, "allocate: tokens_per_unit must be >= 0");
    if (R > 0xffffffffull) return set_error(ctx, CDX_EINVAL, "allocate: at most 2^32-1 requests per call");
    if (!meets_bits && pol->kind != CDX_POL_EVEN) return set_error(ctx, CDX_EINVAL, "allocate: null meets bits");

    AllocParams p{};
    p.meets = meets_bits;
    p.exit_knob = exit_knob;
    p.reason = reason;
    p.granted = granted;
    p.offsets = offsets;
    p.kept = kept;
    p.n_kept = n_kept;
    p.tokens_saved = tokens_saved;
    p.total_budget = total_budget;
    p.R = R;
    p.words = (P + 31) / 32;
    p.cap = cap;
    p.detect = pol->kind == CDX_POL_EVEN ? 0 : pol->detect_at;
    p.tpu = pol->tokens_per_unit;
    p.base_offset = base_offset;
    p.kept_base = kept_base;
    if (pol->kind != CDX_POL_EVEN) {
        const int32_t step = pol->kind == CDX_POL_K_STEP_THRESHOLD ? pol->recheck_every : cap + 1;
        for (int32_t k = pol->detect_at; k <= cap; k += step) p.chk[(k - 1) / 32] |= 1u << ((k - 1) % 32);
    }
    if (R == 0) {
        if (n_kept) cudaMemsetAsync(n_kept, 0, 8, ctx->stream);
        if (tokens_saved) cudaMemsetAsync(tokens_saved, 0, 8, ctx->stream);
        if (total_budget) cudaMemsetAsync(total_budget, 0, 8, ctx->stream);
        return CDX_OK;
    }
    if (!meets_bits) p.meets = nullptr;
    p.ntiles = static_cast<uint32_t>((R + AL_TILE - 1) / AL_TILE);
    // scratch: counter + flags + aggregates
    const size_t n = p.ntiles;
    const size_t bytes = 256 + n * 4 + n * 8 * 2 + n * 4 * 2 + 64;
    uint8_t* s = static_cast<uint8_t*>(scratch(ctx, bytes));
    if (!s) return set_error(ctx, CDX_ECUDA, "allocate: scratch allocation failed");
    p.tile_counter = reinterpret_cast<uint32_t*>(s);
    p.flags = reinterpret_cast<uint32_t*>(s + 256);
    p.agg_b = reinterpret_cast<int64_t*>(s + 256 + ((n * 4 + 15) / 16) * 16);
    p.inc_b = p.agg_b + n;
    p.agg_k = reinterpret_cast<uint32_t*>(p.inc_b + n);
    p.inc_k = p.agg_k + n;
    cudaMemsetAsync(s, 0, 256 + n * 4, ctx->stream);
    if (tokens_saved) cudaMemsetAsync(tokens_saved, 0, 8, ctx->stream);
    if (pol->kind == CDX_POL_EVEN) {
        // no meets bits needed: the chk mask is empty, point at a harmless word
        p.meets = reinterpret_cast<const uint32_t*>(s);
        p.words = 0;
    }
    allocate_scan_kernel<<<p.ntiles, AL_THREADS, 0, ctx->stream>>>(p);
    CDX_CHECK_LAUNCH(ctx, "allocate_scan");
    return CDX_OK;
}

namespace cdx {
namespace {
__global__ void rebase_kernel(int64_t* __restrict__ off, uint64_t n, const int64_t* __restrict__ totals,
                              uint32_t rank) {
    int64_t b = 0;
    for (uint32_t q = 0; q < rank; ++q) b += totals[q];
    for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<uint64_t>(gridDim.x) * blockDim.x)
        off[i] += b;
}
}  // namespace
}  // namespace cdx

extern "C" int cdx_offsets_rebase(cdx_ctx* ctx, int64_t* offsets, uint64_t R, const int64_t* shard_totals,
                                  uint32_t rank) {
    using namespace cdx;
    if (!ctx) return CDX_EINVAL;
    if (R == 0 || rank == 0) return CDX_OK;
    if (!offsets || !shard_totals) return set_error(ctx, CDX_EINVAL, "offsets_rebase: null pointer");
    const uint64_t want = (R / 2 + 255) / 256;  // 2 x int64 per thread-iteration is plenty for 8 B/request
    const unsigned grid = static_cast<unsigned>(std::max<uint64_t>(1, std::min<uint64_t>(want, ctx->sm_count * 4ull)));
    rebase_kernel<<<grid, 256, 0, ctx->stream>>>(offsets, R, shard_totals, rank);
    CDX_CHECK_LAUNCH(ctx, "offsets_rebase");
    return CDX_OK;
}
