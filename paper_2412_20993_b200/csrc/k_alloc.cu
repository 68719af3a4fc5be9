// k_alloc.cu — K5: certaindex-driven allocation decision + exclusive scan of token budgets
// + stable compaction of continuing requests, in ONE single-pass kernel with no helper
// launches (decoupled look-back scan: each tile publishes its aggregate, then resolves its
// exclusive prefix from its predecessors' published state, 32 tiles per look-back step;
// tiles take tickets from a persistent counter so every predecessor is resident or done —
// the last tile to finish rewinds it and advances a device-side epoch that tags the tile
// records, so nothing is cleared between calls and a captured CUDA graph replays correctly).
//
// Semantics restated from SPEC.md:404-412 (scheduler.allocate; no reference code exists):
//   even               -> grant to the cap
//   static_threshold   -> at detect_at, terminate iff the thresholds hold, else grant to cap
//   k_step_threshold   -> re-test every recheck_every units from detect_at on
//   always terminate at resource_cap.
// token budget = granted * tokens_per_unit; kept = requests granted past detect_at.
#include <algorithm>
#include <cstdlib>

#include <cooperative_groups.h>

#include "cdx_internal.cuh"

namespace cdx {

constexpr int AL_THREADS = 256;
constexpr int AL_WARPS = AL_THREADS / 32;
constexpr int AL_ITEMS = 8;
constexpr int AL_TILE = AL_THREADS * AL_ITEMS;  // 2048 requests per tile
constexpr int AL_MAX_WORDS = 128;               // P <= 4096

// Per-tile look-back record.  `flag` = epoch << 2 | state (1 aggregate, 2 inclusive):
// records from earlier calls carry an older epoch and read as "not yet published".  The
// scan carries granted units and kept counts only: budgets are units x tokens_per_unit and
// the tokens saved are (valid requests x cap - units) x tokens_per_unit, both equal to the
// per-request int64 sums bit for bit (multiplication distributes over sums mod 2^64).
struct AlTile {
    uint64_t agg_e, inc_e;
    uint32_t agg_k, inc_k;
    uint32_t flag;
    uint32_t _pad;
};

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
    uint32_t* tickets;  // [0] tile tickets, [1] finished tiles, [2] epoch; the last tile resets
                        // [0] and [1] and advances [2]
    AlTile* tiles;
    uint64_t R;
    uint32_t ntiles;
    uint32_t words;      // meets words per request
    uint32_t chk_words;  // words that hold a test point (the rest is never read)
    int32_t cap, detect;
    int64_t tpu;
    int64_t base_offset;
    uint32_t kept_base;
    int coop;  // cooperative launch: every tile resident, prefixes by grid barrier (no look-back)
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
template <typename T>
__device__ __forceinline__ T warp_sum(T v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// Striped layout: item i of thread t is request base + i*256 + t, so every load/store
// instruction is coalesced; request order = (item, warp, lane), which the block scan
// over (item, warp) totals follows.  Per item one u32 warp scan carries both the granted
// units and the kept flag (units << 12 | kept: a warp's units <= 32 * 4096 = 2^17).  Tiles
// take tickets in launch order, so a tile only ever waits for tiles that are running or
// done.
__global__ void __launch_bounds__(AL_THREADS) allocate_scan_kernel(const __grid_constant__ AllocParams p) {
    __shared__ uint32_t s_tile;
    __shared__ uint32_t s_we[AL_ITEMS * AL_WARPS];  // exclusive units before (item, warp) in the tile
    __shared__ uint32_t s_wk[AL_ITEMS * AL_WARPS];
    __shared__ uint64_t s_excl_e, s_red_e[AL_WARPS];
    __shared__ uint32_t s_excl_k, s_tot_e, s_tot_k, s_red_k[AL_WARPS], s_first[AL_WARPS];

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    __shared__ uint32_t s_epoch;
    // a one-tile call (small batches) needs no ticket, no records and no look-back
    const bool single = p.ntiles == 1;
    const bool coop = p.coop != 0;  // tiles in block order, no tickets, no epochs
    if (tid == 0) {
        s_tile = (single || coop) ? blockIdx.x : atomicAdd(&p.tickets[0], 1u);
        s_epoch = (single || coop) ? 0u : ld_acquire(&p.tickets[2]);  // constant until every tile of this call is done
    }
    __syncthreads();
    const uint32_t tile = s_tile;
    if (tile >= p.ntiles) __trap();  // a stale ticket counter must fail loudly, never scribble
    const uint64_t base = static_cast<uint64_t>(tile) * AL_TILE;

    // ---- per-request decision, coalesced.  The first meets word of
    // every item is loaded before any is used: one memory round trip for the tile, not one
    // per item (the scan loop below has a data-dependent exit the compiler will not hoist
    // loads across).  Further words (P > 32 with test points past probe 32) load on demand.
    uint32_t m0[AL_ITEMS];
#pragma unroll
    for (int i = 0; i < AL_ITEMS; ++i) {
        const uint64_t r = base + static_cast<uint64_t>(i) * AL_THREADS + tid;
        m0[i] = (p.chk_words && r < p.R) ? __ldg(p.meets + r * p.words) : 0u;
    }
    // No global store happens before the tile's aggregate is published: the flag is a
    // release store, and a release waits for every earlier store of its thread.  The
    // per-request outputs are written in the last phase instead.
    uint32_t pk[AL_ITEMS];  // inclusive warp scan of (units << 12 | kept)
    uint32_t certain = 0;   // bit i: item i terminated on a threshold
#pragma unroll
    for (int i = 0; i < AL_ITEMS; ++i) {
        const uint64_t r = base + static_cast<uint64_t>(i) * AL_THREADS + tid;
        if (base + static_cast<uint64_t>(i) * AL_THREADS >= p.R) {  // whole item row past R (CTA-uniform)
            pk[i] = 0;
            if (lane == 31) s_we[i * AL_WARPS + warp] = 0;
            continue;
        }
        uint32_t e = 0;
        if (r < p.R) {
            e = static_cast<uint32_t>(p.cap);
            uint8_t why = CDX_EXIT_BUDGET;
            for (uint32_t w = 0; w < p.chk_words; ++w) {
                const uint32_t x = (w ? __ldg(p.meets + r * p.words + w) : m0[i]) & p.chk[w];
                if (x) {
                    e = w * 32 + static_cast<uint32_t>(__ffs(x));  // knob = probe index + 1
                    why = CDX_EXIT_CERTAIN;
                    break;
                }
            }
            certain |= (why == CDX_EXIT_CERTAIN ? 1u : 0u) << i;
        }
        const uint32_t k = (r < p.R && static_cast<int32_t>(e) > p.detect) ? 1u : 0u;
        pk[i] = warp_incl_scan<uint32_t>((e << 12) | k, lane);
        if (lane == 31) s_we[i * AL_WARPS + warp] = pk[i];
    }
    __syncthreads();
    // ---- exclusive prefix over the (item, warp) totals: 64 entries, 2 per lane of warp 0
    if (warp == 0) {
        const int a0 = 2 * lane, a1 = 2 * lane + 1;
        const uint32_t x0 = s_we[a0], x1 = s_we[a1];
        const uint32_t e0 = x0 >> 12, e1 = x1 >> 12, k0 = x0 & 0xfffu, k1 = x1 & 0xfffu;
        const uint32_t ince = warp_incl_scan<uint32_t>(e0 + e1, lane);  // tile units <= 2^23
        const uint32_t inck = warp_incl_scan<uint32_t>(k0 + k1, lane);
        const uint32_t tot_e = __shfl_sync(0xffffffffu, ince, 31);
        const uint32_t tot_k = __shfl_sync(0xffffffffu, inck, 31);
        __syncwarp();
        s_we[a0] = ince - e0 - e1;
        s_we[a1] = ince - e1;
        s_wk[a0] = inck - k0 - k1;
        s_wk[a1] = inck - k1;

        if (lane == 0) {
            s_tot_e = tot_e;
            s_tot_k = tot_k;
        }
        if (lane == 0 && coop) {  // aggregates only: read after the grid barrier, never by flag
            p.tiles[tile].agg_e = tot_e;
            p.tiles[tile].agg_k = tot_k;
        }
        if (lane == 0 && !single && !coop) {
            AlTile* T = p.tiles;
            const uint32_t ep = (s_epoch & 0x3fffffffu) << 2;
            if (tile == 0) {  // the first tile's aggregate is its inclusive prefix
                T[0].inc_e = tot_e;
                T[0].inc_k = tot_k;
            } else {
                T[tile].agg_e = tot_e;
                T[tile].agg_k = tot_k;
            }
            st_release(&T[tile].flag, ep | (tile == 0 ? 2u : 1u));
        }
    }
    __syncthreads();
    // ---- decoupled look-back over earlier tiles with the whole CTA, 256 records per round.
    // When a wave of tiles publishes its aggregates together, a tile walks back until it
    // meets an inclusive record — up to its distance from the wave's start — so the window
    // width, not the chain, sets the cost: 256 wide, a 512-tile grid needs at most 2 rounds.
    {
        const AlTile* T = p.tiles;
        const uint32_t ep = (s_epoch & 0x3fffffffu) << 2;
        uint64_t ee = 0;
        uint32_t ekk = 0;
        int64_t j = static_cast<int64_t>(tile) - 1;
        if (coop) {  // every tile's aggregate is written: one grid barrier, then sum the predecessors
            cooperative_groups::this_grid().sync();
            uint64_t ve = 0;
            uint32_t vk = 0;
            for (uint32_t q = tid; q < tile; q += AL_THREADS) {
                ve += __ldcg(reinterpret_cast<const unsigned long long*>(&T[q].agg_e));
                vk += __ldcg(&T[q].agg_k);
            }
            ve = warp_sum<uint64_t>(ve);
            vk = warp_sum<uint32_t>(vk);
            if (lane == 0) {
                s_red_e[warp] = ve;
                s_red_k[warp] = vk;
            }
            __syncthreads();
#pragma unroll
            for (int w = 0; w < AL_WARPS; ++w) {
                ee += s_red_e[w];
                ekk += s_red_k[w];
            }
            j = -1;  // skip the look-back
        }
        while (j >= 0) {  // block-uniform
            const int64_t idx = j - tid;
            uint32_t st = 2;  // before tile 0: an inclusive zero
            if (idx >= 0) {
                uint32_t f;
                do {
                    f = ld_acquire(&T[idx].flag);
                } while ((f & ~3u) != ep || (f & 3u) == 0);
                st = f & 3u;
            }
            const uint32_t incl = __ballot_sync(0xffffffffu, st == 2);
            if (lane == 0) s_first[warp] = incl ? static_cast<uint32_t>(warp * 32 + __ffs(incl) - 1) : 0xffffffffu;
            __syncthreads();
            uint32_t stop = 0xffffffffu;  // nearest inclusive predecessor in this window
#pragma unroll
            for (int w = 0; w < AL_WARPS; ++w) stop = min(stop, s_first[w]);
            uint64_t ve = 0;
            uint32_t vk = 0;
            if (static_cast<uint32_t>(tid) <= stop && idx >= 0) {
                const volatile AlTile* tv = T + idx;
                ve = st == 2 ? tv->inc_e : tv->agg_e;
                vk = st == 2 ? tv->inc_k : tv->agg_k;
            }
            ve = warp_sum<uint64_t>(ve);
            vk = warp_sum<uint32_t>(vk);
            if (lane == 0) {
                s_red_e[warp] = ve;
                s_red_k[warp] = vk;
            }
            __syncthreads();
#pragma unroll
            for (int w = 0; w < AL_WARPS; ++w) {
                ee += s_red_e[w];
                ekk += s_red_k[w];
            }
            __syncthreads();  // s_first / s_red are rewritten next round
            if (stop != 0xffffffffu) break;
            j -= AL_THREADS;
        }
        if (tid == 0) {
            const uint32_t tot_e = s_tot_e, tot_k = s_tot_k;
            if (tile != 0 && !single && !coop) {
                AlTile* Tw = p.tiles;
                Tw[tile].inc_e = ee + tot_e;
                Tw[tile].inc_k = ekk + tot_k;
                st_release(&Tw[tile].flag, ep | 2u);
            }
            s_excl_e = ee;
            s_excl_k = ekk;
            if (tile == p.ntiles - 1) {
                const uint64_t units = ee + tot_e;
                if (p.n_kept) *p.n_kept = static_cast<uint64_t>(ekk) + tot_k;
                if (p.total_budget) *p.total_budget = static_cast<int64_t>(units * static_cast<uint64_t>(p.tpu));
                if (p.tokens_saved)
                    *p.tokens_saved = static_cast<int64_t>(
                        (p.R * static_cast<uint64_t>(p.cap) - units) * static_cast<uint64_t>(p.tpu));
            }
        }
    }
    __syncthreads();

    // ---- global offsets and the stable kept list
    const uint64_t tpu = static_cast<uint64_t>(p.tpu);
    const uint64_t ebase = s_excl_e;
    const uint32_t kbase = s_excl_k;
#pragma unroll
    for (int i = 0; i < AL_ITEMS; ++i) {
        if (base + static_cast<uint64_t>(i) * AL_THREADS >= p.R) break;  // CTA-uniform: rows past R
        const uint64_t r = base + static_cast<uint64_t>(i) * AL_THREADS + tid;
        const uint32_t x = pk[i];
        const uint32_t own = __shfl_up_sync(0xffffffffu, x, 1);  // exclusive = inclusive of lane - 1
        const uint32_t ex = lane ? own : 0u;
        if (r >= p.R) continue;
        const int32_t e = static_cast<int32_t>((x - ex) >> 12);  // this request's granted units
        if (p.exit_knob) p.exit_knob[r] = e;
        if (p.reason) p.reason[r] = ((certain >> i) & 1u) ? CDX_EXIT_CERTAIN : CDX_EXIT_BUDGET;
        if (p.granted) p.granted[r] = e;
        const uint64_t units = ebase + s_we[i * AL_WARPS + warp] + (ex >> 12);
        if (p.offsets) p.offsets[r] = p.base_offset + static_cast<int64_t>(units * tpu);
        if (p.kept && ((x - ex) & 1u)) {
            const uint32_t pos = kbase + s_wk[i * AL_WARPS + warp] + (ex & 0xfffu);
            p.kept[pos] = p.kept_base + static_cast<uint32_t>(r);
        }
    }
    // every tile has drawn its ticket before any tile finishes: the last one to finish
    // rewinds the counters for the next call (no host-side bookkeeping, no memset launch)
    if (tid == 0 && !single && !coop) {
        __threadfence();
        if (atomicAdd(&p.tickets[1], 1u) == p.ntiles - 1) {
            p.tickets[0] = 0;
            p.tickets[1] = 0;
            p.tickets[2] = (p.tickets[2] + 1u) & 0x3fffffffu;  // next call's records are new
            __threadfence();
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
    CDX_NVTX("cdx_allocate_scan");
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
    p.ntiles = static_cast<uint32_t>((R + AL_TILE - 1) / AL_TILE);
    // persistent look-back state: zeroed only when (re)allocated; every call uses a new
    // epoch and a fresh range of tickets, so no per-call clearing launches are needed
    if (ctx->al_tiles < p.ntiles) {
        cudaStreamSynchronize(ctx->stream);
        if (ctx->al_state) cudaFree(ctx->al_state);
        ctx->al_state = nullptr;
        const size_t cap_tiles = std::max<size_t>(p.ntiles, 1024);
        if (cudaMalloc(&ctx->al_state, 256 + cap_tiles * sizeof(AlTile)) != cudaSuccess) {
            ctx->al_tiles = 0;
            return set_error(ctx, CDX_ECUDA, "allocate: state allocation failed");
        }
        cudaMemsetAsync(ctx->al_state, 0, 256 + cap_tiles * sizeof(AlTile), ctx->stream);
        ctx->al_tiles = cap_tiles;
    }
    p.tickets = static_cast<uint32_t*>(ctx->al_state);
    p.tiles = reinterpret_cast<AlTile*>(static_cast<uint8_t*>(ctx->al_state) + 256);
    p.chk_words = 0;
    for (uint32_t w = 0; w < p.words; ++w)
        if (p.chk[w]) p.chk_words = w + 1;
    if (pol->kind == CDX_POL_EVEN) p.meets = nullptr;  // no test points: meets is never read
    // every tile resident at once (C: 512 tiles, D: 128): cooperative launch, prefixes after
    // one grid barrier instead of a look-back chain; larger grids use the ticketed look-back
    static thread_local int coop_cap = -1, coop_dev = -1;
    if (coop_dev != ctx->device) {
        int per_sm = 0, attr = 0;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, allocate_scan_kernel, AL_THREADS, 0);
        cudaDeviceGetAttribute(&attr, cudaDevAttrCooperativeLaunch, ctx->device);
        coop_cap = attr ? per_sm * ctx->sm_count : 0;
        coop_dev = ctx->device;
    }
    p.coop = (p.ntiles > 1 && static_cast<int64_t>(p.ntiles) <= coop_cap && !getenv("CDX_ALLOC_LOOKBACK")) ? 1 : 0;
    if (p.coop) {
        void* args[] = {&p};
        const cudaError_t e = cudaLaunchCooperativeKernel(reinterpret_cast<const void*>(allocate_scan_kernel),
                                                          dim3(p.ntiles), dim3(AL_THREADS), args, 0, ctx->stream);
        if (e != cudaSuccess) {  // e.g. fewer SMs than queried (MPS limits): ticketed look-back instead
            (void)cudaGetLastError();
            p.coop = 0;
        }
    }
    if (!p.coop) allocate_scan_kernel<<<p.ntiles, AL_THREADS, 0, ctx->stream>>>(p);
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
