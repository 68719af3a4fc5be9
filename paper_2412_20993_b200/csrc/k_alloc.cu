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

#include "k_alloc.cuh"

namespace cdx {

using namespace al;

// Tiles take tickets in launch order (a tile only ever waits for tiles that are running or
// done); a one-tile call and a cooperative launch use the block index.
__global__ void __launch_bounds__(AL_THREADS) allocate_scan_kernel(const __grid_constant__ AllocParams p) {
    __shared__ uint32_t s_tile, s_epoch;
    const int tid = threadIdx.x;
    const bool single = p.ntiles == 1;  // no ticket, no records, no look-back
    const bool coop = p.coop != 0;      // tiles in block order, no tickets, no epochs
    if (tid == 0) {
        s_tile = (single || coop) ? blockIdx.x : atomicAdd(&p.tickets[0], 1u);
        s_epoch = (single || coop) ? 0u : ld_acquire(&p.tickets[2]);  // constant until every tile of this call is done
    }
    __syncthreads();
    const uint32_t tile = s_tile;
    if (tile >= p.ntiles) __trap();  // a stale ticket counter must fail loudly, never scribble
    alloc_tile(p, tile, s_epoch, single, coop);
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

namespace cdx {

int alloc_prepare(cdx_ctx* ctx, const uint32_t* meets_bits, uint64_t R, uint32_t P, const cdx_alloc_policy* pol,
                  int64_t base_offset, uint32_t kept_base, int32_t* exit_knob, uint8_t* reason, int32_t* granted,
                  int64_t* offsets, uint32_t* kept, uint64_t* n_kept, int64_t* tokens_saved, int64_t* total_budget,
                  al::AllocParams* out, bool* empty) {
    using namespace al;
    *empty = false;
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

    AllocParams& p = *out;
    p = AllocParams{};
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
        *empty = true;
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
        const size_t bytes = 256 + cap_tiles * sizeof(AlTile);
        if (cudaMalloc(&ctx->al_state, bytes) != cudaSuccess) {
            ctx->al_tiles = 0;
            return set_error(ctx, CDX_ECUDA, "allocate: state allocation failed");
        }
        cudaMemsetAsync(ctx->al_state, 0, bytes, ctx->stream);
        ctx->al_tiles = cap_tiles;
    }
    p.tickets = static_cast<uint32_t*>(ctx->al_state);
    p.tiles = reinterpret_cast<AlTile*>(static_cast<uint8_t*>(ctx->al_state) + 256);
    p.chk_words = 0;
    for (uint32_t w = 0; w < p.words; ++w)
        if (p.chk[w]) p.chk_words = w + 1;
    if (pol->kind == CDX_POL_EVEN) p.meets = nullptr;  // no test points: meets is never read
    return CDX_OK;
}

}  // namespace cdx

extern "C" int cdx_allocate_scan(cdx_ctx* ctx, const uint32_t* meets_bits, uint64_t R, uint32_t P,
                                 const cdx_alloc_policy* pol, int64_t base_offset, uint32_t kept_base,
                                 int32_t* exit_knob, uint8_t* reason, int32_t* granted, int64_t* offsets,
                                 uint32_t* kept, uint64_t* n_kept, int64_t* tokens_saved,
                                 int64_t* total_budget) {
    using namespace cdx;
    using namespace cdx::al;
    CDX_NVTX("cdx_allocate_scan");
    if (!ctx) return CDX_EINVAL;
    AllocParams p;
    bool empty = false;
    if (int st = alloc_prepare(ctx, meets_bits, R, P, pol, base_offset, kept_base, exit_knob, reason, granted, offsets,
                               kept, n_kept, tokens_saved, total_budget, &p, &empty))
        return st;
    if (empty) return CDX_OK;
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
