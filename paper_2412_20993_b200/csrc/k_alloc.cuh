#pragma once
// k_alloc.cuh — K5's tile (allocation decision + budget scan + kept compaction), shared by the
// allocate_scan kernel (k_alloc.cu) and any kernel that runs K5 tiles itself.
#include <cooperative_groups.h>

#include "cdx_internal.cuh"

namespace cdx {
namespace al {

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

// One tile of requests: decision, block scan, look-back (or the cooperative barrier), global
// offsets and the stable kept list.  `tile` and `epoch` come from the caller (a ticket, or the
// block index when single / coop); every thread of a 256-thread CTA calls it.  The shared
// memory is the function's own.  The meets words are read through L2 (ld.global.cg), so a
// caller may run it on words other SMs wrote earlier in the same launch.
__device__ __forceinline__ void alloc_tile(const AllocParams& p, uint32_t tile, uint32_t epoch, bool single,
                                           bool coop) {
    __shared__ uint32_t s_we[AL_ITEMS * AL_WARPS];  // exclusive units before (item, warp) in the tile
    __shared__ uint32_t s_wk[AL_ITEMS * AL_WARPS];
    __shared__ uint64_t s_excl_e, s_red_e[AL_WARPS];
    __shared__ uint32_t s_excl_k, s_tot_e, s_tot_k, s_red_k[AL_WARPS], s_first[AL_WARPS];

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const uint32_t s_epoch = epoch;
    const uint64_t base = static_cast<uint64_t>(tile) * AL_TILE;

    // ---- per-request decision, coalesced.  The first meets word of
    // every item is loaded before any is used: one memory round trip for the tile, not one
    // per item (the scan loop below has a data-dependent exit the compiler will not hoist
    // loads across).  Further words (P > 32 with test points past probe 32) load on demand.
    uint32_t m0[AL_ITEMS];
#pragma unroll
    for (int i = 0; i < AL_ITEMS; ++i) {
        const uint64_t r = base + static_cast<uint64_t>(i) * AL_THREADS + tid;
        m0[i] = (p.chk_words && r < p.R) ? __ldcg(p.meets + r * p.words) : 0u;
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
                const uint32_t x = (w ? __ldcg(p.meets + r * p.words + w) : m0[i]) & p.chk[w];
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
    __syncthreads();  // the shared arrays are rewritten by the caller's next tile
}

}  // namespace al

// Host side of K5 (k_alloc.cu): validates the policy exactly as cdx_allocate_scan does and
// fills *p (persistent look-back state included).  *empty: R == 0, the scalars were zeroed
// and nothing is to be launched.
int alloc_prepare(cdx_ctx* ctx, const uint32_t* meets_bits, uint64_t R, uint32_t P, const cdx_alloc_policy* pol,
                  int64_t base_offset, uint32_t kept_base, int32_t* exit_knob, uint8_t* reason, int32_t* granted,
                  int64_t* offsets, uint32_t* kept, uint64_t* n_kept, int64_t* tokens_saved, int64_t* total_budget,
                  al::AllocParams* p, bool* empty);

}  // namespace cdx
