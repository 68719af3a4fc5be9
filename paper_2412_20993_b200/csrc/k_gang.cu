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
// which all keys agree are skipped.  Key build and compaction of live programs are one
// single-pass kernel (gang_prepare); the sort is onesweep: one histogram read for all 8
// digits (fused into the key-build sync), then one kernel per digit whose tiles rank
// stably (warp match + a shared-memory atomic per digit group), sort themselves by digit in
// shared memory, resolve their offsets by windowed decoupled look-back and write digit
// runs; the last pass writes program ids directly.
#include <algorithm>
#include <atomic>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

#include <cooperative_groups.h>

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
    const int32_t* knob;
    const int32_t* cap;
    const uint8_t* terminated;
    const uint32_t* program_id;  // nullable: id_base + index
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

// ---- key build + compaction of live programs, one pass ---------------------------------
// Per program: escalated = now - last_service >= limit (inclusive);
// est = mean completed iteration tokens or the prior; key = arrival when escalated or
// fifo, else est * remaining knob; hi = (escalated ? 0 : 1) << 63 | bits(key).  Live
// (non-terminated) programs are compacted in id order (reduce-then-scan: per-tile live
// counts from the terminated bytes, one-CTA scan, then this pass), writing hi / arrival
// bits / id / the identity permutation.  The same pass flags invalid times and whether arrivals are
// non-decreasing (the (arrival, id) pre-sort can then be skipped).
constexpr int GP_THREADS = 256, GP_ITEMS = 4, GP_TILE = GP_THREADS * GP_ITEMS;
// live programs per tile (reads only the terminated bytes)
// One warp per 1-KB tile of flags (8 tiles per CTA): 32 B per lane as two 16-byte loads when
// the tile is full and aligned, live = zero bytes; a warp reduction, no shared memory.
__device__ __forceinline__ uint32_t zero_bytes(uint32_t w) {
    return 4u - static_cast<uint32_t>(__popc((((w & 0x7f7f7f7fu) + 0x7f7f7f7fu) | w) & 0x80808080u));
}
__global__ void __launch_bounds__(256) gang_count(const uint8_t* __restrict__ term, uint64_t N,
                                                  uint32_t* __restrict__ tile_cnt, uint32_t ntiles) {
    const uint32_t tile = blockIdx.x * 8u + (threadIdx.x >> 5), lane = threadIdx.x & 31u;
    if (tile >= ntiles) return;
    const uint64_t base = static_cast<uint64_t>(tile) * GP_TILE;
    uint32_t c = 0;
    if (base + GP_TILE <= N && (reinterpret_cast<uintptr_t>(term) & 15) == 0) {
        static_assert(GP_TILE == 32 * 32, "two uint4 per lane");
        const uint4* q = reinterpret_cast<const uint4*>(term + base);
#pragma unroll
        for (int j = 0; j < 2; ++j) {
            const uint4 w = __ldg(q + lane + 32 * j);
            c += zero_bytes(w.x) + zero_bytes(w.y) + zero_bytes(w.z) + zero_bytes(w.w);
        }
    } else {
        for (uint32_t j = lane; j < GP_TILE; j += 32) {
            const uint64_t i = base + j;
            c += (i < N && term[i] == 0) ? 1u : 0u;
        }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
    if (lane == 0) tile_cnt[tile] = c;
}

// exclusive scan of the tile counts in place (one CTA), total -> misc[0]; 4 counts per thread
// per pass (uint4 when aligned), so config E's 4096 tile counts take one pass.
__global__ void __launch_bounds__(1024) gang_scan_tiles(uint32_t* __restrict__ v, uint32_t n, uint32_t* misc) {
    __shared__ uint32_t ws[32];
    const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    uint32_t carry = 0;
    for (uint32_t b = 0; b < n; b += 4096) {
        const uint32_t i = b + 4 * threadIdx.x;
        uint32_t x[4];
        const bool vec = i + 4 <= n && (reinterpret_cast<uintptr_t>(v + i) & 15) == 0;
        if (vec) {
            const uint4 q = *reinterpret_cast<const uint4*>(v + i);
            x[0] = q.x; x[1] = q.y; x[2] = q.z; x[3] = q.w;
        } else {
#pragma unroll
            for (int j = 0; j < 4; ++j) x[j] = i + j < n ? v[i + j] : 0u;
        }
        const uint32_t t = x[0] + x[1] + x[2] + x[3];
        uint32_t inc = t;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, inc, o);
            if (lane >= static_cast<uint32_t>(o)) inc += y;
        }
        if (lane == 31) ws[warp] = inc;
        __syncthreads();
        if (warp == 0) {
            uint32_t w = ws[lane];
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const uint32_t y = __shfl_up_sync(0xffffffffu, w, o);
                if (lane >= static_cast<uint32_t>(o)) w += y;
            }
            ws[lane] = w;  // inclusive over warps
        }
        __syncthreads();
        uint32_t e = carry + (warp ? ws[warp - 1] : 0u) + inc - t;
        uint32_t o4[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) { o4[j] = e; e += x[j]; }
        if (vec) {
            *reinterpret_cast<uint4*>(v + i) = make_uint4(o4[0], o4[1], o4[2], o4[3]);
        } else {
#pragma unroll
            for (int j = 0; j < 4; ++j)
                if (i + j < n) v[i + j] = o4[j];
        }
        carry += ws[31];
        __syncthreads();  // ws reused by the next pass
    }
    if (threadIdx.x == 0) misc[0] = carry;
}

// misc: [0] live count (from gang_scan_tiles), [1] arrivals not sorted, [2] bad time/key
__global__ void __launch_bounds__(GP_THREADS, 6) gang_prepare(const GangParams p, uint64_t* __restrict__ khi,
                                                           uint64_t* __restrict__ karr, uint32_t* __restrict__ kid,
                                                           uint32_t* __restrict__ perm,
                                                           const uint32_t* __restrict__ tile_excl,
                                                           uint32_t* __restrict__ misc, uint32_t lean) {
    __shared__ uint32_t s_excl;
    __shared__ uint32_t s_cnt[GP_ITEMS * (GP_THREADS / 32)];
    const uint32_t tid = threadIdx.x, lane = tid & 31u, warp = tid >> 5;
    const uint32_t tile = blockIdx.x;
    const uint64_t base = static_cast<uint64_t>(tile) * GP_TILE;
    uint64_t hk[GP_ITEMS], ak[GP_ITEMS];
    uint32_t rank[GP_ITEMS], ids[GP_ITEMS];
    bool lv[GP_ITEMS];
    bool bad = false, unsorted = false;
#pragma unroll
    for (int j = 0; j < GP_ITEMS; ++j) {
        const uint64_t i = base + static_cast<uint64_t>(j) * GP_THREADS + tid;  // striped: coalesced
        bool live = false;
        if (i < p.N) {
            // every field is loaded up front (one memory round trip per item, not two)
            const double a = __ldg(p.arrival + i), ls = __ldg(p.last_service + i);
            const double an = i + 1 < p.N ? __ldg(p.arrival + i + 1) : a;
            const uint32_t id = p.program_id ? __ldg(p.program_id + i) : p.id_base + static_cast<uint32_t>(i);
            const uint32_t idn = p.program_id && i + 1 < p.N ? __ldg(p.program_id + i + 1) : id + 1u;
            ids[j] = id;
            const int64_t sum = __ldg(p.iter_tok_sum + i);
            const uint32_t c = __ldg(p.iter_count + i);
            const int64_t rem = static_cast<int64_t>(__ldg(p.cap + i)) - static_cast<int64_t>(__ldg(p.knob + i));
            live = __ldg(p.terminated + i) == 0;
            bad = bad || !(a >= 0.0) || !(ls >= 0.0) || isinf(a) || isinf(ls);
            // index order is the (arrival, id) order unless arrivals descend or, with explicit
            // ids, an equal arrival is followed by a smaller id
            unsorted = unsorted || a > an || (a == an && idn <= id);
            const bool esc = (p.now - ls) >= p.limit;  // inclusive escalation
            if (p.escalated) p.escalated[i] = esc ? 1 : 0;
            double key;
            if (esc || p.order == CDX_ORDER_FIFO) {
                key = a;
            } else {
                const double est = c ? __ddiv_rn(static_cast<double>(sum), static_cast<double>(c)) : p.prior;
                key = __dmul_rn(est, static_cast<double>(rem > 0 ? rem : 0));
                bad = bad || !(key >= 0.0) || isinf(key);
            }
            hk[j] = (esc ? 0ull : (1ull << 63)) | dbits(key);
            ak[j] = dbits(a);
        }
        lv[j] = live;
    }
    // ranks after all loads are issued (no warp vote between the items' loads)
#pragma unroll
    for (int j = 0; j < GP_ITEMS; ++j) {
        const uint32_t m = __ballot_sync(0xffffffffu, lv[j]);
        rank[j] = __popc(m & ((1u << lane) - 1u));
        if (lane == 0) s_cnt[j * (GP_THREADS / 32) + warp] = __popc(m);
    }
    if (__any_sync(0xffffffffu, bad) && lane == 0) atomicExch(misc + 2, 1u);
    if (__any_sync(0xffffffffu, unsorted) && lane == 0) atomicExch(misc + 1, 1u);
    __syncthreads();
    if (warp == 0) {  // exclusive prefix over the (item, warp) counts of this tile
        static_assert(GP_ITEMS * (GP_THREADS / 32) <= 64, "two counts per lane");
        const bool h0 = 2 * lane < GP_ITEMS * (GP_THREADS / 32), h1 = 2 * lane + 1 < GP_ITEMS * (GP_THREADS / 32);
        const uint32_t a0 = h0 ? s_cnt[2 * lane] : 0u, a1 = h1 ? s_cnt[2 * lane + 1] : 0u;
        uint32_t inc = a0 + a1;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, inc, o);
            if (lane >= static_cast<uint32_t>(o)) inc += y;
        }
        if (h0) s_cnt[2 * lane] = inc - a0 - a1;
        if (h1) s_cnt[2 * lane + 1] = inc - a1;
        if (lane == 0) s_excl = tile_excl[tile];
    }
    __syncthreads();
#pragma unroll
    for (int j = 0; j < GP_ITEMS; ++j) {
        if (!lv[j]) continue;
        const uint64_t i = base + static_cast<uint64_t>(j) * GP_THREADS + tid;
        const uint32_t pos = s_excl + s_cnt[j * (GP_THREADS / 32) + warp] + rank[j];
        khi[pos] = hk[j];
        if (lean) {  // the sort carries the program id itself; arrival keys are not needed
            perm[pos] = ids[j];
        } else {
            karr[pos] = ak[j];
            kid[pos] = ids[j];
            perm[pos] = pos;
        }
    }
}

// keys[i] = {hi, arrival bits, id} of the i-th program in priority order (merge input)
__global__ void pack_keys(const uint64_t* __restrict__ shi, const uint64_t* __restrict__ karr,
                          const uint32_t* __restrict__ kid, const uint32_t* __restrict__ fin, uint64_t* __restrict__ keys,
                          uint64_t n, const uint32_t* __restrict__ n_dev = nullptr) {
    if (n_dev) n = *n_dev;
    for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
        const uint32_t j = fin[i];
        keys[3 * i] = shi[i];
        keys[3 * i + 1] = karr[j];
        keys[3 * i + 2] = kid[j];
    }
}


// ---- Onesweep LSD radix sort of (u64 key, u32 value) -------------------------------------
// One histogram kernel reads the keys once and counts all 8 digits (global digit counts do
// not depend on the order), then ONE kernel per non-trivial digit: each tile ranks its keys
// stably (warp match + popc, warps in tile order), publishes its per-digit counts and
// resolves its exclusive per-digit offsets by decoupled look-back over earlier tiles
// (flag and count packed in one 32-bit word), then scatters.  Tiles take tickets in
// launch order, so look-back only ever waits on running or finished tiles.
constexpr uint32_t LB_AGG = 1u << 30, LB_INC = 2u << 30, LB_CNT = (1u << 30) - 1u;

// The look-back records carry their payload in the flag word itself (flag | count), so no
// other memory is published through them: relaxed gpu-scope accesses suffice, and skip
// the fence a release store implies.
__device__ __forceinline__ uint32_t ld_rlx_u32(const uint32_t* p) {
    uint32_t v;
    asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_rlx_u32(uint32_t* p, uint32_t v) {
    asm volatile("st.relaxed.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
// Exclusive prefix of digit d over tiles [0, tile): the records of `win` predecessors are
// loaded together and consumed in order up to the first inclusive one; an unpublished
// record restarts the window there.
constexpr int LB_WIN = 8;  // measured on config E: 4 and 8 equal, 16 slower, 1 (serial) 25 % slower
template <int WIN>
__device__ __forceinline__ uint32_t lookback_win(const uint32_t* look, uint32_t tile, uint32_t d) {
    uint32_t excl = 0;
    int64_t j = static_cast<int64_t>(tile) - 1;
    while (j >= 0) {
        uint32_t f[WIN];
#pragma unroll
        for (int q = 0; q < WIN; ++q)
            f[q] = j - q >= 0 ? ld_rlx_u32(look + static_cast<uint64_t>(j - q) * 256 + d) : LB_INC;
        int used = 0;
        bool done = false;
#pragma unroll
        for (int q = 0; q < WIN; ++q) {
            if (done || used != q || (f[q] & ~LB_CNT) == 0) continue;
            excl += f[q] & LB_CNT;
            used = q + 1;
            done = (f[q] & LB_INC) != 0;
        }
        if (done) break;
        j -= used;
    }
    return excl;
}

// n_dev (nullable): the key count is read on the device (the gang path histograms its
// compacted keys before the host has learned how many there are: one sync, not two)
// DLO: digits below it are not counted (their rows stay zero; the upper-half sort skips them)
template <int DLO = 0>
__global__ void __launch_bounds__(RS_THREADS) os_histogram(const uint64_t* __restrict__ keys, uint64_t n,
                                                           uint32_t* __restrict__ ghist,
                                                           const uint32_t* __restrict__ n_dev) {
    __shared__ uint32_t h[8][256];
    if (n_dev) n = *n_dev;
    for (int i = threadIdx.x; i < 8 * 256; i += RS_THREADS) (&h[0][0])[i] = 0;
    __syncthreads();
    // eight keys in flight per thread per round: the loop is load-latency bound, not atomic bound
    // (warp-aggregating the skewed top digits with MATCH was measured slower: 19 -> 27 us)
    constexpr uint32_t U = 8;
    const uint64_t stride = static_cast<uint64_t>(gridDim.x) * RS_THREADS * U;
    for (uint64_t b = blockIdx.x * static_cast<uint64_t>(RS_THREADS) * U + threadIdx.x; b < n; b += stride) {
        uint64_t k[U];
#pragma unroll
        for (uint32_t u = 0; u < U; ++u) {
            const uint64_t i = b + u * RS_THREADS;
            k[u] = i < n ? __ldg(keys + i) : 0ull;
        }
#pragma unroll
        for (uint32_t u = 0; u < U; ++u) {
            if (b + u * RS_THREADS >= n) break;
#pragma unroll
            for (int d = DLO; d < 8; ++d) atomicAdd(&h[d][(k[u] >> (8 * d)) & 0xff], 1u);
        }
    }
    __syncthreads();
    for (int i = threadIdx.x; i < 8 * 256; i += RS_THREADS) {
        const uint32_t c = (&h[0][0])[i];
        if (c) atomicAdd(ghist + i, c);
    }
}

// Same pass with a tile-local counting sort through shared memory: after ranking, every
// key goes to its digit-sorted slot in the tile (smem), and the global scatter then walks
// the tile in sorted order, so consecutive threads write consecutive addresses of one
// digit run (~16 keys per digit per tile) instead of 32 unrelated sectors per store.  The
// tile's aggregate is published before the local shuffle and the look-back runs after it,
// so waiting on a predecessor overlaps this tile's own work.  Ranking: per item, the warp's
// lanes with equal digits find each other with MATCH; the group's first lane adds the group
// size to the warp's private counter with a shared-memory atomic (a warp's atomics on one
// address are performed in issue order, so ranks stay stable across items without a warp
// barrier per item) and the base is broadcast back with one shuffle.  Full tiles (all but
// the last) run without bounds checks.
constexpr int RS2_SMEM = RS_TILE * 12 + RS_WARPS * 256 * 4 + 2 * 256 * 4 + 64;

template <bool FULL, int WIN>
__device__ __forceinline__ void os_tile(const uint64_t* __restrict__ kin, const uint32_t* __restrict__ vin,
                                        uint64_t* __restrict__ kout, uint32_t* __restrict__ vout, uint64_t n,
                                        int shift, const uint32_t* __restrict__ ghist, uint32_t* __restrict__ look,
                                        uint32_t tile, uint8_t* rs2_smem, const uint32_t* __restrict__ vmap) {
    uint64_t* sk = reinterpret_cast<uint64_t*>(rs2_smem);
    uint32_t* sv = reinterpret_cast<uint32_t*>(sk + RS_TILE);
    uint32_t(*wcnt)[256] = reinterpret_cast<uint32_t(*)[256]>(sv + RS_TILE);
    uint32_t* s_gbase = &wcnt[RS_WARPS][0];
    uint32_t* s_wsum = s_gbase + 256;  // [RS_WARPS] x 2
    const uint32_t tid = threadIdx.x, lane = tid & 31u, warp = tid >> 5;
#pragma unroll
    for (int i = 0; i < RS_WARPS; ++i) wcnt[i][tid] = 0;
    // global exclusive base of digit `tid`
    const uint32_t g = ghist[tid];
    uint32_t incl = g;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= static_cast<uint32_t>(o)) incl += y;
    }
    if (lane == 31) s_wsum[warp] = incl;
    __syncthreads();
    uint32_t wpre = 0;
#pragma unroll
    for (uint32_t w = 0; w < RS_WARPS; ++w) wpre += w < warp ? s_wsum[w] : 0u;
    const uint32_t gbase = wpre + incl - g;
    const uint64_t tbase = static_cast<uint64_t>(tile) * RS_TILE;
    const uint32_t tile_n = FULL ? RS_TILE : static_cast<uint32_t>(n - tbase);
    const uint64_t* tk = kin + tbase + warp * 32 * RS_ITEMS + lane;
    const uint32_t* tv = vin + tbase + warp * 32 * RS_ITEMS + lane;
    const uint32_t wofs = warp * 32 * RS_ITEMS + lane;  // item j of this thread: tile index wofs + 32 j
    uint64_t k[RS_ITEMS];
    uint32_t v[RS_ITEMS], rank[RS_ITEMS];
    const uint32_t lt = (1u << lane) - 1u;
#pragma unroll
    for (int j = 0; j < RS_ITEMS; ++j) {
        if (FULL || wofs + 32 * j < tile_n) {
            k[j] = tk[32 * j];
            v[j] = tv[32 * j];
        } else {
            k[j] = 0;
            v[j] = 0;
        }
    }
#pragma unroll
    for (int j = 0; j < RS_ITEMS; ++j) {
        const bool ok = FULL || wofs + 32 * j < tile_n;
        const uint32_t d = ok ? static_cast<uint32_t>((k[j] >> shift) & 0xff) : 256u + lane;  // unique dummy
        const uint32_t peers = __match_any_sync(0xffffffffu, d);
        const uint32_t below = peers & lt;
        uint32_t old = 0;
        if (ok && below == 0) old = atomicAdd(&wcnt[warp][d], static_cast<uint32_t>(__popc(peers)));
        rank[j] = __shfl_sync(0xffffffffu, old, __ffs(peers) - 1) + __popc(below);
    }
    __syncthreads();
    // thread d: tile count of digit d, publish the aggregate, tile offsets by digit, and
    // per-warp slots: wcnt[w][d] = first tile-sorted index of warp w's digit-d keys
    const uint32_t d = tid;
    uint32_t cw[RS_WARPS];
    uint32_t c = 0;
#pragma unroll
    for (int w = 0; w < RS_WARPS; ++w) {
        cw[w] = wcnt[w][d];
        c += cw[w];
    }
    if (tile == 0)
        st_rlx_u32(look + d, LB_INC | c);
    else
        st_rlx_u32(look + static_cast<uint64_t>(tile) * 256 + d, LB_AGG | c);
    incl = c;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= static_cast<uint32_t>(o)) incl += y;
    }
    if (lane == 31) s_wsum[RS_WARPS + warp] = incl;
    __syncthreads();
    wpre = 0;
#pragma unroll
    for (uint32_t w = 0; w < RS_WARPS; ++w) wpre += w < warp ? s_wsum[RS_WARPS + w] : 0u;
    const uint32_t toff = wpre + incl - c;
    {
        uint32_t run = toff;
#pragma unroll
        for (int w = 0; w < RS_WARPS; ++w) {
            wcnt[w][d] = run;
            run += cw[w];
        }
    }
    __syncthreads();
    // digit-sorted tile in shared memory
#pragma unroll
    for (int j = 0; j < RS_ITEMS; ++j) {
        if (FULL || wofs + 32 * j < tile_n) {
            const uint32_t lp = wcnt[warp][(k[j] >> shift) & 0xff] + rank[j];
            sk[lp] = k[j];
            sv[lp] = v[j];
        }
    }
    // look-back for digit d over earlier tiles
    uint32_t excl = 0;
    if (tile != 0) {
        excl = lookback_win<WIN>(look, tile, d);
        st_rlx_u32(look + static_cast<uint64_t>(tile) * 256 + d, LB_INC | (excl + c));
    }
    s_gbase[d] = gbase + excl - toff;  // position = s_gbase[digit] + sorted tile index
    __syncthreads();
#pragma unroll 4
    for (uint32_t j = 0; j < RS_ITEMS; ++j) {
        const uint32_t i = j * RS_THREADS + tid;
        if (FULL || i < tile_n) {
            const uint64_t key = sk[i];
            const uint32_t pos = s_gbase[(key >> shift) & 0xff] + i;
            kout[pos] = key;
            vout[pos] = vmap ? vmap[sv[i]] : sv[i];
        }
    }
}

// Tiles take tickets in launch order (look-back only waits on running or finished tiles);
// every tile but the last is full.
// n_dev (nullable): the key count lives on the device and `n` only bounds it (the grid is
// sized for the bound; tiles past the count exit).  The host has then not seen the digit
// counts either, so a digit on which every key agrees is detected here and the pass
// degenerates to a copy (the ping-pong parity stays what the host planned).
__global__ void __launch_bounds__(RS_THREADS, 2)
    os_pass2(const uint64_t* __restrict__ kin, const uint32_t* __restrict__ vin, uint64_t* __restrict__ kout,
             uint32_t* __restrict__ vout, uint64_t n, int shift, const uint32_t* __restrict__ ghist,
             uint32_t* __restrict__ look, uint32_t* __restrict__ counter, const uint32_t* __restrict__ vmap,
             const uint32_t* __restrict__ n_dev) {
    extern __shared__ __align__(16) uint8_t rs2_smem[];
    uint32_t* s_tile = reinterpret_cast<uint32_t*>(rs2_smem + RS2_SMEM - 16);
    if (threadIdx.x == 0) *s_tile = atomicAdd(counter, 1u);
    if (n_dev) n = *n_dev;
    __syncthreads();
    const uint32_t tile = *s_tile;
    const uint64_t tb = static_cast<uint64_t>(tile) * RS_TILE;
    if (tb >= n) return;
    if (n_dev && __syncthreads_or(ghist[threadIdx.x] == n)) {  // trivial digit: copy the tile
        const uint64_t te = tb + RS_TILE < n ? tb + RS_TILE : n;
        for (uint64_t i = tb + threadIdx.x; i < te; i += RS_THREADS) {
            kout[i] = kin[i];
            vout[i] = vmap ? vmap[vin[i]] : vin[i];
        }
        return;
    }
    if ((static_cast<uint64_t>(tile) + 1) * RS_TILE <= n)
        os_tile<true, LB_WIN>(kin, vin, kout, vout, n, shift, ghist, look, tile, rs2_smem, vmap);
    else
        os_tile<false, LB_WIN>(kin, vin, kout, vout, n, shift, ghist, look, tile, rs2_smem, vmap);
}

__global__ void widen_u32(const uint32_t* __restrict__ src, uint64_t* __restrict__ dst, uint64_t n) {
    for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<uint64_t>(gridDim.x) * blockDim.x)
        dst[i] = src[i];
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

// ---- Range LSD radix pass (reduce-then-scan, no look-back) -------------------------------
// Block b owns a contiguous range of RS_RANGE_TILES tiles.  Per pass: (1) each range counts
// its digits (hist[b][256]); (2) one CTA turns the counts into exclusive offsets in
// (digit, range) order; (3) each range re-reads its tiles in order, ranks every tile
// stably (warp match + popc, warps in order) and scatters at running per-digit offsets.
__global__ void __launch_bounds__(RS_THREADS) rr_hist(const uint64_t* __restrict__ keys, uint64_t n, uint64_t range,
                                                      int shift, uint32_t* __restrict__ hist) {
    __shared__ uint32_t h[256];
    h[threadIdx.x] = 0;
    __syncthreads();
    const uint64_t b = static_cast<uint64_t>(blockIdx.x) * range;
    const uint64_t e = min(b + range, n);
    for (uint64_t i = b + threadIdx.x; i < e; i += RS_THREADS) atomicAdd(&h[(keys[i] >> shift) & 0xff], 1u);
    __syncthreads();
    hist[static_cast<uint64_t>(blockIdx.x) * 256 + threadIdx.x] = h[threadIdx.x];
}

// thread d: exclusive prefix over ranges of digit d, then the digit bases (one CTA of 256)
__global__ void __launch_bounds__(256) rr_scan(uint32_t* __restrict__ hist, uint32_t nr) {
    __shared__ uint32_t tot[256];
    __shared__ uint32_t ws[8];
    const uint32_t d = threadIdx.x, lane = d & 31, warp = d >> 5;
    uint32_t acc = 0;
    for (uint32_t b = 0; b < nr; ++b) {
        const uint32_t c = hist[static_cast<uint64_t>(b) * 256 + d];
        hist[static_cast<uint64_t>(b) * 256 + d] = acc;
        acc += c;
    }
    uint32_t inc = acc;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, inc, o);
        if (lane >= static_cast<uint32_t>(o)) inc += y;
    }
    if (lane == 31) ws[warp] = inc;
    __syncthreads();
    uint32_t base = inc - acc;
    for (uint32_t w = 0; w < warp; ++w) base += ws[w];
    tot[d] = base;
    __syncthreads();
    for (uint32_t b = 0; b < nr; ++b) hist[static_cast<uint64_t>(b) * 256 + d] += tot[d];
}

__global__ void __launch_bounds__(RS_THREADS) rr_scatter(const uint64_t* __restrict__ kin,
                                                         const uint32_t* __restrict__ vin, uint64_t* __restrict__ kout,
                                                         uint32_t* __restrict__ vout, uint64_t n, uint64_t range,
                                                         int shift, const uint32_t* __restrict__ offs) {
    __shared__ uint32_t run[256];
    __shared__ uint32_t wcnt[RS_WARPS][256];
    const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    run[threadIdx.x] = offs[static_cast<uint64_t>(blockIdx.x) * 256 + threadIdx.x];
    const uint64_t rb = static_cast<uint64_t>(blockIdx.x) * range;
    const uint64_t re = min(rb + range, n);
    const uint32_t lt = (1u << lane) - 1u;
    for (uint64_t tb = rb; tb < re; tb += RS_TILE) {
        for (int i = threadIdx.x; i < RS_WARPS * 256; i += RS_THREADS) (&wcnt[0][0])[i] = 0;
        __syncthreads();
        const uint64_t base = tb + static_cast<uint64_t>(warp) * 32 * RS_ITEMS;
        uint64_t k[RS_ITEMS];
        uint32_t v[RS_ITEMS], rank[RS_ITEMS], dig[RS_ITEMS];
#pragma unroll
        for (int j = 0; j < RS_ITEMS; ++j) {
            const uint64_t i = base + j * 32 + lane;
            const bool ok = i < re;
            k[j] = ok ? kin[i] : 0;
            v[j] = ok ? vin[i] : 0;
        }
#pragma unroll
        for (int j = 0; j < RS_ITEMS; ++j) {
            const bool ok = base + j * 32 + lane < re;
            const uint32_t d = ok ? static_cast<uint32_t>((k[j] >> shift) & 0xff) : 256u + lane;
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
        {  // warps' exclusive prefixes per digit, and this tile's total
            const uint32_t d = threadIdx.x;
            uint32_t c = 0;
            for (int w = 0; w < RS_WARPS; ++w) {
                const uint32_t x = wcnt[w][d];
                wcnt[w][d] = c + run[d];
                c += x;
            }
            __syncthreads();
            run[d] += c;
        }
#pragma unroll
        for (int j = 0; j < RS_ITEMS; ++j) {
            const uint64_t i = base + j * 32 + lane;
            if (i < re) {
                const uint64_t pos = static_cast<uint64_t>(wcnt[warp][dig[j]]) + rank[j];
                kout[pos] = k[j];
                vout[pos] = v[j];
            }
        }
        __syncthreads();
    }
}

// Stable LSD radix sort of (keys, vals) over 8-bit digits (onesweep).  `lb` is scratch of
// 8*256 + 16 + 8*ntiles*256 u32 (global digit counts, pass tickets, look-back records);
// digits where every key agrees are skipped (decided on the host from the global counts).
// `hh` (nullable): the caller already histogrammed the keys into lb[0, 2048) and holds the
// counts on the host (saves a launch and a sync).  `vmap`/`vfinal` (nullable): the last
// pass writes vmap[value] to vfinal instead of the value (folds the caller's final gather).
// *which: 0 result in k0/v0, 1 in k1/v1, 2 keys in k0/k1 as for (pass count & 1) and the
// mapped values in vfinal.  dlo: sort by digits [dlo, 8) only (the upper bytes).
int radix_sort(cdx_ctx* ctx, uint64_t* k0, uint32_t* v0, uint64_t* k1, uint32_t* v1, uint64_t n, uint32_t* lb,
               int* which, const uint32_t* hh, const uint32_t* vmap, uint32_t* vfinal, int dlo = 0) {
    *which = 0;
    if (n <= 1) return CDX_OK;
    const uint32_t ntiles = static_cast<uint32_t>((n + RS_TILE - 1) / RS_TILE);
    uint32_t* ghist = lb;
    uint32_t* tickets = lb + 8 * 256;
    uint32_t* look = tickets + 16;
    const size_t clear = (16 + static_cast<size_t>(8) * ntiles * 256) * 4;
    cudaError_t e = hh ? cudaMemsetAsync(tickets, 0, clear, ctx->stream)
                       : cudaMemsetAsync(lb, 0, clear + 8 * 256 * 4, ctx->stream);
    if (e != cudaSuccess) return cuda_fail(ctx, e, "radix(clear)");
    uint32_t h[8 * 256];
    if (!hh) {
        const unsigned hgrid =
            static_cast<unsigned>(std::min<uint64_t>(ntiles, static_cast<uint64_t>(ctx->sm_count) * 4));
        os_histogram<0><<<hgrid, RS_THREADS, 0, ctx->stream>>>(k0, n, ghist, nullptr);
        CDX_CHECK_LAUNCH(ctx, "radix(histogram)");
        e = cudaMemcpyAsync(h, ghist, sizeof(h), cudaMemcpyDeviceToHost, ctx->stream);
        if (e == cudaSuccess) e = cudaStreamSynchronize(ctx->stream);
        if (e != cudaSuccess) return cuda_fail(ctx, e, "radix(histogram)");
        hh = h;
    }
    uint64_t* kin = k0;
    uint32_t* vin = v0;
    uint64_t* kout = k1;
    uint32_t* vout = v1;
    // onesweep look-back passes by default; CDX_RADIX=ranges selects the reduce-then-scan
    // range passes (ranges of several tiles, no tile waits on another) — measured slower on
    // config E (three launches and a serial one-CTA scan per digit)
    const char* impl = getenv("CDX_RADIX");
    const bool ranges = impl && std::strcmp(impl, "ranges") == 0;
    if (!ranges) {  // per call: cheap, and correct for every device of the process
        e = cudaFuncSetAttribute(os_pass2, cudaFuncAttributeMaxDynamicSharedMemorySize, RS2_SMEM);
        if (e != cudaSuccess) return cuda_fail(ctx, e, "radix(smem attribute)");
    }
    const uint64_t want = static_cast<uint64_t>(ctx->sm_count) * 2;
    const uint64_t range = std::max<uint64_t>(RS_TILE, ((n + want - 1) / want + RS_TILE - 1) / RS_TILE * RS_TILE);
    const uint32_t nr = static_cast<uint32_t>((n + range - 1) / range);
    int last = -1;
    bool nontrivial[8];
    for (int d = 0; d < 8; ++d) {
        nontrivial[d] = d >= dlo;  // digits below dlo are left to the caller
        if (!nontrivial[d]) continue;
        for (int b = 0; b < 256; ++b)
            if (hh[d * 256 + b]) {
                nontrivial[d] = hh[d * 256 + b] != n;
                break;
            }
        if (nontrivial[d]) last = d;
    }
    bool mapped = false;
    for (int d = 0; d < 8; ++d) {
        if (!nontrivial[d]) continue;
        if (ranges) {
            uint32_t* rh = look;  // [nr][256], reused every pass (stream-ordered)
            rr_hist<<<nr, RS_THREADS, 0, ctx->stream>>>(kin, n, range, 8 * d, rh);
            CDX_CHECK_LAUNCH(ctx, "radix(range hist)");
            rr_scan<<<1, 256, 0, ctx->stream>>>(rh, nr);
            CDX_CHECK_LAUNCH(ctx, "radix(range scan)");
            rr_scatter<<<nr, RS_THREADS, 0, ctx->stream>>>(kin, vin, kout, vout, n, range, 8 * d, rh);
            CDX_CHECK_LAUNCH(ctx, "radix(range scatter)");
        } else {
            const bool fold = vmap && vfinal && d == last;
            os_pass2<<<ntiles, RS_THREADS, RS2_SMEM, ctx->stream>>>(
                kin, vin, kout, fold ? vfinal : vout, n, 8 * d, ghist + d * 256,
                look + static_cast<size_t>(d) * ntiles * 256, tickets + d, fold ? vmap : nullptr, nullptr);
            CDX_CHECK_LAUNCH(ctx, "radix(pass)");
            mapped = fold;
        }
        std::swap(kin, kout);
        std::swap(vin, vout);
    }
    *which = mapped ? 2 : (kin == k0 ? 0 : 1);
    return CDX_OK;
}

// ---- upper-half sort + run fix-up --------------------------------------------------------
// The priority word is first sorted (stably, over the (arrival, id) pre-order) by its upper
// 32 bits only: 4 radix passes instead of 8.  Keys then differ from the full order only
// inside runs of equal upper halves, and only where the lower halves descend.  Pass A
// writes order[i] = id of position i for everyone and lists each run that holds a descent
// (its first descent reports the run start, found by a backward scan of at most 64 keys);
// pass B sorts each listed run by the full key (insertion sort: stable, so ties keep the
// pre-order) and rewrites its order entries.  A descending run longer than 64 raises the
// fallback flag and the caller re-sorts with all 8 digits: only adversarial inputs get
// there.  With no descents (integer-valued keys, distinct upper halves) pass B is skipped.
constexpr uint32_t FIX_RUN = 64;

// fix[0] fallback flag, fix[1] listed runs, fix[2..] run starts
__global__ void gang_fix_a(const uint64_t* __restrict__ k, const uint32_t* __restrict__ v,
                           const uint32_t* __restrict__ kid, uint64_t n, uint32_t* __restrict__ order,
                           uint32_t* __restrict__ fix, uint32_t list_cap, const uint32_t* __restrict__ n_dev) {
    if (n_dev) n = *n_dev;
    for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
        order[i] = kid ? kid[v[i]] : v[i];
        if (i == 0) continue;
        const uint64_t ki = k[i], kp = k[i - 1];
        const uint32_t h = static_cast<uint32_t>(ki >> 32);
        if (static_cast<uint32_t>(kp >> 32) != h || ki >= kp) continue;
        // a descent inside a run: the first one of its run lists the run start
        uint64_t j = i - 1;
        bool first = true;
        while (j > 0 && static_cast<uint32_t>(k[j - 1] >> 32) == h) {
            if (i - j >= FIX_RUN) break;
            first = first && !(k[j] < k[j - 1]);
            --j;
        }
        const bool reach = j == 0 || static_cast<uint32_t>(k[j - 1] >> 32) != h;
        if (!reach) {
            atomicOr(fix, 1u);  // the run is longer than the fix-up handles
        } else if (first) {
            uint64_t e = i + 1;  // the run must also end within reach
            while (e < n && e - j <= FIX_RUN && static_cast<uint32_t>(k[e] >> 32) == h) ++e;
            if (e - j > FIX_RUN) {
                atomicOr(fix, 1u);
                continue;
            }
            const uint32_t slot = atomicAdd(fix + 1, 1u);
            if (slot < list_cap) fix[2 + slot] = static_cast<uint32_t>(j);
            else atomicOr(fix, 1u);
        }
    }
}

__global__ void gang_fix_b(uint64_t* __restrict__ k, uint32_t* __restrict__ v, const uint32_t* __restrict__ kid,
                           uint64_t n, uint32_t* __restrict__ order, const uint32_t* __restrict__ fix,
                           const uint32_t* __restrict__ n_dev) {
    if (n_dev) n = *n_dev;
    if (fix[0]) return;  // the caller falls back to the full sort
    const uint32_t cnt = fix[1];
    for (uint32_t t = blockIdx.x * blockDim.x + threadIdx.x; t < cnt; t += gridDim.x * blockDim.x) {
        const uint64_t i = fix[2 + t];
        const uint32_t h = static_cast<uint32_t>(k[i] >> 32);
        uint64_t e = i + 1;
        while (e < n && static_cast<uint32_t>(k[e] >> 32) == h) ++e;
        if (e - i > FIX_RUN) continue;  // flagged by pass A; the caller falls back
        for (uint64_t a = i + 1; a < e; ++a) {  // stable insertion sort by the full key
            const uint64_t ka = k[a];
            const uint32_t va = v[a];
            uint64_t b = a;
            while (b > i && k[b - 1] > ka) {
                k[b] = k[b - 1];
                v[b] = v[b - 1];
                --b;
            }
            k[b] = ka;
            v[b] = va;
        }
        for (uint64_t a = i; a < e; ++a) order[a] = kid ? kid[v[a]] : v[a];
    }
}

// ---- persistent gang order: key build, radix passes and the run fix-up in ONE launch -------
// The lean fast path (no key output, arrivals assumed non-decreasing) as a cooperative kernel
// with one 1024-thread CTA per SM.  The sort moves 4-byte upper halves and 4-byte program
// indices (the low halves stay in lo[program], read only by the fix-up), and every pass is
// reduce-then-scan across the grid instead of a look-back chain:
//   phase 0   CTA c builds the keys of programs [c*Q0, (c+1)*Q0) (as
//             gang_prepare), writes lo[i] and the upper half (PG_DEAD when terminated),
//             counts all 4 digits of its live upper halves and ORs / ANDs the live keys'
//             halves;                                                           grid barrier
//   plan      digits on which every live key agrees are skipped (the OR / AND of all CTAs);
//   pass      every CTA reads the digit's counts of all CTAs (G x 256, L2) and derives its
//             exclusive base per digit value; then, tile by tile over its input range (the
//             first pass: its programs, dead ones dropped; later passes: positions
//             [c*Q, (c+1)*Q) of the previous output), ranks stably (ballot digit match + a
//             shared atomic per group of equal digits), sorts the tile by digit in shared
//             memory and writes whole digit runs;                                grid barrier
//             then counts the next digit over its next input range;             grid barrier
//   fix-up    only when the low halves differ at all: runs of equal upper halves whose low
//             halves descend are listed (gang_fix_a's rule) and insertion-sorted by the low
//             half (gang_fix_b's rule);                                         grid barrier
// On this path arrivals are non-decreasing and ids increase with the index (the flag that
// says otherwise sends the call to the checked path), so the (arrival, id) tie-break IS the
// index order, which every pass keeps.  An escalated program's key is its arrival, so the
// escalated programs' order is the index order too: their key is canonicalised to 0 (they
// still precede every other program, whose key has bit 63 set); under FIFO the others' keys
// are arrivals as well and become the constant 1 << 63.  The order is unchanged, and digits
// that no longer vary are skipped (FIFO sorts nothing: one compaction pass).
// No ticket counters, no look-back records, nothing cleared before the launch: flags and
// bit masks are per-CTA records reduced after the first barrier; the run counter is zeroed
// in phase 0.
constexpr int PG_THREADS = 1024, PG_WARPS = PG_THREADS / 32, PG_ITEMS = 8, PG_TILE = PG_THREADS * PG_ITEMS;
constexpr uint32_t PG_DEAD = 0xffffffffu;
constexpr int PG_FEW = 24;  // never a live upper half: a finite key's exponent is <= 0x7fe
// dynamic shared memory: sk, sv, stk, stv [PG_TILE] (phase 0: the program-field ring) | wcnt
// [PG_WARPS][256] | s_q [4][256] | s_red [4][256] | s_base, s_gb, s_toff [256] | s_ws [32] |
// scalars [16] | mbarriers [PG_NST + 1]
// Phase 0 ring: PG_NST stages of PG_CH programs, every SoA field bulk-copied (arrival, last
// service, token sum: 8 B; count, knob, cap, id: 4 B; terminated: 1 B)
constexpr int PG_CH = 1024, PG_NST = 3;  // (6 x 512 with two chunks per step measured slower: 40 -> 52 us)
constexpr int PG_ST_ARR = 0, PG_ST_LS = PG_CH * 8, PG_ST_SUM = PG_CH * 16, PG_ST_CNT = PG_CH * 24,
              PG_ST_KNOB = PG_CH * 28, PG_ST_CAP = PG_CH * 32, PG_ST_TERM = PG_CH * 36, PG_ST_PID = PG_CH * 37,
              PG_ST_BYTES = PG_CH * 41;
static_assert(PG_NST * PG_ST_BYTES <= PG_TILE * 16, "the phase-0 ring lives in the tile buffers");
constexpr int PG_SMEM = PG_TILE * 16 + PG_WARPS * 256 * 4 + 2 * 4 * 256 * 4 + 3 * 256 * 4 + 32 * 4 + 16 * 4 +
                        8 * (PG_NST + 1);  // + the mbarriers

struct PgArgs {
    GangParams p;
    uint32_t* lo;                  // [N] low half of program i's key
    uint32_t *ka, *va, *kb, *vb;   // [N] ping-pong (kb holds phase 0's per-program upper halves)
    uint32_t* hist;                // [4 digits][G][256] counts of each CTA's input range
    uint32_t* crec;                // [G][8] phase-0 record per CTA: flags, OR / AND of upper and low halves
    uint32_t* misc;                // [0] live count [1] unsorted [2] bad [3] fix-up fallback [4] listed runs
    uint32_t* order;
    unsigned long long* prof;      // nullable: per-CTA %globaltimer stamps at each phase end (CDX_GANG_PS_PROF)
    int bulk0;                     // every SoA pointer 16-byte aligned: phase 0 streams them by bulk copies
};

__device__ __forceinline__ void pg_stamp(const PgArgs& a, uint32_t slot) {
    if (a.prof && threadIdx.x == 0) {
        unsigned long long t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        a.prof[blockIdx.x * 16 + slot] = t;
    }
}
__device__ __forceinline__ uint64_t umin64(uint64_t x, uint64_t y) { return x < y ? x : y; }
__device__ __forceinline__ uint64_t policy_evict_last() {
    uint64_t q;
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(q));
    return q;
}
__device__ __forceinline__ void fence_proxy_async_all() { asm volatile("fence.proxy.async;" ::: "memory"); }
__device__ __forceinline__ uint32_t warp_incl_scan(uint32_t x, uint32_t lane) {
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= static_cast<uint32_t>(o)) x += y;
    }
    return x;
}
// Lanes holding the same 8-bit digit: one vote when the warp agrees, else MATCH.ANY or 8
// ballots (one per bit).  MATCH.ANY's cost grows with the number of distinct values (1.6 to
// 12.7 cycles per warp per SM on this part, tools/mb_match.cu) while the ballots cost the
// same for any digit, so a pass whose digit takes few values (skewed exponent bytes, integer
// mantissas) matches and the others vote.  An invalid lane matches only itself.
__device__ __forceinline__ uint32_t match_digit(uint32_t d, bool ok, uint32_t lane, bool few) {
    const uint32_t vm = __ballot_sync(0xffffffffu, ok);
    const uint32_t d0 = __shfl_sync(0xffffffffu, d, vm ? __ffs(vm) - 1 : 0);
    uint32_t m = vm;
    if (!__all_sync(0xffffffffu, !ok || d == d0)) {
        if (few) {
            m = __match_any_sync(0xffffffffu, ok ? d : 256u + lane);
        } else {
#pragma unroll
            for (int b = 0; b < 8; ++b) {
                const bool bit = (d >> b) & 1u;
                const uint32_t bb = __ballot_sync(0xffffffffu, bit);
                m &= bit ? bb : ~bb;
            }
        }
    }
    return ok ? m : (1u << lane);
}
// digit count: one atomic when the warp's valid lanes agree, else one per lane (distinct
// digits rarely collide within a warp)
__device__ __forceinline__ void cnt_add(uint32_t* h, uint32_t d, bool ok, uint32_t lane) {
    const uint32_t vm = __ballot_sync(0xffffffffu, ok);
    if (!vm) return;
    const int src = __ffs(vm) - 1;
    const uint32_t d0 = __shfl_sync(0xffffffffu, d, src);
    if (__all_sync(0xffffffffu, !ok || d == d0)) {
        if (lane == static_cast<uint32_t>(src)) atomicAdd(h + d0, static_cast<uint32_t>(__popc(vm)));
    } else if (ok) {
        atomicAdd(h + d, 1u);
    }
}

__global__ void __launch_bounds__(PG_THREADS, 1) gang_order_persistent(const PgArgs a) {
    namespace cg = cooperative_groups;
    cg::grid_group grid = cg::this_grid();
    extern __shared__ __align__(16) uint8_t pg_smem[];
    uint32_t* sk = reinterpret_cast<uint32_t*>(pg_smem);
    uint32_t* sv = sk + PG_TILE;
    uint32_t* stk = sv + PG_TILE;    // staging: the next tile's keys / values, bulk-copied while the
    uint32_t* stv = stk + PG_TILE;   // current tile is scanned, sorted and written
    uint32_t(*wcnt)[256] = reinterpret_cast<uint32_t(*)[256]>(stv + PG_TILE);
    uint32_t(*s_q)[256] = reinterpret_cast<uint32_t(*)[256]>(&wcnt[PG_WARPS][0]);
    uint32_t(*s_red)[256] = s_q + 4;
    uint32_t* s_base = &s_red[4][0];
    uint32_t* s_gb = s_base + 256;
    uint32_t* s_toff = s_gb + 256;
    uint32_t* s_ws = s_toff + 256;
    uint32_t* s_sc = s_ws + 32;  // [0] live count, [1] tile live count, [2..6] reduced phase-0 record
    uint64_t* bars = reinterpret_cast<uint64_t*>(s_sc + 16);  // [0, PG_NST) phase-0 ring, [PG_NST] tile staging
    uint64_t* bar = bars + PG_NST;
    const GangParams& p = a.p;
    const uint32_t G = gridDim.x, c = blockIdx.x, tid = threadIdx.x, lane = tid & 31u, warp = tid >> 5;
    const uint32_t lt = (1u << lane) - 1u;
    const uint64_t N = p.N;
    // ranges start on 16-byte boundaries (bulk copies of every field); buffers are padded past N
    const uint64_t Q0 = ((N + G - 1) / G + 15) & ~15ull;
    const uint64_t b0 = umin64(N, static_cast<uint64_t>(c) * Q0), e0 = umin64(N, b0 + Q0);

    pg_stamp(a, 0);
    // ---- phase 0: keys of programs [b0, e0); digit counts and bit masks of the live ones
    wcnt[tid >> 8][tid & 255u] = 0;  // rows 0..3: the 4 digit counts
    if (c == 0 && tid == 0) {
        a.misc[3] = 0;
        a.misc[4] = 0;
    }
    if (tid == 0) {
        for (int q = 0; q <= PG_NST; ++q) mbar_init(bars + q, 1);
        fence_mbar_init();
    }
    __syncthreads();
    bool bad = false, unsorted = false;
    uint32_t oh = 0, ah = ~0u, ol = 0, al = ~0u;
    // one program: key, flags, masks, digit-0 count (every thread calls it the same number of
    // times: the count uses warp votes)
    auto program = [&](uint64_t i, bool has, double a_, double ls, double an, uint32_t id, uint32_t idn,
                       int64_t sum, uint32_t cntv, int64_t rem, bool live) {
        uint32_t k32 = PG_DEAD;
        if (has) {
            bad = bad || !(a_ >= 0.0) || !(ls >= 0.0) || isinf(a_) || isinf(ls);
            unsorted = unsorted || a_ > an || (a_ == an && idn <= id);
            const bool esc = (p.now - ls) >= p.limit;  // inclusive escalation
            if (p.escalated) p.escalated[i] = esc ? 1 : 0;
            uint64_t hk = 0;  // escalated: arrival order == index order here
            if (!esc) {
                hk = 1ull << 63;  // fifo: arrival order == index order here
                if (p.order != CDX_ORDER_FIFO) {
                    const double est =
                        cntv ? __ddiv_rn(static_cast<double>(sum), static_cast<double>(cntv)) : p.prior;
                    const double key = __dmul_rn(est, static_cast<double>(rem > 0 ? rem : 0));
                    bad = bad || !(key >= 0.0) || isinf(key);
                    hk |= dbits(key);
                }
            }
            const uint32_t h32 = static_cast<uint32_t>(hk >> 32), l32 = static_cast<uint32_t>(hk);
            a.lo[i] = l32;
            if (live) {
                k32 = h32;
                oh |= h32;
                ah &= h32;
                ol |= l32;
                al &= l32;
            }
            a.kb[i] = k32;
        }
        cnt_add(wcnt[0], k32 & 0xffu, has && k32 != PG_DEAD, lane);  // digit 0 (see the plan)
    };
    uint64_t dstart = b0;  // programs from here on take the direct-load loop
    if (a.bulk0) {
        // whole chunks of PG_CH programs through a PG_NST-stage ring of bulk copies (thread 0
        // refills a stage once every thread has read it); the partial last chunk loads directly
        uint8_t* ring = reinterpret_cast<uint8_t*>(pg_smem);
        const uint32_t nfull = static_cast<uint32_t>((e0 - b0) / PG_CH);
        const uint64_t pol0 = policy_evict_first();
        auto issue0 = [&](uint32_t j) {
            uint8_t* st = ring + (j % PG_NST) * PG_ST_BYTES;
            uint64_t* br = bars + (j % PG_NST);
            const uint64_t i = b0 + static_cast<uint64_t>(j) * PG_CH;
            mbar_expect_tx(br, PG_CH * (8 * 3 + 4 * 3 + 1) + (p.program_id ? PG_CH * 4 : 0));
            bulk_g2s(st + PG_ST_ARR, p.arrival + i, PG_CH * 8, br, pol0);
            bulk_g2s(st + PG_ST_LS, p.last_service + i, PG_CH * 8, br, pol0);
            bulk_g2s(st + PG_ST_SUM, p.iter_tok_sum + i, PG_CH * 8, br, pol0);
            bulk_g2s(st + PG_ST_CNT, p.iter_count + i, PG_CH * 4, br, pol0);
            bulk_g2s(st + PG_ST_KNOB, p.knob + i, PG_CH * 4, br, pol0);
            bulk_g2s(st + PG_ST_CAP, p.cap + i, PG_CH * 4, br, pol0);
            bulk_g2s(st + PG_ST_TERM, p.terminated + i, PG_CH, br, pol0);
            if (p.program_id) bulk_g2s(st + PG_ST_PID, p.program_id + i, PG_CH * 4, br, pol0);
        };
        if (tid == 0)
            for (uint32_t j = 0; j < nfull && j < static_cast<uint32_t>(PG_NST); ++j) issue0(j);
        for (uint32_t j = 0; j < nfull; ++j) {
            const uint8_t* st = ring + (j % PG_NST) * PG_ST_BYTES;
            mbar_wait(bars + (j % PG_NST), (j / PG_NST) & 1u);
            const uint64_t i = b0 + static_cast<uint64_t>(j) * PG_CH + tid;
            const double* sa = reinterpret_cast<const double*>(st + PG_ST_ARR);
            const uint32_t* sp = reinterpret_cast<const uint32_t*>(st + PG_ST_PID);
            const double a_ = sa[tid];
            const double an = tid + 1 < PG_CH ? sa[tid + 1] : (i + 1 < N ? __ldg(p.arrival + i + 1) : a_);
            const uint32_t id = p.program_id ? sp[tid] : p.id_base + static_cast<uint32_t>(i);
            const uint32_t idn = !p.program_id ? id + 1u
                                 : tid + 1 < PG_CH ? sp[tid + 1]
                                 : (i + 1 < N ? __ldg(p.program_id + i + 1) : id + 1u);
            const int64_t rem = static_cast<int64_t>(reinterpret_cast<const int32_t*>(st + PG_ST_CAP)[tid]) -
                                static_cast<int64_t>(reinterpret_cast<const int32_t*>(st + PG_ST_KNOB)[tid]);
            program(i, true, a_, reinterpret_cast<const double*>(st + PG_ST_LS)[tid], an, id, idn,
                    reinterpret_cast<const int64_t*>(st + PG_ST_SUM)[tid],
                    reinterpret_cast<const uint32_t*>(st + PG_ST_CNT)[tid], rem, (st + PG_ST_TERM)[tid] == 0);
            __syncthreads();  // the stage is read: refill it
            if (tid == 0 && j + PG_NST < nfull) {
                fence_proxy_async();
                issue0(j + PG_NST);
            }
        }
        dstart = b0 + static_cast<uint64_t>(nfull) * PG_CH;
    }
    // every thread runs the same trip count (the digit counts use warp votes)
    const uint64_t span0 = (e0 - dstart + 2 * PG_THREADS - 1) / (2 * PG_THREADS) * (2 * PG_THREADS);
    for (uint64_t i0 = dstart + tid; i0 < dstart + span0; i0 += 2 * PG_THREADS) {
        double av[2], lsv[2], anv[2];
        uint32_t idv[2], idnv[2], cntv[2];
        int64_t sumv[2], remv[2];
        bool has[2], live[2];
#pragma unroll
        for (int u = 0; u < 2; ++u) {  // every field of both items loaded before any is used
            const uint64_t i = i0 + static_cast<uint64_t>(u) * PG_THREADS;
            has[u] = i < e0;
            const uint64_t k = has[u] ? i : dstart;
            av[u] = __ldg(p.arrival + k);
            lsv[u] = __ldg(p.last_service + k);
            anv[u] = k + 1 < N ? __ldg(p.arrival + k + 1) : av[u];
            idv[u] = p.program_id ? __ldg(p.program_id + k) : p.id_base + static_cast<uint32_t>(k);
            idnv[u] = p.program_id && k + 1 < N ? __ldg(p.program_id + k + 1) : idv[u] + 1u;
            sumv[u] = __ldg(p.iter_tok_sum + k);
            cntv[u] = __ldg(p.iter_count + k);
            remv[u] = static_cast<int64_t>(__ldg(p.cap + k)) - static_cast<int64_t>(__ldg(p.knob + k));
            live[u] = __ldg(p.terminated + k) == 0;
        }
#pragma unroll
        for (int u = 0; u < 2; ++u)
            program(i0 + static_cast<uint64_t>(u) * PG_THREADS, has[u], av[u], lsv[u], anv[u], idv[u], idnv[u],
                    sumv[u], cntv[u], remv[u], live[u]);
    }
    {  // this CTA's record: flags and the live keys' bit masks
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            oh |= __shfl_xor_sync(0xffffffffu, oh, o);
            ah &= __shfl_xor_sync(0xffffffffu, ah, o);
            ol |= __shfl_xor_sync(0xffffffffu, ol, o);
            al &= __shfl_xor_sync(0xffffffffu, al, o);
        }
        uint32_t* rec = &s_red[0][0];  // [PG_WARPS][4]
        if (lane == 0) {
            rec[warp * 4 + 0] = oh;
            rec[warp * 4 + 1] = ah;
            rec[warp * 4 + 2] = ol;
            rec[warp * 4 + 3] = al;
        }
        const int fl = (__syncthreads_or(unsorted) ? 1 : 0) | (__syncthreads_or(bad) ? 2 : 0);
        if (warp == 0) {
            oh = rec[lane * 4 + 0];
            ah = rec[lane * 4 + 1];
            ol = rec[lane * 4 + 2];
            al = rec[lane * 4 + 3];
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) {
                oh |= __shfl_xor_sync(0xffffffffu, oh, o);
                ah &= __shfl_xor_sync(0xffffffffu, ah, o);
                ol |= __shfl_xor_sync(0xffffffffu, ol, o);
                al &= __shfl_xor_sync(0xffffffffu, al, o);
            }
            if (lane == 0) {
                uint32_t* r = a.crec + static_cast<uint64_t>(c) * 8;
                r[0] = static_cast<uint32_t>(fl);
                r[1] = oh;
                r[2] = ah;
                r[3] = ol;
                r[4] = al;
            }
        }
    }
    if (tid < 256) a.hist[static_cast<uint64_t>(c) * 256 + tid] = wcnt[0][tid];
    pg_stamp(a, 1);
    grid.sync();
    if (warp == 0) {  // every CTA's record, reduced (each CTA plans the same passes)
        uint32_t f = 0;
        oh = 0, ah = ~0u, ol = 0, al = ~0u;
        for (uint32_t q = lane; q < G; q += 32) {
            const uint32_t* r = a.crec + static_cast<uint64_t>(q) * 8;
            f |= __ldcg(r);
            oh |= __ldcg(r + 1);
            ah &= __ldcg(r + 2);
            ol |= __ldcg(r + 3);
            al &= __ldcg(r + 4);
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            f |= __shfl_xor_sync(0xffffffffu, f, o);
            oh |= __shfl_xor_sync(0xffffffffu, oh, o);
            ah &= __shfl_xor_sync(0xffffffffu, ah, o);
            ol |= __shfl_xor_sync(0xffffffffu, ol, o);
            al &= __shfl_xor_sync(0xffffffffu, al, o);
        }
        if (lane == 0) {
            s_sc[2] = f;
            s_sc[3] = oh ^ ah;  // varying bits of the upper halves (0 when no key is live)
            s_sc[4] = ol ^ al;  // ... and of the low halves
            if (c == 0) {
                a.misc[1] = f & 1u;
                a.misc[2] = (f >> 1) & 1u;
            }
        }
    }
    __syncthreads();
    const uint32_t vary_hi = s_sc[3], vary_lo = s_sc[4];
    uint32_t dlist = 0, np = 0;  // digits to sort, 4 bits each in pass order
#pragma unroll
    for (uint32_t d = 0; d < 4; ++d)
        if ((vary_hi >> (8 * d)) & 0xffu) dlist |= d << (4 * np++);
    if (np == 0) np = 1;  // every live key equal: one pass is the stable compaction
    if ((dlist & 0xfu) != 0) {  // the first pass is not digit 0: count its digit over the programs
        const uint32_t d0 = dlist & 0xfu;
        __syncthreads();
        if (tid < 256) wcnt[0][tid] = 0;
        __syncthreads();
        const uint64_t span = (e0 - b0 + PG_THREADS - 1) / PG_THREADS * PG_THREADS;
        for (uint64_t i = b0 + tid; i < b0 + span; i += PG_THREADS) {
            const uint32_t key = i < e0 ? __ldcg(a.kb + i) : PG_DEAD;
            cnt_add(wcnt[0], (key >> (8 * d0)) & 0xffu, key != PG_DEAD, lane);
        }
        __syncthreads();
        if (tid < 256) a.hist[(static_cast<uint64_t>(d0) * G + c) * 256 + tid] = wcnt[0][tid];
        grid.sync();
    }

    uint32_t n = 0;  // live programs (known after the first pass's offsets)
    uint32_t phase = 0;
    bool few = false;  // this pass's digit takes at most PG_FEW values: rank by MATCH.ANY
    const uint64_t pol = policy_evict_last();
    for (uint32_t k = 0; k < np; ++k) {
        const uint32_t dg = (dlist >> (4 * k)) & 0xfu;
        const int shift = 8 * static_cast<int>(dg);
        const uint32_t* hp = a.hist + static_cast<uint64_t>(dg) * G * 256;
        // this pass's input range (the first pass: this CTA's programs)
        const uint32_t* kin = (k & 1) ? a.ka : a.kb;
        const uint32_t* vin = (k & 1) ? a.va : a.vb;
        uint32_t* kout = (k & 1) ? a.kb : a.ka;
        uint32_t* vout = (k & 1) ? a.vb : a.va;
        const bool last = k + 1 == np;
        // thread 0 bulk-copies tile tb of the range into the staging buffers (keys; values
        // after the first pass), completion on `bar`; whole 16-byte chunks (padding past the
        // range is never read)
        auto issue = [&](uint64_t tb, uint64_t re_) {
            const uint32_t cnt = static_cast<uint32_t>(umin64(PG_TILE, re_ - tb));
            const uint32_t bytes = (cnt * 4 + 15) & ~15u;
            fence_proxy_async_all();  // generic writes of earlier passes -> async-proxy reads
            mbar_expect_tx(bar, k ? 2 * bytes : bytes);
            bulk_g2s(stk, kin + tb, bytes, bar, pol);
            if (k) bulk_g2s(stv, vin + tb, bytes, bar, pol);
        };
        // the first pass reads this CTA's programs; later ones positions [c*Q, (c+1)*Q) of the
        // previous output (n is known from the first pass on)
        const uint64_t Q = ((static_cast<uint64_t>(n) + G - 1) / G + 3) & ~3ull;
        const uint64_t rb = k == 0 ? b0 : umin64(n, c * Q);
        const uint64_t re = k == 0 ? e0 : umin64(n, rb + Q);
        if (tid == 0 && rb < re) issue(rb, re);  // overlaps the offsets below
        // ---- this CTA's exclusive base per digit: all CTAs' counts before it + smaller digits
        {  // thread: 4 digits (one 16-byte load) of every 16th CTA's row; partial sums in wcnt
            const uint32_t rg = tid >> 6, cc = tid & 63u;
            uint4 all4 = make_uint4(0, 0, 0, 0), bef4 = make_uint4(0, 0, 0, 0);
#pragma unroll 4
            for (uint32_t q = rg; q < G; q += 16) {
                const uint4 x = __ldcg(reinterpret_cast<const uint4*>(hp + static_cast<uint64_t>(q) * 256) + cc);
                all4.x += x.x, all4.y += x.y, all4.z += x.z, all4.w += x.w;
                if (q < c) bef4.x += x.x, bef4.y += x.y, bef4.z += x.z, bef4.w += x.w;
            }
            reinterpret_cast<uint4*>(wcnt[rg])[cc] = all4;
            reinterpret_cast<uint4*>(wcnt[16 + rg])[cc] = bef4;
        }
        __syncthreads();
        {
            uint32_t all = 0, before = 0;
            if (tid < 256) {
#pragma unroll
                for (int q = 0; q < 16; ++q) {
                    all += wcnt[q][tid];
                    before += wcnt[16 + q][tid];
                }
            }
            const uint32_t incl = warp_incl_scan(all, lane);
            if (lane == 31 && warp < 8) s_ws[warp] = incl;
            few = __syncthreads_count(all != 0) <= PG_FEW;  // values the digit takes over all keys
            if (tid < 256) {
                uint32_t wpre = 0;
                for (uint32_t w = 0; w < warp; ++w) wpre += s_ws[w];
                s_base[tid] = wpre + incl - all + before;
                if (tid == 255) s_sc[0] = wpre + incl;  // every live key counted once
            }
            __syncthreads();
        }
        pg_stamp(a, 2 + 3 * k);
        if (k == 0) {
            n = s_sc[0];
            if (c == 0 && tid == 0) a.misc[0] = n;
        }
        // ---- rank, sort by digit in shared memory, write digit runs; tile by tile in order
#pragma unroll
        for (int w = 0; w < PG_WARPS; w += 4) wcnt[w + (tid >> 8)][tid & 255u] = 0;
        __syncthreads();
        for (uint64_t tb = rb; tb < re; tb += PG_TILE) {
            const uint32_t tile_n = static_cast<uint32_t>(umin64(PG_TILE, re - tb));
            mbar_wait(bar, phase);
            phase ^= 1u;
            uint32_t kk[PG_ITEMS], v[PG_ITEMS], rank[PG_ITEMS];
            const uint32_t wofs = warp * 32 * PG_ITEMS + lane;  // item j: tile index wofs + 32 j
#pragma unroll
            for (int j = 0; j < PG_ITEMS; ++j) {
                const uint32_t li = wofs + 32 * j;
                const bool ok = li < tile_n;
                kk[j] = ok ? stk[li] : PG_DEAD;
                v[j] = k == 0 ? static_cast<uint32_t>(tb + li) : stv[li];
            }
#pragma unroll
            for (int j = 0; j < PG_ITEMS; ++j) {
                const bool ok = kk[j] != PG_DEAD;  // out of range or terminated (first pass)
                const uint32_t d = (kk[j] >> shift) & 0xffu;
                const uint32_t peers = match_digit(d, ok, lane, few);
                const uint32_t below = peers & lt;
                // the row is this warp's own and the group leaders hold distinct digits: a plain
                // read-modify-write, ordered against the next item by the warp barrier
                uint32_t old = 0;
                if (ok && below == 0) {
                    old = wcnt[warp][d];
                    wcnt[warp][d] = old + static_cast<uint32_t>(__popc(peers));
                }
                rank[j] = __shfl_sync(0xffffffffu, old, __ffs(peers) - 1) + __popc(below);
                __syncwarp();
            }
            __syncthreads();  // the staging buffers are consumed: fetch the next tile behind this one
            if (tid == 0 && tb + PG_TILE < re) issue(tb + PG_TILE, re);
            // thread d < 256: the tile's count of digit d over the warps, the digit scan, then the
            // warps' first tile-sorted index per digit (two CTA barriers)
            uint32_t cnt = 0;
            if (tid < 256) {
#pragma unroll 8
                for (int w = 0; w < PG_WARPS; ++w) cnt += wcnt[w][tid];
            }
            const uint32_t incl = warp_incl_scan(cnt, lane);
            if (lane == 31 && warp < 8) s_ws[warp] = incl;
            __syncthreads();
            if (tid < 256) {
                uint32_t wpre = 0;
                for (uint32_t w = 0; w < warp; ++w) wpre += s_ws[w];
                const uint32_t toff = wpre + incl - cnt;
                s_gb[tid] = s_base[tid] - toff;  // global position = s_gb[digit] + tile-sorted index
                s_base[tid] += cnt;
                if (tid == 255) s_sc[1] = wpre + incl;
                uint32_t run = toff;  // wcnt[w][d] = first tile-sorted index of warp w's digit-d keys
#pragma unroll 8
                for (int w = 0; w < PG_WARPS; ++w) {
                    const uint32_t x = wcnt[w][tid];
                    wcnt[w][tid] = run;
                    run += x;
                }
            }
            __syncthreads();
#pragma unroll
            for (int j = 0; j < PG_ITEMS; ++j) {
                if (kk[j] == PG_DEAD) continue;
                const uint32_t lp = wcnt[warp][(kk[j] >> shift) & 0xffu] + rank[j];
                sk[lp] = kk[j];
                sv[lp] = v[j];
            }
            __syncthreads();
#pragma unroll
            for (int w = 0; w < PG_WARPS; w += 4) wcnt[w + (tid >> 8)][tid & 255u] = 0;  // next tile's counts
            const uint32_t tl = s_sc[1];
            for (uint32_t li = tid; li < tl; li += PG_THREADS) {
                const uint32_t key = sk[li], val = sv[li];
                const uint32_t pos = s_gb[(key >> shift) & 0xffu] + li;
                kout[pos] = key;
                vout[pos] = val;
                if (last) a.order[pos] = p.program_id ? __ldg(p.program_id + val) : p.id_base + val;
            }
            __syncthreads();  // sk / sv / wcnt / s_gb / s_sc are reused by the next tile
        }
        pg_stamp(a, 3 + 3 * k);
        grid.sync();
        if (last) break;
        // ---- next digit's counts over this CTA's next input range (positions [c*Q, (c+1)*Q))
        if (tid < 256) wcnt[0][tid] = 0;
        __syncthreads();
        {
            const uint32_t dn = (dlist >> (4 * (k + 1))) & 0xfu;
            const int nshift = 8 * static_cast<int>(dn);
            const uint64_t Qn = ((static_cast<uint64_t>(n) + G - 1) / G + 3) & ~3ull;  // n is known now
            const uint64_t nb = umin64(n, c * Qn), ne = umin64(n, nb + Qn);  // the next pass's range
            constexpr int U = 8;  // keys in flight per thread per round trip
            const uint64_t span = (ne - nb + U * PG_THREADS - 1) / (U * PG_THREADS) * (U * PG_THREADS);
            for (uint64_t i0 = nb + tid; i0 < nb + span; i0 += U * PG_THREADS) {
                uint32_t key[U];
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    const uint64_t i = i0 + static_cast<uint64_t>(u) * PG_THREADS;
                    key[u] = i < ne ? __ldcg(kout + i) : 0u;
                }
#pragma unroll
                for (int u = 0; u < U; ++u)
                    cnt_add(wcnt[0], (key[u] >> nshift) & 0xffu, i0 + static_cast<uint64_t>(u) * PG_THREADS < ne, lane);
            }
            __syncthreads();
            if (tid < 256) a.hist[(static_cast<uint64_t>(dn) * G + c) * 256 + tid] = wcnt[0][tid];
        }
        pg_stamp(a, 4 + 3 * k);
        grid.sync();
    }
    if (vary_lo == 0) {  // every live low half equal: the upper halves decide alone
        pg_stamp(a, 15);
        return;
    }

    // ---- fix-up: runs of equal upper halves whose low halves descend
    const bool odd = ((np - 1) & 1u) != 0;  // the last pass wrote kb / vb when odd, ka / va when even
    const uint32_t* kf = odd ? a.kb : a.ka;
    const uint32_t* vf = odd ? a.vb : a.va;
    uint32_t* runs = odd ? a.va : a.vb;  // free after the last pass
    {
        const uint64_t Q = ((static_cast<uint64_t>(n) + G - 1) / G + 3) & ~3ull;
        const uint64_t nb = umin64(n, c * Q), ne = umin64(n, nb + Q);
        constexpr int U = 8;  // positions per thread per round: the key / value / low-half loads
                              // of all U are in flight together
        for (uint64_t i0 = nb + tid; i0 < ne; i0 += U * PG_THREADS) {
            uint32_t hk[U], hq[U], vi[U], vp[U], li[U], lp[U];
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const uint64_t i = i0 + static_cast<uint64_t>(u) * PG_THREADS;
                const bool in = i < ne && i > 0;
                hk[u] = in ? __ldcg(kf + i) : 0u;
                hq[u] = in ? __ldcg(kf + i - 1) : 1u;
            }
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const uint64_t i = i0 + static_cast<uint64_t>(u) * PG_THREADS;
                const bool eq = hk[u] == hq[u];
                vi[u] = eq ? __ldcg(vf + i) : 0u;
                vp[u] = eq ? __ldcg(vf + i - 1) : 0u;
            }
            uint32_t desc = 0;  // bit u: a descent at position i0 + u * PG_THREADS
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const bool eq = hk[u] == hq[u];
                li[u] = eq ? __ldcg(a.lo + vi[u]) : 1u;
                lp[u] = eq ? __ldcg(a.lo + vp[u]) : 0u;
            }
#pragma unroll
            for (int u = 0; u < U; ++u) desc |= (li[u] < lp[u] ? 1u : 0u) << u;
            while (desc) {  // a descent inside a run: the first one of its run lists the run start
                const int u = __ffs(desc) - 1;
                desc &= desc - 1;
                const uint64_t i = i0 + static_cast<uint64_t>(u) * PG_THREADS;
                const uint32_t h = __ldcg(kf + i);
                uint64_t j = i - 1;
                bool first = true;
                while (j > 0 && __ldcg(kf + j - 1) == h) {
                    if (i - j >= FIX_RUN) break;
                    first = first && !(__ldcg(a.lo + __ldcg(vf + j)) < __ldcg(a.lo + __ldcg(vf + j - 1)));
                    --j;
                }
                const bool reach = j == 0 || __ldcg(kf + j - 1) != h;
                if (!reach) {
                    atomicOr(a.misc + 3, 1u);  // the run is longer than the fix-up handles
                } else if (first) {
                    uint64_t e = i + 1;  // the run must also end within reach
                    while (e < n && e - j <= FIX_RUN && __ldcg(kf + e) == h) ++e;
                    if (e - j > FIX_RUN) atomicOr(a.misc + 3, 1u);
                    else runs[atomicAdd(a.misc + 4, 1u)] = static_cast<uint32_t>(j);  // at most n/2 runs
                }
            }
        }
    }
    pg_stamp(a, 14);
    grid.sync();
    if (__ldcg(a.misc + 3)) return;  // the caller re-sorts all 8 digits
    const uint32_t cnt = __ldcg(a.misc + 4);
    for (uint32_t t = c * PG_THREADS + tid; t < cnt; t += G * PG_THREADS) {
        const uint64_t i = __ldcg(runs + t);
        const uint32_t h = __ldcg(kf + i);
        uint32_t rv[FIX_RUN], rl[FIX_RUN];
        uint32_t m = 0;
        for (uint64_t e = i; e < n && m < FIX_RUN && __ldcg(kf + e) == h; ++e, ++m) {
            const uint32_t val = __ldcg(vf + e), l = __ldcg(a.lo + val);
            uint32_t b = m;  // stable insertion by the low half
            while (b > 0 && rl[b - 1] > l) {
                rl[b] = rl[b - 1];
                rv[b] = rv[b - 1];
                --b;
            }
            rl[b] = l;
            rv[b] = val;
        }
        for (uint32_t q = 0; q < m; ++q)
            a.order[i + q] = p.program_id ? __ldg(p.program_id + rv[q]) : p.id_base + rv[q];
    }
    pg_stamp(a, 15);
}

// Digits [dlo, 8) with the key count on the device (n_dev; nmax bounds it): the caller has
// histogrammed the keys into lb[0, 2048) already.  No host round trip: every digit gets a
// pass (trivial ones copy), so the result lands in k0/v0 for an even pass count.
int radix_sort_dev(cdx_ctx* ctx, uint64_t* k0, uint32_t* v0, uint64_t* k1, uint32_t* v1, uint64_t nmax,
                   const uint32_t* n_dev, uint32_t* lb, int dlo, int* which) {
    const uint32_t ntiles = static_cast<uint32_t>((nmax + RS_TILE - 1) / RS_TILE);
    *which = 0;
    if (nmax == 0) return CDX_OK;
    uint32_t* ghist = lb;
    uint32_t* tickets = lb + 8 * 256;
    uint32_t* look = tickets + 16;
    cudaError_t e = cudaMemsetAsync(tickets, 0, (16 + static_cast<size_t>(8) * ntiles * 256) * 4, ctx->stream);
    if (e == cudaSuccess) e = cudaFuncSetAttribute(os_pass2, cudaFuncAttributeMaxDynamicSharedMemorySize, RS2_SMEM);
    if (e != cudaSuccess) return cuda_fail(ctx, e, "radix(device count)");
    uint64_t* kin = k0;
    uint32_t* vin = v0;
    uint64_t* kout = k1;
    uint32_t* vout = v1;
    for (int d = dlo; d < 8; ++d) {
        os_pass2<<<ntiles, RS_THREADS, RS2_SMEM, ctx->stream>>>(kin, vin, kout, vout, nmax, 8 * d, ghist + d * 256,
                                                                look + static_cast<size_t>(d) * ntiles * 256,
                                                                tickets + d, nullptr, n_dev);
        CDX_CHECK_LAUNCH(ctx, "radix(pass)");
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

// stable LSD radix sort of (u64 key, u32 value) pairs for other kernels (k_jsonl.cu)
size_t radix_scratch_words(uint64_t n) {
    return static_cast<size_t>(8) * 256 * ((n + RS_TILE - 1) / RS_TILE) + 8 * 256 + 16;
}
int radix_sort_pairs(cdx_ctx* ctx, uint64_t* k0, uint32_t* v0, uint64_t* k1, uint32_t* v1, uint64_t n, uint32_t* lb,
                     int* which) {
    return radix_sort(ctx, k0, v0, k1, v1, n, lb, which, nullptr, nullptr, nullptr);
}

}  // namespace cdx

namespace cdx {
namespace {
enum GangMode { GANG_FAST = 0, GANG_CHECKED = 1, GANG_FULL = 2 };
// The persistent one-launch order (gang_order_persistent).  *used = false when this device
// cannot host the cooperative grid (no cooperative launch, an SM limit leaving no room), or
// CDX_GANG_PS=0 asks for the multi-launch path; the caller then takes that path.
int gang_persistent(cdx_ctx* ctx, const GangParams& p, uint64_t N, uint32_t* order, uint64_t* n_out, int* redo,
                    bool* used) {
    *used = false;
    const char* env = getenv("CDX_GANG_PS");
    if (env && env[0] == '0') return CDX_OK;
    // resident CTAs per SM, queried once per device (-1: not yet, 0: no cooperative launch)
    static std::atomic<int> occ_cache[64];
    static std::atomic<int> occ_set[64];
    const int dev = ctx->device & 63;
    int occ = 0;
    if (occ_set[dev].load(std::memory_order_acquire)) {
        occ = occ_cache[dev].load(std::memory_order_relaxed);
    } else {
        int coop = 0;
        cudaDeviceGetAttribute(&coop, cudaDevAttrCooperativeLaunch, ctx->device);
        cudaError_t e = cudaFuncSetAttribute(gang_order_persistent, cudaFuncAttributeMaxDynamicSharedMemorySize, PG_SMEM);
        if (e == cudaSuccess && coop)
            e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, gang_order_persistent, PG_THREADS, PG_SMEM);
        if (e != cudaSuccess || !coop) {
            cudaGetLastError();
            occ = 0;
        }
        occ_cache[dev].store(occ, std::memory_order_relaxed);
        occ_set[dev].store(1, std::memory_order_release);
    }
    if (occ < 1) return CDX_OK;
    const uint64_t want = std::max<uint64_t>(1, (N + PG_TILE - 1) / PG_TILE);
    const uint32_t G = static_cast<uint32_t>(std::min<uint64_t>(want, static_cast<uint64_t>(ctx->sm_count) * occ));
    // scratch: lo ka va kb vb [NP] | hist [4][G][256] | crec [G][8] | misc [16]; NP pads N to whole
    // 16-byte chunks plus one (the bulk copies read whole chunks)
    const size_t NP = ((N + 3) & ~3ull) + 4;
    const size_t words = NP * 5 + static_cast<size_t>(4) * G * 256 + static_cast<size_t>(G) * 8 + 16;
    uint32_t* s = static_cast<uint32_t*>(scratch(ctx, words * 4));
    if (!s) return set_error(ctx, CDX_ECUDA, "gang_priority: scratch allocation failed");
    PgArgs a{p, s, s + NP, s + 2 * NP, s + 3 * NP, s + 4 * NP, s + 5 * NP, nullptr, nullptr, order, nullptr, 0};
    auto al16 = [](const void* q) { return (reinterpret_cast<uintptr_t>(q) & 15) == 0; };
    a.bulk0 = al16(p.arrival) && al16(p.last_service) && al16(p.iter_tok_sum) && al16(p.iter_count) &&
              al16(p.knob) && al16(p.cap) && al16(p.terminated) && al16(p.program_id);
    a.crec = a.hist + static_cast<size_t>(4) * G * 256;
    a.misc = a.crec + static_cast<size_t>(G) * 8;
    const bool prof = getenv("CDX_GANG_PS_PROF") != nullptr;  // phase timings to stderr (tuning only)
    if (prof) {
        a.prof = static_cast<unsigned long long*>(scratch2(ctx, static_cast<size_t>(G) * 16 * 8));
        cudaMemsetAsync(a.prof, 0, static_cast<size_t>(G) * 16 * 8, ctx->stream);
    }
    void* args[] = {&a};
    cudaError_t e = cudaLaunchCooperativeKernel(reinterpret_cast<const void*>(gang_order_persistent), dim3(G),
                                                dim3(PG_THREADS), args, PG_SMEM, ctx->stream);
    if (e == cudaErrorCooperativeLaunchTooLarge) {  // e.g. an MPS SM limit below the occupancy query
        cudaGetLastError();
        return CDX_OK;
    }
    if (e != cudaSuccess) return cuda_fail(ctx, e, "gang_priority(persistent)");
    CDX_LAUNCHED(ctx);
    *used = true;
    uint32_t* hm = ctx->h_small;  // pinned: an asynchronous copy, then one stream sync
    e = cudaMemcpyAsync(hm, a.misc, 5 * 4, cudaMemcpyDeviceToHost, ctx->stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize(ctx->stream);
    if (e != cudaSuccess) return cuda_fail(ctx, e, "gang_priority");
    if (prof) {  // per phase: the latest CTA's stamp minus the earliest start
        std::vector<unsigned long long> t(static_cast<size_t>(G) * 16);
        cudaMemcpy(t.data(), a.prof, t.size() * 8, cudaMemcpyDeviceToHost);
        unsigned long long t0 = ~0ull, mx[16] = {};
        for (uint32_t c = 0; c < G; ++c) {
            t0 = std::min(t0, t[c * 16]);
            for (int k = 0; k < 16; ++k) mx[k] = std::max(mx[k], t[c * 16 + k]);
        }
        fprintf(stderr, "gang_ps G=%u N=%llu:", G, static_cast<unsigned long long>(N));
        for (int k = 1; k < 16; ++k) fprintf(stderr, " %d:%.1f", k, mx[k] >= t0 ? (mx[k] - t0) / 1e3 : -1.0);
        fprintf(stderr, " us  (runs %u fallback %u)\n", hm[4], hm[3]);
    }
    if (hm[2]) return set_error(ctx, CDX_EINVAL, "gang_priority: times and keys must be finite and >= 0");
    *n_out = hm[0];
    if (hm[0] == 0) return CDX_OK;
    if (hm[1]) *redo = GANG_CHECKED;
    else if (hm[3]) *redo = GANG_FULL;
    return CDX_OK;
}

// One evaluation.  GANG_FAST: no pre-sort, device-side count, one sync (see below).
// GANG_CHECKED: host-driven, with the (arrival, id) pre-sort when arrivals are unsorted and
// the upper-half sort + run fix-up.  GANG_FULL: all 8 digits.  *redo names the path the
// caller must run instead when this one could not finish (unsorted arrivals, a long run).
int gang_priority_run(cdx_ctx* ctx, const cdx_prog_soa* progs, uint64_t N, const cdx_inter_policy* pol, double now,
                      uint32_t* order, uint64_t* n_out, uint8_t* escalated, uint64_t* keys, int mode, int* redo) {
    *redo = GANG_FAST;
    const bool full = mode == GANG_FULL;
    GangParams p{progs->arrival, progs->last_service, progs->iter_tok_sum, progs->iter_count, progs->knob,
                 progs->cap, progs->terminated, progs->program_id, escalated, N, progs->id_base, pol->order, now,
                 pol->starvation_limit, pol->prior_tokens};
    if (mode == GANG_FAST && !keys) {
        bool used = false;
        if (int st = gang_persistent(ctx, p, N, order, n_out, redo, &used)) return st;
        if (used) return CDX_OK;
    }
    const uint32_t ntiles = static_cast<uint32_t>((N + RS_TILE - 1) / RS_TILE);
    const uint32_t gtiles = static_cast<uint32_t>((N + GP_TILE - 1) / GP_TILE);
    const uint64_t nh = static_cast<uint64_t>(8) * 256 * ntiles + 8 * 256 + 16;  // radix look-back scratch
    // scratch: khi karr t0 t1 (u64) | kid va vb perm (u32) | misc | prepare look-back | radix
    const size_t bytes = N * 8 * 4 + N * 4 * 4 + 64 + (gtiles + 16) * 4 + nh * 4 + 256;
    uint8_t* s = static_cast<uint8_t*>(scratch(ctx, bytes));
    if (!s) return set_error(ctx, CDX_ECUDA, "gang_priority: scratch allocation failed");
    uint64_t* khi = reinterpret_cast<uint64_t*>(s);
    uint64_t* karr = khi + N;
    uint64_t* t0 = karr + N;
    uint64_t* t1 = t0 + N;
    uint32_t* kid = reinterpret_cast<uint32_t*>(t1 + N);
    uint32_t* va = kid + N;
    uint32_t* vb = va + N;
    uint32_t* perm = vb + N;
    uint32_t* misc = perm + N;  // 16 words
    uint32_t* plook = misc + 16;
    uint32_t* hist = plook + gtiles + 16;
    cudaMemsetAsync(misc, 0, 16 * 4, ctx->stream);
    Launch L{ctx};
    gang_count<<<(gtiles + 7) / 8, 256, 0, ctx->stream>>>(progs->terminated, N, plook, gtiles);
    CDX_CHECK_LAUNCH(ctx, "gang_priority(count)");
    gang_scan_tiles<<<1, 1024, 0, ctx->stream>>>(plook, gtiles, misc);
    CDX_CHECK_LAUNCH(ctx, "gang_priority(scan)");
    // lean: the fast path without key output sorts the ids themselves (no position -> id
    // gather afterwards, no arrival keys or id table written); any redo re-runs prepare
    const uint32_t lean = mode == GANG_FAST && !keys ? 1u : 0u;
    gang_prepare<<<gtiles, GP_THREADS, 0, ctx->stream>>>(p, khi, karr, kid, va, plook, misc, lean);
    CDX_CHECK_LAUNCH(ctx, "gang_priority(prepare)");
    // digit counts of the live hi keys (count read on the device), fetched with the flags
    cudaMemsetAsync(hist, 0, 8 * 256 * 4, ctx->stream);
    const unsigned hgrid = static_cast<unsigned>(std::min<uint64_t>(ntiles, static_cast<uint64_t>(ctx->sm_count) * 4));
    if (full)
        os_histogram<0><<<hgrid, RS_THREADS, 0, ctx->stream>>>(khi, N, hist, misc);
    else
        os_histogram<4><<<hgrid, RS_THREADS, 0, ctx->stream>>>(khi, N, hist, misc);
    CDX_CHECK_LAUNCH(ctx, "gang_priority(histogram)");
    if (mode == GANG_FAST) {
        // Optimistic single-round-trip path: arrivals assumed non-decreasing (no pre-sort),
        // the key count stays on the device, 4 upper-half passes (even count: the result is
        // back in khi/va), the run fix-up, then ONE sync that fetches the count and every
        // flag.  Unsorted arrivals or a long descending run send the caller to the checked /
        // full path, which recomputes everything.
        int which = 0;
        if (int st = radix_sort_dev(ctx, khi, va, t0, vb, N, misc, hist, 4, &which)) return st;
        uint32_t* fix = hist;  // the digit counts are consumed: reuse for the run list
        const uint32_t list_cap = static_cast<uint32_t>(std::min<uint64_t>(nh - 2, 0xffffffffull));
        cudaMemsetAsync(fix, 0, 8, ctx->stream);
        const uint32_t* vid = lean ? nullptr : kid;  // values are ids already when lean
        gang_fix_a<<<L.grid(N), 256, 0, ctx->stream>>>(khi, va, vid, N, order, fix, list_cap, misc);
        CDX_CHECK_LAUNCH(ctx, "gang_priority(order)");
        gang_fix_b<<<ctx->sm_count * 2, 256, 0, ctx->stream>>>(khi, va, vid, N, order, fix, misc);
        CDX_CHECK_LAUNCH(ctx, "gang_priority(runs)");
        if (keys) {
            pack_keys<<<L.grid(N), 256, 0, ctx->stream>>>(khi, karr, kid, va, keys, N, misc);
            CDX_CHECK_LAUNCH(ctx, "gang_priority(keys)");
        }
        uint32_t hm[3], fb[2];
        cudaError_t e = cudaMemcpyAsync(hm, misc, 12, cudaMemcpyDeviceToHost, ctx->stream);
        if (e == cudaSuccess) e = cudaMemcpyAsync(fb, fix, 8, cudaMemcpyDeviceToHost, ctx->stream);
        if (e == cudaSuccess) e = cudaStreamSynchronize(ctx->stream);
        if (e != cudaSuccess) return cuda_fail(ctx, e, "gang_priority");
        if (hm[2]) return set_error(ctx, CDX_EINVAL, "gang_priority: times and keys must be finite and >= 0");
        *n_out = hm[0];
        if (hm[0] == 0) return CDX_OK;
        if (hm[1]) *redo = GANG_CHECKED;
        else if (fb[0]) *redo = GANG_FULL;
        return CDX_OK;
    }
    uint32_t hm[3];
    std::vector<uint32_t> hh(8 * 256);
    cudaError_t e = cudaMemcpyAsync(hm, misc, 12, cudaMemcpyDeviceToHost, ctx->stream);
    if (e == cudaSuccess)
        e = cudaMemcpyAsync(hh.data(), hist, 8 * 256 * 4, cudaMemcpyDeviceToHost, ctx->stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize(ctx->stream);
    if (e != cudaSuccess) return cuda_fail(ctx, e, "gang_priority");
    if (hm[2]) return set_error(ctx, CDX_EINVAL, "gang_priority: times and keys must be finite and >= 0");
    const uint64_t n = hm[0];
    *n_out = n;
    if (n == 0) return CDX_OK;
    // 1) (arrival, id): programs are compacted in id order, so a stable sort on arrival
    //    bits yields the tie-break order; skipped when arrivals are non-decreasing.
    uint32_t* p1 = va;  // permutation: position -> compacted index (identity from prepare)
    if (hm[1] && progs->program_id) {
        // explicit ids: stable sort by id, then stably by arrival bits -> (arrival, id) order
        widen_u32<<<L.grid(n), 256, 0, ctx->stream>>>(kid, t0, n);
        CDX_CHECK_LAUNCH(ctx, "gang_priority(ids)");
        int which = 0;
        if (int st = radix_sort(ctx, t0, va, t1, vb, n, hist, &which, nullptr, nullptr, nullptr)) return st;
        uint32_t* by_id = which ? vb : va;
        uint32_t* other = which ? va : vb;
        gather<uint64_t><<<L.grid(n), 256, 0, ctx->stream>>>(karr, by_id, t0, n);
        CDX_CHECK_LAUNCH(ctx, "gang_priority(gather)");
        if (int st = radix_sort(ctx, t0, by_id, t1, other, n, hist, &which, nullptr, nullptr, nullptr)) return st;
        p1 = which ? other : by_id;  // va or vb; the hi sort below ping-pongs it with perm
    } else if (hm[1]) {
        cudaMemcpyAsync(t0, karr, n * 8, cudaMemcpyDeviceToDevice, ctx->stream);
        int which = 0;
        if (int st = radix_sort(ctx, t0, va, t1, vb, n, hist, &which, nullptr, nullptr, nullptr)) return st;
        p1 = which ? vb : va;
    }
    // 2) stable sort on hi over the (arrival, id) order
    uint64_t* hin = khi;  // already in (arrival, id) order when the pre-sort was skipped
    uint32_t* pa = p1;
    uint32_t* pb = perm;
    if (hm[1]) {
        gather<uint64_t><<<L.grid(n), 256, 0, ctx->stream>>>(khi, p1, t0, n);
        CDX_CHECK_LAUNCH(ctx, "gang_priority(gather)");
        hin = t0;
    }
    int which = 0;
    uint64_t* hout = hin == t0 ? t1 : t0;
    // the hi counts on the device are still valid unless the pre-sort overwrote them
    const uint32_t* hhp = hm[1] ? nullptr : hh.data();
    if (!full) {
        if (int st = radix_sort(ctx, hin, pa, hout, pb, n, hist, &which, hhp, nullptr, nullptr, 4)) return st;
        uint64_t* ks = which ? hout : hin;
        uint32_t* vs = which ? pb : pa;  // position -> compacted index
        // run list: the radix look-back scratch is free again (>= 8*256*ntiles words)
        uint32_t* fix = hist;
        const uint32_t list_cap = static_cast<uint32_t>(std::min<uint64_t>(nh - 2, 0xffffffffull));
        cudaMemsetAsync(fix, 0, 8, ctx->stream);
        gang_fix_a<<<L.grid(n), 256, 0, ctx->stream>>>(ks, vs, kid, n, order, fix, list_cap, nullptr);
        CDX_CHECK_LAUNCH(ctx, "gang_priority(order)");
        uint32_t fb[2] = {0, 0};
        e = cudaMemcpyAsync(fb, fix, 8, cudaMemcpyDeviceToHost, ctx->stream);
        if (e == cudaSuccess) e = cudaStreamSynchronize(ctx->stream);
        if (e != cudaSuccess) return cuda_fail(ctx, e, "gang_priority(runs)");
        if (fb[0]) {
            *redo = GANG_FULL;
            return CDX_OK;
        }
        if (fb[1]) {
            gang_fix_b<<<L.grid(fb[1]), 256, 0, ctx->stream>>>(ks, vs, kid, n, order, fix, nullptr);
            CDX_CHECK_LAUNCH(ctx, "gang_priority(runs)");
        }
        if (keys) {
            pack_keys<<<L.grid(n), 256, 0, ctx->stream>>>(ks, karr, kid, vs, keys, n);
            CDX_CHECK_LAUNCH(ctx, "gang_priority(keys)");
        }
        return CDX_OK;
    }
    // all 8 digits; the last pass writes program ids straight into `order` unless the keys
    // are wanted too
    if (int st = radix_sort(ctx, hin, pa, hout, pb, n, hist, &which, hhp, keys ? nullptr : kid,
                            keys ? nullptr : order))
        return st;
    if (which == 2) return CDX_OK;
    uint32_t* fin = which ? pb : pa;  // position -> compacted index
    gather<uint32_t><<<L.grid(n), 256, 0, ctx->stream>>>(kid, fin, order, n);
    CDX_CHECK_LAUNCH(ctx, "gang_priority(order)");
    if (keys) {
        pack_keys<<<L.grid(n), 256, 0, ctx->stream>>>(which ? hout : hin, karr, kid, fin, keys, n);
        CDX_CHECK_LAUNCH(ctx, "gang_priority(keys)");
    }
    return CDX_OK;
}
}  // namespace
}  // namespace cdx


extern "C" int cdx_gang_priority(cdx_ctx* ctx, const cdx_prog_soa* progs, uint64_t N, const cdx_inter_policy* pol,
                                 double now, uint32_t* order, uint64_t* n_out, uint8_t* escalated, uint64_t* keys) {
    using namespace cdx;
    CDX_NVTX("cdx_gang_priority");
    if (!ctx) return CDX_EINVAL;
    if (!progs || !pol || !order || !n_out) return set_error(ctx, CDX_EINVAL, "gang_priority: null pointer");
    if (!(pol->starvation_limit > 0.0))
        return set_error(ctx, CDX_EINVAL, "scheduler: starvation_limit must be > 0");
    if (pol->order != CDX_ORDER_FIFO && pol->order != CDX_ORDER_SJF)
        return set_error(ctx, CDX_EINVAL, "scheduler: order must be fifo or sjf_estimated");
    if (N >= 0xffffffffull) return set_error(ctx, CDX_EINVAL, "gang_priority: at most 2^32-2 programs");
    *n_out = 0;
    if (N == 0) return CDX_OK;
    // CDX_GANG_MODE=checked|full pins the path (A/B timing, tests of the fallbacks)
    const char* fm = getenv("CDX_GANG_MODE");
    int mode = fm && !std::strcmp(fm, "full") ? GANG_FULL : (fm && !std::strcmp(fm, "checked") ? GANG_CHECKED : GANG_FAST);
    for (;;) {
        int redo = GANG_FAST;
        if (int st = gang_priority_run(ctx, progs, N, pol, now, order, n_out, escalated, keys, mode, &redo)) return st;
        if (redo == GANG_FAST || redo <= mode) return CDX_OK;
        mode = redo;
    }
}

extern "C" int cdx_gang_merge(cdx_ctx* ctx, const uint64_t* keys, const uint64_t* run_len, uint32_t runs,
                              uint64_t stride, uint32_t* order_out, uint64_t* total) {
    using namespace cdx;
    CDX_NVTX("cdx_gang_merge");
    if (!ctx) return CDX_EINVAL;
    if (!keys || !run_len || !order_out || runs == 0) return set_error(ctx, CDX_EINVAL, "gang_merge: bad args");
    if (stride == 0) return CDX_OK;
    Launch L{ctx};
    merge_rank<<<L.grid(static_cast<uint64_t>(runs) * stride), 256, 0, ctx->stream>>>(keys, run_len, runs, stride,
                                                                                      order_out, total);
    CDX_CHECK_LAUNCH(ctx, "gang_merge");
    return CDX_OK;
}
