#pragma once
// k_scan.cuh — single-pass exclusive scan of a loaded u32 sequence into Out (u32 / u64),
// shared by the JSONL ingestion (k_jsonl.cu) and the answer interning (k_intern.cu).
// Every tile resident: one cooperative launch, tile aggregates summed after one grid
// barrier.  Otherwise: tiles take tickets and resolve their prefix by decoupled look-back.
#include <cooperative_groups.h>

#include <algorithm>

#include "cdx_internal.cuh"

namespace cdx {
namespace scan {

// ---- single-pass exclusive scan (decoupled look-back) --------------------------------------
// out[i] = sum of ld(j) for j < i; with `total_slot`, out[n] = the grand total as well (arena
// offsets are n + 1 long).  Tiles of 2048 elements, 8 consecutive per thread; the tile
// records pack state (bits 62-63: 1 aggregate, 2 inclusive) with a 62-bit value, so one
// 64-bit store publishes both.  Tickets order the tiles; records and ticket are cleared by
// the caller before each call.
constexpr int SL_THREADS = 256, SL_ITEMS = 8, SL_TILE = SL_THREADS * SL_ITEMS;
constexpr uint64_t SL_AGG = 1ull << 62, SL_INC = 2ull << 62, SL_VAL = (1ull << 62) - 1;

struct LoadU32 {
    const uint32_t* v;
    __device__ uint32_t operator()(uint64_t i) const { return v[i]; }
};

// coop: launched cooperatively with every tile resident; tile aggregates are summed after
// one grid barrier (no tickets, no look-back chain)
template <class Load, typename Out>
__global__ void __launch_bounds__(SL_THREADS) scan_lb(Load ld, uint64_t n, Out* __restrict__ out, bool total_slot,
                                                      uint64_t* __restrict__ rec, uint32_t* __restrict__ ticket,
                                                      uint64_t* __restrict__ total, int coop) {
    __shared__ uint32_t s_tile;
    __shared__ uint64_t s_w[SL_THREADS / 32];
    __shared__ uint64_t s_excl;
    const uint32_t tid = threadIdx.x, lane = tid & 31u, warp = tid >> 5;
    if (tid == 0) s_tile = coop ? blockIdx.x : atomicAdd(ticket, 1u);
    __syncthreads();
    const uint32_t tile = s_tile;
    const uint64_t b = static_cast<uint64_t>(tile) * SL_TILE + static_cast<uint64_t>(tid) * SL_ITEMS;
    uint32_t v[SL_ITEMS];
    uint64_t sum = 0;
#pragma unroll
    for (int j = 0; j < SL_ITEMS; ++j) {
        v[j] = b + j < n ? ld(b + j) : 0u;
        sum += v[j];
    }
    uint64_t inc = sum;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint64_t y = __shfl_up_sync(0xffffffffu, inc, o);
        if (lane >= static_cast<uint32_t>(o)) inc += y;
    }
    if (lane == 31) s_w[warp] = inc;
    __syncthreads();
    uint64_t tot = 0, wpre = 0;
#pragma unroll
    for (int w = 0; w < SL_THREADS / 32; ++w) {
        wpre += w < static_cast<int>(warp) ? s_w[w] : 0ull;
        tot += s_w[w];
    }
    if (coop) {
        if (tid == 0) rec[tile] = tot;
        cooperative_groups::this_grid().sync();
        uint64_t sv = 0;
        for (uint32_t q = tid; q < tile; q += SL_THREADS) sv += __ldcg(reinterpret_cast<const unsigned long long*>(rec + q));
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) sv += __shfl_xor_sync(0xffffffffu, sv, o);
        __shared__ uint64_t s_red[SL_THREADS / 32];
        if (lane == 0) s_red[warp] = sv;
        __syncthreads();
        if (tid == 0) {
            uint64_t ex = 0;
            for (int w = 0; w < SL_THREADS / 32; ++w) ex += s_red[w];
            s_excl = ex;
            if (static_cast<uint64_t>(tile + 1) * SL_TILE >= n) {  // the last tile
                if (total) *total = ex + tot;
                if (total_slot) out[n] = static_cast<Out>(ex + tot);
            }
        }
    } else if (warp == 0) {
        if (lane == 0) {
            volatile uint64_t* r = rec + tile;
            __threadfence();
            *r = (tile == 0 ? SL_INC : SL_AGG) | tot;
        }
        uint64_t ex = 0;
        int64_t j = static_cast<int64_t>(tile) - 1;
        while (j >= 0) {
            const int64_t idx = j - lane;
            uint64_t f = SL_INC;  // before tile 0: an inclusive zero
            if (idx >= 0) {
                do {
                    f = *reinterpret_cast<volatile uint64_t*>(rec + idx);
                } while ((f >> 62) == 0);
            }
            const uint32_t incl = __ballot_sync(0xffffffffu, (f >> 62) == 2);
            const int stop = incl ? __ffs(incl) - 1 : 31;
            uint64_t val = (lane <= static_cast<uint32_t>(stop) && idx >= 0) ? (f & SL_VAL) : 0ull;
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) val += __shfl_xor_sync(0xffffffffu, val, o);
            ex += val;
            if (incl) break;
            j -= 32;
        }
        if (lane == 0) {
            if (tile != 0) {
                __threadfence();
                *reinterpret_cast<volatile uint64_t*>(rec + tile) = SL_INC | (ex + tot);
            }
            s_excl = ex;
            if (static_cast<uint64_t>(tile + 1) * SL_TILE >= n) {  // the last tile
                if (total) *total = ex + tot;
                if (total_slot) out[n] = static_cast<Out>(ex + tot);
            }
        }
    }
    __syncthreads();
    uint64_t run = s_excl + wpre + inc - sum;
#pragma unroll
    for (int j = 0; j < SL_ITEMS; ++j) {
        if (b + j < n) out[b + j] = static_cast<Out>(run);
        run += v[j];
    }
}

// one single-pass scan launch (records + ticket cleared first)
template <class Load, typename Out>
inline int scan_excl(cdx_ctx* ctx, Load ld, uint64_t n, Out* out, bool total_slot, uint64_t* rec, uint64_t* total) {
    const uint64_t tiles = (n + SL_TILE - 1) / SL_TILE;
    if (n == 0) {
        if (total) cudaMemsetAsync(total, 0, 8, ctx->stream);
        if (total_slot) cudaMemsetAsync(out, 0, sizeof(Out), ctx->stream);
        return CDX_OK;
    }
    uint32_t* ticket = reinterpret_cast<uint32_t*>(rec + tiles);
    static thread_local int cap = -1, cap_dev = -1;
    if (cap_dev != ctx->device) {
        int per_sm = 0, attr = 0;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, scan_lb<Load, Out>, SL_THREADS, 0);
        cudaDeviceGetAttribute(&attr, cudaDevAttrCooperativeLaunch, ctx->device);
        cap = attr ? per_sm * ctx->sm_count : 0;
        cap_dev = ctx->device;
    }
    int coop = tiles > 1 && static_cast<int64_t>(tiles) <= cap;
    if (coop) {
        void* args[] = {&ld, &n, &out, &total_slot, &rec, &ticket, &total, &coop};
        const cudaError_t e = cudaLaunchCooperativeKernel(reinterpret_cast<const void*>(scan_lb<Load, Out>),
                                                          dim3(static_cast<unsigned>(tiles)), dim3(SL_THREADS), args, 0,
                                                          ctx->stream);
        if (e != cudaSuccess) {  // e.g. fewer SMs than queried (MPS limits): the look-back form below
            (void)cudaGetLastError();
            coop = 0;
        }
    }
    if (!coop) {
        cudaMemsetAsync(rec, 0, tiles * 8 + 8, ctx->stream);
        scan_lb<Load, Out><<<static_cast<unsigned>(tiles), SL_THREADS, 0, ctx->stream>>>(ld, n, out, total_slot, rec,
                                                                                          ticket, total, 0);
    }
    CDX_CHECK_LAUNCH(ctx, "jsonl(scan)");
    return CDX_OK;
}


}  // namespace scan
}  // namespace cdx
