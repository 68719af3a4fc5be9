// shard.cu — the multi-GPU exchange steps behind the C-ABI.
//
// Requests and programs are independent units: each rank owns a contiguous slice and scores
// it with the single-GPU kernels, no data-path exchange.  Two results are global and need an
// exchange step, run here through the context's communicator:
//
//   * K5 global token offsets (cdx_allocate_scan_sharded): the local scan, then ONE allgather
//     of 32 bytes per rank {requests, budget total, kept, tokens saved}, then one kernel adds
//     the rank's base to its offsets and kept indices and writes the global sums.  Nothing
//     syncs with the host: the allgather is stream-ordered.
//   * K6 global gang order (cdx_gang_priority_sharded): a distributed sample sort.  Every rank
//     sorts its own composite keys (K6), allgathers 256 regular samples of its run (+ its
//     count), derives the same world-1 splitters on the host (count-weighted quantiles of the
//     samples), finds its bucket bounds by binary search, and sends each bucket's keys to the
//     rank that owns it (alltoallv).  A rank then merges the world sorted runs it received
//     (merge-path ranks: one binary search per other run, no global synchronisation) and the
//     buckets' program ids are allgathered in bucket order.  Per rank that moves the keys once
//     ((world-1)/world x 24 B per local program) plus 4 B per program of the global order,
//     instead of every rank gathering and merging every key.  The composite key (priority
//     word, arrival bits, program id) is a total order, so the result equals the 1-GPU sort.
//
// Transports: an NCCL communicator the context creates and owns (libnccl.so.2 loaded at run
// time: ncclAllGather and grouped ncclSend/ncclRecv over NVLink / NVSwitch), or the caller's
// callbacks (tests/cpp/shard_world2.cpp stages through host memory between two threads).
#include <dlfcn.h>
#include <nccl.h>  // types only; the symbols are resolved with dlsym

#include <algorithm>
#include <cstring>
#include <mutex>
#include <vector>

#include "cdx_internal.cuh"

namespace cdx {
namespace {

constexpr uint32_t SHARD_SAMPLES = 256;

struct NcclApi {
    bool ok = false;
    ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
    ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
    ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*GroupStart)() = nullptr;
    ncclResult_t (*GroupEnd)() = nullptr;
    const char* (*GetErrorString)(ncclResult_t) = nullptr;
};

// libnccl.so.2 by soname: the copy already loaded in the process (torch's) when there is one
const NcclApi& nccl_api() {
    static NcclApi api;
    static std::once_flag once;
    std::call_once(once, [] {
        void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
        if (!h) return;
        auto sym = [&](auto& f, const char* name) {
            f = reinterpret_cast<std::remove_reference_t<decltype(f)>>(dlsym(h, name));
            return f != nullptr;
        };
        api.ok = sym(api.GetUniqueId, "ncclGetUniqueId") && sym(api.CommInitRank, "ncclCommInitRank") &&
                 sym(api.CommDestroy, "ncclCommDestroy") && sym(api.AllGather, "ncclAllGather") &&
                 sym(api.Send, "ncclSend") && sym(api.Recv, "ncclRecv") && sym(api.GroupStart, "ncclGroupStart") &&
                 sym(api.GroupEnd, "ncclGroupEnd") && sym(api.GetErrorString, "ncclGetErrorString");
    });
    return api;
}

int nccl_fail(cdx_ctx* ctx, ncclResult_t r, const char* what) {
    const auto& api = nccl_api();
    return set_error(ctx, CDX_ENCCL, std::string(what) + ": " + (api.ok ? api.GetErrorString(r) : "nccl unavailable"));
}

int do_allgather(cdx_ctx* ctx, const void* send, void* recv, uint64_t bytes) {
    if (bytes == 0) return CDX_OK;
    if (ctx->nccl) {
        const ncclResult_t r = nccl_api().AllGather(send, recv, bytes, ncclUint8, static_cast<ncclComm_t>(ctx->nccl),
                                                    ctx->stream);
        return r == ncclSuccess ? CDX_OK : nccl_fail(ctx, r, "allgather");
    }
    if (ctx->comm.allgather) {
        if (ctx->comm.allgather(ctx->comm.user, send, recv, bytes, ctx->stream) != 0)
            return set_error(ctx, CDX_ENCCL, "allgather: communicator callback failed");
        return CDX_OK;
    }
    // world 1 without a communicator: the gather is a copy
    const cudaError_t e = cudaMemcpyAsync(recv, send, bytes, cudaMemcpyDeviceToDevice, ctx->stream);
    return e == cudaSuccess ? CDX_OK : cuda_fail(ctx, e, "allgather");
}

int do_alltoallv(cdx_ctx* ctx, const void* send, const uint64_t* sb, const uint64_t* so, void* recv,
                 const uint64_t* rb, const uint64_t* ro) {
    const uint32_t W = ctx->world;
    if (ctx->nccl) {
        const auto& api = nccl_api();
        auto* comm = static_cast<ncclComm_t>(ctx->nccl);
        ncclResult_t r = api.GroupStart();
        for (uint32_t q = 0; q < W && r == ncclSuccess; ++q) {
            if (sb[q]) r = api.Send(static_cast<const char*>(send) + so[q], sb[q], ncclUint8, static_cast<int>(q), comm,
                                    ctx->stream);
            if (r == ncclSuccess && rb[q])
                r = api.Recv(static_cast<char*>(recv) + ro[q], rb[q], ncclUint8, static_cast<int>(q), comm, ctx->stream);
        }
        const ncclResult_t r2 = api.GroupEnd();
        if (r != ncclSuccess) return nccl_fail(ctx, r, "alltoallv");
        return r2 == ncclSuccess ? CDX_OK : nccl_fail(ctx, r2, "alltoallv");
    }
    if (ctx->comm.alltoallv) {
        if (ctx->comm.alltoallv(ctx->comm.user, send, sb, so, recv, rb, ro, ctx->stream) != 0)
            return set_error(ctx, CDX_ENCCL, "alltoallv: communicator callback failed");
        return CDX_OK;
    }
    if (rb[0] == 0) return CDX_OK;
    const cudaError_t e = cudaMemcpyAsync(static_cast<char*>(recv) + ro[0], static_cast<const char*>(send) + so[0],
                                          rb[0], cudaMemcpyDeviceToDevice, ctx->stream);
    return e == cudaSuccess ? CDX_OK : cuda_fail(ctx, e, "alltoallv");
}

__device__ __forceinline__ bool key_lt(const uint64_t* k, uint64_t i, uint64_t a0, uint64_t a1, uint64_t a2) {
    const uint64_t b0 = k[3 * i], b1 = k[3 * i + 1], b2 = k[3 * i + 2];
    if (b0 != a0) return b0 < a0;
    if (b1 != a1) return b1 < a1;
    return b2 < a2;
}

// first index of the sorted run keys[lo, hi) whose key is >= (a0, a1, a2)
__device__ __forceinline__ uint64_t lower_bound3(const uint64_t* k, uint64_t lo, uint64_t hi, uint64_t a0, uint64_t a1,
                                                 uint64_t a2) {
    while (lo < hi) {
        const uint64_t mid = (lo + hi) >> 1;
        if (key_lt(k, mid, a0, a1, a2)) lo = mid + 1;
        else hi = mid;
    }
    return lo;
}

// s samples at the midpoints of s equal ranges of the run (+ the run length after them)
__global__ void samples_kernel(const uint64_t* __restrict__ keys, uint64_t n, uint32_t s, uint64_t* __restrict__ out) {
    for (uint32_t j = blockIdx.x * blockDim.x + threadIdx.x; j < s; j += gridDim.x * blockDim.x) {
        if (n == 0) {
            out[3 * j] = out[3 * j + 1] = out[3 * j + 2] = ~0ull;
        } else {
            const uint64_t i = ((2ull * j + 1ull) * n) / (2ull * s);
            out[3 * j] = keys[3 * i];
            out[3 * j + 1] = keys[3 * i + 1];
            out[3 * j + 2] = keys[3 * i + 2];
        }
    }
}

__global__ void bounds_kernel(const uint64_t* __restrict__ keys, uint64_t n, const uint64_t* __restrict__ split,
                              uint32_t world, uint64_t* __restrict__ bounds) {
    const uint32_t b = blockIdx.x * blockDim.x + threadIdx.x;
    if (b > world) return;
    if (b == 0) bounds[0] = 0;
    else if (b == world) bounds[world] = n;
    else bounds[b] = lower_bound3(keys, 0, n, split[3 * (b - 1)], split[3 * (b - 1) + 1], split[3 * (b - 1) + 2]);
}

// element i of run q lands at (i - run_off[q]) + sum over other runs of their keys < it
__global__ void merge_runs_kernel(const uint64_t* __restrict__ keys, const uint64_t* __restrict__ run_off, uint32_t runs,
                                  uint32_t* __restrict__ out) {
    const uint64_t total = run_off[runs];
    for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < total;
         i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
        uint32_t r = 0;
        while (i >= run_off[r + 1]) ++r;
        const uint64_t a0 = keys[3 * i], a1 = keys[3 * i + 1], a2 = keys[3 * i + 2];
        uint64_t pos = i - run_off[r];
        for (uint32_t q = 0; q < runs; ++q)
            if (q != r) pos += lower_bound3(keys, run_off[q], run_off[q + 1], a0, a1, a2) - run_off[q];
        out[pos] = static_cast<uint32_t>(a2);
    }
}

__global__ void shard_pack_kernel(uint64_t* pk, uint64_t R) { pk[0] = R; }

// all = u64[world][4] {requests, budget total, kept, tokens saved}: rebase this rank's
// offsets and kept indices, write the global sums
__global__ void shard_finish_kernel(const uint64_t* __restrict__ all, uint32_t rank, uint32_t world, uint64_t R,
                                    int64_t* __restrict__ offsets, uint32_t* __restrict__ kept,
                                    uint64_t* __restrict__ n_kept, int64_t* __restrict__ tokens_saved,
                                    int64_t* __restrict__ total_budget, uint64_t* __restrict__ shard_info) {
    uint64_t base_req = 0, base_off = 0, saved = 0, budget = 0;
    for (uint32_t q = 0; q < world; ++q) {
        if (q < rank) {
            base_req += all[4 * q];
            base_off += all[4 * q + 1];
        }
        budget += all[4 * q + 1];
        saved += all[4 * q + 3];
    }
    const uint64_t nk = all[4 * rank + 2];
    const uint64_t tid = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
    const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
    if (offsets && base_off)
        for (uint64_t i = tid; i < R; i += stride) offsets[i] += static_cast<int64_t>(base_off);
    if (kept && base_req)
        for (uint64_t i = tid; i < nk; i += stride) kept[i] += static_cast<uint32_t>(base_req);
    if (tid == 0) {
        if (n_kept) *n_kept = nk;
        if (tokens_saved) *tokens_saved = static_cast<int64_t>(saved);
        if (total_budget) *total_budget = static_cast<int64_t>(budget);
    }
    if (shard_info)
        for (uint64_t i = tid; i < 4ull * world; i += stride) shard_info[i] = all[i];
}

unsigned grid_for(cdx_ctx* ctx, uint64_t n, unsigned t = 256) {
    return static_cast<unsigned>(std::max<uint64_t>(1, std::min<uint64_t>((n + t - 1) / t, ctx->sm_count * 8ull)));
}

// pinned host staging of `words` u64 (grown on demand)
uint64_t* host_stage(cdx_ctx* ctx, size_t words) {
    const size_t want = words * 8;
    if (ctx->sh_host && ctx->sh_host[-1] >= want) return ctx->sh_host;
    if (ctx->sh_host) {
        cudaStreamSynchronize(ctx->stream);
        cudaFreeHost(ctx->sh_host - 1);
        ctx->sh_host = nullptr;
    }
    uint64_t* p = nullptr;
    const size_t cap = std::max<size_t>(want, 1 << 16);
    if (cudaMallocHost(&p, cap + 8) != cudaSuccess) return nullptr;
    p[0] = cap;
    ctx->sh_host = p + 1;
    return ctx->sh_host;
}

}  // namespace

void comm_destroy(cdx_ctx* ctx) {
    if (ctx->nccl) {
        nccl_api().CommDestroy(static_cast<ncclComm_t>(ctx->nccl));
        ctx->nccl = nullptr;
    }
    if (ctx->sh_host) {
        cudaFreeHost(ctx->sh_host - 1);
        ctx->sh_host = nullptr;
    }
}

}  // namespace cdx

extern "C" {

int cdx_nccl_unique_id(uint8_t id[128]) {
    using namespace cdx;
    if (!id) return CDX_EINVAL;
    const auto& api = nccl_api();
    if (!api.ok) return CDX_ENCCL;
    ncclUniqueId u;
    if (api.GetUniqueId(&u) != ncclSuccess) return CDX_ENCCL;
    static_assert(sizeof(u) == 128, "ncclUniqueId is 128 bytes");
    std::memcpy(id, &u, 128);
    return CDX_OK;
}

int cdx_ctx_create_comm(int device, const cdx_comm* comm, cdx_ctx** out) {
    using namespace cdx;
    if (comm && (comm->world < 1 || comm->rank >= comm->world)) return CDX_EINVAL;
    if (comm && !comm->nccl_id && comm->world > 1 && (!comm->allgather || !comm->alltoallv)) return CDX_EINVAL;
    if (int st = cdx_ctx_create(device, out)) return st;
    cdx_ctx* c = *out;
    if (!comm) return CDX_OK;
    c->rank = comm->rank;
    c->world = comm->world;
    c->comm = *comm;
    c->comm.nccl_id = nullptr;
    if (comm->nccl_id) {
        c->comm.allgather = nullptr;
        c->comm.alltoallv = nullptr;
        const auto& api = nccl_api();
        if (!api.ok) {
            cdx_ctx_destroy(c);
            *out = nullptr;
            return CDX_ENCCL;
        }
        ncclUniqueId u;
        std::memcpy(&u, comm->nccl_id, sizeof(u));
        ncclComm_t nc = nullptr;
        cudaSetDevice(device);
        if (api.CommInitRank(&nc, static_cast<int>(comm->world), u, static_cast<int>(comm->rank)) != ncclSuccess) {
            cdx_ctx_destroy(c);
            *out = nullptr;
            return CDX_ENCCL;
        }
        c->nccl = nc;
    }
    return CDX_OK;
}

int cdx_ctx_comm_info(const cdx_ctx* ctx, uint32_t* rank, uint32_t* world) {
    if (!ctx) return CDX_EINVAL;
    if (rank) *rank = ctx->rank;
    if (world) *world = ctx->world;
    return CDX_OK;
}

int cdx_allgather(cdx_ctx* ctx, const void* send, void* recv, uint64_t bytes) {
    using namespace cdx;
    CDX_NVTX("cdx_allgather");
    if (!ctx) return CDX_EINVAL;
    if (bytes && (!send || !recv)) return set_error(ctx, CDX_EINVAL, "allgather: null buffer");
    return do_allgather(ctx, send, recv, bytes);
}

int cdx_allocate_scan_sharded(cdx_ctx* ctx, const uint32_t* meets_bits, uint64_t R, uint32_t P,
                              const cdx_alloc_policy* pol, int32_t* exit_knob, uint8_t* reason, int32_t* granted,
                              int64_t* offsets, uint32_t* kept, uint64_t* n_kept, int64_t* tokens_saved,
                              int64_t* total_budget, uint64_t* shard_info) {
    using namespace cdx;
    CDX_NVTX("cdx_allocate_scan_sharded");
    if (!ctx) return CDX_EINVAL;
    const uint32_t W = ctx->world;
    // [0, 4): this rank's packed totals; [4, 4 + 4W): every rank's
    auto* pk = static_cast<uint64_t*>(grow_buffer(ctx, &ctx->sh_buf2, &ctx->sh_bytes2, (4 + 4ull * W) * 8));
    if (!pk) return set_error(ctx, CDX_ECUDA, "allocate_scan_sharded: scratch");
    uint64_t* all = pk + 4;
    cudaMemsetAsync(pk, 0, 32, ctx->stream);
    if (R > 0) {
        if (int st = cdx_allocate_scan(ctx, meets_bits, R, P, pol, 0, 0, exit_knob, reason, granted, offsets, kept,
                                       pk + 2, reinterpret_cast<int64_t*>(pk + 3), reinterpret_cast<int64_t*>(pk + 1)))
            return st;
    } else if (!pol) {
        return set_error(ctx, CDX_EINVAL, "allocate: null policy");
    }
    shard_pack_kernel<<<1, 1, 0, ctx->stream>>>(pk, R);
    CDX_CHECK_LAUNCH(ctx, "allocate_scan_sharded(pack)");
    if (int st = do_allgather(ctx, pk, all, 32)) return st;
    shard_finish_kernel<<<grid_for(ctx, R), 256, 0, ctx->stream>>>(all, ctx->rank, W, R, offsets, kept, n_kept,
                                                                   tokens_saved, total_budget, shard_info);
    CDX_CHECK_LAUNCH(ctx, "allocate_scan_sharded(finish)");
    return CDX_OK;
}

int cdx_shard_samples(cdx_ctx* ctx, const uint64_t* keys, uint64_t n, uint32_t s, uint64_t* samples) {
    using namespace cdx;
    if (!ctx) return CDX_EINVAL;
    if (s == 0 || !samples || (n && !keys)) return set_error(ctx, CDX_EINVAL, "shard_samples: bad arguments");
    samples_kernel<<<grid_for(ctx, s), 256, 0, ctx->stream>>>(keys, n, s, samples);
    CDX_CHECK_LAUNCH(ctx, "shard_samples");
    return CDX_OK;
}

int cdx_shard_splitters(const uint64_t* samples, const uint64_t* counts, uint32_t world, uint32_t s,
                        uint64_t* splitters) {
    if (world == 0 || s == 0 || !samples || !counts || (world > 1 && !splitters)) return CDX_EINVAL;
    struct Sample {
        uint64_t k[3];
        uint32_t q;
    };
    std::vector<Sample> v;
    v.reserve(static_cast<size_t>(world) * s);
    unsigned __int128 total = 0;
    for (uint32_t q = 0; q < world; ++q) {
        total += counts[q];
        if (counts[q] == 0) continue;  // sentinel samples of an empty run carry no weight
        for (uint32_t j = 0; j < s; ++j) {
            const uint64_t* p = samples + (static_cast<uint64_t>(q) * s + j) * 3;
            v.push_back(Sample{{p[0], p[1], p[2]}, q});
        }
    }
    std::sort(v.begin(), v.end(), [](const Sample& a, const Sample& b) {
        if (a.k[0] != b.k[0]) return a.k[0] < b.k[0];
        if (a.k[1] != b.k[1]) return a.k[1] < b.k[1];
        if (a.k[2] != b.k[2]) return a.k[2] < b.k[2];
        return a.q < b.q;
    });
    // weights in units of 1/s keys: sample of run q weighs counts[q]; target b = b*total*s/world
    unsigned __int128 cum = 0;
    uint32_t b = 1;
    for (const Sample& x : v) {
        while (b < world && cum * world >= static_cast<unsigned __int128>(b) * total * s) {
            std::memcpy(splitters + 3 * (b - 1), x.k, 24);
            ++b;
        }
        cum += counts[x.q];
    }
    for (; b < world; ++b) std::memset(splitters + 3 * (b - 1), 0xff, 24);  // trailing buckets empty
    return CDX_OK;
}

int cdx_shard_bounds(cdx_ctx* ctx, const uint64_t* keys, uint64_t n, const uint64_t* splitters, uint32_t world,
                     uint64_t* bounds) {
    using namespace cdx;
    if (!ctx) return CDX_EINVAL;
    if (world == 0 || !bounds || (world > 1 && !splitters) || (n && !keys))
        return set_error(ctx, CDX_EINVAL, "shard_bounds: bad arguments");
    bounds_kernel<<<(world + 1 + 127) / 128, 128, 0, ctx->stream>>>(keys, n, splitters, world, bounds);
    CDX_CHECK_LAUNCH(ctx, "shard_bounds");
    return CDX_OK;
}

int cdx_gang_merge_runs(cdx_ctx* ctx, const uint64_t* keys, const uint64_t* run_off, uint32_t runs,
                        uint32_t* order_out) {
    using namespace cdx;
    CDX_NVTX("cdx_gang_merge_runs");
    if (!ctx) return CDX_EINVAL;
    if (runs == 0 || !run_off || !order_out) return set_error(ctx, CDX_EINVAL, "gang_merge_runs: bad arguments");
    merge_runs_kernel<<<ctx->sm_count * 8, 256, 0, ctx->stream>>>(keys, run_off, runs, order_out);
    CDX_CHECK_LAUNCH(ctx, "gang_merge_runs");
    return CDX_OK;
}

int cdx_gang_priority_sharded(cdx_ctx* ctx, const cdx_prog_soa* progs, uint64_t N, const cdx_inter_policy* pol,
                              double now, uint32_t* order, uint64_t* n_out) {
    using namespace cdx;
    CDX_NVTX("cdx_gang_priority_sharded");
    if (!ctx) return CDX_EINVAL;
    if (!order || !n_out) return set_error(ctx, CDX_EINVAL, "gang_priority: null pointer");
    const uint32_t W = ctx->world, me = ctx->rank, s = SHARD_SAMPLES;
    const uint64_t rec = 3 * s + 1;  // samples + the run length, per rank
    // device layout (sh_buf): local keys u64[N][3] | local order u32[N] | samples u64[rec] |
    // gathered samples u64[W][rec] | splitters u64[W-1][3] | bounds u64[W+1] | all bounds
    // u64[W][W+1] | run offsets u64[W+1]
    const uint64_t keys_w = 3 * N, ord_w = (N + 1) / 2;
    const uint64_t words = keys_w + ord_w + rec + W * rec + 3ull * W + (W + 1) + W * (W + 1ull) + (W + 1);
    auto* base = static_cast<uint64_t*>(grow_buffer(ctx, &ctx->sh_buf, &ctx->sh_bytes, words * 8 + 64));
    if (!base) return set_error(ctx, CDX_ECUDA, "gang_priority_sharded: scratch");
    uint64_t* keys = base;
    auto* lorder = reinterpret_cast<uint32_t*>(keys + keys_w);
    uint64_t* samp = keys + keys_w + ord_w;
    uint64_t* gsamp = samp + rec;
    uint64_t* split = gsamp + W * rec;
    uint64_t* bnd = split + 3ull * W;
    uint64_t* gbnd = bnd + (W + 1);
    uint64_t* roff = gbnd + W * (W + 1ull);
    uint64_t* h = host_stage(ctx, W * rec + 3ull * W + W * (W + 1ull) + 4ull * (W + 1) + 8);
    if (!h) return set_error(ctx, CDX_ECUDA, "gang_priority_sharded: host staging");
    uint64_t* h_samp = h;                      // [W][rec]
    uint64_t* h_split = h_samp + W * rec;      // [W-1][3]
    uint64_t* h_bnd = h_split + 3ull * W;      // [W][W+1]
    uint64_t* h_roff = h_bnd + W * (W + 1ull); // [W+1]
    uint64_t* h_sb = h_roff + (W + 1);         // send bytes / offsets, recv bytes / offsets
    uint64_t* h_so = h_sb + (W + 1);
    uint64_t* h_rb = h_so + (W + 1);
    uint64_t* h_ro = h_rb + (W + 1);

    // 1. this rank's run: K6 with composite keys (one host round trip for the live count)
    uint64_t n = 0;
    if (N > 0) {
        if (int st = cdx_gang_priority(ctx, progs, N, pol, now, lorder, &n, nullptr, keys)) return st;
    } else if (!pol) {
        return set_error(ctx, CDX_EINVAL, "gang_priority: null pointer");
    }
    // 2. regular samples + run length, allgathered
    if (int st = cdx_shard_samples(ctx, keys, n, s, samp)) return st;
    shard_pack_kernel<<<1, 1, 0, ctx->stream>>>(samp + 3 * s, n);
    CDX_CHECK_LAUNCH(ctx, "gang_priority_sharded(pack)");
    if (int st = do_allgather(ctx, samp, gsamp, rec * 8)) return st;
    cudaMemcpyAsync(h_samp, gsamp, W * rec * 8, cudaMemcpyDeviceToHost, ctx->stream);
    cudaError_t e = cudaStreamSynchronize(ctx->stream);
    if (e != cudaSuccess) return cuda_fail(ctx, e, "gang_priority_sharded: samples");
    // 3. the same splitters on every rank
    std::vector<uint64_t> sm(static_cast<size_t>(W) * 3 * s), cnt(W);
    uint64_t total = 0;
    for (uint32_t q = 0; q < W; ++q) {
        std::memcpy(sm.data() + static_cast<size_t>(q) * 3 * s, h_samp + q * rec, 3 * s * 8);
        cnt[q] = h_samp[q * rec + 3 * s];
        total += cnt[q];
    }
    if (W > 1) {
        cdx_shard_splitters(sm.data(), cnt.data(), W, s, h_split);
        cudaMemcpyAsync(split, h_split, 3ull * (W - 1) * 8, cudaMemcpyHostToDevice, ctx->stream);
    }
    // 4. bucket bounds of this run, allgathered: rank b receives bucket b of every run
    if (int st = cdx_shard_bounds(ctx, keys, n, split, W, bnd)) return st;
    if (int st = do_allgather(ctx, bnd, gbnd, (W + 1) * 8)) return st;
    cudaMemcpyAsync(h_bnd, gbnd, W * (W + 1ull) * 8, cudaMemcpyDeviceToHost, ctx->stream);
    e = cudaStreamSynchronize(ctx->stream);
    if (e != cudaSuccess) return cuda_fail(ctx, e, "gang_priority_sharded: bounds");
    const uint64_t* mine = h_bnd + me * (W + 1ull);
    uint64_t recv_n = 0;
    for (uint32_t q = 0; q < W; ++q) {
        h_sb[q] = (mine[q + 1] - mine[q]) * 24;
        h_so[q] = mine[q] * 24;
        const uint64_t* theirs = h_bnd + q * (W + 1ull);
        h_rb[q] = (theirs[me + 1] - theirs[me]) * 24;
        h_ro[q] = recv_n * 24;
        h_roff[q] = recv_n;
        recv_n += theirs[me + 1] - theirs[me];
    }
    h_roff[W] = recv_n;
    // bucket sizes (every rank's merged run) for the final gather
    std::vector<uint64_t> bucket(W, 0);
    for (uint32_t b = 0; b < W; ++b)
        for (uint32_t q = 0; q < W; ++q) bucket[b] += h_bnd[q * (W + 1ull) + b + 1] - h_bnd[q * (W + 1ull) + b];
    // 5. keys to their bucket's rank
    auto* rkeys = static_cast<uint64_t*>(grow_buffer(ctx, &ctx->sh_buf2, &ctx->sh_bytes2, recv_n * 24 + recv_n * 4 + 64));
    if (!rkeys) return set_error(ctx, CDX_ECUDA, "gang_priority_sharded: receive buffer");
    auto* bids = reinterpret_cast<uint32_t*>(rkeys + 3 * recv_n);
    if (int st = do_alltoallv(ctx, keys, h_sb, h_so, rkeys, h_rb, h_ro)) return st;
    // 6. merge the W runs of this bucket
    cudaMemcpyAsync(roff, h_roff, (W + 1) * 8, cudaMemcpyHostToDevice, ctx->stream);
    if (recv_n) {
        if (int st = cdx_gang_merge_runs(ctx, rkeys, roff, W, bids)) return st;
    }
    // 7. program ids of every bucket, in bucket order, to every rank
    uint64_t off = 0;
    for (uint32_t q = 0; q < W; ++q) {
        h_sb[q] = recv_n * 4;
        h_so[q] = 0;
        h_rb[q] = bucket[q] * 4;
        h_ro[q] = off * 4;
        off += bucket[q];
    }
    if (int st = do_alltoallv(ctx, bids, h_sb, h_so, order, h_rb, h_ro)) return st;
    e = cudaStreamSynchronize(ctx->stream);  // the host staging is reused by the next call
    if (e != cudaSuccess) return cuda_fail(ctx, e, "gang_priority_sharded");
    *n_out = total;
    return CDX_OK;
}

}  // extern "C"
