// shard_world2.cpp — the multi-GPU exchange steps through the C-ABI with a caller-supplied
// communicator: `world` ranks as host threads, each with its own context (cdx_ctx_create_comm)
// on device 0, whose allgather / alltoallv callbacks stage through host memory between the
// threads.  The same protocol runs over NCCL when the context owns an NCCL communicator
// (tests/test_gpu_sharding_nccl.py); only one GPU is reachable here, so the multi-rank run
// shares it.
//
//   usage: shard_world2 <dir> <world>
//   <dir>/gang_*.bin: program SoA written by tests/test_gpu_shard_cabi.py (N programs)
//   writes <dir>/rank<q>_{offsets,kept,exit,scalars,info,order}.bin
//
// Per rank q: requests [q*R/W, (q+1)*R/W) of the SC trace (cdx_gen_sc at r0) through K2 +
// cdx_allocate_scan_sharded; programs [q*N/W, (q+1)*N/W) through cdx_gang_priority_sharded.
#include <barrier>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <fstream>
#include <string>
#include <thread>
#include <vector>

#include <cuda_runtime.h>

#include "cdx_c.h"

namespace {

struct Hub {
    explicit Hub(int w) : world(w), bar(w), slot(w), so(w), sb(w) {}
    int world;
    std::barrier<> bar;
    std::vector<std::vector<char>> slot;
    std::vector<std::vector<uint64_t>> so, sb;
};

struct User {
    Hub* hub;
    int rank;
};

int cb_allgather(void* user, const void* send, void* recv, uint64_t bytes, void* stream) {
    auto* u = static_cast<User*>(user);
    Hub& h = *u->hub;
    if (cudaStreamSynchronize(static_cast<cudaStream_t>(stream)) != cudaSuccess) return 1;
    h.slot[u->rank].resize(bytes);
    if (cudaMemcpy(h.slot[u->rank].data(), send, bytes, cudaMemcpyDeviceToHost) != cudaSuccess) return 1;
    h.bar.arrive_and_wait();
    int bad = 0;
    for (int q = 0; q < h.world; ++q)
        bad |= cudaMemcpy(static_cast<char*>(recv) + q * bytes, h.slot[q].data(), bytes, cudaMemcpyHostToDevice) !=
               cudaSuccess;
    h.bar.arrive_and_wait();  // every rank has read the slots before they are reused
    return bad;
}

int cb_alltoallv(void* user, const void* send, const uint64_t* sb, const uint64_t* so, void* recv, const uint64_t* rb,
                 const uint64_t* ro, void* stream) {
    auto* u = static_cast<User*>(user);
    Hub& h = *u->hub;
    const int me = u->rank, W = h.world;
    if (cudaStreamSynchronize(static_cast<cudaStream_t>(stream)) != cudaSuccess) return 1;
    uint64_t end = 0;
    for (int q = 0; q < W; ++q) end = std::max(end, so[q] + sb[q]);
    h.slot[me].resize(end);
    if (end && cudaMemcpy(h.slot[me].data(), send, end, cudaMemcpyDeviceToHost) != cudaSuccess) return 1;
    h.so[me].assign(so, so + W);
    h.sb[me].assign(sb, sb + W);
    h.bar.arrive_and_wait();
    int bad = 0;
    for (int q = 0; q < W; ++q) {
        if (rb[q] != h.sb[q][me]) bad = 1;  // the sizes both sides derived must agree
        else if (rb[q])
            bad |= cudaMemcpy(static_cast<char*>(recv) + ro[q], h.slot[q].data() + h.so[q][me], rb[q],
                              cudaMemcpyHostToDevice) != cudaSuccess;
    }
    h.bar.arrive_and_wait();
    return bad;
}

template <class T>
std::vector<T> load(const std::string& path) {
    std::ifstream f(path, std::ios::binary | std::ios::ate);
    const auto n = static_cast<size_t>(f.tellg());
    std::vector<T> v(n / sizeof(T));
    f.seekg(0);
    f.read(reinterpret_cast<char*>(v.data()), static_cast<std::streamsize>(n));
    return v;
}

template <class T>
void dump(const std::string& path, const T* p, size_t n) {
    std::ofstream f(path, std::ios::binary);
    f.write(reinterpret_cast<const char*>(p), static_cast<std::streamsize>(n * sizeof(T)));
}

template <class T>
T* up(const std::vector<T>& h, size_t lo, size_t n) {
    T* d = nullptr;
    cudaMalloc(&d, std::max<size_t>(n, 1) * sizeof(T));
    if (n) cudaMemcpy(d, h.data() + lo, n * sizeof(T), cudaMemcpyHostToDevice);
    return d;
}

constexpr uint64_t R = 6000;
constexpr uint32_t P = 64, S = 32;

int run_rank(Hub* hub, int rank, const std::string& dir) {
    const int W = hub->world;
    User user{hub, rank};
    cdx_comm comm{};
    comm.rank = static_cast<uint32_t>(rank);
    comm.world = static_cast<uint32_t>(W);
    comm.user = &user;
    comm.allgather = cb_allgather;
    comm.alltoallv = cb_alltoallv;
    cdx_ctx* ctx = nullptr;
    if (cdx_ctx_create_comm(0, &comm, &ctx) != CDX_OK) {
        std::printf("rank %d: cdx_ctx_create_comm failed\n", rank);
        return 1;
    }
    auto fail = [&](int st, const char* what) {
        std::printf("rank %d: %s failed (%d): %s\n", rank, what, st, cdx_last_error(ctx));
        return 1;
    };
    const std::string pre = dir + "/rank" + std::to_string(rank) + "_";
    // ---- SC: K2 + sharded K5
    const uint64_t r0 = R * rank / W, rn = R * (rank + 1) / W - r0;
    cdx_gen_params g{};
    g.seed = 91;
    g.groups = 5;
    g.conv_lo = 1;
    g.conv_hi = 64;
    g.noise_level = 0.5;
    g.solvable_fraction = 0.9;
    uint32_t *ids, *meets, *kept;
    int32_t *ek, *gr;
    uint8_t* why;
    int64_t *off, *sc;
    uint64_t* info;
    cudaMalloc(&ids, std::max<uint64_t>(rn, 1) * P * S * 4);
    cudaMalloc(&meets, std::max<uint64_t>(rn, 1) * 8);
    cudaMalloc(&kept, std::max<uint64_t>(rn, 1) * 4);
    cudaMalloc(&ek, std::max<uint64_t>(rn, 1) * 4);
    cudaMalloc(&gr, std::max<uint64_t>(rn, 1) * 4);
    cudaMalloc(&why, std::max<uint64_t>(rn, 1));
    cudaMalloc(&off, std::max<uint64_t>(rn, 1) * 8);
    cudaMalloc(&sc, 3 * 8);
    cudaMalloc(&info, W * 4 * 8);
    cdx_threshold th{};
    th.signal = CDX_SIG_ENTROPY;
    th.dir = CDX_DIR_GE;
    th.cutoff = 0.7;
    cdx_alloc_policy pol{};
    pol.kind = CDX_POL_STATIC_THRESHOLD;
    pol.detect_at = 5;
    pol.recheck_every = 1;
    pol.resource_cap = 64;
    pol.tokens_per_unit = 64 * S;
    int st = CDX_OK;
    if (rn) {
        if ((st = cdx_gen_sc(ctx, &g, r0, rn, P, S, ids))) return fail(st, "gen_sc");
        if ((st = cdx_sc_certaindex(ctx, ids, rn, P, S, &th, 1, nullptr, meets))) return fail(st, "sc_certaindex");
    }
    if ((st = cdx_allocate_scan_sharded(ctx, meets, rn, P, &pol, ek, why, gr, off, kept,
                                        reinterpret_cast<uint64_t*>(sc), sc + 1, sc + 2, info)))
        return fail(st, "allocate_scan_sharded");
    if ((st = cdx_sync(ctx))) return fail(st, "sync");
    std::vector<int64_t> h_off(rn), h_sc(3);
    std::vector<int32_t> h_ek(rn);
    std::vector<uint64_t> h_info(W * 4);
    cudaMemcpy(h_off.data(), off, rn * 8, cudaMemcpyDeviceToHost);
    cudaMemcpy(h_ek.data(), ek, rn * 4, cudaMemcpyDeviceToHost);
    cudaMemcpy(h_sc.data(), sc, 24, cudaMemcpyDeviceToHost);
    cudaMemcpy(h_info.data(), info, W * 32, cudaMemcpyDeviceToHost);
    std::vector<uint32_t> h_kept(static_cast<size_t>(h_sc[0]));
    cudaMemcpy(h_kept.data(), kept, h_kept.size() * 4, cudaMemcpyDeviceToHost);
    dump(pre + "offsets.bin", h_off.data(), rn);
    dump(pre + "exit.bin", h_ek.data(), rn);
    dump(pre + "scalars.bin", h_sc.data(), 3);
    dump(pre + "info.bin", h_info.data(), h_info.size());
    dump(pre + "kept.bin", h_kept.data(), h_kept.size());
    // ---- gang order: this rank's programs, global ids, the global order back
    const auto arrival = load<double>(dir + "/gang_arrival.bin");
    const auto last = load<double>(dir + "/gang_last_service.bin");
    const auto tok = load<int64_t>(dir + "/gang_iter_tok_sum.bin");
    const auto cnt = load<uint32_t>(dir + "/gang_iter_count.bin");
    const auto knob = load<int32_t>(dir + "/gang_knob.bin");
    const auto cap = load<int32_t>(dir + "/gang_cap.bin");
    const auto term = load<uint8_t>(dir + "/gang_terminated.bin");
    const auto par = load<double>(dir + "/gang_params.bin");  // now, limit, prior, order
    const uint64_t N = arrival.size();
    const uint64_t g0 = N * rank / W, gn = N * (rank + 1) / W - g0;
    cdx_prog_soa soa{};
    soa.arrival = up(arrival, g0, gn);
    soa.last_service = up(last, g0, gn);
    soa.iter_tok_sum = up(tok, g0, gn);
    soa.iter_count = up(cnt, g0, gn);
    soa.knob = up(knob, g0, gn);
    soa.cap = up(cap, g0, gn);
    soa.terminated = up(term, g0, gn);
    soa.id_base = static_cast<uint32_t>(g0);
    cdx_inter_policy ip{};
    ip.gang = 1;
    ip.order = static_cast<uint8_t>(par[3]);
    ip.starvation_limit = par[1];
    ip.prior_tokens = par[2];
    uint32_t* order = nullptr;
    cudaMalloc(&order, std::max<uint64_t>(N, 1) * 4);
    uint64_t n_out = 0;
    for (int rep = 0; rep < 2; ++rep)  // twice: buffers and host staging are reused
        if ((st = cdx_gang_priority_sharded(ctx, &soa, gn, &ip, par[0], order, &n_out)))
            return fail(st, "gang_priority_sharded");
    std::vector<uint32_t> h_order(n_out);
    cudaMemcpy(h_order.data(), order, n_out * 4, cudaMemcpyDeviceToHost);
    dump(pre + "order.bin", h_order.data(), n_out);
    cdx_ctx_destroy(ctx);
    return 0;
}

}  // namespace

int main(int argc, char** argv) {
    if (argc < 3) {
        std::fprintf(stderr, "usage: shard_world2 <dir> <world>\n");
        return 2;
    }
    const std::string dir = argv[1];
    const int W = std::atoi(argv[2]);
    Hub hub(W);
    std::vector<int> rc(W, 0);
    std::vector<std::thread> th;
    for (int q = 0; q < W; ++q) th.emplace_back([&, q] { rc[q] = run_rank(&hub, q, dir); });
    for (auto& t : th) t.join();
    for (int q = 0; q < W; ++q)
        if (rc[q]) return 1;
    std::printf("ok\n");
    return 0;
}
