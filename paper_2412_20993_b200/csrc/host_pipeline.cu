// host_pipeline.cu — end-to-end entries from HOST buffers (the reference-facing calls a serving
// loop makes with traces that live in host memory):
//
//   cdx_sc_decide_host      K2 sc_certaindex + K5 allocate_scan   (configs A, C)
//   cdx_cot_decide_host     K3 cot_exit                           (config B)
//   cdx_reward_decide_host  K4 reward_certaindex + K5             (config D)
//
// All three share one pipeline: the inputs stream through the device in chunks of whole
// requests / programs on a copy stream, double buffered against the kernels on the compute
// stream; results come back with one D2H per output per chunk; token-budget offsets are made
// global across chunks on the device.  Each call returns when every result is in the
// caller's host buffers (pinned buffers give full PCIe bandwidth; pageable ones work too).
#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "cdx_internal.cuh"

namespace cdx {
namespace {

__global__ void add_base(int64_t* __restrict__ off, uint64_t n, const int64_t* __restrict__ base) {
    const int64_t b = *base;
    for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<uint64_t>(gridDim.x) * blockDim.x)
        off[i] += b;
}
// scal = {n_kept, tokens_saved, total_budget}; acc = {running base, saved sum}
__global__ void accumulate(const int64_t* __restrict__ scal, int64_t* __restrict__ acc) {
    acc[0] += scal[2];
    acc[1] += scal[1];
}

// one host array streamed per chunk: `unit` bytes per request / program
struct Stream {
    const void* in;  // host input (nullptr: an output)
    void* out;       // host output
    uint64_t unit;
};

// Chunked, double-buffered host pipeline.  `arrays` lists every host input and output with
// its bytes per unit; `scratch_unit` is per-unit device scratch the kernels may use (not
// copied).  compute(r0, nr, dev, scratch, acc) enqueues the kernels of one chunk on
// ctx->stream (the compute stream) reading dev[k] for inputs and writing dev[k] for outputs;
// acc is 16 bytes of device state carried across chunks (zeroed once).
template <class F>
int pipeline(cdx_ctx* ctx, const char* name, uint64_t n, const std::vector<Stream>& arrays, uint64_t scratch_unit,
             int64_t* acc_out, F compute) {
    uint64_t in_unit = 0;
    for (const auto& a : arrays) in_unit += a.in ? a.unit : 0;
    // ~256 MB of inputs per chunk (CDX_PIPE_CHUNK_KB overrides: tests of the chunk seams)
    uint64_t chunk_bytes = 256ull << 20;
    if (const char* e = getenv("CDX_PIPE_CHUNK_KB")) chunk_bytes = std::max<uint64_t>(1, strtoull(e, nullptr, 10)) << 10;
    uint64_t chunk = std::max<uint64_t>(1, chunk_bytes / std::max<uint64_t>(1, in_unit));
    chunk = std::min<uint64_t>(chunk, n);
    auto al = [](uint64_t b) { return (b + 255) / 256 * 256; };
    uint64_t per = al(chunk * scratch_unit) + 256;
    for (const auto& a : arrays) per += al(chunk * a.unit);
    const uint64_t need = 2 * per + 256;
    if (ctx->pipe_bytes < need) {
        if (ctx->pipe_buf) {
            cudaStreamSynchronize(ctx->stream);
            cudaFree(ctx->pipe_buf);
        }
        ctx->pipe_buf = nullptr;
        ctx->pipe_bytes = 0;
        if (cudaMalloc(&ctx->pipe_buf, need) != cudaSuccess)
            return set_error(ctx, CDX_ECUDA, std::string(name) + ": pipeline buffer allocation failed");
        ctx->pipe_bytes = need;
    }
    uint8_t* base = static_cast<uint8_t*>(ctx->pipe_buf);
    int64_t* acc = reinterpret_cast<int64_t*>(base + 2 * per);
    std::vector<void*> dev[2];
    void* scr[2];
    for (int i = 0; i < 2; ++i) {
        uint8_t* q = base + i * per;
        for (const auto& a : arrays) {
            dev[i].push_back(q);
            q += al(chunk * a.unit);
        }
        scr[i] = q;
    }
    cudaStream_t user = ctx->stream;
    cudaStream_t comp = ctx->own_stream, copy = ctx->copy_stream;
    cudaEvent_t loaded[2], consumed[2];
    for (int i = 0; i < 2; ++i) {
        cudaEventCreateWithFlags(&loaded[i], cudaEventDisableTiming);
        cudaEventCreateWithFlags(&consumed[i], cudaEventDisableTiming);
    }
    cudaMemsetAsync(acc, 0, 16, comp);
    int st = CDX_OK;
    ctx->stream = comp;
    const uint64_t nchunks = (n + chunk - 1) / chunk;
    auto upload = [&](uint64_t c) {
        const uint64_t r0 = c * chunk, nr = std::min(chunk, n - r0);
        cudaStreamWaitEvent(copy, consumed[c & 1], 0);
        for (size_t k = 0; k < arrays.size(); ++k)
            if (arrays[k].in)
                cudaMemcpyAsync(dev[c & 1][k], static_cast<const uint8_t*>(arrays[k].in) + r0 * arrays[k].unit,
                                nr * arrays[k].unit, cudaMemcpyHostToDevice, copy);
        cudaEventRecord(loaded[c & 1], copy);
    };
    for (int i = 0; i < 2; ++i) cudaEventRecord(consumed[i], comp);
    upload(0);
    for (uint64_t c = 0; c < nchunks && st == CDX_OK; ++c) {
        if (c + 1 < nchunks) upload(c + 1);
        const uint64_t r0 = c * chunk, nr = std::min(chunk, n - r0);
        cudaStreamWaitEvent(comp, loaded[c & 1], 0);
        st = compute(r0, nr, dev[c & 1], scr[c & 1], acc);
        if (st) break;
        cudaEventRecord(consumed[c & 1], comp);
        for (size_t k = 0; k < arrays.size(); ++k)
            if (arrays[k].out)
                cudaMemcpyAsync(static_cast<uint8_t*>(arrays[k].out) + r0 * arrays[k].unit, dev[c & 1][k],
                                nr * arrays[k].unit, cudaMemcpyDeviceToHost, comp);
    }
    int64_t hacc[2] = {0, 0};
    if (st == CDX_OK) {
        cudaMemcpyAsync(hacc, acc, 16, cudaMemcpyDeviceToHost, comp);
        cudaError_t e = cudaStreamSynchronize(comp);
        if (e != cudaSuccess) st = cuda_fail(ctx, e, name);
    } else {
        cudaStreamSynchronize(comp);
    }
    cudaStreamSynchronize(copy);
    for (int i = 0; i < 2; ++i) {
        cudaEventDestroy(loaded[i]);
        cudaEventDestroy(consumed[i]);
    }
    ctx->stream = user;
    if (st == CDX_OK && acc_out) {
        acc_out[0] = hacc[0];
        acc_out[1] = hacc[1];
    }
    if (st == CDX_OK) st = cdx_sync(ctx);  // device-side validation errors of the whole call
    return st;
}

// K5 on a chunk's meets bits, offsets made global with the running base in acc[0]
int allocate_chunk(cdx_ctx* ctx, const char* name, const uint32_t* meets, uint64_t nr, uint32_t P,
                   const cdx_alloc_policy* pol, uint64_t r0, int32_t* exit, uint8_t* reason, int64_t* off,
                   uint8_t* scr, int64_t* acc) {
    int32_t* granted = reinterpret_cast<int32_t*>(scr);
    uint32_t* kept = reinterpret_cast<uint32_t*>(scr + (nr * 4 + 255) / 256 * 256);
    int64_t* scal = reinterpret_cast<int64_t*>(scr + 2 * ((nr * 4 + 255) / 256 * 256));
    if (int st = cdx_allocate_scan(ctx, meets, nr, P, pol, 0, static_cast<uint32_t>(r0), exit, reason, granted, off,
                                   kept, reinterpret_cast<uint64_t*>(scal), scal + 1, scal + 2))
        return st;
    add_base<<<static_cast<unsigned>(std::min<uint64_t>((nr + 255) / 256, 1184)), 256, 0, ctx->stream>>>(off, nr, acc);
    CDX_CHECK_LAUNCH(ctx, name);
    accumulate<<<1, 1, 0, ctx->stream>>>(scal, acc);
    CDX_CHECK_LAUNCH(ctx, name);
    return CDX_OK;
}
constexpr uint64_t ALLOC_SCRATCH_UNIT = 8 + 64;  // granted + kept per unit (+ alignment slack)

}  // namespace
}  // namespace cdx

extern "C" int cdx_sc_decide_host(cdx_ctx* ctx, const uint32_t* ids_host, uint64_t R, uint32_t P, uint32_t S,
                                  const cdx_threshold* th, uint32_t n_th, const cdx_alloc_policy* pol,
                                  int32_t* exit_knob_host, uint8_t* reason_host, int64_t* offsets_host,
                                  float* hcert_host, int64_t* tokens_saved_host) {
    using namespace cdx;
    CDX_NVTX("cdx_sc_decide_host");
    if (!ctx) return CDX_EINVAL;
    if (!ids_host || !pol || !exit_knob_host || !reason_host || !offsets_host)
        return set_error(ctx, CDX_EINVAL, "sc_decide_host: null pointer");
    if (P == 0 || S == 0) return set_error(ctx, CDX_EINVAL, "sc_decide_host: empty shape");
    if (R == 0) {
        if (tokens_saved_host) *tokens_saved_host = 0;
        return CDX_OK;
    }
    const uint32_t words = (P + 31) / 32;
    // arrays: ids in | meets (device only) | exit | reason | offsets | hcert
    std::vector<Stream> arr = {{ids_host, nullptr, static_cast<uint64_t>(P) * S * 4},
                               {nullptr, nullptr, static_cast<uint64_t>(words) * 4},
                               {nullptr, exit_knob_host, 4},
                               {nullptr, reason_host, 1},
                               {nullptr, offsets_host, 8},
                               {nullptr, hcert_host, hcert_host ? static_cast<uint64_t>(P) * 4 : 0}};
    int64_t acc[2];
    const int st = pipeline(ctx, "sc_decide_host", R, arr, ALLOC_SCRATCH_UNIT, acc,
                            [&](uint64_t r0, uint64_t nr, std::vector<void*>& d, void* scr, int64_t* dacc) {
                                auto* meets = static_cast<uint32_t*>(d[1]);
                                if (int s = cdx_sc_certaindex(ctx, static_cast<const uint32_t*>(d[0]), nr, P, S, th, n_th,
                                                              hcert_host ? static_cast<float*>(d[5]) : nullptr, meets))
                                    return s;
                                return allocate_chunk(ctx, "sc_decide_host", meets, nr, P, pol, r0,
                                                      static_cast<int32_t*>(d[2]), static_cast<uint8_t*>(d[3]),
                                                      static_cast<int64_t*>(d[4]), static_cast<uint8_t*>(scr), dacc);
                            });
    if (st == CDX_OK && tokens_saved_host) *tokens_saved_host = acc[1];
    return st;
}

extern "C" int cdx_cot_decide_host(cdx_ctx* ctx, const uint32_t* ids_host, const uint64_t* hes_host,
                                   const int64_t* offsets_host, uint64_t R, uint32_t P, const cdx_probe_cfg* cfg,
                                   int32_t* exit_step_host, uint8_t* reason_host, uint32_t* final_id_host,
                                   uint8_t* low_conf_host) {
    using namespace cdx;
    CDX_NVTX("cdx_cot_decide_host");
    if (!ctx) return CDX_EINVAL;
    if (!ids_host || !hes_host || !cfg || !exit_step_host || !reason_host)
        return set_error(ctx, CDX_EINVAL, "cot_decide_host: null pointer");
    if (P == 0) return set_error(ctx, CDX_EINVAL, "final_answer: empty trace");
    if (R == 0) return CDX_OK;
    const uint32_t hw = (P + 63) / 64;
    // arrays: ids | hes | offsets | exit | reason | final | low
    std::vector<Stream> arr = {{ids_host, nullptr, static_cast<uint64_t>(P) * 4},
                               {hes_host, nullptr, static_cast<uint64_t>(hw) * 8},
                               {offsets_host, nullptr, offsets_host ? static_cast<uint64_t>(P) * 8 : 0},
                               {nullptr, exit_step_host, 4},
                               {nullptr, reason_host, 1},
                               {nullptr, final_id_host, final_id_host ? 4u : 0u},
                               {nullptr, low_conf_host, low_conf_host ? 1u : 0u}};
    return pipeline(ctx, "cot_decide_host", R, arr, 0, nullptr,
                    [&](uint64_t, uint64_t nr, std::vector<void*>& d, void*, int64_t*) {
                        return cdx_cot_exit(ctx, static_cast<const uint32_t*>(d[0]), static_cast<const uint64_t*>(d[1]),
                                            offsets_host ? static_cast<const int64_t*>(d[2]) : nullptr, nr, P, cfg,
                                            static_cast<int32_t*>(d[3]), static_cast<uint8_t*>(d[4]),
                                            final_id_host ? static_cast<uint32_t*>(d[5]) : nullptr,
                                            low_conf_host ? static_cast<uint8_t*>(d[6]) : nullptr, nullptr);
                    });
}

extern "C" int cdx_reward_decide_host(cdx_ctx* ctx, const float* rewards_host, const uint32_t* ids_host,
                                      const uint8_t* agg_host, uint64_t G, uint32_t T, uint32_t W,
                                      const cdx_threshold* th_mean, uint32_t n_th_mean, const cdx_threshold* th_max,
                                      uint32_t n_th_max, const cdx_alloc_policy* pol, int32_t* exit_knob_host,
                                      uint8_t* reason_host, int64_t* offsets_host, float* R_host,
                                      int64_t* tokens_saved_host) {
    using namespace cdx;
    CDX_NVTX("cdx_reward_decide_host");
    if (!ctx) return CDX_EINVAL;
    if (!rewards_host || !agg_host || !pol || !exit_knob_host || !reason_host || !offsets_host)
        return set_error(ctx, CDX_EINVAL, "reward_decide_host: null pointer");
    if (T == 0 || W == 0) return set_error(ctx, CDX_EINVAL, "certaindex_reward: empty reward set");
    if (G == 0) {
        if (tokens_saved_host) *tokens_saved_host = 0;
        return CDX_OK;
    }
    const uint64_t node = static_cast<uint64_t>(T) * W;
    const uint32_t words = (T + 31) / 32;
    // arrays: rewards | ids | agg | meets (device) | exit | reason | offsets | R
    std::vector<Stream> arr = {{rewards_host, nullptr, node * 4},
                               {ids_host, nullptr, ids_host ? node * 4 : 0},
                               {agg_host, nullptr, 1},
                               {nullptr, nullptr, static_cast<uint64_t>(words) * 4},
                               {nullptr, exit_knob_host, 4},
                               {nullptr, reason_host, 1},
                               {nullptr, offsets_host, 8},
                               {nullptr, R_host, R_host ? static_cast<uint64_t>(T) * 4 : 0}};
    int64_t acc[2];
    const int st = pipeline(ctx, "reward_decide_host", G, arr, ALLOC_SCRATCH_UNIT, acc,
                            [&](uint64_t r0, uint64_t nr, std::vector<void*>& d, void* scr, int64_t* dacc) {
                                auto* meets = static_cast<uint32_t*>(d[3]);
                                if (int s = cdx_reward_certaindex(
                                        ctx, static_cast<const float*>(d[0]),
                                        ids_host ? static_cast<const uint32_t*>(d[1]) : nullptr,
                                        static_cast<const uint8_t*>(d[2]), nr, T, W, th_mean, n_th_mean, th_max,
                                        n_th_max, R_host ? static_cast<float*>(d[7]) : nullptr, nullptr, meets))
                                    return s;
                                return allocate_chunk(ctx, "reward_decide_host", meets, nr, T, pol, r0,
                                                      static_cast<int32_t*>(d[4]), static_cast<uint8_t*>(d[5]),
                                                      static_cast<int64_t*>(d[6]), static_cast<uint8_t*>(scr), dacc);
                            });
    if (st == CDX_OK && tokens_saved_host) *tokens_saved_host = acc[1];
    return st;
}
