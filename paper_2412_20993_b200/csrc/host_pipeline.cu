// host_pipeline.cu — end-to-end entry from HOST buffers: cdx_sc_decide_host.
//
// The reference-facing call a serving loop makes with answers that live in host memory:
// ids stream through the device in chunks of whole requests on a copy stream, double
// buffered against K2 (sc_certaindex) + K5 (allocate_scan) on the compute stream; budget
// offsets are made global across chunks on the device; results come back with one D2H per
// chunk.  Returns when every result is in the caller's host buffers.
#include <algorithm>
#include <cstring>

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

}  // namespace
}  // namespace cdx

extern "C" int cdx_sc_decide_host(cdx_ctx* ctx, const uint32_t* ids_host, uint64_t R, uint32_t P, uint32_t S,
                                  const cdx_threshold* th, uint32_t n_th, const cdx_alloc_policy* pol,
                                  int32_t* exit_knob_host, uint8_t* reason_host, int64_t* offsets_host,
                                  float* hcert_host, int64_t* tokens_saved_host) {
    using namespace cdx;
    if (!ctx) return CDX_EINVAL;
    if (!ids_host || !pol || !exit_knob_host || !reason_host || !offsets_host)
        return set_error(ctx, CDX_EINVAL, "sc_decide_host: null pointer");
    if (P == 0 || S == 0) return set_error(ctx, CDX_EINVAL, "sc_decide_host: empty shape");
    if (R == 0) {
        if (tokens_saved_host) *tokens_saved_host = 0;
        return CDX_OK;
    }
    const uint64_t req_bytes = static_cast<uint64_t>(P) * S * 4u;
    uint64_t chunk = std::max<uint64_t>(1, (256ull << 20) / req_bytes);  // ~256 MB of ids per chunk
    chunk = std::min<uint64_t>(chunk, R);
    const uint32_t words = (P + 31) / 32;
    // per buffer: ids | hcert | meets | exit | reason | granted | offsets | kept | scalars
    auto al = [](uint64_t b) { return (b + 255) / 256 * 256; };
    const uint64_t b_ids = al(chunk * req_bytes), b_h = al(chunk * P * 4), b_m = al(chunk * words * 4);
    const uint64_t b_e = al(chunk * 4), b_r = al(chunk), b_g = al(chunk * 4), b_o = al(chunk * 8), b_k = al(chunk * 4);
    const uint64_t per = b_ids + b_h + b_m + b_e + b_r + b_g + b_o + b_k + 256;
    const uint64_t need = 2 * per + 256;
    if (ctx->pipe_bytes < need) {
        if (ctx->pipe_buf) {
            cudaStreamSynchronize(ctx->stream);
            cudaFree(ctx->pipe_buf);
        }
        ctx->pipe_buf = nullptr;
        ctx->pipe_bytes = 0;
        if (cudaMalloc(&ctx->pipe_buf, need) != cudaSuccess) return set_error(ctx, CDX_ECUDA, "sc_decide_host: alloc");
        ctx->pipe_bytes = need;
    }
    uint8_t* base = static_cast<uint8_t*>(ctx->pipe_buf);
    int64_t* acc = reinterpret_cast<int64_t*>(base + 2 * per);
    struct Buf {
        uint32_t* ids;
        float* h;
        uint32_t* meets;
        int32_t* exit;
        uint8_t* reason;
        int32_t* granted;
        int64_t* off;
        uint32_t* kept;
        int64_t* scal;
    } buf[2];
    for (int i = 0; i < 2; ++i) {
        uint8_t* q = base + i * per;
        buf[i].ids = reinterpret_cast<uint32_t*>(q);
        q += b_ids;
        buf[i].h = reinterpret_cast<float*>(q);
        q += b_h;
        buf[i].meets = reinterpret_cast<uint32_t*>(q);
        q += b_m;
        buf[i].exit = reinterpret_cast<int32_t*>(q);
        q += b_e;
        buf[i].reason = q;
        q += b_r;
        buf[i].granted = reinterpret_cast<int32_t*>(q);
        q += b_g;
        buf[i].off = reinterpret_cast<int64_t*>(q);
        q += b_o;
        buf[i].kept = reinterpret_cast<uint32_t*>(q);
        q += b_k;
        buf[i].scal = reinterpret_cast<int64_t*>(q);
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
    const uint64_t nchunks = (R + chunk - 1) / chunk;
    auto upload = [&](uint64_t c) {
        const uint64_t r0 = c * chunk, nr = std::min(chunk, R - r0);
        cudaStreamWaitEvent(copy, consumed[c & 1], 0);
        cudaMemcpyAsync(buf[c & 1].ids, ids_host + r0 * P * S, nr * req_bytes, cudaMemcpyHostToDevice, copy);
        cudaEventRecord(loaded[c & 1], copy);
    };
    for (int i = 0; i < 2; ++i) cudaEventRecord(consumed[i], comp);
    upload(0);
    for (uint64_t c = 0; c < nchunks && st == CDX_OK; ++c) {
        if (c + 1 < nchunks) upload(c + 1);
        const uint64_t r0 = c * chunk, nr = std::min(chunk, R - r0);
        Buf& b = buf[c & 1];
        cudaStreamWaitEvent(comp, loaded[c & 1], 0);
        st = cdx_sc_certaindex(ctx, b.ids, nr, P, S, th, n_th, hcert_host ? b.h : nullptr, b.meets);
        if (st) break;
        cudaEventRecord(consumed[c & 1], comp);  // ids buffer free once K2 has read it
        st = cdx_allocate_scan(ctx, b.meets, nr, P, pol, 0, static_cast<uint32_t>(r0), b.exit, b.reason, b.granted,
                               b.off, b.kept, reinterpret_cast<uint64_t*>(b.scal), b.scal + 1, b.scal + 2);
        if (st) break;
        add_base<<<static_cast<unsigned>(std::min<uint64_t>((nr + 255) / 256, 1184)), 256, 0, comp>>>(b.off, nr, acc);
        CDX_CHECK_LAUNCH(ctx, "sc_decide_host(offsets)");
        accumulate<<<1, 1, 0, comp>>>(b.scal, acc);
        CDX_CHECK_LAUNCH(ctx, "sc_decide_host(totals)");
        cudaMemcpyAsync(exit_knob_host + r0, b.exit, nr * 4, cudaMemcpyDeviceToHost, comp);
        cudaMemcpyAsync(reason_host + r0, b.reason, nr, cudaMemcpyDeviceToHost, comp);
        cudaMemcpyAsync(offsets_host + r0, b.off, nr * 8, cudaMemcpyDeviceToHost, comp);
        if (hcert_host) cudaMemcpyAsync(hcert_host + r0 * P, b.h, nr * P * 4, cudaMemcpyDeviceToHost, comp);
    }
    int64_t hacc[2] = {0, 0};
    if (st == CDX_OK) {
        cudaMemcpyAsync(hacc, acc, 16, cudaMemcpyDeviceToHost, comp);
        cudaError_t e = cudaStreamSynchronize(comp);
        if (e != cudaSuccess) st = cuda_fail(ctx, e, "sc_decide_host");
    } else {
        cudaStreamSynchronize(comp);
    }
    cudaStreamSynchronize(copy);
    for (int i = 0; i < 2; ++i) {
        cudaEventDestroy(loaded[i]);
        cudaEventDestroy(consumed[i]);
    }
    ctx->stream = user;
    if (st == CDX_OK && tokens_saved_host) *tokens_saved_host = hacc[1];
    return st;
}
