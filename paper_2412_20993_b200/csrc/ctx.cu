// ctx.cu — C-ABI context: device selection, stream, scratch, error reporting.
#include <cmath>
#include <cstring>
#include <mutex>
#include <vector>

#include "cdx_internal.cuh"

namespace cdx {

int set_error(cdx_ctx* ctx, int code, const std::string& msg) {
    if (ctx) ctx->err = msg;
    return code;
}

int take_dev_err(cdx_ctx* ctx) {
    const int code = *ctx->h_err;
    if (code == 0) return CDX_OK;
    cudaMemsetAsync(ctx->d_err, 0, sizeof(int), ctx->stream);
    const int st = (code == DEV_REWARD_RANGE || code == DEV_BAD_CLUSTERING || code == DEV_EMPTY_REWARDS ||
                    code == DEV_EMPTY_CLUSTER || code == DEV_MIXED_PROGRAM ||
                    (code >= DEV_ABSENT_SIGNAL && code < DEV_ABSENT_SIGNAL + 4))
                       ? CDX_EINVAL
                       : CDX_ERUNTIME;
    return set_error(ctx, st, dev_err_message(code));
}

int cuda_fail(cdx_ctx* ctx, cudaError_t e, const char* what) {
    return set_error(ctx, CDX_ECUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

static void* grow(cdx_ctx* ctx, void** buf, size_t* have, size_t bytes) {
    if (bytes <= *have) return *buf;
    if (*buf) {
        cudaStreamSynchronize(ctx->stream);
        cudaFree(*buf);
        *buf = nullptr;
        *have = 0;
    }
    size_t want = bytes < (1u << 20) ? (1u << 20) : bytes + bytes / 4;
    if (cudaMalloc(buf, want) != cudaSuccess) {
        *buf = nullptr;
        return nullptr;
    }
    *have = want;
    return *buf;
}

void* grow_buffer(cdx_ctx* ctx, void** buf, size_t* have, size_t bytes) { return grow(ctx, buf, have, bytes); }

void* scratch(cdx_ctx* ctx, size_t bytes) { return grow(ctx, &ctx->scratch, &ctx->scratch_bytes, bytes); }
void* scratch2(cdx_ctx* ctx, size_t bytes) {
    return grow(ctx, &ctx->scratch2, &ctx->scratch2_bytes, bytes);
}
void* scratch3(cdx_ctx* ctx, size_t bytes) {
    return grow(ctx, &ctx->scratch3, &ctx->scratch3_bytes, bytes);
}

const char* dev_err_message(int code) {
    switch (code) {
        case DEV_REWARD_RANGE: return "certaindex_reward: reward outside [0,1]";
        case DEV_INTERN_COLLISION: return "canon_intern: 64-bit hash collision between distinct answers";
        case DEV_INTERN_FULL: return "canon_intern: intern table full";
        case DEV_BAD_CLUSTERING: return "semantic_entropy: invalid clustering";
        case DEV_EMPTY_REWARDS: return "certaindex_reward: empty reward set";
        case DEV_EMPTY_CLUSTER: return "semantic_entropy: empty cluster";
        case DEV_MIXED_PROGRAM: return "mixed_allocate: archetype, slot or knob out of range";
        case DEV_ABSENT_SIGNAL + 0: return "combined_meets_thresholds: signal 'certaindex_entropy' absent";
        case DEV_ABSENT_SIGNAL + 1: return "combined_meets_thresholds: signal 'certaindex_reward' absent";
        case DEV_ABSENT_SIGNAL + 2: return "combined_meets_thresholds: signal 'mean_output_length' absent";
        case DEV_ABSENT_SIGNAL + 3: return "combined_meets_thresholds: signal 'mean_norm_logprob' absent";
    }
    return "device error";
}

static PFN_cuTensorMapEncodeTiled_v12000 tmap_fn() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    static std::once_flag once;
    std::call_once(once, [] {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
    });
    return fn;
}

bool encode_tmap(CUtensorMap* map, const void* base, uint32_t rank, const uint64_t* dims,
                 const uint64_t* strides_bytes, const uint32_t* box, CUtensorMapDataType dtype,
                 CUtensorMapSwizzle swz) {
    auto fn = tmap_fn();
    if (!fn || rank < 1 || rank > 5) return false;
    cuuint64_t d[5], st[4];
    cuuint32_t b[5], es[5];
    for (uint32_t i = 0; i < rank; ++i) {
        d[i] = dims[i];
        b[i] = box[i];
        es[i] = 1;
    }
    for (uint32_t i = 0; i + 1 < rank; ++i) st[i] = strides_bytes[i];
    CUresult r = fn(map, dtype, rank, const_cast<void*>(base), d, st, b, es, CU_TENSOR_MAP_INTERLEAVE_NONE, swz,
                    CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS;
}

double host_term(uint32_t c, uint32_t n) {
    // p * log(p) with p = c/n, exactly as metrics.cpp:113-116 rounds it (no contraction)
    volatile double p = static_cast<double>(c) / static_cast<double>(n);
    volatile double lg = std::log(p);
    return p * lg;
}

int build_term_tables(cdx_ctx* ctx, const uint32_t* ns, uint32_t count, TermTables* out) {
    std::string key(reinterpret_cast<const char*>(ns), count * sizeof(uint32_t));
    if (ctx->tt_dev && key == ctx->tt_key) {
        out->row_off = reinterpret_cast<const uint64_t*>(ctx->tt_dev);
        out->logs = ctx->tt_dev + count;
        out->tab = ctx->tt_dev + 2 * count;
        return CDX_OK;
    }
    std::vector<double> host(2 * count);
    uint64_t off = 0;
    for (uint32_t i = 0; i < count; ++i) {
        std::memcpy(&host[i], &off, 8);
        off += static_cast<uint64_t>(ns[i]) + 1;
    }
    for (uint32_t i = 0; i < count; ++i) host[count + i] = std::log(static_cast<double>(ns[i]));
    host.reserve(2 * count + off);
    for (uint32_t i = 0; i < count; ++i) {
        host.push_back(0.0);
        for (uint32_t c = 1; c <= ns[i]; ++c) host.push_back(host_term(c, ns[i]));
    }
    const size_t bytes = host.size() * sizeof(double);
    cudaStreamSynchronize(ctx->stream);
    if (bytes > ctx->tt_bytes) {
        if (ctx->tt_dev) cudaFree(ctx->tt_dev);
        ctx->tt_dev = nullptr;
        ctx->tt_bytes = 0;
        if (cudaMalloc(&ctx->tt_dev, bytes) != cudaSuccess) return set_error(ctx, CDX_ECUDA, "term table alloc");
        ctx->tt_bytes = bytes;
    }
    cudaError_t e = cudaMemcpy(ctx->tt_dev, host.data(), bytes, cudaMemcpyHostToDevice);
    if (e != cudaSuccess) return cuda_fail(ctx, e, "term table upload");
    ctx->tt_key = key;
    out->row_off = reinterpret_cast<const uint64_t*>(ctx->tt_dev);
    out->logs = ctx->tt_dev + count;
    out->tab = ctx->tt_dev + 2 * count;
    return CDX_OK;
}

bool encode_tmap_2d(CUtensorMap* map, const void* base, uint64_t inner, uint64_t outer,
                    uint64_t row_stride_bytes, uint32_t box_inner, uint32_t box_outer,
                    CUtensorMapDataType dtype, CUtensorMapSwizzle swz) {
    auto fn = tmap_fn();
    if (!fn) return false;
    cuuint64_t dims[2] = {inner, outer};
    cuuint64_t strides[1] = {row_stride_bytes};
    cuuint32_t box[2] = {box_inner, box_outer};
    cuuint32_t estr[2] = {1, 1};
    CUresult r = fn(map, dtype, 2, const_cast<void*>(base), dims, strides, box, estr,
                    CU_TENSOR_MAP_INTERLEAVE_NONE, swz, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                    CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS;
}

}  // namespace cdx

extern "C" {

int cdx_abi_version(void) { return CDX_ABI_VERSION; }

int cdx_ctx_create(int device, cdx_ctx** out) {
    if (!out) return CDX_EINVAL;
    *out = nullptr;
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess || n == 0) return CDX_ECUDA;
    if (device < 0 || device >= n) return CDX_EINVAL;
    cudaDeviceProp prop;
    if (cudaGetDeviceProperties(&prop, device) != cudaSuccess) return CDX_ECUDA;
    if (prop.major != 10) return CDX_ECUDA;  // sm_100a kernels only
    if (cudaSetDevice(device) != cudaSuccess) return CDX_ECUDA;
    auto* c = new cdx_ctx();
    c->device = device;
    c->sm_count = prop.multiProcessorCount;
    if (cudaStreamCreateWithFlags(&c->own_stream, cudaStreamNonBlocking) != cudaSuccess ||
        cudaStreamCreateWithFlags(&c->copy_stream, cudaStreamNonBlocking) != cudaSuccess ||
        cudaMalloc(&c->d_err, sizeof(int)) != cudaSuccess ||
        cudaMallocHost(&c->h_err, 64 * sizeof(int)) != cudaSuccess) {
        delete c;
        return CDX_ECUDA;
    }
    cudaMemset(c->d_err, 0, sizeof(int));
    c->h_small = reinterpret_cast<uint32_t*>(c->h_err) + 16;
    // K2's group-claim counters (k_sc_fast.cu): zeroed once here, rewound by the kernel
    if (cudaMalloc(&c->sc_counter, 2 * sizeof(unsigned long long)) == cudaSuccess)
        cudaMemset(c->sc_counter, 0, 2 * sizeof(unsigned long long));
    else
        c->sc_counter = nullptr;
    cudaDeviceSynchronize();
    c->stream = c->own_stream;
    *out = c;
    return CDX_OK;
}

int cdx_ctx_destroy(cdx_ctx* ctx) {
    if (!ctx) return CDX_OK;
    cudaSetDevice(ctx->device);
    cudaStreamSynchronize(ctx->stream);
    if (ctx->scratch) cudaFree(ctx->scratch);
    if (ctx->scratch2) cudaFree(ctx->scratch2);
    if (ctx->scratch3) cudaFree(ctx->scratch3);
    if (ctx->pipe_buf) cudaFree(ctx->pipe_buf);
    if (ctx->tt_dev) cudaFree(ctx->tt_dev);
    if (ctx->al_state) cudaFree(ctx->al_state);
    for (double* t : ctx->comp_tab)
        if (t) cudaFree(t);
    if (ctx->jl_buf) cudaFree(ctx->jl_buf);
    cdx::comm_destroy(ctx);
    if (ctx->sh_buf) cudaFree(ctx->sh_buf);
    if (ctx->sh_buf2) cudaFree(ctx->sh_buf2);
    if (ctx->sh_host) cudaFreeHost(ctx->sh_host);
    if (ctx->d_err) cudaFree(ctx->d_err);
    if (ctx->h_err) cudaFreeHost(ctx->h_err);
    if (ctx->sc_d) cudaFree(ctx->sc_d);
    if (ctx->sc_counter) cudaFree(ctx->sc_counter);
    if (ctx->sc_h) cudaFreeHost(ctx->sc_h);
    for (int q = 0; q < 2; ++q) {
        if (ctx->aux[q]) cudaStreamDestroy(ctx->aux[q]);
        if (ctx->ev_join[q]) cudaEventDestroy(ctx->ev_join[q]);
    }
    if (ctx->ev_fork) cudaEventDestroy(ctx->ev_fork);
    if (ctx->own_stream) cudaStreamDestroy(ctx->own_stream);
    if (ctx->copy_stream) cudaStreamDestroy(ctx->copy_stream);
    delete ctx;
    return CDX_OK;
}

int cdx_ctx_set_stream(cdx_ctx* ctx, void* s) {
    if (!ctx) return CDX_EINVAL;
    // NULL is the (legacy) default stream of the device, shared with every runtime in the
    // process (e.g. torch's default stream); cdx_ctx_use_own_stream() restores the private one
    ctx->stream = static_cast<cudaStream_t>(s);
    return CDX_OK;
}

int cdx_ctx_use_own_stream(cdx_ctx* ctx) {
    if (!ctx) return CDX_EINVAL;
    ctx->stream = ctx->own_stream;
    return CDX_OK;
}

void* cdx_ctx_stream(cdx_ctx* ctx) { return ctx ? ctx->stream : nullptr; }

uint64_t cdx_launch_count(const cdx_ctx* ctx) { return ctx ? ctx->launches : 0; }

const char* cdx_last_error(const cdx_ctx* ctx) { return ctx ? ctx->err.c_str() : "null context"; }

int cdx_sync(cdx_ctx* ctx) {
    if (!ctx) return CDX_EINVAL;
    cudaSetDevice(ctx->device);
    cudaError_t e = cudaStreamSynchronize(ctx->stream);
    if (e != cudaSuccess) return cdx::cuda_fail(ctx, e, "cdx_sync");
    e = cudaMemcpy(ctx->h_err, ctx->d_err, sizeof(int), cudaMemcpyDeviceToHost);
    if (e != cudaSuccess) return cdx::cuda_fail(ctx, e, "cdx_sync");
    return cdx::take_dev_err(ctx);
}

}  // extern "C"

// ---- CUDA graphs of a call sequence on the context stream (launch-bound small batches) ----
struct cdx_graph {
    cudaGraph_t graph = nullptr;
    cudaGraphExec_t exec = nullptr;
    uint64_t launches = 0;  // kernels per replay (for cdx_launch_count)
};

extern "C" {

int cdx_graph_begin(cdx_ctx* ctx) {
    if (!ctx) return CDX_EINVAL;
    if (ctx->stream == nullptr || ctx->stream == cudaStreamLegacy || ctx->stream == cudaStreamPerThread)
        return cdx::set_error(ctx, CDX_EINVAL, "graph: capture needs a non-default stream (cdx_ctx_set_stream)");
    ctx->graph_mark = ctx->launches;
    cudaError_t e = cudaStreamBeginCapture(ctx->stream, cudaStreamCaptureModeThreadLocal);
    if (e != cudaSuccess) return cdx::cuda_fail(ctx, e, "graph: begin capture");
    return CDX_OK;
}

int cdx_graph_end(cdx_ctx* ctx, cdx_graph** out) {
    if (!ctx || !out) return CDX_EINVAL;
    *out = nullptr;
    auto* g = new cdx_graph();
    cudaError_t e = cudaStreamEndCapture(ctx->stream, &g->graph);
    if (e == cudaSuccess) e = cudaGraphInstantiate(&g->exec, g->graph, 0);
    if (e != cudaSuccess) {
        if (g->graph) cudaGraphDestroy(g->graph);
        delete g;
        return cdx::cuda_fail(ctx, e, "graph: end capture / instantiate");
    }
    g->launches = ctx->launches - ctx->graph_mark;
    ctx->launches = ctx->graph_mark;  // captured launches count when replayed
    *out = g;
    return CDX_OK;
}

int cdx_graph_launch(cdx_ctx* ctx, cdx_graph* g) {
    if (!ctx || !g) return CDX_EINVAL;
    cudaError_t e = cudaGraphLaunch(g->exec, ctx->stream);
    if (e != cudaSuccess) return cdx::cuda_fail(ctx, e, "graph: launch");
    ctx->launches += g->launches;
    return CDX_OK;
}

int cdx_graph_destroy(cdx_graph* g) {
    if (!g) return CDX_OK;
    if (g->exec) cudaGraphExecDestroy(g->exec);
    if (g->graph) cudaGraphDestroy(g->graph);
    delete g;
    return CDX_OK;
}

}  // extern "C"
