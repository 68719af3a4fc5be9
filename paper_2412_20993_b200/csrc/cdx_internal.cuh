// cdx_internal.cuh — context, error plumbing and the sm_100a async-copy primitives
// (TMA tensor loads, 1-D bulk copies, mbarriers) shared by the Certaindex kernels.
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <cstdint>
#include <string>

#include "../../include/cdx_c.h"

// NVTX ranges (header-only NVTX v3): every C-ABI entry that launches work opens a named
// range, so ncu --nvtx / nsys timelines group kernels by the reference function they replace.
#include <nvtx3/nvToolsExt.h>
namespace cdx {
struct NvtxRange {
    explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
    ~NvtxRange() { nvtxRangePop(); }
    NvtxRange(const NvtxRange&) = delete;
    NvtxRange& operator=(const NvtxRange&) = delete;
};
}  // namespace cdx
#define CDX_NVTX(name) ::cdx::NvtxRange cdx_nvtx_range_(name)

#define CDX_SMS 148

struct cdx_ctx {
    int device = 0;
    int sm_count = CDX_SMS;
    cudaStream_t own_stream = nullptr;
    cudaStream_t stream = nullptr;
    std::string err;
    uint64_t launches = 0;
    uint64_t graph_mark = 0;  // launches before the current graph capture
    // device error word: 0 ok, else a CDX_E* code set by a kernel (validated on sync)
    int* d_err = nullptr;
    int* h_err = nullptr;  // pinned mirror (a 64-word pinned block)
    uint32_t* h_small = nullptr;  // pinned staging for small results read back by a call (h_err + 16, 48 words)
    std::string pending_err_msg[8];
    // growable scratch (look-back tile state, counters, tables)
    void* scratch = nullptr;
    size_t scratch_bytes = 0;
    void* scratch2 = nullptr;
    size_t scratch2_bytes = 0;
    void* scratch3 = nullptr;
    size_t scratch3_bytes = 0;
    // host-entry pipeline buffers
    void* pipe_buf = nullptr;
    size_t pipe_bytes = 0;
    cudaStream_t copy_stream = nullptr;
    // K5 look-back state, persistent across calls: tile ticket counter + per-tile flags /
    // aggregates, tagged with a per-call epoch so nothing is cleared between calls
    void* al_state = nullptr;
    size_t al_tiles = 0;      // capacity in tiles
    // JSONL ingestion working buffer (k_jsonl.cu)
    void* jl_buf = nullptr;
    size_t jl_bytes = 0;
    double* comp_tab[17] = {};  // K2: H~ per first-seen cluster-size composition, S <= 16 (k_sc.cu)
    // term-table cache (device): keyed by the list of n values it was built for
    double* tt_dev = nullptr;
    size_t tt_bytes = 0;
    std::string tt_key;
    // communicator (shard.cu): rank / world, the caller's callbacks or an owned NCCL comm
    uint32_t rank = 0, world = 1;
    cdx_comm comm{};
    void* nccl = nullptr;  // ncclComm_t
    // sharded paths' buffers (shard.cu)
    void* sh_buf = nullptr;
    size_t sh_bytes = 0;
    void* sh_buf2 = nullptr;
    size_t sh_bytes2 = 0;
    uint64_t* sh_host = nullptr;  // pinned host staging (counts, bounds)
    uint64_t it_cap = 0;          // K1 global table capacity of the last call (k_intern.cu)
    // one-round-trip scalar calls (k_scalar.cu): pinned host / device staging pair
    void* sc_counter = nullptr;   // K2 fast path: group claims + CTAs done (k_sc_fast.cu)
    uint8_t* sc_h = nullptr;
    uint8_t* sc_d = nullptr;
    size_t sc_cap = 0;
    // the mixed step's side streams (k_mixed.cu): the archetype engines run concurrently
    cudaStream_t aux[2] = {nullptr, nullptr};
    cudaEvent_t ev_fork = nullptr, ev_join[2] = {nullptr, nullptr};
    uint32_t sc_ctas_per_sm = 0;  // K2 fast path: resident CTAs per SM cap while sharing the GPU (0: none)
};

namespace cdx {

int set_error(cdx_ctx* ctx, int code, const std::string& msg);
int cuda_fail(cdx_ctx* ctx, cudaError_t e, const char* what);
void* scratch(cdx_ctx* ctx, size_t bytes);
void* scratch2(cdx_ctx* ctx, size_t bytes);
void* scratch3(cdx_ctx* ctx, size_t bytes);  // the mixed step's own buffers (K2/K4 use scratch, scratch2)
void* grow_buffer(cdx_ctx* ctx, void** buf, size_t* have, size_t bytes);
void comm_destroy(cdx_ctx* ctx);  // shard.cu
// device-side validation error codes (set via atomicCAS on ctx->d_err)
enum DevErr : int {
    DEV_OK = 0,
    DEV_REWARD_RANGE = 1,   // "certaindex_reward: reward outside [0,1]"
    DEV_INTERN_COLLISION = 2,
    DEV_INTERN_FULL = 3,
    DEV_BAD_CLUSTERING = 4,  // "semantic_entropy: invalid clustering"
    DEV_EMPTY_REWARDS = 5,   // "certaindex_reward: empty reward set"
    DEV_EMPTY_CLUSTER = 6,   // "semantic_entropy: empty cluster"
    DEV_MIXED_PROGRAM = 7,   // "mixed_allocate: archetype, slot or knob out of range"
    DEV_ABSENT_SIGNAL = 16,  // + SignalKind: "combined_meets_thresholds: signal '<name>' absent"
};
const char* dev_err_message(int code);
// the device error word already copied to *ctx->h_err (stream synchronised): CDX_OK, or the
// mapped status with the message (the word is cleared for the next call)
int take_dev_err(cdx_ctx* ctx);
// k_rows.cu helpers shared with the one-round-trip entries (k_scalar.cu)
int check_probe_cfg_c(cdx_ctx* ctx, const cdx_probe_cfg* cfg);
int entropy_terms_launch(cdx_ctx* ctx, const double* terms, uint32_t m, double log_n, bool n_is_one, double* H,
                         double* Hc);
// cuTensorMapEncodeTiled through the runtime's driver entry point (no -lcuda needed)
bool encode_tmap_2d(CUtensorMap* map, const void* base, uint64_t inner, uint64_t outer,
                    uint64_t row_stride_bytes, uint32_t box_inner, uint32_t box_outer,
                    CUtensorMapDataType dtype, CUtensorMapSwizzle swz);
// rank-N tiled tensor map: dims/box innermost first, strides_bytes has rank-1 entries
bool encode_tmap(CUtensorMap* map, const void* base, uint32_t rank, const uint64_t* dims,
                 const uint64_t* strides_bytes, const uint32_t* box, CUtensorMapDataType dtype,
                 CUtensorMapSwizzle swz);
// Host-built entropy term tables: for each n in ns, T_n[c] = (c/n)*log(c/n), c = 0..n
// (metrics.cpp:113-116 with the host libm), uploaded to device scratch.  Returns device
// pointers: tab (rows concatenated), row_off[i] = offset of n_i's row, logs[i] = log(n_i).
struct TermTables {
    const double* tab = nullptr;
    const uint64_t* row_off = nullptr;
    const double* logs = nullptr;
};
int build_term_tables(cdx_ctx* ctx, const uint32_t* ns, uint32_t count, TermTables* out);
double host_term(uint32_t c, uint32_t n);
// K1 for inputs with many distinct keys (k_intern.cu): dense first-seen ids of the trimmed
// bytes with one thread per answer against one global table; no markers / hesitation
int canon_intern_direct(cdx_ctx* ctx, const char* bytes, const uint64_t* offsets, uint64_t n, uint32_t* ids,
                        uint64_t* first_index, uint64_t* n_unique);
// stable LSD radix sort of (u64 key, u32 value) (k_gang.cu); lb = radix_scratch_words(n)
// u32 of device scratch; *which = 1 when the result is in (k1, v1)
size_t radix_scratch_words(uint64_t n);
int radix_sort_pairs(cdx_ctx* ctx, uint64_t* k0, uint32_t* v0, uint64_t* k1, uint32_t* v1, uint64_t n, uint32_t* lb,
                     int* which);

#define CDX_LAUNCHED(ctx) ((ctx)->launches++)

__device__ __forceinline__ void set_dev_err(int* d_err, int code) { atomicCAS(d_err, 0, code); }

// The reference's host arithmetic is x86-64 SSE2: a + b / a / b with a NaN operand returns
// that NaN (quieted, sign and payload kept), the first operand's when both are NaN.  The GPU
// returns a canonical NaN instead; these keep the host's bits where a NaN reaches an f64
// output of the scalar API (e.g. certaindex_reward's mean over a NaN reward).
__device__ __forceinline__ double x86_nan(double a) {
    return __longlong_as_double(__double_as_longlong(a) | 0x0008000000000000ll);
}
__device__ __forceinline__ double x86_add(double a, double b) {
    return isnan(a) ? x86_nan(a) : (isnan(b) ? x86_nan(b) : __dadd_rn(a, b));
}
__device__ __forceinline__ double x86_div(double a, double b) {
    return isnan(a) ? x86_nan(a) : (isnan(b) ? x86_nan(b) : __ddiv_rn(a, b));
}

// ---------------------------------------------------------------------------------------
// mbarrier / bulk-copy / TMA (PTX for sm_90+/sm_100a; SASS: SYNCS.*, UBLKCP, UTMALDG)
// ---------------------------------------------------------------------------------------
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}

__device__ __forceinline__ void fence_mbar_init() {
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

__device__ __forceinline__ void fence_proxy_async() {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
                 "r"(bytes)
                 : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    asm volatile(
        "{\n"
        ".reg .pred P1;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
        "@!P1 bra WAIT_%=;\n"
        "}\n" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}

// 1-D bulk global->shared copy, completion counted on `bar` (bytes % 16 == 0, 16B aligned)
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar,
                                         uint64_t policy) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint "
        "[%0], [%1], %2, [%3], %4;" ::"r"(smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(policy)
        : "memory");
}

// 2-D TMA tile load at (c0 = inner coordinate, c1 = outer coordinate)
__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, int32_t c0, int32_t c1,
                                            uint64_t* bar, uint64_t policy) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes.L2::cache_hint "
        "[%0], [%1, {%2, %3}], [%4], %5;" ::"r"(smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(smem_u32(bar)), "l"(policy)
        : "memory");
}

__device__ __forceinline__ void tma_load_3d(void* dst, const CUtensorMap* map, int32_t c0, int32_t c1,
                                            int32_t c2, uint64_t* bar, uint64_t policy) {
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes.L2::cache_hint "
        "[%0], [%1, {%2, %3, %4}], [%5], %6;" ::"r"(smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(bar)), "l"(policy)
        : "memory");
}

__device__ __forceinline__ void tma_prefetch_desc(const CUtensorMap* map) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(map)) : "memory");
}

__device__ __forceinline__ uint64_t policy_evict_first() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
    return p;
}

// streaming stores that do not allocate in L1
__device__ __forceinline__ void st_na_f32(float* p, float v) {
    asm volatile("st.global.L1::no_allocate.f32 [%0], %1;" ::"l"(p), "f"(v) : "memory");
}

// 128B-swizzle: 16-byte chunk c of smem row r lives at chunk c ^ (r & 7)
__device__ __forceinline__ uint32_t swz128(uint32_t row, uint32_t chunk) {
    return row * 128u + ((chunk ^ (row & 7u)) << 4);
}

}  // namespace cdx

// kernel-launch helper: records the launch and surfaces launch errors
#define CDX_CHECK_LAUNCH(ctx, name)                                         \
    do {                                                                    \
        (ctx)->launches++;                                                  \
        cudaError_t _e = cudaGetLastError();                                \
        if (_e != cudaSuccess) return cdx::cuda_fail((ctx), _e, name);      \
    } while (0)
