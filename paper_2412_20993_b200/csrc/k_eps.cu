// k_eps.cu — the batched epsilon-accuracy stop test: the
// appendix-E alternative CoT stop rule probe::stationary_by_epsilon_test (probe.cpp:104-120)
// over theory::epsilon_stop_test (theory.cpp:100-146), evaluated at every prefix of every
// request's probe trace.
//
// Per prefix: the non-hesitant answers map to group indices in first-seen order (the
// reference's std::find over `seen`); with n of them, nullopt while n < 2k; else, anchored
// at a = n - 2k, every window of length k (and k-1 when k >= 2) starting at a+j must stay
// within total variation eps/3 of the window at a:  TV = 0.5 * sum_g |c_a(g)/L - c_j(g)/L|
// summed over group index g ascending (groups absent from both windows add +0.0, which
// leaves the sum's bits unchanged, so only the <= 2L groups present are visited).  All FP64
// ops are IEEE-rounded in the reference's order, so the decisions are the reference's.

#include "cdx_internal.cuh"

namespace cdx {
namespace {

constexpr int EPS_MAX_P = 64;     // probes per request held per thread (batched kernel)
constexpr int EPS_MAX_ROW = 1024;  // usable records per ragged row (scalar API)

// TV between the windows [a, a+L) and [b, b+L) of g[], group-ascending sum
__device__ __forceinline__ double tv_windows(const uint16_t* g, int a, int b, int L) {
    const double len = static_cast<double>(L);
    double l1 = 0.0;
    int last = -1;
    for (;;) {  // next group index above `last` present in either window
        int nxt = 1 << 30;
        for (int i = 0; i < L; ++i) {
            const int x = g[a + i], y = g[b + i];
            if (x > last && x < nxt) nxt = x;
            if (y > last && y < nxt) nxt = y;
        }
        if (nxt == (1 << 30)) break;
        int ca = 0, cb = 0;
        for (int i = 0; i < L; ++i) {
            ca += g[a + i] == nxt;
            cb += g[b + i] == nxt;
        }
        const double pa = __ddiv_rn(static_cast<double>(ca), len), pb = __ddiv_rn(static_cast<double>(cb), len);
        l1 = __dadd_rn(l1, fabs(__dsub_rn(pa, pb)));
        last = nxt;
    }
    return __dmul_rn(0.5, l1);
}

// theory.cpp:117-146 on g[0..n): 0 nullopt, 1 false, 2 true
__device__ __forceinline__ uint8_t eps_test(const uint16_t* g, int n, int k, double limit) {
    if (n < 2 * k) return 0;
    const int anchor = n - 2 * k;
    for (int j = 1; j <= k; ++j)
        if (tv_windows(g, anchor, anchor + j, k) > limit) return 1;
    if (k >= 2)
        for (int j = 1; j <= k - 1; ++j)
            if (tv_windows(g, anchor, anchor + j, k - 1) > limit) return 1;
    return 2;
}

// first-seen group index of answer v among seen[0..m), appending when new
__device__ __forceinline__ uint16_t group_of(uint32_t* seen, int* m, uint32_t v) {
    for (int i = 0; i < *m; ++i)
        if (seen[i] == v) return static_cast<uint16_t>(i);
    seen[*m] = v;
    return static_cast<uint16_t>((*m)++);
}

__global__ void eps_stop_kernel(const uint32_t* __restrict__ ids, const uint64_t* __restrict__ hes, uint64_t R,
                                uint32_t P, uint32_t hw, int k, double limit, int32_t* __restrict__ eps_step,
                                uint8_t* __restrict__ state) {
    for (uint64_t r = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; r < R;
         r += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
        uint16_t g[EPS_MAX_P];
        uint32_t seen[EPS_MAX_P];
        int n = 0, m = 0;
        int32_t first = -1;
        for (uint32_t p = 0; p < P; ++p) {
            const bool h = (__ldg(hes + r * hw + p / 64) >> (p % 64)) & 1ull;
            if (!h) {
                g[n] = group_of(seen, &m, __ldg(ids + r * P + p));
                ++n;
            }
            const uint8_t st = eps_test(g, n, k, limit);
            if (state) state[r * P + p] = st;
            if (st == 2 && first < 0) {
                first = static_cast<int32_t>(p);
                if (!state) break;
            }
        }
        eps_step[r] = first;
    }
}

// one ragged row = one whole record span (the scalar probe::stationary_by_epsilon_test)
__global__ void eps_rows_kernel(const uint32_t* __restrict__ ids, const uint8_t* __restrict__ hes,
                                const uint64_t* __restrict__ row_off, uint64_t rows, int k, double limit,
                                uint8_t* __restrict__ state, int* err) {
    for (uint64_t r = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; r < rows;
         r += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
        uint16_t g[EPS_MAX_ROW];
        uint32_t seen[EPS_MAX_ROW];
        int n = 0, m = 0;
        bool over = false;
        for (uint64_t i = row_off[r]; i < row_off[r + 1]; ++i) {
            if (hes[i]) continue;
            if (n == EPS_MAX_ROW) {
                over = true;
                break;
            }
            g[n] = group_of(seen, &m, ids[i]);
            ++n;
        }
        if (over) {
            set_dev_err(err, DEV_BAD_CLUSTERING);
            continue;
        }
        state[r] = eps_test(g, n, k, limit);
    }
}

unsigned grid_n(const cdx_ctx* ctx, uint64_t n) {
    const uint64_t want = (n + 127) / 128;
    const uint64_t cap = static_cast<uint64_t>(ctx->sm_count) * 16;
    return static_cast<unsigned>(want < 1 ? 1 : (want < cap ? want : cap));
}

int check_eps(cdx_ctx* ctx, int32_t k, double epsilon) {  // theory.cpp:118-119
    if (k < 1) return set_error(ctx, CDX_EINVAL, "epsilon_stop_test: k must be >= 1");
    if (epsilon <= 0.0) return set_error(ctx, CDX_EINVAL, "epsilon_stop_test: epsilon must be > 0");
    return CDX_OK;
}

}  // namespace
}  // namespace cdx

extern "C" int cdx_cot_eps_stop(cdx_ctx* ctx, const uint32_t* ids, const uint64_t* hes, uint64_t R, uint32_t P,
                                int32_t k, double epsilon, int32_t* eps_step, uint8_t* state) {
    using namespace cdx;
    CDX_NVTX("cdx_cot_eps_stop");
    if (!ctx) return CDX_EINVAL;
    if (int st = check_eps(ctx, k, epsilon)) return st;
    if (P == 0 || P > static_cast<uint32_t>(EPS_MAX_P))
        return set_error(ctx, CDX_EINVAL, "cot_eps_stop: probes must be 1..64");
    if (R == 0) return CDX_OK;
    if (!ids || !hes || !eps_step) return set_error(ctx, CDX_EINVAL, "cot_eps_stop: null pointer");
    const double limit = epsilon / 3.0;  // theory.cpp:129, host IEEE division
    eps_stop_kernel<<<grid_n(ctx, R), 128, 0, ctx->stream>>>(ids, hes, R, P, (P + 63) / 64, k, limit, eps_step, state);
    CDX_CHECK_LAUNCH(ctx, "cot_eps_stop");
    return CDX_OK;
}

extern "C" int cdx_probe_eps_stop_rows(cdx_ctx* ctx, const uint32_t* ids, const uint8_t* hes, const uint64_t* row_off,
                                       uint64_t rows, int32_t k, double epsilon, uint8_t* state) {
    using namespace cdx;
    if (!ctx) return CDX_EINVAL;
    if (int st = check_eps(ctx, k, epsilon)) return st;
    if (rows == 0) return CDX_OK;
    if (!ids || !hes || !row_off || !state) return set_error(ctx, CDX_EINVAL, "eps_stop_rows: null pointer");
    eps_rows_kernel<<<grid_n(ctx, rows), 128, 0, ctx->stream>>>(ids, hes, row_off, rows, k, epsilon / 3.0, state,
                                                                ctx->d_err);
    CDX_CHECK_LAUNCH(ctx, "eps_stop_rows");
    return CDX_OK;
}
