// k_aggregate.cu — the final answer of a terminated program per archetype (SURVEY.md §8(f)
// rank 1): ProgramDriver::aggregate_prefix, runtime.cpp:318-403 (weighted_plurality
// :316-336), for whole batches of programs.
//
//   SC      plurality over the exit row's S answers, earliest-seen cluster wins ties (the
//           reference scans clusters in first-seen order with a strict `>`).
//   MCTS    the answer of the first path with the maximum reward over every path so far
//           (strict `>` over reward.value_or(0.0) in path order).
//   Rebase  softmax-weighted plurality over the last full layer: weight(cluster) = sum of
//           exp(reward) over its members in path order (double), earliest-seen wins ties.
//           exp() is the host libm's own algorithm restated bit for bit on the device
//           (libm_exp.cuh), so the weights are the reference's bits for every reward, on or
//           off any grid.  When no weight beats the reference's initial -1.0 (NaN rewards)
//           the reference returns an empty string; the answer id is then CDX_NO_ANSWER.
// Rewards are f32 (the synthetic traces) or f64 (RewardSet holds doubles, metrics.hpp:74-77).
// CoT's final answer is K3's final_id (probe::final_answer).  Answers are interned ids
// (equal id <=> equal trimmed bytes), so the winner's id is the reference's trimmed answer.

#include <cmath>
#include <vector>

#include "cdx_internal.cuh"
#include "libm_exp.cuh"

namespace cdx {
namespace {

constexpr int AG_MAX_W = 256;  // Rebase layer width handled per thread (shared-memory table)
constexpr int AG_THREADS = 64;

// SC: thread per request, the exit row's S ids; first-seen peel, strict > on counts
__global__ void sc_aggregate_kernel(const uint32_t* __restrict__ ids, uint64_t R, uint32_t P, uint32_t S,
                                    const int32_t* __restrict__ exit_knob, uint32_t* __restrict__ answer, int* err) {
    for (uint64_t r = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; r < R;
         r += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
        const int32_t k = exit_knob[r];
        if (k < 1 || static_cast<uint32_t>(k) > P) {
            set_dev_err(err, DEV_BAD_CLUSTERING);
            continue;
        }
        const uint32_t* row = ids + (r * P + static_cast<uint64_t>(k - 1)) * S;
        uint32_t best = row[0];
        uint32_t best_c = 0;
        // clusters in first-seen order: sample s leads iff no earlier sample holds its id
        for (uint32_t s = 0; s < S; ++s) {
            const uint32_t v = __ldg(row + s);
            bool seen = false;
            for (uint32_t q = 0; q < s && !seen; ++q) seen = __ldg(row + q) == v;
            if (seen) continue;
            uint32_t c = 1;
            for (uint32_t q = s + 1; q < S; ++q) c += __ldg(row + q) == v ? 1u : 0u;
            if (c > best_c) {  // weight[key] > best_w with weights = counts (exact in double)
                best_c = c;
                best = v;
            }
        }
        answer[r] = best;
    }
}

// MCTS / Rebase: thread per program, exit step t (0-based): paths = steps 0..t
template <typename RT>
__global__ void __launch_bounds__(AG_THREADS) reward_aggregate_kernel(
    const RT* __restrict__ rw, const uint32_t* __restrict__ ids, const uint8_t* __restrict__ agg, uint64_t G,
    uint32_t T, uint32_t W, const int32_t* __restrict__ exit_step, uint32_t* __restrict__ answer, int* err) {
    extern __shared__ __align__(16) uint8_t ag_smem[];  // per thread: W weights (f64) then W keys (u32)
    const uint64_t g = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
    if (g >= G) return;
    const int32_t t = exit_step[g];
    if (t < 0 || static_cast<uint32_t>(t) >= T) {
        set_dev_err(err, DEV_BAD_CLUSTERING);
        return;
    }
    const uint64_t base = g * T * W;
    if (agg[g] == CDX_AGG_MEAN) {  // MCTS: first maximum over every path so far
        const uint64_t n = static_cast<uint64_t>(t + 1) * W;
        uint64_t best = 0;
        double bv = static_cast<double>(__ldg(rw + base));
        for (uint64_t i = 1; i < n; ++i) {
            const double v = static_cast<double>(__ldg(rw + base + i));
            if (v > bv) {  // strict >, NaN never wins (runtime.cpp:386-388)
                bv = v;
                best = i;
            }
        }
        answer[g] = __ldg(ids + base + best);
        return;
    }
    // Rebase: last full layer = step t; clusters in first-seen order with summed weights
    double* wt = reinterpret_cast<double*>(ag_smem) + static_cast<size_t>(threadIdx.x) * W;
    uint32_t* key = reinterpret_cast<uint32_t*>(reinterpret_cast<double*>(ag_smem) + static_cast<size_t>(blockDim.x) * W) +
                    static_cast<size_t>(threadIdx.x) * W;
    uint32_t m = 0;
    const uint64_t l0 = base + static_cast<uint64_t>(t) * W;
    for (uint32_t i = 0; i < W; ++i) {
        const uint32_t v = __ldg(ids + l0 + i);
        const double e = libm::exp(static_cast<double>(__ldg(rw + l0 + i)));  // std::exp, runtime.cpp:324
        uint32_t c = 0;
        while (c < m && key[c] != v) ++c;
        if (c == m) {
            key[m] = v;
            wt[m] = 0.0;
            ++m;
        }
        wt[c] = __dadd_rn(wt[c], e);
    }
    uint32_t best = CDX_NO_ANSWER;  // std::string best; stays empty if nothing beats -1.0
    double bw = -1.0;
    for (uint32_t c = 0; c < m; ++c)
        if (wt[c] > bw) {
            bw = wt[c];
            best = key[c];
        }
    answer[g] = best;
}

__global__ void libm_exp_kernel(const double* __restrict__ x, uint64_t n, double* __restrict__ y) {
    for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<uint64_t>(gridDim.x) * blockDim.x)
        y[i] = libm::exp(x[i]);
}

unsigned grid_of(const cdx_ctx* ctx, uint64_t n, unsigned t) {
    const uint64_t want = (n + t - 1) / t;
    const uint64_t cap = static_cast<uint64_t>(ctx->sm_count) * 16;
    return static_cast<unsigned>(want < 1 ? 1 : (want < cap ? want : cap));
}

}  // namespace
}  // namespace cdx

extern "C" int cdx_sc_aggregate(cdx_ctx* ctx, const uint32_t* ids, uint64_t R, uint32_t P, uint32_t S,
                                const int32_t* exit_knob, uint32_t* answer) {
    using namespace cdx;
    CDX_NVTX("cdx_sc_aggregate");
    if (!ctx) return CDX_EINVAL;
    if (P == 0 || S == 0) return set_error(ctx, CDX_ERUNTIME, "aggregate: empty program");  // runtime.cpp:347
    if (R == 0) return CDX_OK;
    if (!ids || !exit_knob || !answer) return set_error(ctx, CDX_EINVAL, "sc_aggregate: null pointer");
    sc_aggregate_kernel<<<grid_of(ctx, R, 128), 128, 0, ctx->stream>>>(ids, R, P, S, exit_knob, answer, ctx->d_err);
    CDX_CHECK_LAUNCH(ctx, "sc_aggregate");
    return CDX_OK;
}

namespace cdx {
namespace {
template <typename RT>
int reward_aggregate_impl(cdx_ctx* ctx, const RT* rewards, const uint32_t* ids, const uint8_t* agg, uint64_t G,
                          uint32_t T, uint32_t W, const int32_t* exit_step, uint32_t* answer, uint64_t* inexact) {
    if (!ctx) return CDX_EINVAL;
    if (T == 0 || W == 0) return set_error(ctx, CDX_ERUNTIME, "aggregate: empty program");
    if (W > static_cast<uint32_t>(AG_MAX_W)) return set_error(ctx, CDX_EINVAL, "reward_aggregate: width above 256");
    if (inexact) {  // ABI v2 counter of approximated weights: every weight is exact now
        cudaError_t e = cudaMemsetAsync(inexact, 0, 8, ctx->stream);
        if (e != cudaSuccess) return cuda_fail(ctx, e, "reward_aggregate");
    }
    if (G == 0) return CDX_OK;
    if (!rewards || !ids || !agg || !exit_step || !answer)
        return set_error(ctx, CDX_EINVAL, "reward_aggregate: null pointer");
    const unsigned threads = W > 128 ? 32u : static_cast<unsigned>(AG_THREADS);
    const size_t smem = static_cast<size_t>(threads) * W * 12u;
    cudaFuncSetAttribute(reward_aggregate_kernel<RT>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         static_cast<int>(smem));
    const unsigned grid = static_cast<unsigned>((G + threads - 1) / threads);
    reward_aggregate_kernel<RT><<<grid, threads, smem, ctx->stream>>>(rewards, ids, agg, G, T, W, exit_step, answer,
                                                                      ctx->d_err);
    CDX_CHECK_LAUNCH(ctx, "reward_aggregate");
    return CDX_OK;
}
}  // namespace
}  // namespace cdx

extern "C" int cdx_reward_aggregate(cdx_ctx* ctx, const float* rewards, const uint32_t* ids, const uint8_t* agg,
                                    uint64_t G, uint32_t T, uint32_t W, const int32_t* exit_step, uint32_t* answer,
                                    uint64_t* inexact) {
    CDX_NVTX("cdx_reward_aggregate");
    return cdx::reward_aggregate_impl(ctx, rewards, ids, agg, G, T, W, exit_step, answer, inexact);
}

extern "C" int cdx_reward_aggregate_f64(cdx_ctx* ctx, const double* rewards, const uint32_t* ids, const uint8_t* agg,
                                        uint64_t G, uint32_t T, uint32_t W, const int32_t* exit_step,
                                        uint32_t* answer) {
    CDX_NVTX("cdx_reward_aggregate_f64");
    return cdx::reward_aggregate_impl(ctx, rewards, ids, agg, G, T, W, exit_step, answer, nullptr);
}

extern "C" int cdx_libm_exp(cdx_ctx* ctx, const double* x, uint64_t n, double* y) {
    using namespace cdx;
    CDX_NVTX("cdx_libm_exp");
    if (!ctx) return CDX_EINVAL;
    if (n == 0) return CDX_OK;
    if (!x || !y) return set_error(ctx, CDX_EINVAL, "libm_exp: null pointer");
    const unsigned grid = grid_of(ctx, n, 256);
    libm_exp_kernel<<<grid, 256, 0, ctx->stream>>>(x, n, y);
    CDX_CHECK_LAUNCH(ctx, "libm_exp");
    return CDX_OK;
}
