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
//           exp() is the host libm's: rewards on the 2^-24 grid (the synthetic traces and
//           every value k/2^24) read a table of std::exp(k * 2^-24) built on the host once
//           per context, so the weights are the reference's bits; a reward off that grid
//           uses the device exp (<= 1 ulp from the host's) and is counted in *inexact.
// CoT's final answer is K3's final_id (probe::final_answer).  Answers are interned ids
// (equal id <=> equal trimmed bytes), so the winner's id is the reference's trimmed answer.

#include <cmath>
#include <vector>

#include "cdx_internal.cuh"

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

__device__ __forceinline__ double exp_ref(float r, const double* __restrict__ tab, unsigned long long* inexact) {
    const float s = r * 16777216.0f;  // exact scaling by 2^24
    if (r >= 0.0f && r <= 1.0f && s == truncf(s)) return __ldg(tab + static_cast<uint32_t>(s));
    atomicAdd(inexact, 1ull);
    return exp(static_cast<double>(r));
}

// MCTS / Rebase: thread per program, exit step t (0-based): paths = steps 0..t
__global__ void __launch_bounds__(AG_THREADS) reward_aggregate_kernel(
    const float* __restrict__ rw, const uint32_t* __restrict__ ids, const uint8_t* __restrict__ agg, uint64_t G,
    uint32_t T, uint32_t W, const int32_t* __restrict__ exit_step, const double* __restrict__ tab,
    uint32_t* __restrict__ answer, unsigned long long* inexact, int* err) {
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
        float bv = __ldg(rw + base);
        for (uint64_t i = 1; i < n; ++i) {
            const float v = __ldg(rw + base + i);
            if (static_cast<double>(v) > static_cast<double>(bv)) {
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
        const double e = exp_ref(__ldg(rw + l0 + i), tab, inexact);
        uint32_t c = 0;
        while (c < m && key[c] != v) ++c;
        if (c == m) {
            key[m] = v;
            wt[m] = 0.0;
            ++m;
        }
        wt[c] = __dadd_rn(wt[c], e);
    }
    uint32_t best = key[0];
    double bw = -1.0;
    for (uint32_t c = 0; c < m; ++c)
        if (wt[c] > bw) {
            bw = wt[c];
            best = key[c];
        }
    answer[g] = best;
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

extern "C" int cdx_reward_aggregate(cdx_ctx* ctx, const float* rewards, const uint32_t* ids, const uint8_t* agg,
                                    uint64_t G, uint32_t T, uint32_t W, const int32_t* exit_step, uint32_t* answer,
                                    uint64_t* inexact) {
    using namespace cdx;
    CDX_NVTX("cdx_reward_aggregate");
    if (!ctx) return CDX_EINVAL;
    if (T == 0 || W == 0) return set_error(ctx, CDX_ERUNTIME, "aggregate: empty program");
    if (W > static_cast<uint32_t>(AG_MAX_W)) return set_error(ctx, CDX_EINVAL, "reward_aggregate: width above 256");
    if (!inexact) return set_error(ctx, CDX_EINVAL, "reward_aggregate: null inexact counter");
    cudaError_t e = cudaMemsetAsync(inexact, 0, 8, ctx->stream);
    if (e != cudaSuccess) return cuda_fail(ctx, e, "reward_aggregate");
    if (G == 0) return CDX_OK;
    if (!rewards || !ids || !agg || !exit_step || !answer)
        return set_error(ctx, CDX_EINVAL, "reward_aggregate: null pointer");
    // std::exp on the 2^-24 grid of [0,1], from the host libm (the reference's exp)
    if (!ctx->exp_tab) {
        const size_t n = (1u << 24) + 1;
        std::vector<double> h(n);
        for (size_t k = 0; k < n; ++k) h[k] = std::exp(std::ldexp(static_cast<double>(k), -24));
        if (cudaMalloc(&ctx->exp_tab, n * sizeof(double)) != cudaSuccess)
            return set_error(ctx, CDX_ECUDA, "reward_aggregate: exp table allocation failed");
        e = cudaMemcpy(ctx->exp_tab, h.data(), n * sizeof(double), cudaMemcpyHostToDevice);
        if (e != cudaSuccess) return cuda_fail(ctx, e, "reward_aggregate: exp table upload");
    }
    const unsigned threads = W > 128 ? 32u : static_cast<unsigned>(AG_THREADS);
    const size_t smem = static_cast<size_t>(threads) * W * 12u;
    cudaFuncSetAttribute(reward_aggregate_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    const unsigned grid = static_cast<unsigned>((G + threads - 1) / threads);
    reward_aggregate_kernel<<<grid, threads, smem, ctx->stream>>>(rewards, ids, agg, G, T, W, exit_step, ctx->exp_tab,
                                                                  answer,
                                                                  reinterpret_cast<unsigned long long*>(inexact),
                                                                  ctx->d_err);
    CDX_CHECK_LAUNCH(ctx, "reward_aggregate");
    return CDX_OK;
}
