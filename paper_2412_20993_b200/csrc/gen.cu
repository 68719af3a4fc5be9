// gen.cu — synthetic reasoning-program traces generated on the device.
//
// Counter-based restatement of the reference's synthetic oracle (runtime.cpp:91-117,
// generate_workload :430-460): every draw is a pure function of (seed, program, sample,
// knob) built from the reference's own splitmix64 mixing (rng.hpp:25-34), so the device
// and the host checker (oracle/cdx_oracle.c) produce identical traces.  Integer math and
// exact double compares only.  Generation is never part of a timed region.
#include "cdx_internal.cuh"

namespace cdx {
namespace {

constexpr uint64_t TAG_SOLVABLE = 0x50175ULL;
constexpr uint64_t TAG_CONV = 0xC0117ULL;
constexpr uint64_t TAG_DISTRACT = 0xD15ULL;
constexpr uint64_t TAG_JITTER = 0x8E3AULL;
constexpr uint64_t HES_DOMAIN = 1ULL << 63;

__device__ __forceinline__ uint64_t mix64(uint64_t x) {
    x += 0x9e3779b97f4a7c15ULL;
    x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
    x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
    return x ^ (x >> 31);
}
__device__ __forceinline__ uint64_t derive_seed(uint64_t m, uint64_t a, uint64_t b) {
    return mix64(mix64(m ^ mix64(a)) ^ mix64(b ^ 0xa5a5a5a5a5a5a5a5ULL));
}
__device__ __forceinline__ double unit53(uint64_t h) {
    return __dmul_rn(static_cast<double>(h >> 11), 0x1.0p-53);
}

struct ProgState {
    bool solvable;
    uint32_t conv;
};

__device__ __forceinline__ ProgState prog_state(const cdx_gen_params& g, uint64_t r) {
    ProgState s;
    s.solvable = unit53(derive_seed(g.seed, r, TAG_SOLVABLE)) < g.solvable_fraction;
    const uint64_t span = static_cast<uint64_t>(g.conv_hi - g.conv_lo) + 1;
    s.conv = g.conv_lo + static_cast<uint32_t>(mix64(derive_seed(g.seed, r, TAG_CONV)) % span);
    return s;
}

__device__ __forceinline__ uint32_t answer(const cdx_gen_params& g, const ProgState& ps, uint64_t r,
                                           uint64_t j, uint32_t knob) {
    const uint64_t h = derive_seed(g.seed, r, (j << 32) | knob);
    const uint32_t distractor = 1 + static_cast<uint32_t>(mix64(h ^ TAG_DISTRACT) % (g.groups - 1));
    if (!ps.solvable) return distractor;
    const double noise = knob < ps.conv ? g.noise_level : g.residual_noise;
    if (noise > 0.0 && unit53(h) < noise) return distractor;
    return 0;
}

__device__ __forceinline__ uint32_t reward_k(const cdx_gen_params& g, const ProgState& ps, uint64_t r,
                                             uint64_t j, uint32_t knob) {
    int64_t mean;
    if (!ps.solvable) {
        mean = g.reward_unsolvable_k;
    } else {
        const uint32_t k = knob < ps.conv ? knob : ps.conv;
        mean = static_cast<int64_t>(g.reward_start_k) +
               (static_cast<int64_t>(g.reward_final_k) - static_cast<int64_t>(g.reward_start_k)) * k / ps.conv;
    }
    const uint64_t h = derive_seed(g.seed, r, (j << 32) | knob);
    const int64_t span = 2 * static_cast<int64_t>(g.reward_jitter_k) + 1;
    const int64_t jit = static_cast<int64_t>(mix64(h ^ TAG_JITTER) % static_cast<uint64_t>(span)) -
                        static_cast<int64_t>(g.reward_jitter_k);
    int64_t v = mean + jit;
    v = v < 0 ? 0 : (v > (1 << 24) ? (1 << 24) : v);
    return static_cast<uint32_t>(v);
}

// ids[r][p][s]
__global__ void gen_sc_kernel(cdx_gen_params g, uint64_t r0, uint64_t R, uint32_t P, uint32_t S,
                              uint32_t* __restrict__ ids) {
    const uint64_t total = R * P * S;
    for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < total;
         i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
        const uint32_t s = static_cast<uint32_t>(i % S);
        const uint64_t row = i / S;
        const uint32_t p = static_cast<uint32_t>(row % P);
        const uint64_t r = r0 + row / P;
        const ProgState ps = prog_state(g, r);
        ids[i] = answer(g, ps, r, s, p + 1);
    }
}

// one thread per request: ids[r][p] and hesitation words hes[r][ceil(P/64)]
__global__ void gen_cot_kernel(cdx_gen_params g, uint64_t r0, uint64_t R, uint32_t P,
                               uint32_t* __restrict__ ids, uint64_t* __restrict__ hes) {
    const uint32_t words = (P + 63) / 64;
    for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < R;
         i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
        const uint64_t r = r0 + i;
        const ProgState ps = prog_state(g, r);
        uint64_t word = 0;
        for (uint32_t p = 0; p < P; ++p) {
            const uint32_t a = answer(g, ps, r, 0, p + 1);
            const bool h = g.hesitation_prob > 0.0 &&
                           unit53(derive_seed(g.seed, r, HES_DOMAIN | p)) < g.hesitation_prob;
            ids[i * P + p] = h ? g.groups + a : a;
            if (h) word |= 1ULL << (p % 64);
            if (p % 64 == 63 || p == P - 1) {
                hes[i * words + p / 64] = word;
                word = 0;
            }
        }
    }
}

// rewards[g][t][w], ids[g][t][w]
__global__ void gen_reward_kernel(cdx_gen_params gp, uint64_t g0, uint64_t G, uint32_t T, uint32_t W,
                                  float* __restrict__ rewards, uint32_t* __restrict__ ids) {
    const uint64_t total = G * T * W;
    for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < total;
         i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
        const uint32_t w = static_cast<uint32_t>(i % W);
        const uint64_t gt = i / W;
        const uint32_t t = static_cast<uint32_t>(gt % T);
        const uint64_t g = g0 + gt / T;
        const ProgState ps = prog_state(gp, g);
        if (rewards) rewards[i] = static_cast<float>(reward_k(gp, ps, g, w, t + 1)) * 0x1.0p-24f;
        if (ids) ids[i] = answer(gp, ps, g, w, t + 1);
    }
}

int check_gen(cdx_ctx* ctx, const cdx_gen_params* g) {
    if (!ctx) return CDX_EINVAL;
    if (!g || g->groups < 2) return set_error(ctx, CDX_EINVAL, "spec: answer groups must be >= 2");
    if (g->conv_lo < 1 || g->conv_hi < g->conv_lo)
        return set_error(ctx, CDX_EINVAL, "workload: bad convergence range");
    if (g->noise_level < 0.0 || g->noise_level > 1.0)
        return set_error(ctx, CDX_EINVAL, "spec: noise_level outside [0,1]");
    if (g->residual_noise < 0.0 || g->residual_noise > 1.0)
        return set_error(ctx, CDX_EINVAL, "spec: residual_noise outside [0,1]");
    if (g->hesitation_prob < 0.0 || g->hesitation_prob > 1.0)
        return set_error(ctx, CDX_EINVAL, "spec: hesitation_prob outside [0,1]");
    if (g->solvable_fraction < 0.0 || g->solvable_fraction > 1.0)
        return set_error(ctx, CDX_EINVAL, "workload: solvable_fraction outside [0,1]");
    return CDX_OK;
}

uint32_t gen_grid(cdx_ctx* ctx, uint64_t work) {
    const uint64_t want = (work + 255) / 256;
    const uint64_t cap = static_cast<uint64_t>(ctx->sm_count) * 16;
    return static_cast<uint32_t>(want < cap ? (want ? want : 1) : cap);
}

}  // namespace
}  // namespace cdx

extern "C" {

int cdx_gen_sc(cdx_ctx* ctx, const cdx_gen_params* g, uint64_t r0, uint64_t R, uint32_t P,
               uint32_t S, uint32_t* ids) {
    if (int st = cdx::check_gen(ctx, g)) return st;
    if (!ids || P == 0 || S == 0) return cdx::set_error(ctx, CDX_EINVAL, "gen_sc: bad shape");
    if (R == 0) return CDX_OK;
    cdx::gen_sc_kernel<<<cdx::gen_grid(ctx, R * P * S), 256, 0, ctx->stream>>>(*g, r0, R, P, S, ids);
    CDX_CHECK_LAUNCH(ctx, "gen_sc");
    return CDX_OK;
}

int cdx_gen_cot(cdx_ctx* ctx, const cdx_gen_params* g, uint64_t r0, uint64_t R, uint32_t P,
                uint32_t* ids, uint64_t* hes) {
    if (int st = cdx::check_gen(ctx, g)) return st;
    if (!ids || !hes || P == 0) return cdx::set_error(ctx, CDX_EINVAL, "gen_cot: bad shape");
    if (R == 0) return CDX_OK;
    cdx::gen_cot_kernel<<<cdx::gen_grid(ctx, R), 256, 0, ctx->stream>>>(*g, r0, R, P, ids, hes);
    CDX_CHECK_LAUNCH(ctx, "gen_cot");
    return CDX_OK;
}

int cdx_gen_reward(cdx_ctx* ctx, const cdx_gen_params* g, uint64_t g0, uint64_t G, uint32_t T,
                   uint32_t W, float* rewards, uint32_t* ids) {
    if (int st = cdx::check_gen(ctx, g)) return st;
    if ((!rewards && !ids) || T == 0 || W == 0)
        return cdx::set_error(ctx, CDX_EINVAL, "gen_reward: bad shape");
    if (G == 0) return CDX_OK;
    cdx::gen_reward_kernel<<<cdx::gen_grid(ctx, G * T * W), 256, 0, ctx->stream>>>(*g, g0, G, T, W,
                                                                                   rewards, ids);
    CDX_CHECK_LAUNCH(ctx, "gen_reward");
    return CDX_OK;
}

}  // extern "C"
