// k_reward.cu — K4: reward certaindex for MCTS (mean) / Rebase (max), cumulative over steps,
// with the cumulative answer-cluster certaindex beside it.
//
// Replaces the MCTS/Rebase branch of ProgramDriver::update_certaindex (runtime.cpp:279-292)
// evaluated after every step t of every program:
//   R_t  = certaindex_reward(RewardSet{all rewards of steps 0..t})      metrics.cpp:127-137
//   H~_t = certaindex_entropy(cluster_exact(all answers of steps 0..t))  metrics.cpp:21-37,120
//   meets_t = combined_meets_thresholds({H~_t, R_t}, thresholds[agg])   metrics.cpp:159-171
// The reference rebuilds both from scratch at every step (O(T^2 W) per program); here the
// left fold, the running first-maximum and the cluster table are carried across steps.
//
// Bit-exactness: one thread owns one program and folds its rewards in the reference's
// order (std::accumulate left fold in double, then / n; std::max_element's first maximum
// with operator<, so NaN propagation matches too).  Clusters are kept in first-seen order
// in a register table of KM slots; the entropy fold h -= T_n[count] uses host-built term
// rows T_n[c] = (c/n)*log(c/n) for n = (t+1)*W.  Programs with more than KM distinct
// answers are finished by the overflow kernel below: one warp per program with a
// shared-memory hash table (first-seen ordinals assigned by warp match + ballot).
//
// Data path: each step's [programs x W] slice of rewards and ids is staged by 3-D TMA
// (box {32, 1, PROGS}, 128-byte swizzle) so a thread reads its program's row without bank
// conflicts; a CTA walks its tile of programs step by step through a 2-deep ring.
#include <algorithm>
#include <cstdlib>
#include <vector>

#include "k_sc.cuh"

namespace cdx {
namespace {

constexpr int RW_PROGS = 64;   // programs (threads) per CTA
constexpr int RW_KM = 8;       // register cluster slots per program
constexpr int RW_STAGES = 2;
constexpr int RW_MAX_TH = 8;

struct RwParams {
    CUtensorMap tm_r;  // rewards {W, T, G}
    CUtensorMap tm_i;  // ids     {W, T, G}
    const float* rewards;
    const uint32_t* ids;
    const uint8_t* agg;
    float* R;
    float* H;
    uint32_t* meets;
    const double* tab;        // term rows, row t at row_off[t]
    const uint64_t* row_off;
    const double* logs;       // log(n_t)
    uint32_t* ovf_list;       // programs needing the overflow kernel
    uint32_t* ovf_count;
    int* d_err;
    uint64_t G;
    uint32_t T, W, words;     // words = ceil(T/32)
    uint32_t boxes;           // ceil(W/32)
    uint32_t stage_bytes;     // per array
    uint32_t stages;          // ring depth (<= RW_STAGES)
    int tma;
    int n_th[2];
    uint8_t th_sig[2][RW_MAX_TH];
    uint8_t th_dir[2][RW_MAX_TH];
    double th_cut[2][RW_MAX_TH];
};

__device__ __forceinline__ bool meets_th(const RwParams& p, int a, double hc, bool has_h, double rv) {
    bool ok = true;
    for (int t = 0; t < p.n_th[a]; ++t) {
        const double v = p.th_sig[a][t] == CDX_SIG_ENTROPY ? hc : rv;
        (void)has_h;
        const bool o = p.th_dir[a][t] == CDX_DIR_GE ? v >= p.th_cut[a][t] : v <= p.th_cut[a][t];
        ok = ok && o;
    }
    return ok;
}

__global__ void __launch_bounds__(RW_PROGS) reward_kernel(const __grid_constant__ RwParams p) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
    const uint32_t arrays = p.ids ? 2u : 1u;  // rewards (+ ids) staged per step
    uint64_t* bar = reinterpret_cast<uint64_t*>(smem + p.stages * arrays * p.stage_bytes);
    const uint32_t tid = threadIdx.x;
    const uint64_t g = static_cast<uint64_t>(blockIdx.x) * RW_PROGS + tid;
    const bool live = g < p.G;
    const bool with_ids = p.ids != nullptr;
    const uint64_t policy = policy_evict_first();
    const uint32_t T = p.T, W = p.W;

    if (p.tma && tid == 0) {
        tma_prefetch_desc(&p.tm_r);
        if (with_ids) tma_prefetch_desc(&p.tm_i);
        for (uint32_t s = 0; s < p.stages; ++s) mbar_init(&bar[s], 1);
        fence_mbar_init();
    }
    __syncthreads();
    auto issue = [&](uint32_t t, uint32_t stage) {
        uint8_t* dr = smem + stage * arrays * p.stage_bytes;
        uint8_t* di = dr + p.stage_bytes;
        mbar_expect_tx(&bar[stage], p.stage_bytes * (with_ids ? 2u : 1u));
        const int32_t g0 = static_cast<int32_t>(static_cast<uint64_t>(blockIdx.x) * RW_PROGS);
        for (uint32_t b = 0; b < p.boxes; ++b) {
            tma_load_3d(dr + b * RW_PROGS * 128u, &p.tm_r, static_cast<int32_t>(b * 32), static_cast<int32_t>(t), g0,
                        &bar[stage], policy);
            if (with_ids)
                tma_load_3d(di + b * RW_PROGS * 128u, &p.tm_i, static_cast<int32_t>(b * 32), static_cast<int32_t>(t),
                            g0, &bar[stage], policy);
        }
    };
    if (p.tma && tid == 0)
        for (uint32_t s = 0; s < p.stages && s < T; ++s) issue(s, s);

    const uint8_t a = live ? p.agg[g] : 0;
    double sum = 0.0;
    float best = 0.f;
    bool bad = false;
    uint32_t key[RW_KM], cnt[RW_KM];
#pragma unroll
    for (int k = 0; k < RW_KM; ++k) key[k] = cnt[k] = 0;
    uint32_t m = 0;
    bool ovf = false;
    uint32_t mword = 0;

    for (uint32_t t = 0; t < T; ++t) {
        const uint32_t stage = t % p.stages;
        const uint8_t* sr = smem + stage * arrays * p.stage_bytes;
        const uint8_t* si = sr + p.stage_bytes;
        if (p.tma) mbar_wait(&bar[stage], (t / p.stages) & 1u);
        if (live) {
            for (uint32_t w0 = 0; w0 < W; w0 += 4) {
                float rv4[4];
                uint32_t iv4[4] = {0, 0, 0, 0};
                if (p.tma) {
                    const uint32_t b = w0 >> 5, c = (w0 & 31u) >> 2;
                    const uint32_t off = b * RW_PROGS * 128u + swz128(tid, c);
                    const float4 f = *reinterpret_cast<const float4*>(sr + off);
                    rv4[0] = f.x; rv4[1] = f.y; rv4[2] = f.z; rv4[3] = f.w;
                    if (with_ids) {
                        const uint4 u = *reinterpret_cast<const uint4*>(si + off);
                        iv4[0] = u.x; iv4[1] = u.y; iv4[2] = u.z; iv4[3] = u.w;
                    }
                } else {
                    const uint64_t base = (g * T + t) * W + w0;
#pragma unroll
                    for (int e = 0; e < 4; ++e) {
                        rv4[e] = w0 + e < W ? __ldg(p.rewards + base + e) : 0.f;
                        if (with_ids) iv4[e] = w0 + e < W ? __ldg(p.ids + base + e) : 0u;
                    }
                }
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                    if (w0 + e >= W) break;
                    const float r = rv4[e];
                    bad = bad || (r < 0.f || r > 1.f);                 // metrics.cpp:129-132
                    sum = __dadd_rn(sum, static_cast<double>(r));      // std::accumulate
                    if (t == 0 && w0 + e == 0) best = r;               // std::max_element
                    else if (best < r) best = r;
                    if (with_ids && !ovf) {
                        const uint32_t v = iv4[e];
                        bool found = false;
#pragma unroll
                        for (int k = 0; k < RW_KM; ++k) {
                            const bool hit = static_cast<uint32_t>(k) < m && key[k] == v;
                            cnt[k] += hit ? 1u : 0u;
                            found = found || hit;
                        }
                        if (!found) {
                            if (m < RW_KM) {
#pragma unroll
                                for (int k = 0; k < RW_KM; ++k)
                                    if (static_cast<uint32_t>(k) == m) {
                                        key[k] = v;
                                        cnt[k] = 1;
                                    }
                                ++m;
                            } else {
                                ovf = true;  // more than KM clusters: the overflow kernel takes over
                            }
                        }
                    }
                }
            }
            const uint32_t n = (t + 1) * W;
            const double rv = a == CDX_AGG_MAX ? static_cast<double>(best) : __ddiv_rn(sum, static_cast<double>(n));
            if (p.R) p.R[g * T + t] = static_cast<float>(rv);
            double hc = 0.0;
            if (with_ids && !ovf) {
                if (n == 1) {
                    hc = 1.0;
                } else {
                    const double* Tn = p.tab + __ldg(p.row_off + t);
                    double h = 0.0;
#pragma unroll
                    for (int k = 0; k < RW_KM; ++k)
                        if (static_cast<uint32_t>(k) < m) h = __dsub_rn(h, __ldg(Tn + cnt[k]));
                    h = (0.0 < h) ? h : 0.0;
                    const double ln = __ldg(p.logs + t);
                    const double v = __ddiv_rn(__dsub_rn(ln, h), ln);
                    hc = v < 0.0 ? 0.0 : (1.0 < v ? 1.0 : v);
                }
                if (p.H) p.H[g * T + t] = static_cast<float>(hc);
            }
            if (!ovf && meets_th(p, a == CDX_AGG_MAX ? 1 : 0, hc, with_ids, rv)) mword |= 1u << (t & 31u);
            if (p.meets && ((t & 31u) == 31u || t == T - 1)) {
                if (!ovf) p.meets[g * p.words + (t >> 5)] = mword;
                mword = 0;
            }
        }
        if (p.tma) {
            __syncthreads();
            if (tid == 0 && t + p.stages < T) issue(t + p.stages, stage);
        }
    }
    if (live && bad) set_dev_err(p.d_err, DEV_REWARD_RANGE);
    if (live && ovf) {
        const uint32_t slot = atomicAdd(p.ovf_count, 1u);
        p.ovf_list[slot] = static_cast<uint32_t>(g);
    }
}

// ---------------------------------------------------------------------------------------
// Overflow kernel: one warp per program with > KM distinct answers.  A shared-memory hash
// table maps answer id -> first-seen ordinal; counts live per ordinal; the entropy fold
// walks ordinals 0..m-1 (first-seen order) on lane 0.  Rewards are recomputed here too, so
// the program's outputs are written by exactly one kernel.
constexpr int OV_WARPS = 4;

__global__ void __launch_bounds__(OV_WARPS * 32) reward_overflow_kernel(const __grid_constant__ RwParams p,
                                                                        uint32_t cap_log2) {
    extern __shared__ __align__(16) uint8_t smem[];
    const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const uint32_t cap = 1u << cap_log2;  // hash slots (>= 2 * T * W)
    const uint32_t nmax = p.T * p.W;
    uint32_t* hkey = reinterpret_cast<uint32_t*>(smem) + warp * (2 * cap + nmax);
    uint32_t* hord = hkey + cap;
    uint32_t* cnt = hord + cap;
    const uint32_t n_ovf = *p.ovf_count;
    for (uint32_t j = blockIdx.x * OV_WARPS + warp; j < n_ovf; j += gridDim.x * OV_WARPS) {
        const uint64_t g = p.ovf_list[j];
        for (uint32_t i = lane; i < cap; i += 32) hord[i] = 0xffffffffu;  // empty
        __syncwarp();
        uint32_t m = 0;
        double sum = 0.0;
        float best = 0.f;
        uint32_t mword = 0;
        const uint8_t a = p.agg[g];
        for (uint32_t t = 0; t < p.T; ++t) {
            const uint64_t base = (g * p.T + t) * p.W;
            for (uint32_t w0 = 0; w0 < p.W; w0 += 32) {
                const uint32_t w = w0 + lane;
                const bool act = w < p.W;
                const uint32_t v = act ? __ldg(p.ids + base + w) : 0xffffffffu;
                // first occurrence of each value inside this round of 32
                const uint32_t mm = __match_any_sync(0xffffffffu, v) & __ballot_sync(0xffffffffu, act);
                const bool lead = act && (mm & ((1u << lane) - 1u)) == 0u;
                // look the leader's value up; new values take ordinals in lane order
                uint32_t slot = (v * 0x9E3779B1u) >> (32 - cap_log2);
                bool fresh = false;
                if (lead) {
                    while (true) {
                        if (hord[slot] == 0xffffffffu) {
                            fresh = true;
                            break;
                        }
                        if (hkey[slot] == v) break;
                        slot = (slot + 1) & (cap - 1);
                    }
                }
                // new values take ordinals in lane order (= first-seen order); they may probe
                // into the same empty slot, so insert one at a time
                const uint32_t fb = __ballot_sync(0xffffffffu, fresh);
                for (uint32_t bits = fb; bits; bits &= bits - 1) {
                    const uint32_t l = __ffs(bits) - 1;
                    if (lane == l) {
                        uint32_t s2 = slot;
                        while (hord[s2] != 0xffffffffu) s2 = (s2 + 1) & (cap - 1);
                        hkey[s2] = v;
                        hord[s2] = m;
                        cnt[m] = 0;
                        slot = s2;
                    }
                    ++m;
                    __syncwarp();
                }
                if (lead) cnt[hord[slot]] += __popc(mm);
                __syncwarp();
            }
            // rewards: sequential left fold / first maximum on lane 0
            if (lane == 0) {
                for (uint32_t w = 0; w < p.W; ++w) {
                    const float r = __ldg(p.rewards + base + w);
                    sum = __dadd_rn(sum, static_cast<double>(r));
                    if (t == 0 && w == 0) best = r;
                    else if (best < r) best = r;
                }
                const uint32_t n = (t + 1) * p.W;
                const double rv = a == CDX_AGG_MAX ? static_cast<double>(best) : __ddiv_rn(sum, static_cast<double>(n));
                if (p.R) p.R[g * p.T + t] = static_cast<float>(rv);
                const double* Tn = p.tab + __ldg(p.row_off + t);
                double h = 0.0;
                for (uint32_t k = 0; k < m; ++k) h = __dsub_rn(h, __ldg(Tn + cnt[k]));
                h = (0.0 < h) ? h : 0.0;
                const double ln = __ldg(p.logs + t);
                const double v = __ddiv_rn(__dsub_rn(ln, h), ln);
                const double hc = n == 1 ? 1.0 : (v < 0.0 ? 0.0 : (1.0 < v ? 1.0 : v));
                if (p.H) p.H[g * p.T + t] = static_cast<float>(hc);
                if (meets_th(p, a == CDX_AGG_MAX ? 1 : 0, hc, true, rv)) mword |= 1u << (t & 31u);
                if (p.meets && ((t & 31u) == 31u || t == p.T - 1)) {
                    p.meets[g * p.words + (t >> 5)] = mword;
                    mword = 0;
                }
            }
            __syncwarp();
        }
    }
}

}  // namespace
}  // namespace cdx

extern "C" int cdx_reward_certaindex(cdx_ctx* ctx, const float* rewards, const uint32_t* ids, const uint8_t* agg,
                                     uint64_t G, uint32_t T, uint32_t W, const cdx_threshold* th_mean,
                                     uint32_t n_th_mean, const cdx_threshold* th_max, uint32_t n_th_max, float* R,
                                     float* H, uint32_t* meets_bits) {
    using namespace cdx;
    if (!ctx) return CDX_EINVAL;
    if (!rewards || !agg) return set_error(ctx, CDX_EINVAL, "reward_certaindex: null pointer");
    if (T == 0 || W == 0) return set_error(ctx, CDX_EINVAL, "certaindex_reward: empty reward set");
    if (static_cast<uint64_t>(T) * W > (1u << 16))
        return set_error(ctx, CDX_EINVAL, "reward_certaindex: at most 65536 paths per program");
    const bool present[4] = {ids != nullptr, true, false, false};
    if (int st = check_thresholds(ctx, th_mean, n_th_mean, present)) return st;
    if (int st = check_thresholds(ctx, th_max, n_th_max, present)) return st;
    if (G == 0) return CDX_OK;
    if (G > 0xffffffffull) return set_error(ctx, CDX_EINVAL, "reward_certaindex: at most 2^32-1 programs");

    RwParams p{};
    p.rewards = rewards;
    p.ids = ids;
    p.agg = agg;
    p.R = R;
    p.H = H;
    p.meets = meets_bits;
    p.d_err = ctx->d_err;
    p.G = G;
    p.T = T;
    p.W = W;
    p.words = (T + 31) / 32;
    p.boxes = (W + 31) / 32;
    p.stage_bytes = p.boxes * RW_PROGS * 128u;
    p.n_th[0] = static_cast<int>(n_th_mean);
    p.n_th[1] = static_cast<int>(n_th_max);
    for (uint32_t i = 0; i < n_th_mean; ++i) {
        p.th_sig[0][i] = th_mean[i].signal;
        p.th_dir[0][i] = th_mean[i].dir;
        p.th_cut[0][i] = th_mean[i].cutoff;
    }
    for (uint32_t i = 0; i < n_th_max; ++i) {
        p.th_sig[1][i] = th_max[i].signal;
        p.th_dir[1][i] = th_max[i].dir;
        p.th_cut[1][i] = th_max[i].cutoff;
    }
    // term rows for n_t = (t+1)*W
    std::vector<uint32_t> ns(T);
    for (uint32_t t = 0; t < T; ++t) ns[t] = (t + 1) * W;
    TermTables tt;
    if (ids) {
        if (int st = build_term_tables(ctx, ns.data(), T, &tt)) return st;
        p.tab = tt.tab;
        p.row_off = tt.row_off;
        p.logs = tt.logs;
    }
    // overflow list + counter
    auto* ov = static_cast<uint32_t*>(scratch(ctx, 64 + G * 4));
    if (!ov) return set_error(ctx, CDX_ECUDA, "reward_certaindex: scratch allocation failed");
    p.ovf_count = ov;
    p.ovf_list = ov + 16;
    cudaMemsetAsync(ov, 0, 64, ctx->stream);

    bool tma = (W % 4 == 0) && reinterpret_cast<uintptr_t>(rewards) % 16 == 0 &&
               (!ids || reinterpret_cast<uintptr_t>(ids) % 16 == 0) && G < (1ull << 31);
    if (tma) {
        const uint64_t dims[3] = {W, T, G};
        const uint64_t strides[2] = {static_cast<uint64_t>(W) * 4u, static_cast<uint64_t>(T) * W * 4u};
        const uint32_t box[3] = {32, 1, static_cast<uint32_t>(RW_PROGS)};
        tma = encode_tmap(&p.tm_r, rewards, 3, dims, strides, box, CU_TENSOR_MAP_DATA_TYPE_FLOAT32,
                          CU_TENSOR_MAP_SWIZZLE_128B) &&
              (!ids || encode_tmap(&p.tm_i, ids, 3, dims, strides, box, CU_TENSOR_MAP_DATA_TYPE_UINT32,
                                   CU_TENSOR_MAP_SWIZZLE_128B));
    }
    p.tma = tma ? 1 : 0;
    // one step staged per CTA (more resident CTAs beat a deeper ring here: each thread
    // needs its program's whole step row in shared memory); CDX_RW_STAGES=2 for a ring
    p.stages = 1;
    if (const char* e = getenv("CDX_RW_STAGES")) p.stages = std::max(1, std::min(RW_STAGES, atoi(e)));
    const size_t smem = tma ? 1024 + static_cast<size_t>(p.stages) * (ids ? 2 : 1) * p.stage_bytes + 8 * RW_STAGES
                            : 0;
    const unsigned grid = static_cast<unsigned>((G + RW_PROGS - 1) / RW_PROGS);
    if (tma) cudaFuncSetAttribute(reward_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    reward_kernel<<<grid, RW_PROGS, smem, ctx->stream>>>(p);
    CDX_CHECK_LAUNCH(ctx, "reward_certaindex");
    if (ids) {
        uint32_t cap_log2 = 1;
        while ((1u << cap_log2) < 2u * T * W) ++cap_log2;
        const size_t osmem = static_cast<size_t>(OV_WARPS) * ((2u << cap_log2) + T * W) * 4u;
        if (osmem > 200u * 1024u) {
            // very large programs: one warp per CTA
            return set_error(ctx, CDX_EINVAL, "reward_certaindex: T*W too large for the overflow table");
        }
        cudaFuncSetAttribute(reward_overflow_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(osmem));
        reward_overflow_kernel<<<ctx->sm_count, OV_WARPS * 32, osmem, ctx->stream>>>(p, cap_log2);
        CDX_CHECK_LAUNCH(ctx, "reward_certaindex(overflow)");
    }
    return CDX_OK;
}

namespace cdx {
namespace {
// Scalar façade path of metrics::certaindex_reward (metrics.cpp:127-137): one thread per
// RewardSet, the reference's left fold / first maximum in order, range check first.
__global__ void reward_sets_kernel(const double* __restrict__ v, const uint64_t* __restrict__ off,
                                   const uint8_t* __restrict__ agg, uint64_t rows, double* __restrict__ out,
                                   int* d_err) {
    for (uint64_t r = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; r < rows;
         r += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
        const uint64_t b = off[r], e = off[r + 1];
        if (b == e) {
            set_dev_err(d_err, DEV_EMPTY_REWARDS);
            continue;
        }
        bool bad = false;
        for (uint64_t i = b; i < e; ++i) bad = bad || v[i] < 0.0 || v[i] > 1.0;
        if (bad) {
            set_dev_err(d_err, DEV_REWARD_RANGE);
            continue;
        }
        if (agg[r] == CDX_AGG_MAX) {
            uint64_t best = b;
            for (uint64_t i = b + 1; i < e; ++i)
                if (v[best] < v[i]) best = i;
            out[r] = v[best];
        } else {
            double s = 0.0;
            for (uint64_t i = b; i < e; ++i) s = __dadd_rn(s, v[i]);
            out[r] = __ddiv_rn(s, static_cast<double>(e - b));
        }
    }
}
}  // namespace
}  // namespace cdx

extern "C" int cdx_reward_sets(cdx_ctx* ctx, const double* values, const uint64_t* row_off, const uint8_t* agg,
                               uint64_t rows, double* out) {
    using namespace cdx;
    if (!ctx) return CDX_EINVAL;
    if (!row_off || !agg || !out) return set_error(ctx, CDX_EINVAL, "reward_sets: null pointer");
    if (rows == 0) return CDX_OK;
    const uint64_t blocks = std::min<uint64_t>((rows + 127) / 128, static_cast<uint64_t>(ctx->sm_count) * 8);
    reward_sets_kernel<<<static_cast<unsigned>(blocks), 128, 0, ctx->stream>>>(values, row_off, agg, rows, out,
                                                                               ctx->d_err);
    CDX_CHECK_LAUNCH(ctx, "reward_sets");
    return CDX_OK;
}
