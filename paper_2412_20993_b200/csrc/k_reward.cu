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
#include <cmath>
#include <cstring>
#include <cstdlib>
#include <vector>

#include "k_sc.cuh"

namespace cdx {
namespace {

constexpr int RW_PROGS = 64;   // programs (threads) per CTA
constexpr int RW_KM = 8;       // register cluster slots per program
constexpr int RW_STAGES = 2;
constexpr int RW_MAX_TH = 8;
constexpr int RQ_PROGS = 32;   // quad kernel: programs per CTA (4 lanes each)
constexpr int RQ_MAX_T = 256;  // quad kernel: steps staged in the smem output tile (8 B per program-step)
constexpr int RQ_MAX_BOXES = 4;  // quad kernel: W <= 128

struct RwParams {
    CUtensorMap tm_r;  // rewards {W, T, G}, box {32, 1, RW_PROGS}
    CUtensorMap tm_i;  // ids     {W, T, G}
    CUtensorMap tq_r;  // rewards, box {32, 1, RQ_PROGS} (quad kernel)
    CUtensorMap tq_i;  // ids
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
    uint64_t bstride;         // quad kernel: block b takes program block (b * bstride) mod grid (1: in order)
    uint32_t T, W, words;     // words = ceil(T/32)
    uint32_t boxes;           // ceil(W/32)
    uint32_t stage_bytes;     // per array
    uint32_t stages;          // ring depth (<= RW_STAGES)
    int tma;
    int n_th[2];
    // the AND of inclusive thresholds per (aggregation, signal) as one closed interval:
    // lo = max of the >= cutoffs, hi = min of the <= cutoffs; has = any threshold on it
    double box_lo[2][2], box_hi[2][2];
    uint8_t box_has[2][2];
    uint8_t box_never[2];     // a NaN cutoff: every compare false (metrics.cpp:167)
    uint8_t th_sig[2][RW_MAX_TH];
    uint8_t th_dir[2][RW_MAX_TH];
    double th_cut[2][RW_MAX_TH];
};

// combined_meets_thresholds over {H~, R} (metrics.cpp:159-171): an AND of inclusive
// compares is the interval test above (NaN fails either way); signals without a threshold
// are not looked at, as in the reference.
__device__ __forceinline__ bool meets_box(const RwParams& p, int a, double hc, double rv) {
    if (p.box_never[a]) return false;
    const bool okh = !p.box_has[a][0] || (hc >= p.box_lo[a][0] && hc <= p.box_hi[a][0]);
    const bool okr = !p.box_has[a][1] || (rv >= p.box_lo[a][1] && rv <= p.box_hi[a][1]);
    return okh && okr;
}

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
// Quad kernel (W in {32, 48, 64, ..., 128}, T <= 256): FOUR lanes per program, 32 programs per CTA.
//
// Per step every lane takes W/4 of the program's nodes straight from the TMA-staged,
// 128B-swizzled step slice (the half of a box a lane reads alternates with the program's
// parity, so the 8 lanes of a quarter-warp always hit 8 distinct bank groups).  Per node
// the work is kept to a handful of instructions:
//   * rewards: the unsigned max and (min - 1) of the float bits (two min/max ops) and an
//     FP64 add into the lane's partial sum.  On this path summation order does not matter:
//     when every reward is +0 or a float in [2^-(30-L), 1] (n <= 2^L paths), every partial
//     sum is a multiple of 2^-(53-L) below 2^L and exact in double, so the quad's sum equals
//     the reference's left fold (std::accumulate, metrics.cpp:135) bit for bit, and the max
//     of the bits is the max of the values (std::max_element, :133).  Anything else (tiny,
//     -0.0, negative, NaN, > 1) sends the program to the serial overflow kernel, which folds
//     in the reference's order and performs the range check (metrics.cpp:129-132).
//   * clusters: KW compares against the first-seen table (keys replicated in the 4 lanes),
//     KW = the warp's largest table size; each hit is a predicated increment.  Unused slots
//     duplicate key 0, so no slot-validity test sits on the hot compare.  A value in no
//     valid slot is a miss, detected once per step from the hit total; a step with a miss is
//     re-walked by its quad in node order (smem broadcast reads) to append new keys in
//     first-seen order and count their occurrences.  More than KM keys -> overflow kernel.
// After each step the quad sums its counters (packed xor-shuffles), lane 0 folds
// h -= T_n[count] in first-seen order (host term row n = (t+1)W), clamps, applies the
// thresholds and stages R / H~ in a smem tile that is written out coalesced at the end.
struct QuadLane {
    double psum = 0.0;         // exact partial sum of this lane's rewards
    uint32_t maxb = 0;         // max float bits (rewards are >= +0 on the exact path)
    uint32_t minb = 0xffffffffu;  // min of (bits - 1): +0 maps to 0xffffffff
    uint32_t key[RW_KM], cnt[RW_KM];
};

template <int K, int BOXES, bool HALF>
__device__ __forceinline__ void quad_pass(QuadLane& L, const uint8_t* sr, const uint8_t* si, uint32_t box_bytes,
                                          uint32_t prow, uint32_t q, bool with_ids, uint32_t W) {
#pragma unroll
    for (uint32_t j = 0; j < 2 * BOXES; ++j) {
        const uint32_t b = j >> 1, h = (j ^ prow) & 1u;
        if (HALF && b * 32u + h * 16u >= W) continue;  // W % 16 == 0: a half box is all in or all out
        const uint32_t off = b * box_bytes + swz128(prow, h * 4u + q);
        const uint4 f = *reinterpret_cast<const uint4*>(sr + off);
        const uint32_t rb[4] = {f.x, f.y, f.z, f.w};
#pragma unroll
        for (int e = 0; e < 4; ++e) {
            L.maxb = max(L.maxb, rb[e]);
            L.minb = min(L.minb, rb[e] - 1u);
            L.psum = __dadd_rn(L.psum, static_cast<double>(__uint_as_float(rb[e])));
        }
        if (K > 0 && with_ids) {
            const uint4 u = *reinterpret_cast<const uint4*>(si + off);
            const uint32_t iv[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
            for (int e = 0; e < 4; ++e) {
#pragma unroll
                for (int k = 0; k < K; ++k)  // ISETP + predicated IADD per slot
                    asm("{\n\t.reg .pred p;\n\tsetp.eq.u32 p, %1, %2;\n\t@p add.u32 %0, %0, 1;\n\t}"
                        : "+r"(L.cnt[k])
                        : "r"(L.key[k]), "r"(iv[e]));
            }
        }
    }
}

template <int BOXES, bool HALF>
__device__ __forceinline__ void quad_pass_k(int K, QuadLane& L, const uint8_t* sr, const uint8_t* si,
                                            uint32_t box_bytes, uint32_t prow, uint32_t q, bool with_ids, uint32_t W) {
    switch (K) {  // warp-uniform
        case 0: quad_pass<0, BOXES, HALF>(L, sr, si, box_bytes, prow, q, with_ids, W); break;
        case 1: quad_pass<1, BOXES, HALF>(L, sr, si, box_bytes, prow, q, with_ids, W); break;
        case 2: quad_pass<2, BOXES, HALF>(L, sr, si, box_bytes, prow, q, with_ids, W); break;
        case 3: quad_pass<3, BOXES, HALF>(L, sr, si, box_bytes, prow, q, with_ids, W); break;
        case 4: quad_pass<4, BOXES, HALF>(L, sr, si, box_bytes, prow, q, with_ids, W); break;
        case 5: quad_pass<5, BOXES, HALF>(L, sr, si, box_bytes, prow, q, with_ids, W); break;
        case 6: quad_pass<6, BOXES, HALF>(L, sr, si, box_bytes, prow, q, with_ids, W); break;
        case 7: quad_pass<7, BOXES, HALF>(L, sr, si, box_bytes, prow, q, with_ids, W); break;
        default: quad_pass<8, BOXES, HALF>(L, sr, si, box_bytes, prow, q, with_ids, W); break;
    }
}

// HALF: W % 32 == 16 (the last box is half past W: those nodes are skipped)
template <int BOXES, bool HALF>
__global__ void __launch_bounds__(RQ_PROGS * 4) reward_quad_kernel(const __grid_constant__ RwParams p,
                                                                   uint32_t exact_min_bits) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
    const bool with_ids = p.ids != nullptr;
    const uint32_t arrays = with_ids ? 2u : 1u;
    const uint32_t box_bytes = RQ_PROGS * 128u;
    const uint32_t stage_bytes = BOXES * box_bytes;  // per array
    uint64_t* bar = reinterpret_cast<uint64_t*>(smem + p.stages * arrays * stage_bytes);
    float* outR = reinterpret_cast<float*>(smem + p.stages * arrays * stage_bytes + 64);
    float* outH = outR + RQ_PROGS * p.T;
    uint32_t* outM = reinterpret_cast<uint32_t*>(outH + RQ_PROGS * p.T);

    const uint32_t tid = threadIdx.x, lane = tid & 31u;
    const uint32_t prow = tid >> 2, q = tid & 3u;  // program row in the CTA, lane in the quad
    const uint64_t blk = p.bstride == 1 ? blockIdx.x : (static_cast<uint64_t>(blockIdx.x) * p.bstride) % gridDim.x;
    const uint64_t g0 = blk * RQ_PROGS;
    const uint64_t g = g0 + prow;
    const bool live = g < p.G;
    const uint32_t T = p.T, W = p.W;
    const uint32_t per_lane = W / 4;
    const uint64_t policy = policy_evict_first();

    if (tid == 0) {
        tma_prefetch_desc(&p.tq_r);
        if (with_ids) tma_prefetch_desc(&p.tq_i);
        for (uint32_t s = 0; s < p.stages; ++s) mbar_init(&bar[s], 1);
        fence_mbar_init();
    }
    __syncthreads();
    auto issue = [&](uint32_t t, uint32_t stage) {
        uint8_t* dr = smem + stage * arrays * stage_bytes;
        mbar_expect_tx(&bar[stage], stage_bytes * arrays);
        for (uint32_t b = 0; b < BOXES; ++b) {
            tma_load_3d(dr + b * box_bytes, &p.tq_r, static_cast<int32_t>(b * 32), static_cast<int32_t>(t),
                        static_cast<int32_t>(g0), &bar[stage], policy);
            if (with_ids)
                tma_load_3d(dr + stage_bytes + b * box_bytes, &p.tq_i, static_cast<int32_t>(b * 32),
                            static_cast<int32_t>(t), static_cast<int32_t>(g0), &bar[stage], policy);
        }
    };
    if (tid == 0)
        for (uint32_t s = 0; s < p.stages && s < T; ++s) issue(s, s);

    const uint8_t a = live ? p.agg[g] : 0;
    QuadLane L;
#pragma unroll
    for (int k = 0; k < RW_KM; ++k) L.key[k] = L.cnt[k] = 0;
    uint32_t m = 0;
    bool ovf = !live;
    const uint32_t qmask = 0xFu << (lane & ~3u);
    uint32_t before = 0;  // this lane's hits on valid slots so far (a miss = fewer new hits than nodes)
    struct {
        double tot;
        uint32_t mx, m, t;
        uint32_t tc[RW_KM];
        bool ovf, valid;
    } pend{};
    for (uint32_t i = tid; i < RQ_PROGS * p.words; i += blockDim.x) outM[i] = 0;  // bits land by atomicOr
    __syncthreads();

    uint32_t stage = 0, phase = 0;
    for (uint32_t t = 0; t < T; ++t) {
        const uint8_t* sr = smem + stage * arrays * stage_bytes;
        const uint8_t* si = sr + stage_bytes;
        const int kw = with_ids ? static_cast<int>(__reduce_max_sync(0xffffffffu, ovf ? 0u : m)) : 0;
        mbar_wait(&bar[stage], phase);
        quad_pass_k<BOXES, HALF>(kw, L, sr, si, box_bytes, prow, q, with_ids, W);
        if (with_ids) {
            uint32_t after = 0;
#pragma unroll
            for (int k = 0; k < RW_KM; ++k) after += static_cast<uint32_t>(k) < m ? L.cnt[k] : 0u;
            const bool miss = after - before < per_lane;
            uint32_t ins = 0;  // this lane's nodes counted into slots appended this step
            // ---- first-seen insertion.  One scan marks this lane's nodes whose value is in no
            // valid slot (a bit per node, ascending node order); each round the quad takes its
            // earliest marked node (the next cluster in first-seen order), all 4 lanes append
            // it, and each lane counts and clears its own marked nodes holding that value.
            // Rounds run while any quad of the warp has marks (warp-uniform loop).
            bool need = (__ballot_sync(0xffffffffu, miss && !ovf) & qmask) != 0;  // quad-uniform
            if (__any_sync(0xffffffffu, need)) {
                constexpr int NV = 8 * BOXES;  // this lane's nodes per step
                uint32_t iv[NV];
                uint32_t mk = 0;  // bit i: own node i (node w = b*32 + h*16 + q*4 + e, i = (2b+h)*4 + e)
#pragma unroll
                for (uint32_t j = 0; j < 2 * BOXES; ++j) {
                    const uint32_t b = j >> 1, h = j & 1u;
                    const uint4 u = *reinterpret_cast<const uint4*>(si + b * box_bytes + swz128(prow, h * 4u + q));
                    iv[4 * j] = u.x;
                    iv[4 * j + 1] = u.y;
                    iv[4 * j + 2] = u.z;
                    iv[4 * j + 3] = u.w;
                }
                if (need) {
#pragma unroll
                    for (int i = 0; i < NV; ++i) {
                        if (HALF && static_cast<uint32_t>(i >> 3) * 32u + static_cast<uint32_t>((i >> 2) & 1) * 16u >= W)
                            continue;  // node past W (zero-filled by TMA): never a cluster
                        bool in = false;  // unused slots duplicate key 0, so no validity test
#pragma unroll
                        for (int k = 0; k < RW_KM; ++k) in = in || L.key[k] == iv[i];
                        if (!(in && m > 0)) mk |= 1u << i;
                    }
                }
                while (__any_sync(0xffffffffu, need)) {
                    uint32_t wmin = 0xffffffffu, vmin = 0;
                    if (mk) {
                        const uint32_t i = static_cast<uint32_t>(__ffs(mk) - 1);
                        wmin = (i >> 3) * 32u + ((i >> 2) & 1u) * 16u + q * 4u + (i & 3u);
#pragma unroll
                        for (int k = 0; k < NV; ++k)
                            if (static_cast<uint32_t>(k) == i) vmin = iv[k];
                    }
#pragma unroll
                    for (int o = 1; o <= 2; o <<= 1) {  // quad min over (w, value of w)
                        const uint32_t w2 = __shfl_xor_sync(0xffffffffu, wmin, o);
                        const uint32_t v2 = __shfl_xor_sync(0xffffffffu, vmin, o);
                        if (w2 < wmin) {
                            wmin = w2;
                            vmin = v2;
                        }
                    }
                    need = need && wmin != 0xffffffffu;
                    if (need && m == RW_KM) {  // a ninth cluster: the overflow kernel finishes it
                        ovf = true;
                        need = false;
                    }
                    if (need) {
                        uint32_t c = 0;
#pragma unroll
                        for (int i = 0; i < NV; ++i) {
                            const bool hit = ((mk >> i) & 1u) && iv[i] == vmin;
                            c += hit ? 1u : 0u;
                            mk &= hit ? ~(1u << i) : 0xffffffffu;
                        }
#pragma unroll
                        for (int k = 0; k < RW_KM; ++k) {
                            if (static_cast<uint32_t>(k) == m || (m == 0 && k > 0)) L.key[k] = vmin;  // dup key 0
                            if (static_cast<uint32_t>(k) == m) L.cnt[k] = c;
                        }
                        ins += c;
                        ++m;
                    }
                }
            }
            before = after + ins;  // the valid slots' total: old slots (after) + appended ones
        }
        // ---- quad totals
        double tot = L.psum;
        tot = __dadd_rn(tot, __shfl_xor_sync(0xffffffffu, tot, 1));
        tot = __dadd_rn(tot, __shfl_xor_sync(0xffffffffu, tot, 2));
        uint32_t mx = L.maxb;
        mx = max(mx, __shfl_xor_sync(0xffffffffu, mx, 1));
        mx = max(mx, __shfl_xor_sync(0xffffffffu, mx, 2));
        uint32_t tc[RW_KM];
        if (with_ids) {
#pragma unroll
            for (int k = 0; k < RW_KM; k += 2) {  // counts <= 65535: two per shuffle
                uint32_t pk = L.cnt[k] | (L.cnt[k + 1] << 16);
                pk += __shfl_xor_sync(0xffffffffu, pk, 1);
                pk += __shfl_xor_sync(0xffffffffu, pk, 2);
                tc[k] = pk & 0xffffu;
                tc[k + 1] = pk >> 16;
            }
        }
        const uint32_t ovf_bal = __ballot_sync(0xffffffffu, ovf);  // every lane votes (no short circuit)
        ovf = ovf || (ovf_bal & qmask) != 0;
        // ---- the fold is deferred: lane t % 4 keeps step t's totals, and every 4 steps the
        // quad's 4 lanes fold 4 steps at once (the fold is serial per step, so it would
        // otherwise run on one lane of four)
        if ((t & 3u) == q) {
            pend.t = t;
            pend.tot = tot;
            pend.mx = mx;
            pend.m = m;
            pend.ovf = ovf;
#pragma unroll
            for (int k = 0; k < RW_KM; ++k) pend.tc[k] = with_ids ? tc[k] : 0u;
            pend.valid = true;
        }
        if ((t & 3u) == 3u || t + 1 == T) {
            if (pend.valid && live) {
                const uint32_t pt = pend.t;
                const uint32_t n = (pt + 1) * W;
                const double rv = a == CDX_AGG_MAX ? static_cast<double>(__uint_as_float(pend.mx))
                                                   : __ddiv_rn(pend.tot, static_cast<double>(n));
                double hc = 0.0;
                if (with_ids && !pend.ovf) {
                    if (n == 1) {
                        hc = 1.0;
                    } else {
                        const double* Tn = p.tab + __ldg(p.row_off + pt);
                        double term[RW_KM];  // every tc[k] <= n (unused slots count key-0 hits)
#pragma unroll
                        for (int k = 0; k < RW_KM; ++k) term[k] = __ldg(Tn + pend.tc[k]);
                        double hh = 0.0;
#pragma unroll
                        for (int k = 0; k < RW_KM; ++k)
                            if (static_cast<uint32_t>(k) < pend.m) hh = __dsub_rn(hh, term[k]);
                        hh = (0.0 < hh) ? hh : 0.0;
                        const double ln = __ldg(p.logs + pt);
                        const double v = __ddiv_rn(__dsub_rn(ln, hh), ln);
                        hc = v < 0.0 ? 0.0 : (1.0 < v ? 1.0 : v);
                    }
                }
                outR[prow * T + pt] = static_cast<float>(rv);
                outH[prow * T + pt] = static_cast<float>(hc);
                if (meets_box(p, a == CDX_AGG_MAX ? 1 : 0, hc, rv))
                    atomicOr(&outM[prow * p.words + (pt >> 5)], 1u << (pt & 31u));
            }
            pend.valid = false;
        }
        __syncthreads();  // every lane is done with this stage
        if (tid == 0 && t + p.stages < T) issue(t + p.stages, stage);
        if (++stage == p.stages) {
            stage = 0;
            phase ^= 1u;
        }
    }
    // ---- programs the fast path cannot finish go to the serial overflow kernel:
    // every reward must be +0 or in [2^-(30-L), 1] (bits in [exact_min_bits, 0x3f800000])
    const bool inexact = L.maxb > 0x3f800000u || (L.minb != 0xffffffffu && L.minb + 1u < exact_min_bits);
    const bool qinexact = (__ballot_sync(0xffffffffu, inexact) & qmask) != 0;
    if (live && q == 0 && (ovf || qinexact)) {
        const uint32_t slot = atomicAdd(p.ovf_count, 1u);
        p.ovf_list[slot] = static_cast<uint32_t>(g);
    }
    __syncthreads();
    // ---- coalesced write-out of the staged tiles (overflow programs are rewritten later)
    const uint64_t nprog = p.G - g0 < RQ_PROGS ? p.G - g0 : RQ_PROGS;
    const uint64_t span = nprog * T;
    for (uint64_t i = tid; i < span; i += blockDim.x) {
        if (p.R) p.R[g0 * T + i] = outR[i];
        if (p.H && with_ids) p.H[g0 * T + i] = outH[i];
    }
    if (p.meets)
        for (uint64_t i = tid; i < nprog * p.words; i += blockDim.x) p.meets[g0 * p.words + i] = outM[i];
}

// ---------------------------------------------------------------------------------------
// Overflow kernel: one warp per program with > KM distinct answers.  A shared-memory hash
// table maps answer id -> first-seen ordinal; counts live per ordinal; the entropy fold
// walks ordinals 0..m-1 (first-seen order) on lane 0.  Rewards are recomputed here too, so
// the program's outputs are written by exactly one kernel.
constexpr int OV_WARPS = 4;

// gtab (nullable): programs too large for a shared-memory table (2 * cap + T * W words per
// warp over ~220 KB) keep it in global memory instead, one slice per warp of the grid.
// RT = double: the f64 entry (cdx_reward_certaindex_f64) runs every program here (all = 1:
// program j of the grid-stride loop is program j, no overflow list).
template <typename RT>
__global__ void __launch_bounds__(OV_WARPS * 32) reward_overflow_kernel(const __grid_constant__ RwParams p,
                                                                        uint32_t cap_log2, uint32_t* gtab,
                                                                        const RT* __restrict__ rw, uint32_t all) {
    extern __shared__ __align__(16) uint8_t smem[];
    const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    const uint32_t cap = 1u << cap_log2;  // hash slots (>= 2 * T * W)
    const uint32_t nmax = p.ids ? p.T * p.W : 0u;
    uint32_t* hkey = gtab ? gtab + static_cast<size_t>(blockIdx.x * nw + warp) * (2 * cap + nmax)
                          : reinterpret_cast<uint32_t*>(smem) + warp * (2 * cap + nmax);
    uint32_t* hord = hkey + cap;
    uint32_t* cnt = hord + cap;
    const uint64_t n_ovf = all ? p.G : *p.ovf_count;
    for (uint64_t j = blockIdx.x * nw + warp; j < n_ovf; j += static_cast<uint64_t>(gridDim.x) * nw) {
        const uint64_t g = all ? j : p.ovf_list[j];
        for (uint32_t i = lane; p.ids && i < cap; i += 32) hord[i] = 0xffffffffu;  // empty
        __syncwarp();
        uint32_t m = 0;
        double sum = 0.0;
        RT best = 0;
        uint32_t mword = 0;
        const uint8_t a = p.agg[g];
        for (uint32_t t = 0; t < p.T; ++t) {
            const uint64_t base = (g * p.T + t) * p.W;
            for (uint32_t w0 = 0; p.ids && w0 < p.W; w0 += 32) {
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
                    const RT r = __ldg(rw + base + w);
                    if (r < RT(0) || r > RT(1)) set_dev_err(p.d_err, DEV_REWARD_RANGE);  // metrics.cpp:129-132
                    sum = __dadd_rn(sum, static_cast<double>(r));
                    if (t == 0 && w == 0) best = r;
                    else if (best < r) best = r;
                }
                const uint32_t n = (t + 1) * p.W;
                const double rv = a == CDX_AGG_MAX ? static_cast<double>(best) : __ddiv_rn(sum, static_cast<double>(n));
                if (p.R) p.R[g * p.T + t] = static_cast<float>(rv);
                double hc = 0.0;
                if (p.ids) {
                    const double* Tn = p.tab + __ldg(p.row_off + t);
                    double h = 0.0;
                    for (uint32_t k = 0; k < m; ++k) h = __dsub_rn(h, __ldg(Tn + cnt[k]));
                    h = (0.0 < h) ? h : 0.0;
                    const double ln = __ldg(p.logs + t);
                    const double v = __ddiv_rn(__dsub_rn(ln, h), ln);
                    hc = n == 1 ? 1.0 : (v < 0.0 ? 0.0 : (1.0 < v ? 1.0 : v));
                    if (p.H) p.H[g * p.T + t] = static_cast<float>(hc);
                }
                if (meets_th(p, a == CDX_AGG_MAX ? 1 : 0, hc, p.ids != nullptr, rv)) mword |= 1u << (t & 31u);
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

namespace cdx {
namespace {
int reward_certaindex_impl(cdx_ctx* ctx, const float* rewards, const double* rewards64, const uint32_t* ids,
                           const uint8_t* agg, uint64_t G, uint32_t T, uint32_t W, const cdx_threshold* th_mean,
                           uint32_t n_th_mean, const cdx_threshold* th_max, uint32_t n_th_max, float* R, float* H,
                           uint32_t* meets_bits);
}  // namespace
}  // namespace cdx

extern "C" int cdx_reward_certaindex(cdx_ctx* ctx, const float* rewards, const uint32_t* ids, const uint8_t* agg,
                                     uint64_t G, uint32_t T, uint32_t W, const cdx_threshold* th_mean,
                                     uint32_t n_th_mean, const cdx_threshold* th_max, uint32_t n_th_max, float* R,
                                     float* H, uint32_t* meets_bits) {
    CDX_NVTX("cdx_reward_certaindex");
    if (!rewards && ctx) return cdx::set_error(ctx, CDX_EINVAL, "reward_certaindex: null pointer");
    return cdx::reward_certaindex_impl(ctx, rewards, nullptr, ids, agg, G, T, W, th_mean, n_th_mean, th_max, n_th_max,
                                       R, H, meets_bits);
}

extern "C" int cdx_reward_certaindex_f64(cdx_ctx* ctx, const double* rewards, const uint32_t* ids,
                                         const uint8_t* agg, uint64_t G, uint32_t T, uint32_t W,
                                         const cdx_threshold* th_mean, uint32_t n_th_mean,
                                         const cdx_threshold* th_max, uint32_t n_th_max, float* R, float* H,
                                         uint32_t* meets_bits) {
    CDX_NVTX("cdx_reward_certaindex_f64");
    if (!rewards && ctx) return cdx::set_error(ctx, CDX_EINVAL, "reward_certaindex: null pointer");
    return cdx::reward_certaindex_impl(ctx, nullptr, rewards, ids, agg, G, T, W, th_mean, n_th_mean, th_max, n_th_max,
                                       R, H, meets_bits);
}

namespace cdx {
namespace {
int reward_certaindex_impl(cdx_ctx* ctx, const float* rewards, const double* rewards64, const uint32_t* ids,
                           const uint8_t* agg, uint64_t G, uint32_t T, uint32_t W, const cdx_threshold* th_mean,
                           uint32_t n_th_mean, const cdx_threshold* th_max, uint32_t n_th_max, float* R, float* H,
                           uint32_t* meets_bits) {
    if (!ctx) return CDX_EINVAL;
    if (!agg) return set_error(ctx, CDX_EINVAL, "reward_certaindex: null pointer");
    if (T == 0 || W == 0) return set_error(ctx, CDX_EINVAL, "certaindex_reward: empty reward set");
    if (static_cast<uint64_t>(T) * W > (1u << 16))
        return set_error(ctx, CDX_EINVAL, "reward_certaindex: at most 65536 paths per program");
    const bool present[5] = {ids != nullptr, true, false, false, false};
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
    for (int a = 0; a < 2; ++a) {
        const cdx_threshold* th = a ? th_max : th_mean;
        const uint32_t n = a ? n_th_max : n_th_mean;
        for (int sg = 0; sg < 2; ++sg) {
            p.box_lo[a][sg] = -INFINITY;
            p.box_hi[a][sg] = INFINITY;
            p.box_has[a][sg] = 0;
        }
        p.box_never[a] = 0;
        for (uint32_t i = 0; i < n; ++i) {
            const int sg = th[i].signal == CDX_SIG_ENTROPY ? 0 : 1;  // validated: entropy or reward
            p.box_has[a][sg] = 1;
            if (std::isnan(th[i].cutoff)) p.box_never[a] = 1;
            if (th[i].dir == CDX_DIR_GE) p.box_lo[a][sg] = std::max(p.box_lo[a][sg], th[i].cutoff);
            else p.box_hi[a][sg] = std::min(p.box_hi[a][sg], th[i].cutoff);
        }
    }
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

    // f64 rewards: every program through the warp-per-program kernel (left fold on lane 0)
    const bool f64 = rewards64 != nullptr;
    bool tma = !f64 && (W % 4 == 0) && reinterpret_cast<uintptr_t>(rewards) % 16 == 0 &&
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
    // W % 32 == 16 above one box (48, 80, 112): the last box runs half empty, still well ahead of
    // the one-thread kernel; W = 16 is not (half of every box would be wasted)
    const bool quad = tma && (W % 32 == 0 || (W % 16 == 0 && W > 32)) && W <= 32u * RQ_MAX_BOXES &&
                      T <= static_cast<uint32_t>(RQ_MAX_T) &&
                      !getenv("CDX_RW_LEGACY");
    bool launched_quad = false;
    if (quad) {
        const uint64_t dims[3] = {W, T, G};
        const uint64_t strides[2] = {static_cast<uint64_t>(W) * 4u, static_cast<uint64_t>(T) * W * 4u};
        const uint32_t box[3] = {32, 1, static_cast<uint32_t>(RQ_PROGS)};
        if (encode_tmap(&p.tq_r, rewards, 3, dims, strides, box, CU_TENSOR_MAP_DATA_TYPE_FLOAT32,
                        CU_TENSOR_MAP_SWIZZLE_128B) &&
            (!ids || encode_tmap(&p.tq_i, ids, 3, dims, strides, box, CU_TENSOR_MAP_DATA_TYPE_UINT32,
                                 CU_TENSOR_MAP_SWIZZLE_128B))) {
            p.stages = 2;  // measured: 2 stages beat 1 (0.51 vs 0.59 ms on config D)
            if (const char* e = getenv("CDX_RQ_STAGES")) p.stages = std::max(1, std::min(RW_STAGES, atoi(e)));
            const size_t stage = static_cast<size_t>(p.boxes) * RQ_PROGS * 128u * (ids ? 2 : 1);
            const size_t smem = 1024 + p.stages * stage + 64 + 2u * RQ_PROGS * T * 4u + RQ_PROGS * p.words * 4u;
            // exact-sum threshold 2^-(30-L), n = T*W <= 2^L (see reward_quad_kernel)
            int L = 0;
            while ((1ull << L) < static_cast<uint64_t>(T) * W) ++L;
            const float exact_min = std::ldexp(1.0f, -(30 - L));
            uint32_t exact_min_bits;
            std::memcpy(&exact_min_bits, &exact_min, 4);
            const unsigned grid = static_cast<unsigned>((G + RQ_PROGS - 1) / RQ_PROGS);
            p.bstride = 1;
            // blocks take program blocks in a permuted order (a stride coprime with the grid): the
            // blocks in flight read scattered slices of the trace (config D 0.382 -> 0.378 ms);
            // CDX_RQ_PERMUTE=0 keeps launch order
            if (const char* pe = getenv("CDX_RQ_PERMUTE"); !(pe && pe[0] == '0') && grid > 2) {
                uint64_t st = static_cast<uint64_t>(static_cast<double>(grid) * 0.6180339887) | 1u;
                auto gcd = [](uint64_t a, uint64_t b) { while (b) { const uint64_t t = a % b; a = b; b = t; } return a; };
                while (gcd(st, grid) != 1) st += 2;
                p.bstride = st;
            }
            const bool half = W % 32 != 0;
            void (*kern)(RwParams, uint32_t) =
                half ? (p.boxes == 2 ? reward_quad_kernel<2, true>
                                     : p.boxes == 3 ? reward_quad_kernel<3, true> : reward_quad_kernel<4, true>)
                     : (p.boxes == 1   ? reward_quad_kernel<1, false>
                        : p.boxes == 2 ? reward_quad_kernel<2, false>
                        : p.boxes == 3 ? reward_quad_kernel<3, false>
                                       : reward_quad_kernel<4, false>);
            cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
            kern<<<grid, RQ_PROGS * 4, smem, ctx->stream>>>(p, exact_min_bits);
            CDX_CHECK_LAUNCH(ctx, "reward_certaindex(quad)");
            launched_quad = true;
        }
    }
    // one step staged per CTA (more resident CTAs beat a deeper ring here: each thread
    // needs its program's whole step row in shared memory); CDX_RW_STAGES=2 for a ring
    p.stages = 1;
    if (const char* e = getenv("CDX_RW_STAGES")) p.stages = std::max(1, std::min(RW_STAGES, atoi(e)));
    const size_t smem = tma ? 1024 + static_cast<size_t>(p.stages) * (ids ? 2 : 1) * p.stage_bytes + 8 * RW_STAGES
                            : 0;
    const unsigned grid = static_cast<unsigned>((G + RW_PROGS - 1) / RW_PROGS);
    if (!launched_quad && !f64) {
        if (tma)
            cudaFuncSetAttribute(reward_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
        reward_kernel<<<grid, RW_PROGS, smem, ctx->stream>>>(p);
        CDX_CHECK_LAUNCH(ctx, "reward_certaindex");
    }
    if (ids || launched_quad || f64) {
        uint32_t cap_log2 = 1;
        while (ids && (1u << cap_log2) < 2u * T * W) ++cap_log2;
        // per-warp table: 2 * cap hash words + T*W counts; as many warps per CTA as fit
        const size_t per_warp = ids ? ((2u << cap_log2) + static_cast<size_t>(T) * W) * 4u : 0u;
        const size_t limit = 220u * 1024u;
        if (per_warp <= limit) {
            const int warps = per_warp ? static_cast<int>(std::min<size_t>(OV_WARPS, limit / per_warp)) : OV_WARPS;
            const size_t osmem = std::max<size_t>(16u, warps * per_warp);
            if (f64) {
                cudaFuncSetAttribute(reward_overflow_kernel<double>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     static_cast<int>(osmem));
                const unsigned blocks = static_cast<unsigned>(
                    std::min<uint64_t>((G + warps - 1) / warps, static_cast<uint64_t>(ctx->sm_count) * 32));
                reward_overflow_kernel<double><<<blocks, warps * 32, osmem, ctx->stream>>>(p, cap_log2, nullptr,
                                                                                           rewards64, 1u);
            } else {
                cudaFuncSetAttribute(reward_overflow_kernel<float>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     static_cast<int>(osmem));
                reward_overflow_kernel<float><<<ctx->sm_count, warps * 32, osmem, ctx->stream>>>(p, cap_log2, nullptr,
                                                                                                 rewards, 0u);
            }
        } else {  // global-memory tables: up to ~256 MB of them, at least one warp
            uint64_t nwarps = std::max<uint64_t>(
                1, std::min<uint64_t>(static_cast<uint64_t>(ctx->sm_count) * OV_WARPS, (256ull << 20) / per_warp));
            const unsigned wpb = static_cast<unsigned>(std::min<uint64_t>(OV_WARPS, nwarps));
            nwarps = nwarps / wpb * wpb;  // whole CTAs: one table slice per launched warp
            const unsigned blocks = static_cast<unsigned>(nwarps / wpb);
            auto* gtab = static_cast<uint32_t*>(scratch2(ctx, nwarps * per_warp));
            if (!gtab) return set_error(ctx, CDX_ECUDA, "reward_certaindex: overflow table allocation failed");
            if (f64)
                reward_overflow_kernel<double><<<blocks, wpb * 32, 16, ctx->stream>>>(p, cap_log2, gtab, rewards64, 1u);
            else
                reward_overflow_kernel<float><<<blocks, wpb * 32, 16, ctx->stream>>>(p, cap_log2, gtab, rewards, 0u);
        }
        CDX_CHECK_LAUNCH(ctx, "reward_certaindex(overflow)");
    }
    return CDX_OK;
}
}  // namespace
}  // namespace cdx

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
            for (uint64_t i = b; i < e; ++i) s = x86_add(s, v[i]);  // NaN bits as the host's
            out[r] = x86_div(s, static_cast<double>(e - b));
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
