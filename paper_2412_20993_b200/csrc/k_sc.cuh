// k_sc.cuh — shared declarations of the K2 (Self-Consistency certaindex) kernels.
#pragma once

#include "cdx_internal.cuh"

namespace cdx {

constexpr int SC_MAX_STAGES = 4;
constexpr int SC_MAX_WARPS = 8;
constexpr int MAX_TH = 8;
constexpr uint32_t SC_GROUP_BYTES = 32u * 32u * 4u;  // 32 rows x S<=32 samples x 4 B

struct ScParams {
    const uint32_t* ids;
    float* hcert;
    uint32_t* meets;
    uint64_t R;
    uint64_t ngroups;  // R * words
    uint32_t P, S, words;
    uint32_t stages;
    int bulk_ok;  // ids base 16B-aligned (the generic kernel then bulk-copies every group whose bytes are 16B units)
    int n_th;
    uint8_t th_dir[MAX_TH];
    double th_cut[MAX_TH];
    double term[33];
    double logn;
    const double* comp;  // S <= 16: H~ of every first-seen size composition (null: fold)
    // the AND of the inclusive thresholds on the one signal as a closed interval
    // (metrics.cpp:159-171): lo = max of the >= cutoffs, hi = min of the <= cutoffs;
    // box_never: a NaN cutoff (every compare false)
    double box_lo, box_hi;
    int box_never;
    // majority fraction (CDX_SIG_MAJORITY): largest cluster size / S.  maj: f32[R][P]
    // output (nullable), maj_tab[c] = fp32 of (double)c / S.  Its thresholds reduce to an
    // integer interval of the largest cluster size [maj_lo, maj_hi] (empty: never met),
    // evaluated on the host with the same double compare, as a_min is for CoT.
    float* maj;
    int maj_th;  // any threshold on the majority signal
    uint32_t maj_lo, maj_hi;
    float maj_tab[33];
};

// meets for an SC certaindex value (finite, in [0, 1]) and the row's largest cluster size:
// the interval form of the AND (metrics.cpp:159-171) on each signal
__device__ __forceinline__ bool sc_meets(const ScParams& p, double hc, uint32_t maxc) {
    return p.n_th == 0 || (!p.box_never && hc >= p.box_lo && hc <= p.box_hi &&
                           (!p.maj_th || (maxc >= p.maj_lo && maxc <= p.maj_hi)));
}

// [lo, hi] = {c in 0..S : every majority threshold holds for (double)c / S} (lo > hi: none).
// metrics.cpp:167's inclusive compares, evaluated on the host exactly as the oracle does.
void majority_interval(const cdx_threshold* th, uint32_t n_th, uint32_t S, uint32_t* lo, uint32_t* hi);

namespace al {
struct AllocParams;
}
// The TMA fast path (S in {4,8,16,32}, P % 32 == 0, 16B-aligned ids).  Returns true when
// it launched; false when the shape needs the generic warp-match kernel.  tail (nullable):
// K5's parameters; *tail_done = true when K5 ran in the same launch (one K5 tile: at most 2048
// requests), else the caller launches it.
bool launch_sc_fast(cdx_ctx* ctx, const ScParams& p, const al::AllocParams* tail = nullptr, bool* tail_done = nullptr);

// Validate a threshold list against the signals an entry point produces (present[kind]);
// an absent signal fails with the reference's message (metrics.cpp:163-166).
int check_thresholds(cdx_ctx* ctx, const cdx_threshold* th, uint32_t n_th, const bool present[5]);

}  // namespace cdx
