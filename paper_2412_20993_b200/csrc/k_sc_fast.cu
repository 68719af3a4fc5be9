// k_sc_fast.cu — K2 fast path: Self-Consistency certaindex over 32-row groups with two
// cluster engines.
//
// Shapes: S in {4,8,16,32}, R*P*S % 32 == 0, 16B-aligned ids (configs A and C).  The ids
// tensor is viewed as 128-byte lines ([R*P*S/32][32] u32); a GROUP = 32 consecutive rows
// of the flat row sequence (32 probes of one request when P % 32 == 0) = S lines at G*S, staged by one TMA box load into a 128B-swizzled
// shared buffer (conflict-free 16-byte reads for both engines); warps pull groups from one
// global work counter through a private 2-deep TMA ring.
//
// Work order: lane 0 of a warp claims chunks of up to 16 groups from one counter; claim slot
// c is chunk (c * stride) mod nchunks for a stride coprime with nchunks, so the groups in
// flight are scattered over the whole id tensor rather than one contiguous front (measured
// 4.5 % faster on config C).
//
// Engines, measured on B200 (tools/mb_match.cu, profiles/):
//   * ALU peel engine (default for every warp): lane = row; the row's S ids sit in
//     registers and clusters are peeled in first-seen order (first unassigned sample =
//     next leader), S compares per cluster at two instructions each (ISETP + predicated
//     OR).  On config C it alone streams at the HBM roofline (1.36 ms, 99.7% of the
//     measured copy bandwidth).
//   * warp-match engine: one __match_any_sync per row (lane = sample); the lowest lane of a
//     match set is the cluster's first-seen answer, popc the size.  MATCH.ANY runs on the
//     divergence unit (~4 + 1.5 cycles per distinct value per SM), and its cost does not
//     grow with the number of clusters, so a group with a row of more than PEEL_MAX
//     clusters is redone here (warp vote), and CDX_SCF_MATCH=k dedicates k warps of a CTA
//     to it (the pipes are independent; both engines pull from the same counter).
//
// Both produce, per row, the largest cluster size (the majority fraction maxc / S, the
// plurality rule of runtime.cpp:317-334) and the first-seen-ordered cluster sizes folded in FP64 exactly as
// metrics.cpp:107-125 (h -= term[size], term[c] = (c/S)*log(c/S) from the host libm;
// max(0,h); clamp((log n - h)/log n)), thresholds on the FP64 value (metrics.cpp:159-171),
// an fp32 store and one meets word per group.
#include <algorithm>
#include <cstdlib>
#include <string>

#include "k_alloc.cuh"
#include "k_sc.cuh"

namespace cdx {
namespace {

constexpr uint32_t FAST_WARPS = 8;  // max warps per CTA

// a |= bit when x == v: ISETP + one predicated LOP3 (the select-and-or form costs three)
__device__ __forceinline__ void or_if_eq(uint32_t& a, uint32_t x, uint32_t v, uint32_t bit) {
    asm("{\n\t.reg .pred p;\n\tsetp.eq.u32 p, %1, %2;\n\t@p or.b32 %0, %0, %3;\n\t}"
        : "+r"(a)
        : "r"(x), "r"(v), "r"(bit));
}

// bit e set iff x[e] == v; four independent accumulators keep the dependency chains short
template <int S>
__device__ __forceinline__ uint32_t eq_mask(const uint32_t (&x)[S], uint32_t v) {
    uint32_t a0 = 0, a1 = 0, a2 = 0, a3 = 0;
#pragma unroll
    for (uint32_t e = 0; e < S; e += 4) {
        or_if_eq(a0, x[e], v, 1u << e);
        or_if_eq(a1, x[e + 1], v, 2u << e);
        or_if_eq(a2, x[e + 2], v, 4u << e);
        or_if_eq(a3, x[e + 3], v, 8u << e);
    }
    return (a0 | a1) | (a2 | a3);
}

// byte offset of flat 16-byte chunk f of a 128B-swizzled group buffer (line f/8)
__device__ __forceinline__ uint32_t chunk_addr(uint32_t f) { return (f >> 3) * 128u + (((f & 7u) ^ ((f >> 3) & 7u)) << 4); }
// byte offset of flat u32 element fe
__device__ __forceinline__ uint32_t elem_addr(uint32_t fe) { return chunk_addr(fe >> 2) + (fe & 3u) * 4u; }

__device__ __forceinline__ double finish_entropy(double h, double logn) {
    h = (0.0 < h) ? h : 0.0;  // std::max(0.0, h)
    const double v = __ddiv_rn(__dsub_rn(logn, h), logn);
    return v < 0.0 ? 0.0 : (1.0 < v ? 1.0 : v);  // std::clamp(v, 0, 1)
}

// ALU peel engine: lane owns row `lane` of the group.  At most PEEL_MAX clusters are peeled
// (each costs S compares); a row with more sets *more and the warp redoes the group with the
// match engine, whose cost does not grow with the cluster count.
constexpr uint32_t PEEL_MAX = 8;

template <int S>
__device__ __forceinline__ double alu_row(const uint8_t* __restrict__ buf, const double* __restrict__ term,
                                          uint32_t lane, double logn, bool* more,
                                          const double* __restrict__ comp, uint32_t& maxc) {
    uint32_t x[S];
#pragma unroll
    for (uint32_t j = 0; j < S / 4; ++j) {
        const uint4 v = *reinterpret_cast<const uint4*>(buf + chunk_addr(lane * (S / 4) + j));
        x[4 * j] = v.x;
        x[4 * j + 1] = v.y;
        x[4 * j + 2] = v.z;
        x[4 * j + 3] = v.w;
    }
    uint32_t un = S >= 32 ? 0xffffffffu : ((1u << S) - 1u);
    // first cluster: its leader is sample 0
    uint32_t eq = eq_mask<S>(x, x[0]);
    un &= ~eq;
    maxc = __popc(eq);  // largest cluster so far (majority fraction = maxc / S)
    if (un == 0) return 1.0;  // one cluster holds every answer: H = 0, H~ = 1 exactly
    if (S <= 16 && comp) {  // composition code: a cut bit after every cluster but the last
        uint32_t cum = maxc, code = 1u << (cum - 1);
        uint32_t peeled = 1;
        while (un) {
            if (peeled == PEEL_MAX) {
                *more = true;
                return 0.0;
            }
            ++peeled;
            const uint32_t l = __ffs(un) - 1;
            const uint32_t v = *reinterpret_cast<const uint32_t*>(buf + elem_addr(lane * S + l));
            eq = eq_mask<S>(x, v);
            un &= ~eq;
            const uint32_t c = __popc(eq);
            maxc = max(maxc, c);
            cum += c;
            code |= 1u << (cum - 1);
        }
        return __ldg(comp + (code & ((1u << (S - 1)) - 1u)));
    }
    double h = __dsub_rn(0.0, term[maxc]);
    uint32_t peeled = 1;
    while (un) {
        if (peeled == PEEL_MAX) {
            *more = true;
            return 0.0;
        }
        ++peeled;
        const uint32_t l = __ffs(un) - 1;  // first unassigned sample = next cluster's leader
        const uint32_t v = *reinterpret_cast<const uint32_t*>(buf + elem_addr(lane * S + l));
        eq = eq_mask<S>(x, v);
        un &= ~eq;
        const uint32_t c = __popc(eq);
        maxc = max(maxc, c);
        h = __dsub_rn(h, term[c]);  // h -= p*log(p), first-seen order
    }
    return finish_entropy(h, logn);
}

// largest byte of a row's size slots (the largest cluster), S/4 words of 4 bytes
__device__ __forceinline__ uint32_t max_byte(const uint32_t* wv, uint32_t nwords) {
    uint32_t m = 0;
    for (uint32_t k = 0; k < nwords; ++k) m = __vmaxu4(m, wv[k]);
    m = __vmaxu4(m, m >> 16);
    m = __vmaxu4(m, m >> 8);
    return m & 0xffu;
}

// warp-match engine: lane = sample of the rows of one match iteration; the fold runs on
// the row's owner lane over the [row][32]-byte size table (0 = not a leader).
template <int S>
__device__ __forceinline__ double match_rows(const uint8_t* __restrict__ buf, uint8_t* __restrict__ cntw,
                                             const double* __restrict__ term, uint32_t lane, double logn,
                                             uint32_t& maxc) {
    constexpr uint32_t rpi = 32u / S;
    constexpr uint32_t smask = S >= 32 ? 0xffffffffu : ((1u << S) - 1u);
    const uint32_t sub = lane / S, s = lane - sub * S;
    const uint32_t subm = smask << (sub * S);
    const uint32_t ltm = (1u << lane) - 1u;
#pragma unroll 8
    for (uint32_t it = 0; it < 32u / rpi; ++it) {
        const uint32_t row = it * rpi + sub;
        const uint32_t v = *reinterpret_cast<const uint32_t*>(buf + elem_addr(row * S + s));
        const uint32_t m = __match_any_sync(0xffffffffu, v) & subm;
        cntw[row * 32u + s] = (m & ltm) == 0u ? static_cast<uint8_t>(__popc(m)) : uint8_t(0);
    }
    __syncwarp();
    const uint4* rowp = reinterpret_cast<const uint4*>(cntw + lane * 32u);
    const uint4 a = rowp[0];
    if ((a.x & 0xffu) == S) {  // sample 0's cluster holds every answer
        maxc = S;
        return 1.0;
    }
    const uint4 b = S > 16 ? rowp[1] : make_uint4(0, 0, 0, 0);
    const uint32_t wv[8] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w};
    maxc = max_byte(wv, S / 4);
    // branch-free fold over every slot in sample order: term[0] = +0.0 and h >= 0, so a
    // non-leader slot leaves h bit-identical
    double h = 0.0;
#pragma unroll
    for (uint32_t k = 0; k < S / 4; ++k)
#pragma unroll
        for (uint32_t j = 0; j < 4; ++j) h = __dsub_rn(h, term[__byte_perm(wv[k], 0, 0x4440 + j)]);
    return finish_entropy(h, logn);
}

// TAIL: a batch of at most one K5 tile (2048 requests, P % 32 == 0): the last CTA out runs
// K5 on it (al::alloc_tile) in the same launch.  Every CTA publishes its meets words with the
// fence before its arrival on the CTAs-done counter, and the last arrival fences again before
// its CTA reads them: one launch for the whole SC decision of a small batch (config A).
template <int S, bool TAIL>
__global__ void __launch_bounds__(FAST_WARPS * 32) sc_fast_kernel(const __grid_constant__ CUtensorMap tmap,
                                                                  const __grid_constant__ ScParams p,
                                                                  unsigned long long* __restrict__ counter,
                                                                  uint32_t match_warps, uint32_t claim,
                                                                  uint64_t nchunks, uint64_t stride,
                                                                  const __grid_constant__ al::AllocParams ap) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    // 128B-swizzled TMA destinations need 1024-byte alignment (offset the shared array, do
    // not cast through an integer, so every access stays an LDS)
    uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
    constexpr uint32_t GB = 32u * S * 4u;  // group bytes
    // stage stride: the 128B swizzle repeats every 1024 B and is keyed on address bits 7-9,
    // so every stage must start 1024-aligned (S = 4 groups are only 512 B)
    constexpr uint32_t GS = GB < 1024u ? 1024u : GB;
    const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const uint32_t nw_cta = blockDim.x >> 5;
    const uint32_t ring = p.stages * GS;
    uint8_t* wbase = smem + warp * ring;
    uint8_t* cnt_all = smem + nw_cta * ring;  // [warp][32 rows][32 B]
    uint8_t* cntw = cnt_all + warp * 1024u;
    double* term = reinterpret_cast<double*>(cnt_all + nw_cta * 1024u);
    uint64_t* bar = reinterpret_cast<uint64_t*>(term + 34) + warp * SC_MAX_STAGES;
    unsigned long long* qG = reinterpret_cast<unsigned long long*>(term + 34 + FAST_WARPS * SC_MAX_STAGES) +
                             warp * SC_MAX_STAGES;

    if (threadIdx.x < 33) term[threadIdx.x] = p.term[threadIdx.x];
    if (lane == 0) {
        if (warp == 0) tma_prefetch_desc(&tmap);
        for (uint32_t s = 0; s < p.stages; ++s) mbar_init(&bar[s], 1);
        fence_mbar_init();
    }
    __syncthreads();

    const uint64_t policy = policy_evict_first();
    const bool use_match = warp < match_warps;
    // lane 0 claims groups from the global counter in chunks of `claim` (one same-address
    // atomic per group would serialise at the L2 at ~2 ns each; small batches claim 1 so
    // every warp gets work) and starts each TMA load
    // Claims are monotone slots; slot chunk c maps to chunk (c * stride) mod nchunks (stride
    // coprime with nchunks: a permutation), so the chunks in flight at any moment sit at
    // scattered addresses instead of one contiguous front (stride 1: the identity).
    unsigned long long chunk_next = 0, chunk_end = 0;
    auto claim_issue = [&](uint32_t stage) {
        if (chunk_next == chunk_end) {
            const unsigned long long c = atomicAdd(counter, static_cast<unsigned long long>(claim)) / claim;
            if (c < nchunks) {
                chunk_next = ((c * stride) % nchunks) * claim;
                chunk_end = min(chunk_next + claim, static_cast<unsigned long long>(p.ngroups));
            } else {
                chunk_next = p.ngroups;  // every chunk is claimed: this warp is done
                chunk_end = p.ngroups + 1;
            }
        }
        const unsigned long long G = chunk_next++;
        qG[stage] = G;
        if (G < p.ngroups) {
            mbar_expect_tx(&bar[stage], GB);
            tma_load_2d(wbase + stage * GS, &tmap, 0, static_cast<int32_t>(G * S), &bar[stage], policy);
        }
    };
    if (lane == 0)
        for (uint32_t s = 0; s < p.stages; ++s) claim_issue(s);
    __syncwarp();

    uint32_t stage = 0, parity = 0;
    while (true) {
        const unsigned long long G = qG[stage];
        if (G >= p.ngroups) break;  // claims are monotone: nothing left for this warp
        mbar_wait(&bar[stage], parity);
        const uint8_t* buf = wbase + stage * GS;
        bool more = false;
        uint32_t maxc = 0;
        double hc = use_match ? 0.0 : alu_row<S>(buf, term, lane, p.logn, &more, p.comp, maxc);
        if (use_match || __any_sync(0xffffffffu, more)) hc = match_rows<S>(buf, cntw, term, lane, p.logn, maxc);
        __syncwarp();  // every lane is done with this stage (and with cntw)
        if (lane == 0) claim_issue(stage);
        const bool meets = sc_meets(p, hc, maxc);
        const uint64_t row = G * 32u + lane;  // flat row r * P + p
        if (p.P % 32u == 0) {  // a group is 32 probes of one request: one meets word
            if (p.hcert) p.hcert[row] = static_cast<float>(hc);
            if (p.maj) p.maj[row] = p.maj_tab[maxc];
            const uint32_t mw = __ballot_sync(0xffffffffu, meets);
            if (lane == 0 && p.meets) p.meets[G] = mw;
        } else {  // flat groups straddle requests: OR each word's bits in (meets zeroed first)
            const bool valid = row < p.R * p.P;
            if (p.hcert && valid) p.hcert[row] = static_cast<float>(hc);
            if (p.maj && valid) p.maj[row] = p.maj_tab[maxc];
            const uint64_t r = row / p.P;
            const uint32_t pp = static_cast<uint32_t>(row - r * p.P);
            const uint64_t word = valid ? r * p.words + (pp >> 5) : ~0ull;
            const uint32_t grp = __match_any_sync(0xffffffffu, word);
            const uint32_t bits = __reduce_or_sync(grp, (valid && meets) ? 1u << (pp & 31u) : 0u);
            if (p.meets && valid && bits && (grp & ((1u << lane) - 1u)) == 0) atomicOr(p.meets + word, bits);
        }
        __syncwarp();  // qG[stage] rewritten by lane 0 is visible before the next lap
        if (++stage == p.stages) {
            stage = 0;
            parity ^= 1u;
        }
    }
    // the last CTA out rewinds the claim counter for the next call (no memset launch): every
    // other CTA has left its loop, so no claim can follow the reset
    __shared__ uint32_t s_last;
    if (TAIL) __threadfence();  // each lane 0's meets words before this CTA's arrival
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence();
        const bool last = atomicAdd(counter + 1, 1ull) == gridDim.x - 1;
        if (last) {
            counter[0] = 0;
            counter[1] = 0;
            __threadfence();
        }
        s_last = last ? 1u : 0u;
    }
    if (TAIL) {
        __syncthreads();
        if (s_last) al::alloc_tile(ap, 0, 0, true, false);  // every meets word is written
    }
}

template <int S, bool TAIL>
void launch_fast(cdx_ctx* ctx, const CUtensorMap& tmap, const ScParams& p, uint32_t wpc, uint32_t match_warps,
                 unsigned long long* counter, const al::AllocParams& ap) {
    const size_t smem = 1024 + static_cast<size_t>(wpc) * (p.stages * std::max(32u * S * 4u, 1024u) + 1024u) + 34 * 8 +
                        FAST_WARPS * SC_MAX_STAGES * 16;
    // attribute + occupancy once per (device, CTA shape): host work per call stays one launch
    struct Occ {
        int dev = -1;
        uint32_t wpc = 0;
        size_t smem = 0;
        int per_sm = 0;
    };
    static thread_local Occ oc;  // one per (S, TAIL)
    int per_sm = 0;
    if (oc.dev == ctx->device && oc.wpc == wpc && oc.smem == smem) {
        per_sm = oc.per_sm;
    } else {
        cudaFuncSetAttribute(sc_fast_kernel<S, TAIL>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, sc_fast_kernel<S, TAIL>, wpc * 32, smem);
        oc = Occ{ctx->device, wpc, smem, per_sm};
    }
    if (per_sm < 1) per_sm = 1;
    if (ctx->sc_ctas_per_sm && per_sm > static_cast<int>(ctx->sc_ctas_per_sm)) per_sm = static_cast<int>(ctx->sc_ctas_per_sm);
    const uint64_t want = (p.ngroups + wpc - 1) / wpc;
    const uint64_t grid = std::min<uint64_t>(want, static_cast<uint64_t>(ctx->sm_count) * per_sm);
    // claim 16 groups per atomic on large batches; fewer when that would leave warps idle
    // (config A: 1024 groups over 1024 warps claims 1: 25 -> ~5 us)
    const uint64_t warps = grid * wpc;
    uint64_t cmax = 16, cdiv = 8;  // tuning: CDX_SCF_CLAIM (largest chunk), CDX_SCF_CLAIM_DIV (chunks per warp)
    if (const char* e = getenv("CDX_SCF_CLAIM")) cmax = std::max(1, atoi(e));
    if (const char* e = getenv("CDX_SCF_CLAIM_DIV")) cdiv = std::max(1, atoi(e));
    const uint32_t claim = static_cast<uint32_t>(std::max<uint64_t>(1, std::min<uint64_t>(cmax, p.ngroups / (warps * cdiv))));
    // chunk order: a permutation by default (config C, 16-group chunks: 1.378 -> 1.316 ms for
    // K2 + K5; contiguous chunks in claim order reach the same only at particular chunk
    // sizes, 1.33-1.38 ms between 40 and 100 groups); CDX_SCF_PERMUTE=0 keeps claim order
    const uint64_t nchunks = (p.ngroups + claim - 1) / claim;
    uint64_t stride = 1;
    const char* pe = getenv("CDX_SCF_PERMUTE");
    if (!(pe && pe[0] == '0') && nchunks > 2) {
        stride = static_cast<uint64_t>(static_cast<double>(nchunks) * 0.6180339887) | 1u;
        auto gcd = [](uint64_t a, uint64_t b) { while (b) { const uint64_t t = a % b; a = b; b = t; } return a; };
        while (gcd(stride, nchunks) != 1) stride += 2;
    }
    sc_fast_kernel<S, TAIL><<<static_cast<unsigned>(grid), wpc * 32, smem, ctx->stream>>>(
        tmap, p, counter, match_warps, claim, nchunks, stride, ap);
}

}  // namespace

bool launch_sc_fast(cdx_ctx* ctx, const ScParams& p0, const al::AllocParams* tail, bool* tail_done) {
    if (tail_done) *tail_done = false;
    const uint32_t S = p0.S;
    // Groups are 32 consecutive rows of the flat [R*P] row sequence.  With P % 32 == 0 a
    // group is 32 probes of one request; otherwise it may straddle requests and each row's
    // meets bit is OR-ed into its word.  The rows must fill whole 128-byte lines.
    const uint64_t rows = p0.R * p0.P;
    const uint64_t lines = rows * S / 32;
    if (!(S == 4 || S == 8 || S == 16 || S == 32) || (rows * S) % 32 != 0 ||
        reinterpret_cast<uintptr_t>(p0.ids) % 16 != 0 || lines >= (1ull << 31))
        return false;
    const char* impl = getenv("CDX_SC_IMPL");
    if (impl && std::string(impl) == "match") return false;
    // the descriptor depends only on (ids, lines, S): re-encode only when they change
    struct Tmc {
        const void* ids = nullptr;
        uint64_t lines = 0;
        uint32_t S = 0;
        CUtensorMap map;
    };
    static thread_local Tmc tc;
    CUtensorMap tmap;
    if (tc.ids == p0.ids && tc.lines == lines && tc.S == S) {
        tmap = tc.map;
    } else {
        const uint64_t dims[2] = {32, lines};
        const uint64_t strides[1] = {128};
        const uint32_t box[2] = {32, S};
        if (!encode_tmap(&tmap, p0.ids, 2, dims, strides, box, CU_TENSOR_MAP_DATA_TYPE_UINT32,
                         CU_TENSOR_MAP_SWIZZLE_128B))
            return false;
        tc = Tmc{p0.ids, lines, S, tmap};
    }
    ScParams p = p0;
    p.ngroups = (rows + 31) / 32;
    if (p.P % 32 != 0 && p.meets) {
        if (cudaMemsetAsync(p.meets, 0, p.R * p.words * 4, ctx->stream) != cudaSuccess) return false;
    }
    // warps per CTA, ring depth per warp and how many warps of a CTA run the match engine
    // (defaults tuned on B200, profiles/)
    // config C sweep: 8 warps x 2 stages, every warp on the ALU engine (match fallback per
    // group): 1.360 ms = 99.7% of the measured copy bandwidth; 1 match warp 1.376, 4 1.422
    uint32_t wpc = 8, stages = 2, mw = 0;
    if (const char* e = getenv("CDX_SCF_WARPS")) wpc = static_cast<uint32_t>(atoi(e));
    if (const char* e = getenv("CDX_SCF_STAGES")) stages = static_cast<uint32_t>(atoi(e));
    if (const char* e = getenv("CDX_SCF_MATCH")) mw = static_cast<uint32_t>(atoi(e));
    if (impl && std::string(impl) == "alu") mw = 0;
    if (impl && std::string(impl) == "matchonly") mw = 64;
    wpc = std::max<uint32_t>(1, std::min<uint32_t>(FAST_WARPS, wpc));
    p.stages = std::max<uint32_t>(1, std::min<uint32_t>(SC_MAX_STAGES, stages));
    // claim counter + CTAs-done counter: the context's own (ctx.cu), zeroed once, rewound in-kernel
    if (!ctx->sc_counter) return false;
    auto* counter = static_cast<unsigned long long*>(ctx->sc_counter);
    // one K5 tile, one meets word per group, a CTA of K5's 256 threads: K5 in K2's last CTA
    const bool tl = tail && tail_done && tail->ntiles == 1 && p.P % 32u == 0 && p.meets &&
                    wpc * 32 == static_cast<uint32_t>(al::AL_THREADS);
    static const al::AllocParams none{};
    if (tl) {
        *tail_done = true;
        switch (S) {
            case 32: launch_fast<32, true>(ctx, tmap, p, wpc, mw, counter, *tail); break;
            case 16: launch_fast<16, true>(ctx, tmap, p, wpc, mw, counter, *tail); break;
            case 8: launch_fast<8, true>(ctx, tmap, p, wpc, mw, counter, *tail); break;
            default: launch_fast<4, true>(ctx, tmap, p, wpc, mw, counter, *tail); break;
        }
        return true;
    }
    switch (S) {
        case 32: launch_fast<32, false>(ctx, tmap, p, wpc, mw, counter, none); break;
        case 16: launch_fast<16, false>(ctx, tmap, p, wpc, mw, counter, none); break;
        case 8: launch_fast<8, false>(ctx, tmap, p, wpc, mw, counter, none); break;
        default: launch_fast<4, false>(ctx, tmap, p, wpc, mw, counter, none); break;
    }
    return true;
}

}  // namespace cdx
