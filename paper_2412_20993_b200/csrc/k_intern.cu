// k_intern.cu — K1: answer canonicalisation, interning and hesitation flags.
//
// Replaces metrics::trim + the unordered_map<string_view> key of cluster_exact (metrics.cpp:
// 12-37) — every comparison of answers in the reference goes through trimmed exact bytes —
// and probe::flag_hesitation (probe.cpp:36-44).  Output ids are DENSE and in first-seen
// order of the trimmed bytes (exactly the cluster order cluster_exact would produce over
// the whole arena), so every downstream kernel compares u32 ids instead of strings.
//
// A serving trace repeats a small set of answers many times, so the design keeps the hot
// keys out of global atomics:
//
//   intern_tiles   persistent CTAs walk tiles of 1024 answers (tile k, k + grid, ...: every
//                  CTA sees its answers in increasing order).  A tile's offsets and arena
//                  bytes arrive by 1-D bulk copies (cp.async.bulk + mbarrier, two stages, the
//                  next tile's copy in flight while this one is processed).  Per answer (one
//                  thread): trim (the 6 ASCII whitespace bytes), a word-at-a-time 64-bit hash
//                  of the trimmed bytes, the hesitation scan (ASCII tolower of the raw answer,
//                  any non-empty marker as a substring, 4 bytes per SIMD compare), then a
//                  lookup in the CTA's shared-memory table of keys it has already resolved.
//                  Only a key new to the CTA goes global — once per CTA, not once per answer:
//                  CAS on the hash into the open-addressing table, atomicMin of its first
//                  arena index (the CTA's first sighting is its smallest index), and a CAS
//                  that elects the key's canonical bytes.  Every answer is then byte-verified
//                  against the canonical bytes (a 64-bit hash collision between distinct
//                  answers is reported, never merged) and its global slot is written as a
//                  provisional id.
//   ranks          the slots' first indices set bits in an n-bit bitmap; a popcount scan of
//                  the bitmap words gives every slot its dense first-seen rank (= id).
//   intern_remap   ids[i] = rank[slot], 16 bytes per thread.
//
// The global table starts at the capacity the context used last (2^20 slots at first); a
// call whose distinct answers exceed half of it is redone with room for every answer.
#include <algorithm>
#include <cstring>
#include <vector>

#include "cdx_internal.cuh"
#include "k_scan.cuh"

namespace cdx {
namespace {

constexpr int MAX_MARKERS = 16;
constexpr int MARKER_BYTES = 1024;
constexpr uint32_t IT_THREADS = 512;
constexpr uint32_t IT_TILE = 1024;               // answers per tile
constexpr uint32_t IT_K = IT_TILE / IT_THREADS;  // answers per thread per tile
constexpr uint32_t IT_ARENA = 14336;             // staged arena bytes per tile
constexpr uint32_t IT_OFFB = (IT_TILE + 2) * 8;  // staged offsets per tile (+1, 16-B rounded)
constexpr uint32_t IT_STAGE = IT_OFFB + IT_ARENA;
constexpr uint32_t LT_CAP = 128;                 // CTA-local key table (trimmed keys)
constexpr uint32_t RC_CAP = 512;                 // CTA-local raw-answer cache (answers <= 16 bytes)
constexpr uint32_t HIT = 0xfffffffeu;            // ent[]: answered from the raw cache
constexpr uint32_t EMPTY32 = 0xffffffffu;
constexpr uint64_t EMPTY64 = ~0ull;

struct Markers {
    uint32_t n;
    uint32_t off[MAX_MARKERS + 1];
    uint64_t word[MAX_MARKERS];  // first 8 bytes, little-endian (short-answer fast path)
    char bytes[MARKER_BYTES];
};

struct InternParams {
    const uint8_t* arena;
    const uint64_t* off;
    uint64_t n;
    unsigned long long* hkey;   // global table: hash (0 = empty)
    uint32_t* first;            //               first arena index (EMPTY32)
    unsigned long long* canon;  //               canonical trimmed bytes: pos << 24 | len (EMPTY64)
    uint64_t cap_mask;
    uint32_t* ids;              // provisional: the global slot
    uint8_t* hes;
    uint32_t* n_keys;           // distinct keys inserted (overflow watch)
    uint32_t key_limit;
    int* status;                // bit 0 overflow
    int* d_err;
    int staged;                 // arena and offsets 16-B aligned: bulk copies
    int local_tables;           // CTA-local tables on (enough tiles per CTA to warm them up)
};

__device__ __forceinline__ bool is_space(uint32_t c) {
    return c == ' ' || c == '\t' || c == '\n' || c == '\r' || c == '\f' || c == '\v';
}

// 64-bit hash of n bytes read as little-endian words (tail zero-padded)
__device__ __forceinline__ uint64_t mix(uint64_t h, uint64_t w) {
    h = (h ^ w) * 0x9E3779B97F4A7C15ull;
    return h ^ (h >> 29);
}
__device__ __forceinline__ uint64_t fmix(uint64_t h) {
    h ^= h >> 33;
    h *= 0xff51afd7ed558ccdull;
    h ^= h >> 33;
    h *= 0xc4ceb9fe1a85ec53ull;
    h ^= h >> 33;
    return h ? h : 1;  // 0 marks an empty slot
}

// 8 bytes at p (little-endian) from a buffer whose word alignment matches p's offset from an
// 8-aligned base: two aligned loads and a funnel shift; bytes past `left` read as 0
__device__ __forceinline__ uint64_t ld8(const uint8_t* p, uint64_t left) {
    const uintptr_t a = reinterpret_cast<uintptr_t>(p), al = a & ~static_cast<uintptr_t>(7);
    const uint32_t sh = static_cast<uint32_t>(a & 7) * 8;
    uint64_t v = *reinterpret_cast<const uint64_t*>(al);
    if (sh) v = (v >> sh) | (left + sh / 8 > 8 ? *reinterpret_cast<const uint64_t*>(al + 8) << (64 - sh) : 0ull);
    return left >= 8 ? v : (v & ((1ull << (8 * left)) - 1ull));
}

// 8 arena bytes from pos of the global arena (any alignment): a 16-byte window inside the
// arena, byte loads at its edges
// (`end` = the arena's end bounds the window; bytes past `left` read as 0)
__device__ __forceinline__ uint64_t gload8(const uint8_t* __restrict__ a, uint64_t pos, uint64_t end, uint64_t left) {
    const uintptr_t base = reinterpret_cast<uintptr_t>(a);
    const uintptr_t addr = base + pos, al = addr & ~static_cast<uintptr_t>(7);
    uint64_t v;
    if (al >= base && al + 16 <= base + end) {
        const uint64_t w0 = *reinterpret_cast<const uint64_t*>(al);
        const uint64_t w1 = *reinterpret_cast<const uint64_t*>(al + 8);
        const uint32_t sh = static_cast<uint32_t>(addr & 7) * 8;
        v = sh ? (w0 >> sh) | (w1 << (64 - sh)) : w0;
    } else {
        v = 0;
        for (uint32_t k = 0; k < 8 && k < left && pos + k < end; ++k) v |= static_cast<uint64_t>(a[pos + k]) << (8 * k);
    }
    return left >= 8 ? v : (v & ((1ull << (8 * left)) - 1ull));
}

// ASCII tolower of four bytes
__device__ __forceinline__ uint32_t lower4(uint32_t x) {
    return x | (__vcmpgeu4(x, 0x41414141u) & __vcmpleu4(x, 0x5a5a5a5au) & 0x20202020u);
}

// SWAR byte tests on 8 bytes (exact per byte: no carries cross byte lanes).  Each returns 0x80
// in the bytes that pass.
constexpr uint64_t L7 = 0x7f7f7f7f7f7f7f7full, H8 = 0x8080808080808080ull, B1 = 0x0101010101010101ull;
__device__ __forceinline__ uint64_t eqflags(uint64_t x, uint32_t c) {  // byte == c
    const uint64_t y = x ^ (B1 * c);
    return ~(((y & L7) + L7) | y) & H8;
}
__device__ __forceinline__ uint64_t rangeflags(uint64_t x, uint32_t lo, uint32_t hi) {  // lo <= byte <= hi < 0x80
    const uint64_t m = x & L7;
    return (m + B1 * (0x80u - lo)) & ~(m + B1 * (0x7fu - hi)) & ~x & H8;
}
// the six whitespace bytes of metrics::trim (metrics.cpp:14): ' ' and '\t' .. '\r'
__device__ __forceinline__ uint64_t spaceflags(uint64_t x) { return eqflags(x, 0x20) | rangeflags(x, 0x09, 0x0d); }
__device__ __forceinline__ uint64_t lower8(uint64_t x) { return x | (rangeflags(x, 'A', 'Z') >> 2); }
// 0x80 in the bytes below n (of 8)
__device__ __forceinline__ uint64_t validflags(int n) { return n >= 8 ? H8 : (n <= 0 ? 0ull : H8 & ((1ull << (8 * n)) - 1ull)); }

// 8 bytes starting at byte p of the 24-byte little-endian value (w0, w1, w2)
__device__ __forceinline__ uint64_t window(uint64_t w0, uint64_t w1, uint64_t w2, uint32_t p) {
    const uint64_t a = p < 8 ? w0 : w1, b = p < 8 ? w1 : w2;
    const uint32_t sh = (p & 7u) * 8u;
    return sh ? (a >> sh) | (b << (64 - sh)) : a;
}
__device__ __forceinline__ uint64_t keep_bytes(uint64_t v, uint32_t n) {
    return n >= 8 ? v : (v & ((1ull << (8 * n)) - 1ull));
}

// One answer of at most 16 bytes from shared memory: trim, hash words, hesitation, all on
// two 8-byte words in registers.  t0/t1 = the trimmed bytes as zero-padded words.
struct Short {
    uint32_t tb, tl;
    uint64_t t0, t1;
    bool hes;
};
__device__ __forceinline__ Short short_answer(uint64_t w0, uint64_t w1, uint32_t len, const Markers& mk,
                                              bool want_hes) {
    const uint64_t v0 = validflags(static_cast<int>(len)), v1 = validflags(static_cast<int>(len) - 8);
    const uint64_t g0 = ~spaceflags(w0) & v0, g1 = ~spaceflags(w1) & v1;  // non-space bytes
    Short r;
    if (g0 | g1) {
        r.tb = g0 ? (__ffsll(static_cast<long long>(g0)) - 1) >> 3 : 8 + ((__ffsll(static_cast<long long>(g1)) - 1) >> 3);
        const uint32_t te = g1 ? 8 + ((63 - __clzll(static_cast<long long>(g1))) >> 3) + 1
                               : ((63 - __clzll(static_cast<long long>(g0))) >> 3) + 1;
        r.tl = te - r.tb;
    } else {
        r.tb = len;
        r.tl = 0;
    }
    r.t0 = keep_bytes(window(w0, w1, 0ull, r.tb), r.tl);
    r.t1 = r.tl > 8 ? keep_bytes(window(w0, w1, 0ull, r.tb + 8), r.tl - 8) : 0ull;
    r.hes = false;
    if (!want_hes) return r;
    // probe::flag_hesitation: tolower(answer) contains a non-empty marker (markers not lowered)
    const uint64_t l0 = lower8(w0), l1 = lower8(w1);
    for (uint32_t k = 0; k < mk.n && !r.hes; ++k) {
        const uint32_t mb = mk.off[k], ml = mk.off[k + 1] - mb;
        if (ml == 0 || ml > len) continue;  // empty markers never match (probe.cpp:41)
        const uint32_t m0 = static_cast<uint8_t>(mk.bytes[mb]);
        const int last = static_cast<int>(len - ml);  // candidate starts 0..last
        uint64_t c0 = eqflags(l0, m0) & validflags(last + 1), c1 = eqflags(l1, m0) & validflags(last + 1 - 8);
        while (c0 | c1) {
            uint32_t pos;
            if (c0) {
                pos = (__ffsll(static_cast<long long>(c0)) - 1) >> 3;
                c0 &= c0 - 1;
            } else {
                pos = 8 + ((__ffsll(static_cast<long long>(c1)) - 1) >> 3);
                c1 &= c1 - 1;
            }
            if (ml <= 8) {
                r.hes = keep_bytes(window(l0, l1, 0ull, pos), ml) == mk.word[k];
            } else {  // longer marker: bytes past the first eight
                bool same = window(l0, l1, 0ull, pos) == mk.word[k];
                for (uint32_t j = 8; same && j < ml; ++j)
                    same = static_cast<uint8_t>(window(l0, l1, 0ull, pos + j - (j & 7u)) >> (8 * (j & 7u))) ==
                           static_cast<uint8_t>(mk.bytes[mb + j]);
                r.hes = same;
            }
            if (r.hes) break;
        }
    }
    return r;
}

// probe::flag_hesitation (probe.cpp:36-44) on bytes s[0, len): tolower(answer) contains a
// non-empty marker (markers are not lowered).  First-byte candidates 4 at a time.
__device__ bool hesitant(const Markers& mk, const uint8_t* s, uint32_t len, bool shared_src) {
    (void)shared_src;
    for (uint32_t k = 0; k < mk.n; ++k) {
        const uint32_t mb = mk.off[k], ml = mk.off[k + 1] - mb;
        if (ml == 0 || ml > len) continue;  // empty markers never match (probe.cpp:41)
        const uint32_t m0 = static_cast<uint8_t>(mk.bytes[mb]) * 0x01010101u;
        for (uint32_t p0 = 0; p0 + ml <= len; p0 += 4) {
            uint32_t w = 0;
#pragma unroll
            for (uint32_t q = 0; q < 4; ++q) w |= (p0 + q < len ? static_cast<uint32_t>(s[p0 + q]) : 0u) << (8 * q);
            uint32_t cand = __vcmpeq4(lower4(w), m0);
            while (cand) {
                const uint32_t q = (__ffs(cand) - 1) >> 3;
                cand &= ~(0xffu << (8 * q));
                const uint32_t p = p0 + q;
                if (p + ml > len) break;
                uint32_t j = 1;
                while (j < ml) {
                    uint32_t c = s[p + j];
                    c = (c >= 'A' && c <= 'Z') ? c + 32 : c;
                    if (c != static_cast<uint8_t>(mk.bytes[mb + j])) break;
                    ++j;
                }
                if (j == ml) return true;
            }
        }
    }
    return false;
}

// global insert of one key: slot (EMPTY32 on overflow), first index and canonical bytes
__device__ uint32_t global_insert(const InternParams& p, uint64_t h, uint32_t idx, unsigned long long cpack,
                                  unsigned long long* canon_out) {
    uint64_t s = h & p.cap_mask;
    for (uint64_t probes = 0;; ++probes) {
        const unsigned long long prev = atomicCAS(p.hkey + s, 0ull, h);
        if (prev == h) break;
        if (prev == 0ull) {
            if (atomicAdd(p.n_keys, 1u) >= p.key_limit) {  // table over half full: redo bigger
                atomicOr(p.status, 1);
                return EMPTY32;
            }
            break;
        }
        s = (s + 1) & p.cap_mask;
        if (probes > p.cap_mask) {
            atomicOr(p.status, 1);
            return EMPTY32;
        }
    }
    atomicMin(p.first + s, idx);
    const unsigned long long c = atomicCAS(p.canon + s, EMPTY64, cpack);
    *canon_out = c == EMPTY64 ? cpack : c;
    return static_cast<uint32_t>(s);
}

// Raw-answer cache: an answer of <= 16 bytes seen before by this CTA (the same bytes,
// whitespace included) has the same slot and hesitation flag, so a repeat skips trim, hash,
// marker scan and verification.  Exact compare of the raw words: no collision possible.
// Structure of arrays, 4-way sets: tags u32[RC_CAP] (a set's four tags in one 16-byte load),
// words u64[RC_CAP][2], meta {len | hes << 8, slot}[RC_CAP].
constexpr uint32_t RC_WAYS = 4;
constexpr size_t RC_BYTES = RC_CAP * (4 + 16 + 8);
// 32-bit hash of a raw answer (a cache filter: hits compare every word)
__device__ __forceinline__ uint32_t raw_hash(uint64_t w0, uint64_t w1, uint32_t len) {
    uint32_t h = len * 0x9E3779B1u;
    h = (h ^ static_cast<uint32_t>(w0)) * 0x85EBCA6Bu;
    h = (h ^ static_cast<uint32_t>(w0 >> 32)) * 0xC2B2AE35u;
    h = (h ^ static_cast<uint32_t>(w1)) * 0x27D4EB2Fu;
    h = (h ^ static_cast<uint32_t>(w1 >> 32)) * 0x165667B1u;
    return h ^ (h >> 15);
}

// The first 16 bytes of an answer staged in shared memory (byte address sa), zero past len:
// three aligned 8-byte loads and 32-bit funnel shifts (no 64-bit variable shifts).
__device__ __forceinline__ void load16_shared(uint32_t sa, uint32_t len, uint64_t& w0, uint64_t& w1) {
    const uint32_t a8 = sa & ~7u;
    uint32_t x0, x1, x2, x3, x4, x5;
    asm volatile("ld.shared.v2.u32 {%0, %1}, [%2];" : "=r"(x0), "=r"(x1) : "r"(a8));
    asm volatile("ld.shared.v2.u32 {%0, %1}, [%2];" : "=r"(x2), "=r"(x3) : "r"(a8 + 8));
    asm volatile("ld.shared.v2.u32 {%0, %1}, [%2];" : "=r"(x4), "=r"(x5) : "r"(a8 + 16));
    const uint32_t o = sa & 7u;
    if (o >= 4) {  // drop one word
        x0 = x1;
        x1 = x2;
        x2 = x3;
        x3 = x4;
        x4 = x5;
    }
    const uint32_t sh = (o & 3u) * 8u;
    const uint32_t y0 = __funnelshift_r(x0, x1, sh), y1 = __funnelshift_r(x1, x2, sh);
    const uint32_t y2 = __funnelshift_r(x2, x3, sh), y3 = __funnelshift_r(x3, x4, sh);
    // bytes past len -> 0
    const uint64_t m0 = len >= 8 ? ~0ull : (1ull << (8 * len)) - 1ull;
    const uint64_t m1 = len >= 16 ? ~0ull : (len <= 8 ? 0ull : (1ull << (8 * (len - 8))) - 1ull);
    w0 = (y0 | (static_cast<uint64_t>(y1) << 32)) & m0;
    w1 = (y2 | (static_cast<uint64_t>(y3) << 32)) & m1;
}

struct alignas(16) LocalEntry {
    unsigned long long h;      // 0 = empty
    unsigned long long canon;  // canonical pack of the resolved key
    uint32_t gslot;            // EMPTY32 until resolved
    uint32_t min_idx;          // smallest answer index seen in the tile that created it
    unsigned long long mine;   // the creating answer's own pack (canonical candidate)
    unsigned long long cb0, cb1;  // the canonical's first 16 trimmed bytes
};

__global__ void __launch_bounds__(IT_THREADS, 2) intern_tiles(const __grid_constant__ InternParams p,
                                                           const __grid_constant__ Markers mk) {
    extern __shared__ __align__(128) uint8_t smem[];
    uint8_t* stage_base = smem;  // [2][IT_STAGE]
    auto* lt = reinterpret_cast<LocalEntry*>(smem + 2 * IT_STAGE);
    auto* rc_w = reinterpret_cast<unsigned long long*>(lt + LT_CAP);  // [RC_CAP][2]
    auto* rc_meta = reinterpret_cast<uint2*>(rc_w + 2 * RC_CAP);       // [RC_CAP]
    auto* rc_tag = reinterpret_cast<uint32_t*>(rc_meta + RC_CAP);      // [RC_CAP]
    auto* newlist = rc_tag + RC_CAP;                                   // [IT_TILE]
    auto* bar = reinterpret_cast<uint64_t*>(newlist + IT_TILE);  // [2]
    __shared__ uint32_t s_new[2], s_fill, s_rfill;  // s_new by tile parity
    // a table that had to be cleared twice is useless for this CTA's answers (many distinct
    // keys): off for good, those answers take the global path directly (no local probing)
    __shared__ uint32_t s_clears_lt, s_clears_rc;
    __shared__ uint64_t s_sb[2];
    const uint32_t tid = threadIdx.x;
    const uint64_t tiles = (p.n + IT_TILE - 1) / IT_TILE;

    for (uint32_t e = tid; e < LT_CAP; e += IT_THREADS) lt[e].h = 0;
    for (uint32_t e = tid; e < RC_CAP; e += IT_THREADS) rc_tag[e] = 0;
    if (tid == 0) {
        s_rfill = 0;
        s_clears_lt = s_clears_rc = p.local_tables ? 0u : 2u;
        s_new[0] = s_new[1] = 0;
        s_fill = 0;
        mbar_init(&bar[0], 1);
        mbar_init(&bar[1], 1);
        fence_mbar_init();
    }
    __syncthreads();
    const uint64_t policy = policy_evict_first();
    // stage `st`: offsets of tile t at [0, IT_OFFB), arena bytes [sb, ...) at IT_OFFB
    auto issue = [&](uint64_t t, uint32_t st) {  // thread 0
        const uint64_t i0 = t * IT_TILE, cnt = min(static_cast<uint64_t>(IT_TILE), p.n - i0);
        uint8_t* sbuf = stage_base + st * IT_STAGE;
        fence_proxy_async();  // the stage's earlier generic reads precede the async writes
        const uint64_t o0 = p.off[i0], oT = p.off[i0 + cnt];
        const uint64_t sb = o0 & ~15ull, sbulk = oT & ~15ull;  // bulk [sb, sbulk), tail bytes by hand
        s_sb[st] = sb;
        const uint32_t obulk = static_cast<uint32_t>(((cnt + 1) / 2) * 16);  // whole 16-B pairs of offsets
        const bool arena_fits = oT - sb <= IT_ARENA;
        uint32_t tx = obulk + (arena_fits && sbulk > sb ? static_cast<uint32_t>(sbulk - sb) : 0u);
        mbar_expect_tx(&bar[st], tx);
        bulk_g2s(sbuf, p.off + i0, obulk, &bar[st], policy);
        if (((cnt + 1) & 1u) != 0) reinterpret_cast<uint64_t*>(sbuf)[cnt] = oT;  // odd count: the last offset
        if (arena_fits) {
            if (sbulk > sb) bulk_g2s(sbuf + IT_OFFB, p.arena + sb, static_cast<uint32_t>(sbulk - sb), &bar[st], policy);
            for (uint64_t b = max(sbulk, sb); b < oT; ++b) sbuf[IT_OFFB + (b - sb)] = p.arena[b];
        } else {
            s_sb[st] = EMPTY64;  // too long for the stage: this tile reads the arena in place
        }
    };
    uint64_t t = blockIdx.x;
    if (p.staged && t < tiles && tid == 0) issue(t, 0);
    __syncthreads();  // thread 0's hand-copied bytes of the first stage
    uint32_t st = 0, phase = 0, par = 0;
    for (; t < tiles; t += gridDim.x, par ^= 1u) {
        const uint64_t nt = t + gridDim.x;
        const uint64_t i0 = t * IT_TILE, cnt = min(static_cast<uint64_t>(IT_TILE), p.n - i0);
        uint8_t* sbuf = stage_base + st * IT_STAGE;
        if (p.staged) {
            if (nt < tiles && tid == 0) issue(nt, st ^ 1u);  // that stage's last user passed the barrier below
            mbar_wait(&bar[st], (phase >> st) & 1u);
            phase ^= 1u << st;
        } else {  // unaligned arena / offsets: offsets staged by hand, bytes read in place
            for (uint64_t q = tid; q <= cnt; q += IT_THREADS) reinterpret_cast<uint64_t*>(sbuf)[q] = p.off[i0 + q];
            if (tid == 0) s_sb[st] = EMPTY64;
            __syncthreads();
        }
        const uint64_t* so = reinterpret_cast<const uint64_t*>(sbuf);
        const uint64_t sb = s_sb[st];
        const bool in_smem = sb != EMPTY64;

        // ---- phase A: trim, hash, hesitation, CTA-local lookup --------------------------
        uint64_t hv[IT_K], pk[IT_K], sw0[IT_K], sw1[IT_K];  // hash, pack, first 16 trimmed bytes
        uint32_t ent[IT_K], gsk[IT_K], hk[IT_K];  // gsk / hk: slot and flag of a cache hit
        bool glob[IT_K];
        const uint64_t aend = p.off[p.n];
#pragma unroll
        for (uint32_t k = 0; k < IT_K; ++k) {
            const uint32_t j = tid + k * IT_THREADS;
            ent[k] = EMPTY32;
            glob[k] = false;
            hv[k] = 0;
            pk[k] = 0;
            sw0[k] = sw1[k] = 0;
            if (j >= cnt) continue;
            const uint64_t b0 = so[j], e0 = so[j + 1];
            const uint32_t len = static_cast<uint32_t>(e0 - b0);
            uint32_t tb, tl;
            uint64_t h = 0;
            const bool use_rc = s_clears_rc < 2, use_lt = s_clears_lt < 2;
            if (in_smem && len <= 16) {  // the common case: two words in registers
                uint64_t w0, w1;
                load16_shared(smem_u32(sbuf + IT_OFFB) + static_cast<uint32_t>(b0 - sb), len, w0, w1);
                // 4-way raw cache: the set's tags in one 16-byte load, then the tag-matching way
                const uint32_t rh = raw_hash(w0, w1, len);
                const uint32_t set = ((rh >> 7) & (RC_CAP / RC_WAYS - 1)) * RC_WAYS;
                const uint32_t tag = rh | 1u;
                const uint4 tg = use_rc ? *reinterpret_cast<const uint4*>(rc_tag + set) : make_uint4(0, 0, 0, 0);
                const uint32_t way = tg.x == tag ? 0u : (tg.y == tag ? 1u : (tg.z == tag ? 2u : (tg.w == tag ? 3u : 4u)));
                if (way < RC_WAYS) {
                    const ulonglong2 ww = *reinterpret_cast<const ulonglong2*>(rc_w + 2 * (set + way));
                    const uint2 mt = rc_meta[set + way];
                    if (ww.x == w0 && ww.y == w1 && (mt.x & 0xffu) == len) {
                        gsk[k] = mt.y;
                        hk[k] = mt.x >> 8;
                        ent[k] = HIT;
                        continue;
                    }
                }
                const Short a = short_answer(w0, w1, len, mk, p.hes != nullptr);
                if (p.hes) p.hes[i0 + j] = a.hes ? 1 : 0;
                tb = a.tb;
                tl = a.tl;
                h = 0xcbf29ce484222325ull ^ (static_cast<uint64_t>(tl) * 0x9E3779B97F4A7C15ull);
                if (tl) h = mix(h, a.t0);
                if (tl > 8) h = mix(h, a.t1);
                sw0[k] = a.t0;
                sw1[k] = a.t1;
            } else {
                const uint8_t* src = in_smem ? sbuf + IT_OFFB + (b0 - sb) : p.arena + b0;
                if (p.hes) p.hes[i0 + j] = hesitant(mk, src, len, in_smem) ? 1 : 0;
                uint32_t te = len;
                tb = 0;
                while (tb < te && is_space(src[tb])) ++tb;
                while (te > tb && is_space(src[te - 1])) --te;
                tl = te - tb;
                h = 0xcbf29ce484222325ull ^ (static_cast<uint64_t>(tl) * 0x9E3779B97F4A7C15ull);
                for (uint32_t q = 0; q < tl; q += 8) {
                    const uint64_t w = in_smem ? ld8(src + tb + q, tl - q) : gload8(p.arena, b0 + tb + q, aend, tl - q);
                    h = mix(h, w);
                    if (q == 0) sw0[k] = w;
                    if (q == 8) sw1[k] = w;
                }
            }
            h = fmix(h);
            hv[k] = h;
            pk[k] = ((b0 + tb) << 24) | tl;
            if (tl >= (1u << 24)) set_dev_err(p.d_err, DEV_INTERN_FULL);  // beyond the 24-bit length field
            // CTA-local table: linear probing, at most 32 probes
            uint32_t s = static_cast<uint32_t>(h) & (LT_CAP - 1);
            for (uint32_t pr = 0; use_lt && pr < 32; ++pr, s = (s + 1) & (LT_CAP - 1)) {
                // a plain read first: hot keys are found without a shared-memory atomic
                const unsigned long long seen = *reinterpret_cast<volatile unsigned long long*>(&lt[s].h);
                if (seen == h) {
                    ent[k] = s;
                    break;
                }
                if (seen != 0ull) continue;
                const unsigned long long prev = atomicCAS(&lt[s].h, 0ull, h);
                if (prev == 0ull) {  // created here: resolved after the barrier
                    lt[s].gslot = EMPTY32;
                    lt[s].min_idx = static_cast<uint32_t>(i0 + j);
                    lt[s].mine = pk[k];
                    newlist[atomicAdd(&s_new[par], 1u)] = s;
                    atomicAdd(&s_fill, 1u);
                    ent[k] = s;
                    break;
                }
                if (prev == h) {
                    ent[k] = s;
                    break;
                }
            }
            if (ent[k] == EMPTY32) glob[k] = true;  // local table crowded: this answer goes global
        }
        __syncthreads();
        const uint32_t nnew = s_new[par];
        if (nnew) {  // keys new to this CTA (rare once the tables are warm)
            // smallest index per new entry (entries created this tile hold this tile's sightings)
#pragma unroll
            for (uint32_t k = 0; k < IT_K; ++k)
                if (ent[k] != EMPTY32 && ent[k] != HIT && lt[ent[k]].gslot == EMPTY32)
                    atomicMin(&lt[ent[k]].min_idx, static_cast<uint32_t>(i0 + tid + k * IT_THREADS));
            __syncthreads();
        }
        // ---- phase B: keys new to this CTA go global (once per CTA) ---------------------
        for (uint32_t q = tid; q < nnew; q += IT_THREADS) {
            LocalEntry& e = lt[newlist[q]];
            unsigned long long c = 0;
            e.gslot = global_insert(p, e.h, e.min_idx, e.mine, &c);
            e.canon = c;
            const uint64_t cl = c & 0xffffffu, cp = c >> 24;  // its first 16 bytes, for short verifies
            e.cb0 = cl ? gload8(p.arena, cp, aend, cl) : 0ull;
            e.cb1 = cl > 8 ? gload8(p.arena, cp + 8, aend, cl - 8) : 0ull;
        }
        if (nnew) __syncthreads();
        // ---- phase C: verify bytes against the canonical copy, write provisional ids ------
#pragma unroll
        for (uint32_t k = 0; k < IT_K; ++k) {
            const uint32_t j = tid + k * IT_THREADS;
            if (j >= cnt) continue;
            if (ent[k] == HIT) {
                p.ids[i0 + j] = gsk[k];
                if (p.hes) p.hes[i0 + j] = static_cast<uint8_t>(hk[k]);
                continue;
            }
            uint32_t gs;
            unsigned long long c;
            bool same;
            const uint32_t tl = static_cast<uint32_t>(pk[k] & 0xffffffu);
            if (glob[k]) {
                gs = global_insert(p, hv[k], static_cast<uint32_t>(i0 + j), pk[k], &c);
                same = c == pk[k] || ((c & 0xffffffu) == tl && (tl == 0 || sw0[k] == gload8(p.arena, c >> 24, aend, tl)) &&
                                      (tl <= 8 || sw1[k] == gload8(p.arena, (c >> 24) + 8, aend, tl - 8)));
            } else {
                const LocalEntry& e = lt[ent[k]];
                gs = e.gslot;
                c = e.canon;
                same = c == pk[k] || ((c & 0xffffffu) == tl && sw0[k] == e.cb0 && sw1[k] == e.cb1);
            }
            p.ids[i0 + j] = gs;
            if (gs == EMPTY32) continue;
            if (in_smem && s_clears_rc < 2) {  // remember the raw answer (<= 16 bytes) for later tiles
                const uint64_t b0 = so[j];
                const uint32_t len = static_cast<uint32_t>(so[j + 1] - b0);
                if (len <= 16) {
                    uint64_t w0, w1;
                    load16_shared(smem_u32(sbuf + IT_OFFB) + static_cast<uint32_t>(b0 - sb), len, w0, w1);
                    const uint32_t rh = raw_hash(w0, w1, len);
                    const uint32_t set = ((rh >> 7) & (RC_CAP / RC_WAYS - 1)) * RC_WAYS;
                    const uint32_t tag = rh | 1u;
                    for (uint32_t w = 0; w < RC_WAYS; ++w) {
                        const uint32_t prev = atomicCAS(&rc_tag[set + w], 0u, tag);
                        if (prev == 0u) {
                            rc_w[2 * (set + w)] = w0;
                            rc_w[2 * (set + w) + 1] = w1;
                            rc_meta[set + w] = make_uint2(len | ((p.hes ? static_cast<uint32_t>(p.hes[i0 + j]) : 0u) << 8), gs);
                            atomicAdd(&s_rfill, 1u);
                            break;
                        }
                        if (prev == tag) break;  // most likely the same answer from another thread
                    }
                }
            }
            const uint64_t mypos = pk[k] >> 24, cpos = c >> 24;
            for (uint32_t q = 16; same && q < tl; q += 8) {  // bytes past the first 16 (long answers)
                const uint64_t a = in_smem ? ld8(sbuf + IT_OFFB + (mypos - sb) + q, tl - q)
                                           : gload8(p.arena, mypos + q, aend, tl - q);
                same = a == gload8(p.arena, cpos + q, aend, tl - q);
            }
            if (!same) set_dev_err(p.d_err, DEV_INTERN_COLLISION);
        }
        __syncthreads();  // stage `st`, the new list and both tables are quiescent
        if (tid == 0) s_new[par] = 0;  // read by everyone before the barrier; next used two tiles on
        const bool cl = s_fill > LT_CAP / 2, cr = s_rfill > RC_CAP / 2;  // crowded: clear
        if (cl || cr) {
            if (cl)
                for (uint32_t e = tid; e < LT_CAP; e += IT_THREADS) lt[e].h = 0;
            if (cr)
                for (uint32_t e = tid; e < RC_CAP; e += IT_THREADS) rc_tag[e] = 0;
            __syncthreads();  // every thread has read the counters and cleared its share
            if (tid == 0) {
                if (cl) {
                    s_fill = 0;
                    ++s_clears_lt;
                }
                if (cr) {
                    s_rfill = 0;
                    ++s_clears_rc;
                }
            }
            __syncthreads();
        }
        st ^= 1u;
    }
}

// slot first indices -> bits of the n-bit first-occurrence bitmap
__global__ void intern_mark(const uint32_t* __restrict__ first, uint64_t cap, uint32_t* __restrict__ bitmap,
                            const int* __restrict__ status) {
    if (*status) return;
    for (uint64_t s = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; s < cap;
         s += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
        const uint32_t f = first[s];
        if (f != EMPTY32) atomicOr(bitmap + (f >> 5), 1u << (f & 31u));
    }
}

struct LoadPopc {
    const uint32_t* w;
    __device__ uint32_t operator()(uint64_t i) const { return __popc(w[i]); }
};

// rank[slot] = first occurrences before the slot's first index (its dense first-seen id)
__global__ void intern_rank(const uint32_t* __restrict__ first, uint64_t cap, const uint32_t* __restrict__ bitmap,
                            const uint32_t* __restrict__ excl, uint32_t* __restrict__ rank,
                            unsigned long long* __restrict__ first_index, const int* __restrict__ status) {
    if (*status) return;
    for (uint64_t s = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; s < cap;
         s += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
        const uint32_t f = first[s];
        if (f == EMPTY32) continue;
        const uint32_t r = excl[f >> 5] + __popc(bitmap[f >> 5] & ((1u << (f & 31u)) - 1u));
        rank[s] = r;
        if (first_index) first_index[r] = f;
    }
}

__global__ void intern_remap(uint32_t* __restrict__ ids, uint64_t n, const uint32_t* __restrict__ rank,
                             const int* __restrict__ status) {
    if (*status) return;
    const uint64_t tid = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
    const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
    const bool vec = (reinterpret_cast<uintptr_t>(ids) & 15u) == 0;
    const uint64_t n4 = vec ? n / 4 : 0;
    for (uint64_t q = tid; q < n4; q += stride) {
        uint4 v = reinterpret_cast<const uint4*>(ids)[q];
        v.x = __ldg(rank + v.x);
        v.y = __ldg(rank + v.y);
        v.z = __ldg(rank + v.z);
        v.w = __ldg(rank + v.w);
        reinterpret_cast<uint4*>(ids)[q] = v;
    }
    for (uint64_t i = n4 * 4 + tid; i < n; i += stride) ids[i] = __ldg(rank + ids[i]);
}

}  // namespace
}  // namespace cdx

extern "C" int cdx_canon_intern(cdx_ctx* ctx, const char* bytes, const uint64_t* offsets, uint64_t n,
                                const char* const* markers, uint32_t n_markers, uint32_t* ids, uint8_t* hes,
                                uint64_t* first_index, uint64_t* n_unique) {
    using namespace cdx;
    CDX_NVTX("cdx_canon_intern");
    if (!ctx) return CDX_EINVAL;
    if (!offsets || !ids || !n_unique) return set_error(ctx, CDX_EINVAL, "canon_intern: null pointer");
    if (n >= 0xffffffffull) return set_error(ctx, CDX_EINVAL, "canon_intern: at most 2^32-2 answers per call");
    if (n_markers > MAX_MARKERS) return set_error(ctx, CDX_EINVAL, "canon_intern: at most 16 markers");
    Markers mk{};
    mk.n = n_markers;
    uint32_t pos = 0;
    for (uint32_t k = 0; k < n_markers; ++k) {
        const size_t len = markers[k] ? std::strlen(markers[k]) : 0;
        if (pos + len > MARKER_BYTES) return set_error(ctx, CDX_EINVAL, "canon_intern: markers exceed 1 KiB");
        mk.off[k] = pos;
        if (len) std::memcpy(mk.bytes + pos, markers[k], len);
        pos += static_cast<uint32_t>(len);
    }
    mk.off[n_markers] = pos;
    for (uint32_t k = 0; k < n_markers; ++k) {
        uint64_t w = 0;
        for (uint32_t j = 0; j < 8 && mk.off[k] + j < mk.off[k + 1]; ++j)
            w |= static_cast<uint64_t>(static_cast<uint8_t>(mk.bytes[mk.off[k] + j])) << (8 * j);
        mk.word[k] = w;
    }
    *n_unique = 0;
    if (n == 0) return CDX_OK;
    if (!bytes) return set_error(ctx, CDX_EINVAL, "canon_intern: null pointer");

    static thread_local int occ_dev = -1, per_sm = 1;
    const size_t smem = 2 * IT_STAGE + LT_CAP * sizeof(LocalEntry) + RC_BYTES + IT_TILE * 4 + 16;
    if (occ_dev != ctx->device) {
        cudaFuncSetAttribute(intern_tiles, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, intern_tiles, IT_THREADS, smem);
        per_sm = std::max(per_sm, 1);
        occ_dev = ctx->device;
    }
    const uint8_t* arena = reinterpret_cast<const uint8_t*>(bytes);
    const int staged = (reinterpret_cast<uintptr_t>(arena) % 16 == 0) && (reinterpret_cast<uintptr_t>(offsets) % 16 == 0);
    for (int attempt = 0; attempt < 2; ++attempt) {
        // capacity: the context's last (distinct answers < cap / 2), or room for every answer
        uint64_t cap = std::max<uint64_t>(ctx->it_cap, 1ull << 20);
        if (attempt == 1) {
            cap = 1ull << 20;
            while (cap < 2 * n) cap <<= 1;
        }
        const uint64_t words = (n + 31) / 32;
        const uint64_t nrec = (words + scan::SL_TILE - 1) / scan::SL_TILE + 2;
        // table: hash u64 | canon u64 (reused as rank u32 after the insert pass) | first u32 |
        // bitmap u32[words] | excl u32[words] | scan records | counters
        const size_t bytes_need = cap * 8 + cap * 8 + cap * 4 + words * 4 + words * 4 + 64 + nrec * 8 + 64;
        uint8_t* s = static_cast<uint8_t*>(scratch(ctx, bytes_need));
        if (!s) return set_error(ctx, CDX_ECUDA, "canon_intern: scratch allocation failed");
        auto* hkey = reinterpret_cast<unsigned long long*>(s);
        auto* canon = hkey + cap;
        auto* first = reinterpret_cast<uint32_t*>(canon + cap);
        auto* bitmap = first + cap;
        auto* excl = bitmap + words;
        auto* counters = reinterpret_cast<uint32_t*>(reinterpret_cast<uintptr_t>(excl + words + 15) & ~uintptr_t(15));
        auto* rec = reinterpret_cast<uint64_t*>(counters + 8);
        auto* total = rec + nrec;
        cudaMemsetAsync(hkey, 0, cap * 8, ctx->stream);
        cudaMemsetAsync(canon, 0xff, cap * 8, ctx->stream);
        cudaMemsetAsync(first, 0xff, cap * 4, ctx->stream);
        cudaMemsetAsync(bitmap, 0, words * 4, ctx->stream);
        cudaMemsetAsync(counters, 0, 32, ctx->stream);
        InternParams p{};
        p.arena = arena;
        p.off = offsets;
        p.n = n;
        p.hkey = hkey;
        p.first = first;
        p.canon = canon;
        p.cap_mask = cap - 1;
        p.ids = ids;
        p.hes = hes;
        p.n_keys = counters;
        p.key_limit = static_cast<uint32_t>(std::min<uint64_t>(cap / 2, 0xffffffffull));
        p.status = reinterpret_cast<int*>(counters + 1);
        p.d_err = ctx->d_err;
        p.staged = staged;
        const uint64_t tiles = (n + IT_TILE - 1) / IT_TILE;
        const unsigned grid = static_cast<unsigned>(std::min<uint64_t>(tiles, static_cast<uint64_t>(ctx->sm_count) * per_sm));
        // a CTA's tables pay off over many tiles; a short call goes straight to the global table
        p.local_tables = tiles >= 8ull * grid;
        intern_tiles<<<grid, IT_THREADS, smem, ctx->stream>>>(p, mk);
        CDX_CHECK_LAUNCH(ctx, "canon_intern(tiles)");
        const unsigned g2 = static_cast<unsigned>(std::min<uint64_t>((cap + 255) / 256, ctx->sm_count * 16ull));
        intern_mark<<<g2, 256, 0, ctx->stream>>>(first, cap, bitmap, p.status);
        CDX_CHECK_LAUNCH(ctx, "canon_intern(mark)");
        if (int st = scan::scan_excl(ctx, LoadPopc{bitmap}, words, excl, false, rec, total)) return st;
        auto* rank = reinterpret_cast<uint32_t*>(canon);  // canonical packs are no longer needed
        intern_rank<<<g2, 256, 0, ctx->stream>>>(first, cap, bitmap, excl, rank,
                                                 reinterpret_cast<unsigned long long*>(first_index), p.status);
        CDX_CHECK_LAUNCH(ctx, "canon_intern(rank)");
        const unsigned g3 = static_cast<unsigned>(std::min<uint64_t>((n / 4 + 255) / 256 + 1, ctx->sm_count * 16ull));
        intern_remap<<<g3, 256, 0, ctx->stream>>>(ids, n, rank, p.status);
        CDX_CHECK_LAUNCH(ctx, "canon_intern(remap)");
        uint64_t h[2] = {0, 0};
        cudaError_t e = cudaMemcpyAsync(&h[0], total, 8, cudaMemcpyDeviceToHost, ctx->stream);
        if (e == cudaSuccess) e = cudaMemcpyAsync(&h[1], counters + 1, 4, cudaMemcpyDeviceToHost, ctx->stream);
        if (e == cudaSuccess) e = cudaStreamSynchronize(ctx->stream);
        if (e != cudaSuccess) return cuda_fail(ctx, e, "canon_intern");
        if (h[1] & 1) continue;  // overflow: redo with room for every answer
        *n_unique = h[0];
        uint64_t want = 1ull << 20;  // next call: a table at least 4x the distinct answers
        while (want < 4 * h[0]) want <<= 1;
        ctx->it_cap = want;
        return CDX_OK;
    }
    return set_error(ctx, CDX_ERUNTIME, "canon_intern: intern table full");
}
