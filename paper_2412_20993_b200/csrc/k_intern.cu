// k_intern.cu — K1: answer canonicalisation, interning and hesitation flags.
//
// Replaces metrics::trim + the unordered_map<string_view> key of cluster_exact (metrics.cpp:
// 12-37) — every comparison of answers in the reference goes through trimmed exact bytes —
// and probe::flag_hesitation (probe.cpp:36-44).  Output ids are DENSE and in first-seen
// order of the trimmed bytes (exactly the cluster order cluster_exact would produce over
// the whole arena), so every downstream kernel compares u32 ids instead of strings.
//
// A serving trace repeats a small set of answers many times, so the hot path never touches
// global atomics and never waits on a CTA barrier:
//
//   intern_ws      one persistent CTA per SM, warp-specialised.  A producer warp streams the
//                  CTA's tiles of 1024 answers (tile c, c + grid, ...) into a 6-stage shared
//                  ring by 1-D bulk copies (offsets window + arena window, mbarrier
//                  complete_tx), reading the tile boundaries for 32 tiles per round trip.
//                  Consumer warps take 32-answer slices of the ring in order (one answer per
//                  lane) and release each slice on the stage's empty barrier.
//                  Per answer of <= 16 bytes the lane builds four masked words from shared
//                  memory and looks the RAW bytes up in the CTA's 4-way raw-answer cache; a
//                  hit (the common case) gives the key's local entry and the hesitation flag
//                  with no trim, hash, marker scan or byte verify.  A miss trims, hashes the
//                  trimmed bytes, scans the markers, finds or creates the key in the CTA's
//                  local table (a created key is inserted globally once per CTA: CAS on the
//                  hash, atomicMin of its first index, CAS electing its canonical bytes),
//                  verifies the bytes against the canonical copy (a 64-bit hash collision is
//                  reported, never merged) and caches the raw answer.
//   first indices  every atomicMin that lowers a key's first index XORs the old and the new
//                  index bit of an n-bit bitmap; XOR commutes, so whatever the interleaving
//                  the bitmap ends as exactly the set of first occurrences.
//   dense ids      a key's dense id is the number of first occurrences before its own.  The
//                  tiles are processed in rounds (round q = the q-th tile of every CTA); once
//                  every CTA has finished round q, the bits in round q's range are final and
//                  the last CTA to finish it publishes their count.  The producer warp turns
//                  its local keys' first indices into dense ids as soon as the rounds up to
//                  them are complete, so a slice whose 32 keys all have one writes FINAL ids;
//                  any other slice writes global slots and sets its bit in a slice bitmap.
//   remap          after a popcount scan of the first-occurrence bitmap, only the flagged
//                  slices are rewritten (ids[i] = rank[slot]); with a warm vocabulary that
//                  is the first few rounds' slices, not the whole id array.
//
// The global table starts at the capacity the context used last (2^20 slots at first); a
// call whose distinct answers exceed half of it is redone with room for every answer.
#include <algorithm>
#include <cstddef>
#include <cstdlib>
#include <cstdio>
#include <cstring>
#include <vector>

#include "cdx_internal.cuh"
#include "k_scan.cuh"

namespace cdx {
namespace {

constexpr int MAX_MARKERS = 16;
constexpr int MARKER_BYTES = 1024;
constexpr uint32_t WS_TILE = 1024;                // answers per tile = 32 slices of 32
constexpr uint32_t WS_CHUNK = 128;                // answers per consumer step: 4 slices, 4 per lane
constexpr uint32_t WS_CHUNKS = WS_TILE / WS_CHUNK;
constexpr uint32_t WS_MAXW = 22;                  // consumer warps per CTA (at most)
constexpr uint32_t WS_ST = 6;                     // ring stages
constexpr uint32_t WS_OFFB = (WS_TILE + 4) * 8;   // offsets window: cnt + 1 values + alignment slack
constexpr uint32_t WS_ARENA = 14368;              // arena window (16-B multiple)
constexpr uint32_t WS_STAGE = WS_OFFB + WS_ARENA;
constexpr uint32_t WS_LT = 256;                   // CTA-local key table
constexpr uint32_t WS_RC = 2048;                  // raw-answer cache entries (4-way sets)
constexpr uint32_t LOCKED = 0xffffffffu;          // raw-cache tag being written (never a real tag)
constexpr uint32_t WS_RAWMAX = 12;                // raw answers cached (three words)
constexpr uint32_t EMPTY32 = 0xffffffffu;
constexpr uint64_t EMPTY64 = ~0ull;
constexpr int64_t INPLACE = INT64_MIN;            // stage holds no arena window: read in place

struct Markers {
    uint32_t n;
    uint32_t off[MAX_MARKERS + 1];
    uint64_t word[MAX_MARKERS];  // first 8 bytes, little-endian (short-answer fast path)
    char bytes[MARKER_BYTES];
};

struct WsParams {
    const uint8_t* arena;
    const uint64_t* off;
    uint64_t n;
    uint64_t tiles;
    unsigned long long* hkey;   // global table: hash (0 = empty)
    uint32_t* first;            //               first arena index (EMPTY32)
    unsigned long long* canon;  //               canonical trimmed bytes: pos << 24 | len (EMPTY64)
    uint64_t cap_mask;
    uint32_t* bitmap;           // n bits: first occurrences (XOR-maintained)
    uint32_t* round_done;       // per round: CTAs that finished their tile of it
    uint32_t* round_cnt;        // per round: 1 + first occurrences in its range (0 = not final)
    uint32_t* slice_flags;      // per 32-answer slice: ids written as global slots
    uint32_t* ids;
    uint8_t* hes;
    uint32_t* n_keys;           // distinct keys inserted (overflow watch)
    uint32_t key_limit;
    int* status;                // bit 0 overflow
    int* d_err;
    unsigned long long* stats;  // diagnostics (CDX_IT_STATS=1): chunks, provisional chunks, misses, early firsts
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


// ---- global table -------------------------------------------------------------------------
// first[s] = min(first[s], idx); a lowering XORs the old and the new bit of the first-
// occurrence bitmap (each key's lowerings form one decreasing chain, so the XORs cancel
// pairwise and leave exactly the final first index of every key)
__device__ __forceinline__ void first_min(const WsParams& p, uint32_t s, uint32_t idx) {
    const uint32_t old = atomicMin(p.first + s, idx);
    if (idx < old) {
        atomicXor(p.bitmap + (idx >> 5), 1u << (idx & 31u));
        if (old != EMPTY32) atomicXor(p.bitmap + (old >> 5), 1u << (old & 31u));
    }
}

// insert one key: slot (EMPTY32 on overflow), first index and canonical bytes
__device__ uint32_t ws_insert(const WsParams& p, uint64_t h, uint32_t idx, unsigned long long cpack,
                              unsigned long long* canon_out) {
    uint64_t s = h & p.cap_mask;
    for (uint64_t probes = 0;; ++probes) {
        unsigned long long prev = __ldcg(p.hkey + s);  // most keys exist: no atomic to find them
        if (prev == 0ull) prev = atomicCAS(p.hkey + s, 0ull, h);
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
    first_min(p, static_cast<uint32_t>(s), idx);
    const unsigned long long c = atomicCAS(p.canon + s, EMPTY64, cpack);
    *canon_out = c == EMPTY64 ? cpack : c;
    return static_cast<uint32_t>(s);
}

// ---- raw-answer cache ---------------------------------------------------------------------
// 32-bit hash of a raw answer's three masked words (hits compare every word and the length)
__device__ __forceinline__ uint32_t raw_hash(uint32_t w0, uint32_t w1, uint32_t w2, uint32_t len) {
    uint32_t h = len * 0x9E3779B1u;
    h = (h ^ w0) * 0x85EBCA6Bu;
    h = (h ^ w1) * 0xC2B2AE35u;
    h = (h ^ w2) * 0x27D4EB2Fu;
    return h;
}
// first entry of a raw hash's 4-way set, and its tag (top bit clear: never LOCKED, never 0).  The
// set comes from the top bits of the last product (its low bits see only the inputs' low bits).
__device__ __forceinline__ uint32_t rc_set(uint32_t h) { return (h >> 23) * 4u; }
__device__ __forceinline__ uint32_t rc_tag_of(uint32_t h) { return (h | 1u) & 0x7fffffffu; }
static_assert(WS_RC == 2048, "rc_set takes the top 9 bits");

// the 12 bytes at base + rel as three words, masked to the answer's length: four aligned
// 4-byte loads (conflict-free for odd word strides) and three funnel shifts.  base is a
// 16-byte aligned shared-memory pointer (pointer arithmetic only, so the loads stay LDS).
__device__ __forceinline__ void load_words(const uint8_t* base, uint32_t rel, const uint4& m, uint32_t& w0, uint32_t& w1,
                                           uint32_t& w2) {
    const uint32_t* a4 = reinterpret_cast<const uint32_t*>(base + (rel & ~3u));
    const uint32_t sh = (rel & 3u) * 8u;
    const uint32_t x0 = a4[0], x1 = a4[1], x2 = a4[2], x3 = a4[3];
    w0 = __funnelshift_r(x0, x1, sh) & m.x;
    w1 = __funnelshift_r(x1, x2, sh) & m.y;
    w2 = __funnelshift_r(x2, x3, sh) & m.z;
}

// release / acquire at GPU scope (lighter than __threadfence's fence.sc)
__device__ __forceinline__ void fence_acq_rel_gpu() { asm volatile("fence.acq_rel.gpu;" ::: "memory"); }
__device__ __forceinline__ void red_relaxed_add(uint32_t* a, uint32_t v) {
    asm volatile("red.relaxed.gpu.global.add.u32 [%0], %1;" ::"l"(a), "r"(v) : "memory");
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

__device__ __forceinline__ uint32_t ld_volatile(const uint32_t* a) { return *reinterpret_cast<const volatile uint32_t*>(a); }
__device__ __forceinline__ uint4 lds128_volatile(const void* a) {
    uint4 v;
    asm volatile("ld.volatile.shared.v4.u32 {%0, %1, %2, %3}, [%4];"
                 : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
                 : "r"(smem_u32(a)));
    return v;
}
__device__ __forceinline__ void sts128_volatile(void* a, uint4 v) {
    asm volatile("st.volatile.shared.v4.u32 [%0], {%1, %2, %3, %4};" ::"r"(smem_u32(a)), "r"(v.x), "r"(v.y), "r"(v.z),
                 "r"(v.w)
                 : "memory");
}
// shared state of one CTA (dynamic shared memory after the ring)
struct WsShared {
    uint4 rc[WS_RC];                      // raw answer: three masked words, len | hes << 8 | local entry << 16
                                          // (written once, by one 16-byte store; w = 0xffffffff: empty)
    uint32_t rc_tag[WS_RC];               // tag of the entry (0 empty, LOCKED being written)
    uint4 lt_info[WS_LT];                 // {global slot, dense id (EMPTY32), smallest index submitted, ready}
    unsigned long long lt_h[WS_LT];       // trimmed-key hash (0 empty)
    unsigned long long lt_canon[WS_LT];   // canonical pack
    ulonglong2 lt_cb[WS_LT];              // canonical's first 16 trimmed bytes
    uint4 lenmask[WS_RAWMAX + 1];         // bytes below len of the three words, by len
    uint64_t full[WS_ST], empty[WS_ST];
    int64_t abase[WS_ST];                 // arena offset of the stage's arena window (INPLACE)
    uint32_t odel[WS_ST];                 // offsets window: element shift of the tile's first offset
    uint32_t lt_fill, rc_fill, cons_done, ranked;
    uint32_t stage_steps[WS_ST];          // consumer steps finished per stage (monotonic)
};
constexpr size_t WS_SMEM = WS_ST * WS_STAGE + sizeof(WsShared);

// A local entry found under creation is published by a thread of this CTA within a global
// round trip: wait for it (bounded) rather than repeat its global insert.
// A true return is followed by a CTA fence: the entry's fields (written before its creator's
// fence and flag store) are read after the flag was seen.
__device__ __forceinline__ bool entry_ready(WsShared& S, int e) {
    bool ready = false;
    for (int spin = 0; spin < 64 && !ready; ++spin) {
        ready = ld_volatile(&S.lt_info[e].w) != 0u;
        if (!ready) __nanosleep(128);
    }
    ready = ready || ld_volatile(&S.lt_info[e].w) != 0u;
    if (ready) __threadfence_block();
    return ready;
}

// The miss path of one answer: trim, hash, hesitation, local/global key, verify, cache.
// Returns {global slot, the key's dense id when already final (else EMPTY32), hes | global atomics << 1}.
__device__ __noinline__ uint3 ws_miss(const WsParams& p, const Markers& mk, WsShared& S, const uint8_t* src,
                                         uint64_t b0, uint64_t len, uint32_t idx, bool cacheable, uint32_t w0_, uint32_t w1_,
                                         uint32_t w2_, uint32_t rh, uint64_t aend) {
    uint32_t tb, tl, hes = 0;
    uint64_t h, sw0 = 0, sw1 = 0;
    if (cacheable) {
        const uint64_t w0 = w0_ | (static_cast<uint64_t>(w1_) << 32), w1 = w2_;
        const Short a = short_answer(w0, w1, static_cast<uint32_t>(len), mk, p.hes != nullptr);
        hes = a.hes;
        tb = a.tb;
        tl = a.tl;
        h = 0xcbf29ce484222325ull ^ (static_cast<uint64_t>(tl) * 0x9E3779B97F4A7C15ull);
        if (tl) h = mix(h, a.t0);
        if (tl > 8) h = mix(h, a.t1);
        sw0 = a.t0;
        sw1 = a.t1;
    } else {
        if (len >= (1ull << 24)) {  // beyond the 24-bit length field of the canonical pack
            set_dev_err(p.d_err, DEV_INTERN_FULL);
            len = (1ull << 24) - 1;
        }
        const uint32_t l32 = static_cast<uint32_t>(len);
        if (p.hes) hes = hesitant(mk, src, l32, false);
        uint32_t te = l32;
        tb = 0;
        while (tb < te && is_space(src[tb])) ++tb;
        while (te > tb && is_space(src[te - 1])) --te;
        tl = te - tb;
        h = 0xcbf29ce484222325ull ^ (static_cast<uint64_t>(tl) * 0x9E3779B97F4A7C15ull);
        const bool shared_src = __isShared(src);
        for (uint32_t q = 0; q < tl; q += 8) {
            const uint64_t x = shared_src ? ld8(src + tb + q, tl - q) : gload8(p.arena, b0 + tb + q, aend, tl - q);
            h = mix(h, x);
            if (q == 0) sw0 = x;
            if (q == 8) sw1 = x;
        }
    }
    h = fmix(h);
    const unsigned long long pk = ((b0 + tb) << 24) | tl;
    // local key table: linear probing, at most 32 probes; creation stops at half full
    int e = -1;
    bool creator = false;
    uint32_t s = static_cast<uint32_t>(h) & (WS_LT - 1);
    for (uint32_t pr = 0; pr < 32; ++pr, s = (s + 1) & (WS_LT - 1)) {
        const unsigned long long seen = *reinterpret_cast<volatile unsigned long long*>(&S.lt_h[s]);
        if (seen == h) {
            e = static_cast<int>(s);
            break;
        }
        if (seen != 0ull) continue;
        if (ld_volatile(&S.lt_fill) >= WS_LT / 2) break;
        const unsigned long long prev = atomicCAS(&S.lt_h[s], 0ull, h);
        if (prev == 0ull) {
            atomicAdd(&S.lt_fill, 1u);
            e = static_cast<int>(s);
            creator = true;
            break;
        }
        if (prev == h) {
            e = static_cast<int>(s);
            break;
        }
    }
    uint32_t gs, rank = EMPTY32;
    unsigned long long c;
    bool same, atom = true;
    if (creator) {  // the CTA's first sighting: one global insert, then the entry is published
        gs = ws_insert(p, h, idx, pk, &c);
        if (gs == EMPTY32) c = pk;  // overflow: the call is redone with a larger table
        const uint64_t cl = c & 0xffffffu, cp = c >> 24;
        const unsigned long long cb0 = cl ? gload8(p.arena, cp, aend, cl) : 0ull;
        const unsigned long long cb1 = cl > 8 ? gload8(p.arena, cp + 8, aend, cl - 8) : 0ull;
        S.lt_canon[e] = c;
        S.lt_cb[e] = make_ulonglong2(cb0, cb1);
        S.lt_info[e].x = gs;
        S.lt_info[e].y = EMPTY32;
        S.lt_info[e].z = idx;
        __threadfence_block();
        *reinterpret_cast<volatile uint32_t*>(&S.lt_info[e].w) = 1u;
        same = c == pk || ((c & 0xffffffu) == tl && (tl == 0 || sw0 == cb0) && (tl <= 8 || sw1 == cb1));
    } else if (e >= 0 && entry_ready(S, e)) {
        gs = ld_volatile(&S.lt_info[e].x);
        rank = ld_volatile(&S.lt_info[e].y);
        c = S.lt_canon[e];
        const ulonglong2 cb = S.lt_cb[e];
        if (idx < ld_volatile(&S.lt_info[e].z)) {  // earlier than anything this CTA submitted
            if (gs != EMPTY32) first_min(p, gs, idx);
            atomicMin(&S.lt_info[e].z, idx);
        } else {
            atom = false;
        }
        same = c == pk || ((c & 0xffffffu) == tl && (tl == 0 || sw0 == cb.x) && (tl <= 8 || sw1 == cb.y));
    } else {  // no local entry (table full) or its creator has not published it yet
        e = -1;
        gs = ws_insert(p, h, idx, pk, &c);
        if (gs == EMPTY32) c = pk;
        same = c == pk || ((c & 0xffffffu) == tl && (tl == 0 || sw0 == gload8(p.arena, c >> 24, aend, tl)) &&
                           (tl <= 8 || sw1 == gload8(p.arena, (c >> 24) + 8, aend, tl - 8)));
    }
    const uint64_t mypos = pk >> 24, cpos = c >> 24;
    const bool shared_src = __isShared(src);
    for (uint32_t q = 16; same && q < tl; q += 8) {  // bytes past the first 16 (long answers)
        const uint64_t a = shared_src ? ld8(src + (mypos - b0) + q, tl - q) : gload8(p.arena, mypos + q, aend, tl - q);
        same = a == gload8(p.arena, cpos + q, aend, tl - q);
    }
    if (!same) set_dev_err(p.d_err, DEV_INTERN_COLLISION);
    // cache the raw answer (<= 16 bytes, verified, with a published local entry)
    if (cacheable && e >= 0 && same && gs != EMPTY32) {
        const uint4 ent = make_uint4(w0_, w1_, w2_, static_cast<uint32_t>(len) | (hes << 8) | (static_cast<uint32_t>(e) << 16));
        const uint32_t set = rc_set(rh), tag = rc_tag_of(rh);
        for (uint32_t way = 0; way < 4; ++way) {
            const uint32_t prev = atomicCAS(&S.rc_tag[set + way], 0u, LOCKED);
            if (prev == 0u) {
                sts128_volatile(&S.rc[set + way], ent);  // the entry, then its tag
                __threadfence_block();
                *reinterpret_cast<volatile uint32_t*>(&S.rc_tag[set + way]) = tag;
                if (p.stats) atomicAdd(p.stats + 8 + 2 * gridDim.x + 3 * blockIdx.x + 1, 1ull);
                break;
            }
            if (prev == tag || prev == LOCKED) break;  // cached, or being cached: no duplicate ways
        }
    }
    return make_uint3(gs, rank, hes | (atom ? 2u : 0u));
}

struct MissOut {
    uint32_t g[4], r[4], h[4];
    bool atom;
};
// the hit path's results for the four answers, handed through the miss call so that none
// of them stays live across it
struct ChunkRes {
    uint32_t g0, g1, g2, g3, r0, r1, r2, r3, hmask;
};

// The chunk's missed answers (bit k of miss: answer j0 + 32k + lane), recomputed from the
// stage and sent through ws_miss; out of line so the hit path keeps its registers.
__device__ __noinline__ MissOut chunk_misses(const WsParams& p, const Markers& mk, WsShared& S, const uint8_t* sbuf,
                                             const uint64_t* so, int64_t abase, uint64_t i0, uint32_t j0, uint64_t aend,
                                             uint32_t miss, ChunkRes in) {
    MissOut o{};
    o.g[0] = in.g0, o.g[1] = in.g1, o.g[2] = in.g2, o.g[3] = in.g3;
    o.r[0] = in.r0, o.r[1] = in.r1, o.r[2] = in.r2, o.r[3] = in.r3;
    for (uint32_t k = 0; k < 4; ++k) o.h[k] = (in.hmask >> k) & 1u;
    const uint32_t lane = threadIdx.x & 31u;
    for (uint32_t k = 0; k < 4; ++k) {
        if (!(miss & (1u << k))) continue;
        const uint32_t j = j0 + k * 32u + lane;
        const uint64_t b0 = so[j], len = so[j + 1] - b0;
        const bool cacheable = abase != INPLACE && len <= WS_RAWMAX;
        uint32_t w0 = 0, w1 = 0, w2 = 0, rh = 0;
        if (cacheable) {
            load_words(sbuf + WS_OFFB, static_cast<uint32_t>(b0) - static_cast<uint32_t>(abase), S.lenmask[len], w0, w1, w2);
            rh = raw_hash(w0, w1, w2, static_cast<uint32_t>(len));
        }
        const uint8_t* src = abase != INPLACE ? sbuf + WS_OFFB + (static_cast<int64_t>(b0) - abase) : p.arena + b0;
        const uint3 r = ws_miss(p, mk, S, src, b0, len, static_cast<uint32_t>(i0 + k * 32u + lane), cacheable, w0, w1, w2,
                                rh, aend);
        o.g[k] = r.x;
        o.r[k] = r.y;
        o.h[k] = r.z & 1u;
        o.atom |= (r.z & 2u) != 0;
    }
    return o;
}

// dense id of a first index whose round is complete: first occurrences in earlier rounds
// (pre) plus those of its own round before it
__device__ uint32_t round_rank(const WsParams& p, uint32_t f, uint64_t round_lo_word, uint32_t pre, uint32_t lane) {
    uint32_t c = 0;
    const uint64_t fw = f >> 5;
    for (uint64_t w = round_lo_word + lane; w < fw; w += 32) c += __popc(__ldcg(p.bitmap + w));
#pragma unroll
    for (int o = 16; o; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
    return pre + c + __popc(__ldcg(p.bitmap + fw) & ((1u << (f & 31u)) - 1u));
}

// Warp roles: warps [0, NW) consume slices, warp NW produces the ring, warp NW + 1 publishes
// round counts and turns the local keys' first indices into dense ids.
__global__ void __launch_bounds__(32 * (WS_MAXW + 2), 1) intern_ws(const __grid_constant__ WsParams p,
                                                     const __grid_constant__ Markers mk) {
    extern __shared__ __align__(128) uint8_t smem[];
    uint8_t* ring = smem;
    WsShared& S = *reinterpret_cast<WsShared*>(smem + WS_ST * WS_STAGE);
    const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31u;
    const uint32_t NW = blockDim.x / 32 - 2;
    const uint32_t G = gridDim.x;
    const uint64_t rounds = (p.tiles + G - 1) / G;
    if (p.stats && threadIdx.x == 0) {
        uint64_t t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        p.stats[8 + 2 * blockIdx.x] = t;
    }

    for (uint32_t e = threadIdx.x; e < WS_RC; e += blockDim.x) {
        S.rc[e] = make_uint4(0u, 0u, 0u, 0xffffffffu);
        S.rc_tag[e] = 0;
    }
    for (uint32_t e = threadIdx.x; e < WS_LT; e += blockDim.x) {
        S.lt_h[e] = 0;
        S.lt_info[e] = make_uint4(EMPTY32, EMPTY32, EMPTY32, 0u);
    }
    if (threadIdx.x <= WS_RAWMAX) {
        const uint32_t l8 = threadIdx.x * 8;
        auto m = [&](uint32_t k) { return l8 >= 32 * (k + 1) ? 0xffffffffu : (l8 <= 32 * k ? 0u : (1u << (l8 - 32 * k)) - 1u); };
        S.lenmask[threadIdx.x] = make_uint4(m(0), m(1), m(2), m(3));
    }
    if (threadIdx.x == 0) {
        S.lt_fill = S.rc_fill = S.cons_done = S.ranked = 0;
        for (uint32_t k = 0; k < WS_ST; ++k) S.stage_steps[k] = 0;
        for (uint32_t k = 0; k < WS_ST; ++k) {
            mbar_init(&S.full[k], 1);
            mbar_init(&S.empty[k], WS_CHUNKS);  // one arrival per consumer step
        }
        fence_mbar_init();
    }
    __syncthreads();

    if (warp == NW) {  // ---- producer -------------------------------------------------------
        const uint64_t policy = policy_evict_first();
        const uint64_t aend = __ldg(p.off + p.n);
        const uintptr_t abeg = reinterpret_cast<uintptr_t>(p.arena), aendp = abeg + aend;
        const uintptr_t obeg = reinterpret_cast<uintptr_t>(p.off), oendp = obeg + (p.n + 1) * 8;
        uint64_t blo = 0, bhi = 0;
        for (uint64_t q = 0;; ++q) {
            const uint64_t t = blockIdx.x + q * G;
            if (t >= p.tiles) break;
            const uint32_t st = static_cast<uint32_t>(q % WS_ST);
            if (q >= WS_ST) {
                mbar_wait(&S.empty[st], static_cast<uint32_t>((q / WS_ST) - 1) & 1u);
            }
            if ((q & 31u) == 0) {  // boundaries of this CTA's next 32 tiles, one round trip
                const uint64_t tq = blockIdx.x + (q + lane) * G;
                if (tq < p.tiles) {
                    const uint64_t i0 = tq * WS_TILE;
                    blo = __ldg(p.off + i0);
                    bhi = __ldg(p.off + min(i0 + WS_TILE, p.n));
                }
            }
            const uint64_t lo = __shfl_sync(0xffffffffu, blo, static_cast<int>(q & 31u));
            const uint64_t hi = __shfl_sync(0xffffffffu, bhi, static_cast<int>(q & 31u));
            const uint64_t i0 = t * WS_TILE, cnt = min(static_cast<uint64_t>(WS_TILE), p.n - i0);
            uint8_t* sbuf = ring + st * WS_STAGE;
            // offsets window [olo, ohi): the bulk part inside the array, the rest (<= 8 B a side) by hand
            const uintptr_t oa = reinterpret_cast<uintptr_t>(p.off + i0), ob = oa + (cnt + 1) * 8;
            const uintptr_t olo = oa & ~static_cast<uintptr_t>(15), ohi = (ob + 15) & ~static_cast<uintptr_t>(15);
            const uintptr_t obl = max(olo, (obeg + 15) & ~static_cast<uintptr_t>(15));
            const uintptr_t obh = min(ohi, oendp & ~static_cast<uintptr_t>(15));
            // arena window [alo, ahi)
            const uintptr_t alo = (abeg + lo) & ~static_cast<uintptr_t>(15);
            const uintptr_t ahi = (abeg + hi + 15) & ~static_cast<uintptr_t>(15);
            const bool fits = ahi - alo <= WS_ARENA;
            const uintptr_t abl = max(alo, (abeg + 15) & ~static_cast<uintptr_t>(15));
            const uintptr_t abh = min(ahi, aendp & ~static_cast<uintptr_t>(15));
            // hand-copied edges: lane k < 16 takes head byte k, lanes 16.. tail bytes
            {
                const uintptr_t x = lane < 16 ? obl - 16 + lane : obh + (lane - 16);
                const bool in = lane < 16 ? (x >= olo && x < obl) : (x < ohi);
                if (in && x >= obeg && x < oendp) sbuf[x - olo] = *reinterpret_cast<const uint8_t*>(x);
                if (fits) {
                    const uintptr_t y = lane < 16 ? abl - 16 + lane : abh + (lane - 16);
                    const bool iny = lane < 16 ? (y >= alo && y < abl) : (y < ahi);
                    if (iny && y >= abeg && y < aendp) sbuf[WS_OFFB + (y - alo)] = *reinterpret_cast<const uint8_t*>(y);
                }
            }
            __syncwarp();
            if (lane == 0) {
                S.odel[st] = static_cast<uint32_t>((oa - olo) / 8);
                S.abase[st] = fits ? static_cast<int64_t>(alo - abeg) : INPLACE;
                const uint32_t otx = obh > obl ? static_cast<uint32_t>(obh - obl) : 0u;
                const uint32_t atx = fits && abh > abl ? static_cast<uint32_t>(abh - abl) : 0u;
                fence_proxy_async();  // the stage's earlier generic reads precede the async writes
                mbar_expect_tx(&S.full[st], otx + atx);
                if (otx) bulk_g2s(sbuf + (obl - olo), reinterpret_cast<const void*>(obl), otx, &S.full[st], policy);
                if (atx)
                    bulk_g2s(sbuf + WS_OFFB + (abl - alo), reinterpret_cast<const void*>(abl), atx, &S.full[st], policy);
            }
        }
        return;
    }

    if (warp == NW + 1) {  // ---- round counts and dense ids -----------------------------------
        uint64_t my_r = blockIdx.x;  // rounds this CTA publishes: blockIdx.x, + G, ...
        uint64_t pre_q = 0;          // rounds [0, pre_q) have published counts summing to pre
        uint32_t pre = 0;
        const uint64_t round_answers = static_cast<uint64_t>(G) * WS_TILE;
        uint64_t q_next = 0;  // this CTA's next tile to report in round_done
        const uint64_t my_tiles = (p.tiles - blockIdx.x + G - 1) / G;
        while (ld_volatile(&S.cons_done) < NW) {
            bool progress = false;
            // tiles whose consumer steps are all done: one fence, then a reduction per tile
            // (at most 64 per pass, so the other duties below are never starved)
            uint64_t q_end = q_next;
            while (q_end < my_tiles && q_end < q_next + 64 &&
                   ld_volatile(&S.stage_steps[q_end % WS_ST]) >= static_cast<uint32_t>(q_end / WS_ST + 1) * WS_CHUNKS)
                ++q_end;
            if (q_end > q_next) {
                fence_acq_rel_gpu();
                for (uint64_t q = q_next + lane; q < q_end; q += 32) red_relaxed_add(p.round_done + q, 1u);
                q_next = q_end;
                progress = true;
            }
            if (my_r < rounds) {
                const uint32_t expect = static_cast<uint32_t>(min(static_cast<uint64_t>(G), p.tiles - my_r * G));
                if (__ldcg(p.round_done + my_r) == expect) {
                    fence_acq_rel_gpu();
                    const uint64_t w0 = my_r * round_answers / 32;
                    const uint64_t w1 = (min(p.n, (my_r + 1) * round_answers) + 31) / 32;
                    uint32_t c = 0;
                    for (uint64_t w = w0 + lane; w < w1; w += 32) c += __popc(__ldcg(p.bitmap + w));
#pragma unroll
                    for (int o = 16; o; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
                    if (lane == 0) {
                        fence_acq_rel_gpu();
                        *reinterpret_cast<volatile uint32_t*>(p.round_cnt + my_r) = c + 1;
                    }
                    my_r += G;
                    progress = true;
                }
            }
            if (pre_q < rounds) {  // extend the published prefix by up to 32 rounds
                const uint32_t v = pre_q + lane < rounds ? __ldcg(p.round_cnt + pre_q + lane) : 0u;
                const uint32_t zero = __ballot_sync(0xffffffffu, v == 0u);
                const uint32_t k = zero ? __ffs(zero) - 1 : 32u;
                uint32_t add = lane < k ? v - 1 : 0u;
#pragma unroll
                for (int o = 16; o; o >>= 1) add += __shfl_xor_sync(0xffffffffu, add, o);
                pre += add;
                pre_q += k;
                if (k) progress = true;
            }
            // dense ids pay off for a small vocabulary (its answers hit the caches); with many
            // keys most answers take the global path and are remapped anyway, so the helper
            // stops ranking there (each rank walks up to a round of bitmap words)
            const uint32_t fill = ld_volatile(&S.lt_fill);
            uint32_t budget = 4;  // ranks per pass: the round counts above keep flowing
            if (fill <= 64 && ld_volatile(&S.ranked) < fill) {
                for (uint32_t base = 0; base < WS_LT && budget; base += 32) {
                    const uint32_t e = base + lane;
                    const uint32_t ready = ld_volatile(&S.lt_info[e].w), gs = ld_volatile(&S.lt_info[e].x);
                    const uint32_t rk = ld_volatile(&S.lt_info[e].y);
                    uint32_t f = ready && rk == EMPTY32 && gs != EMPTY32 ? __ldcg(p.first + gs) : EMPTY32;
                    // final when its round is complete and every earlier round is summed
                    const uint64_t qf = f != EMPTY32 ? (f / WS_TILE) / G : ~0ull;
                    bool cand = qf < pre_q || (qf == pre_q && qf < rounds && __ldcg(p.round_cnt + qf) != 0u);
                    uint32_t m = __ballot_sync(0xffffffffu, cand);
                    if (!m) continue;
                    fence_acq_rel_gpu();
                    while (m && budget && ld_volatile(&S.cons_done) < NW) {
                        const int src = __ffs(m) - 1;
                        m &= m - 1;
                        --budget;
                        const uint32_t ff = __shfl_sync(0xffffffffu, f, src);
                        const uint32_t gsl = __shfl_sync(0xffffffffu, gs, src);
                        if (__ldcg(p.first + gsl) != ff) continue;  // lowered meanwhile: next time
                        const uint64_t q = (ff / WS_TILE) / G;
                        // first occurrences of rounds < q: the prefix sum when q == pre_q, else summed here
                        uint32_t base_cnt = 0;
                        if (q == pre_q) {
                            base_cnt = pre;
                        } else {
                            for (uint64_t r = lane; r < q; r += 32) base_cnt += __ldcg(p.round_cnt + r) - 1;
#pragma unroll
                            for (int o = 16; o; o >>= 1) base_cnt += __shfl_xor_sync(0xffffffffu, base_cnt, o);
                        }
                        const uint32_t r = round_rank(p, ff, q * round_answers / 32, base_cnt, lane);
                        if (lane == 0) {
                            *reinterpret_cast<volatile uint32_t*>(&S.lt_info[base + src].y) = r;
                            atomicAdd(&S.ranked, 1u);
                        }
                    }
                    progress = true;
                }
            }
            if (!progress) __nanosleep(2000);
        }
        return;
    }

    // ---- consumers: one 128-answer chunk per step, four answers per lane -------------------
    const uint64_t aend = __ldg(p.off + p.n);
    for (uint32_t g = warp;; g += NW) {
        const uint32_t q = g / WS_CHUNKS, ch = g % WS_CHUNKS;
        const uint64_t t = blockIdx.x + static_cast<uint64_t>(q) * G;
        if (t >= p.tiles) break;
        const uint32_t st = q % WS_ST;
        mbar_wait(&S.full[st], (q / WS_ST) & 1u);
        const uint64_t i0 = t * WS_TILE;
        const uint32_t cnt = static_cast<uint32_t>(min(static_cast<uint64_t>(WS_TILE), p.n - i0));
        const uint8_t* sbuf = ring + st * WS_STAGE;
        const uint64_t* so = reinterpret_cast<const uint64_t*>(sbuf) + S.odel[st];
        const int64_t abase = S.abase[st];
        // the four answers in lock-step phases, every load unconditional (clamped to the
        // tile), so each phase's shared-memory loads are in flight together
        uint32_t gsl[4], rk[4], hf[4], w0[4], w1[4], w2[4], rh[4], ln[4], ent[4];
        bool atom = false, allfin = true, act[4], cach[4], hit[4];
        uint64_t b0[4];
#pragma unroll
        for (uint32_t k = 0; k < 4; ++k) {
            const uint32_t j = ch * WS_CHUNK + k * 32u + lane;
            act[k] = j < cnt;
            const uint32_t jc = act[k] ? j : 0u;
            b0[k] = so[jc];
            const uint32_t len = static_cast<uint32_t>(so[jc + 1]) - static_cast<uint32_t>(b0[k]);
            cach[k] = act[k] && abase != INPLACE && len <= WS_RAWMAX;  // (a staged tile holds < 2^32 bytes)
            ln[k] = cach[k] ? len : 0u;
        }
#pragma unroll
        for (uint32_t k = 0; k < 4; ++k) {
            const uint32_t rel = cach[k] ? static_cast<uint32_t>(b0[k]) - static_cast<uint32_t>(abase) : 0u;
            load_words(sbuf + WS_OFFB, rel, S.lenmask[ln[k]], w0[k], w1[k], w2[k]);
            rh[k] = raw_hash(w0[k], w1[k], w2[k], ln[k]);
        }
        uint4 tg[4], ce[4];
#pragma unroll
        for (uint32_t k = 0; k < 4; ++k) tg[k] = *reinterpret_cast<const uint4*>(&S.rc_tag[rc_set(rh[k])]);
#pragma unroll
        for (uint32_t k = 0; k < 4; ++k) {
            const uint32_t tag = rc_tag_of(rh[k]);
            const uint32_t way = tg[k].x == tag ? 0u : (tg[k].y == tag ? 1u : (tg[k].z == tag ? 2u : 3u));
            ce[k] = S.rc[rc_set(rh[k]) + way];
            hit[k] = cach[k] && (tg[k].x == tag || tg[k].y == tag || tg[k].z == tag || tg[k].w == tag) &&
                     ((ce[k].x ^ w0[k]) | (ce[k].y ^ w1[k]) | (ce[k].z ^ w2[k]) | ((ce[k].w & 0xffu) ^ ln[k])) == 0u;
        }
        uint4 li[4];
        uint32_t mt[4];
#pragma unroll
        for (uint32_t k = 0; k < 4; ++k) {
            mt[k] = ce[k].w;
            ent[k] = hit[k] ? (mt[k] >> 16) & 0xffu : 0u;
            li[k] = S.lt_info[ent[k]];
        }
        uint32_t miss = 0;
#pragma unroll
        for (uint32_t k = 0; k < 4; ++k) {
            const uint32_t idx = static_cast<uint32_t>(i0 + ch * WS_CHUNK + k * 32u + lane);
            gsl[k] = li[k].x;
            rk[k] = li[k].y;
            hf[k] = (mt[k] >> 8) & 1u;
            if (hit[k] && idx < li[k].z && gsl[k] != EMPTY32) {  // earlier than anything this CTA submitted
                first_min(p, gsl[k], idx);
                atomicMin(&S.lt_info[ent[k]].z, idx);
                atom = true;
            }
            if (act[k] && !hit[k]) miss |= 1u << k;
        }
        if (__any_sync(0xffffffffu, miss != 0u)) {  // rare once the caches are warm: out of line
            const ChunkRes in{gsl[0], gsl[1], gsl[2], gsl[3], rk[0], rk[1], rk[2], rk[3],
                              hf[0] | (hf[1] << 1) | (hf[2] << 2) | (hf[3] << 3)};
            const MissOut r = chunk_misses(p, mk, S, sbuf, so, abase, i0 + ch * WS_CHUNK, ch * WS_CHUNK, aend, miss, in);
#pragma unroll
            for (uint32_t k = 0; k < 4; ++k) {
                gsl[k] = r.g[k];
                rk[k] = r.r[k];
                hf[k] = r.h[k];
            }
            atom |= r.atom;
        }
#pragma unroll
        for (uint32_t k = 0; k < 4; ++k) allfin &= !act[k] || (rk[k] != EMPTY32 && gsl[k] != EMPTY32);
        const bool fin = __all_sync(0xffffffffu, allfin);
#pragma unroll
        for (uint32_t k = 0; k < 4; ++k) {
            const uint32_t j = ch * WS_CHUNK + k * 32u + lane;
            if (j < cnt) {
                p.ids[i0 + j] = fin ? rk[k] : gsl[k];
                if (p.hes) p.hes[i0 + j] = static_cast<uint8_t>(hf[k]);
            }
        }
        if (!fin && lane == 0) atomicOr(p.slice_flags + t, 0xfu << (ch * 4u));  // the chunk's 4 slices
        if (p.stats && lane == 0) {
            atomicAdd(p.stats + 0, 1ull);
            if (!fin) atomicAdd(p.stats + 1, 1ull);
        }
        if (p.stats && miss) {
            atomicAdd(p.stats + 2, static_cast<unsigned long long>(__popc(miss)));
            atomicAdd(p.stats + 8 + 2 * G + 3 * blockIdx.x, static_cast<unsigned long long>(__popc(miss)));
        }
        if (p.stats && atom) atomicAdd(p.stats + 3, 1ull);
        if (atom) fence_acq_rel_gpu();  // global table updates precede the round count
        __syncwarp();
        if (lane == 0) {
            mbar_arrive(&S.empty[st]);
            atomicAdd(&S.stage_steps[st], 1u);  // for the round counts (helper warp)
        }
    }
    __syncwarp();
    if (lane == 0) {
        const uint32_t done = atomicAdd(&S.cons_done, 1u) + 1;
        if (p.stats && done == NW) {  // per-CTA lifetime: [8 + 2c] start, [9 + 2c] end
            uint64_t t;
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
            p.stats[9 + 2 * blockIdx.x] = t;
            p.stats[8 + 2 * G + 3 * blockIdx.x + 2] = S.lt_fill;
        }
    }
}

// first occurrences per 1024-bit chunk of the bitmap (32 words)
__global__ void intern_chunk_popc(const uint32_t* __restrict__ bitmap, uint64_t words, uint32_t* __restrict__ csum,
                                  uint64_t chunks, const int* __restrict__ status) {
    if (*status) return;
    for (uint64_t c = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; c < chunks;
         c += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
        uint32_t n = 0;
        if ((c + 1) * 32 <= words) {
            const uint4* w = reinterpret_cast<const uint4*>(bitmap + c * 32);
#pragma unroll
            for (int q = 0; q < 8; ++q) {
                const uint4 v = w[q];
                n += __popc(v.x) + __popc(v.y) + __popc(v.z) + __popc(v.w);
            }
        } else {
            for (uint64_t q = c * 32; q < words; ++q) n += __popc(bitmap[q]);
        }
        csum[c] = n;
    }
}

// rank[slot] = first occurrences before the slot's first index (its dense first-seen id):
// the chunk prefix plus the words of its own chunk before it
__global__ void intern_rank(const uint32_t* __restrict__ first, uint64_t cap, const uint32_t* __restrict__ bitmap,
                            const uint32_t* __restrict__ cexcl, uint32_t* __restrict__ rank,
                            unsigned long long* __restrict__ first_index, const int* __restrict__ status) {
    if (*status) return;
    for (uint64_t s = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; s < cap;
         s += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
        const uint32_t f = first[s];
        if (f == EMPTY32) continue;
        uint32_t r = cexcl[f >> 10];
        for (uint32_t q = (f >> 10) * 32; q < (f >> 5); ++q) r += __popc(bitmap[q]);
        r += __popc(bitmap[f >> 5] & ((1u << (f & 31u)) - 1u));
        rank[s] = r;
        if (first_index) first_index[r] = f;
    }
}

struct LoadU32Arr {
    const uint32_t* v;
    __device__ uint32_t operator()(uint64_t i) const { return v[i]; }
};

// ids of the flagged slices (written as global slots) -> dense ids.  A warp per flag word
// (32 slices): lane i rewrites id i of each set slice, 8 slices in flight at a time.
__global__ void intern_remap(uint32_t* __restrict__ ids, uint64_t n, const uint32_t* __restrict__ rank,
                             const uint32_t* __restrict__ flags, uint64_t nwords, const int* __restrict__ status) {
    if (*status) return;
    const uint32_t lane = threadIdx.x & 31u;
    const uint64_t fw = (blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x) >> 5;
    if (fw >= nwords) return;
    uint32_t f = flags[fw];
    while (f) {
        uint64_t i[8];
        uint32_t v[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) {
            i[q] = ~0ull;
            if (f) {
                i[q] = (fw * 32 + (__ffs(f) - 1)) * 32 + lane;
                f &= f - 1;
            }
        }
#pragma unroll
        for (int q = 0; q < 8; ++q) v[q] = i[q] < n ? ids[i[q]] : 0u;
#pragma unroll
        for (int q = 0; q < 8; ++q) v[q] = __ldg(rank + v[q]);
#pragma unroll
        for (int q = 0; q < 8; ++q)
            if (i[q] < n) ids[i[q]] = v[q];
    }
}

// ---- direct interning: one thread per answer against one global table ------------------
// For inputs whose distinct keys are many (JSONL program ids: one id per ~P records), the
// CTA-local tables and raw-answer caches of intern_ws fill and every answer takes the global
// path anyway; this form goes there directly: pass 1 trims, hashes (8-byte words) and inserts
// (CAS on the hash, atomicMin of the first index), pass 2 byte-verifies every answer against
// its key's first occurrence (collisions reported, never merged) and flags first
// occurrences, an exclusive scan of the flags gives the dense first-seen ids, pass 3 writes
// them.  No markers, no hesitation flags.
__device__ __forceinline__ uint64_t dload8(const uint8_t* __restrict__ a, uint64_t pos, uint64_t end) {
    const uintptr_t base = reinterpret_cast<uintptr_t>(a);
    const uintptr_t addr = base + pos, al = addr & ~static_cast<uintptr_t>(7);
    if (al >= base && al + 16 <= base + end && pos + 8 <= end) {  // one aligned 16-byte window
        const uint64_t w0 = *reinterpret_cast<const uint64_t*>(al);
        const uint64_t w1 = *reinterpret_cast<const uint64_t*>(al + 8);
        const uint32_t sh = static_cast<uint32_t>(addr & 7) * 8;
        return sh ? (w0 >> sh) | (w1 << (64 - sh)) : w0;
    }
    uint64_t v = 0;
    for (uint32_t k = 0; k < 8 && pos + k < end; ++k) v |= static_cast<uint64_t>(a[pos + k]) << (8 * k);
    return v;
}
__device__ __forceinline__ void dtrim(const uint8_t* a, uint64_t& b, uint64_t& e) {
    while (b < e && is_space(a[b])) ++b;
    while (e > b && is_space(a[e - 1])) --e;
}

__global__ void intern_direct_insert(const uint8_t* __restrict__ arena, const uint64_t* __restrict__ off, uint64_t n,
                                     unsigned long long* __restrict__ keys, uint32_t* __restrict__ first,
                                     uint32_t* __restrict__ slot_of, uint64_t cap_mask, int* d_err) {
    const uint64_t end = off[n];
    for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
        uint64_t b = off[i], e = off[i + 1];
        dtrim(arena, b, e);
        const uint64_t len = e - b;
        uint64_t h = 0xcbf29ce484222325ull ^ (len * 0x9E3779B97F4A7C15ull);
        for (uint64_t q = 0; q < len; q += 8) {
            const uint64_t m = len - q >= 8 ? ~0ull : (1ull << (8 * (len - q))) - 1ull;
            h = mix(h, dload8(arena, b + q, end) & m);
        }
        h = fmix(h);
        uint64_t sl = h & cap_mask;
        for (uint64_t probes = 0;; ++probes) {
            unsigned long long prev = __ldcg(keys + sl);  // most keys exist: no atomic to find them
            if (prev == 0ull) prev = atomicCAS(keys + sl, 0ull, h);
            if (prev == 0ull || prev == h) break;
            sl = (sl + 1) & cap_mask;
            if (probes > cap_mask) {
                set_dev_err(d_err, DEV_INTERN_FULL);
                break;
            }
        }
        atomicMin(first + sl, static_cast<uint32_t>(i));
        slot_of[i] = static_cast<uint32_t>(sl);
    }
}

__global__ void intern_direct_verify(const uint8_t* __restrict__ arena, const uint64_t* __restrict__ off, uint64_t n,
                                     const uint32_t* __restrict__ first, const uint32_t* __restrict__ slot_of,
                                     uint32_t* __restrict__ is_first, int* d_err) {
    const uint64_t end = off[n];
    for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
        const uint32_t rep = first[slot_of[i]];
        is_first[i] = rep == i ? 1u : 0u;
        if (rep != i) {
            uint64_t ab = off[i], ae = off[i + 1], bb = off[rep], be = off[rep + 1];
            dtrim(arena, ab, ae);
            dtrim(arena, bb, be);
            const uint64_t len = ae - ab;
            bool same = len == be - bb;
            for (uint64_t k = 0; same && k < len; k += 8) {  // 8 bytes per compare
                const uint64_t m = len - k >= 8 ? ~0ull : (1ull << (8 * (len - k))) - 1ull;
                same = ((dload8(arena, ab + k, end) ^ dload8(arena, bb + k, end)) & m) == 0;
            }
            if (!same) set_dev_err(d_err, DEV_INTERN_COLLISION);
        }
    }
}

__global__ void intern_direct_finish(uint64_t n, const uint32_t* __restrict__ excl, const uint32_t* __restrict__ first,
                                     const uint32_t* __restrict__ slot_of, uint32_t* __restrict__ ids,
                                     unsigned long long* __restrict__ first_index) {
    for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
        const uint32_t rep = first[slot_of[i]];
        const uint32_t dense = excl[rep];  // first occurrences before rep = its dense id
        ids[i] = dense;
        if (rep == i && first_index) first_index[dense] = i;
    }
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
    if (reinterpret_cast<uintptr_t>(offsets) % 8 != 0)
        return set_error(ctx, CDX_EINVAL, "canon_intern: offsets must be 8-byte aligned");
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

    // consumer warps per CTA (+ the producer and the round/dense-id warp)
    static thread_local int occ_dev = -1, nw = 24;
    if (occ_dev != ctx->device) {
        const char* ev = std::getenv("CDX_IT_WARPS");
        nw = ev ? std::max(1, std::min(static_cast<int>(WS_MAXW), std::atoi(ev))) : static_cast<int>(WS_MAXW);
        cudaFuncSetAttribute(intern_ws, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(WS_SMEM));
        occ_dev = ctx->device;
    }
    const uint8_t* arena = reinterpret_cast<const uint8_t*>(bytes);
    const uint64_t tiles = (n + WS_TILE - 1) / WS_TILE;
    const unsigned grid = static_cast<unsigned>(std::min<uint64_t>(tiles, static_cast<uint64_t>(ctx->sm_count)));
    const uint64_t rounds = (tiles + grid - 1) / grid;
    const uint64_t words = (n + 31) / 32;             // first-occurrence bitmap
    const uint64_t fwords = (words + 31) / 32;        // one flag bit per 32-answer slice
    const uint64_t nrec = ((words + 31) / 32 + scan::SL_TILE - 1) / scan::SL_TILE + 2;
    for (int attempt = 0; attempt < 2; ++attempt) {
        // capacity: the context's last (distinct answers < cap / 2), or room for every answer
        uint64_t cap = std::max<uint64_t>(ctx->it_cap, 1ull << 20);
        if (attempt == 1) {
            cap = 1ull << 20;
            while (cap < 2 * n) cap <<= 1;
        }
        // zero region: hash | bitmap | counters | round_done | round_cnt | slice flags;
        // 0xff region: canonical packs (reused as rank u32 after the insert pass) | first;
        // then the chunk counts, their scan and its records
        const size_t zero_bytes = cap * 8 + words * 4 + 32 + rounds * 8 + fwords * 4;
        const size_t zero_pad = (zero_bytes + 15) & ~size_t(15);
        const size_t ff_bytes = cap * 8 + cap * 4;
        const uint64_t ex_words = 2 * ((words + 31) / 32) + 4;  // chunk counts + their exclusive scan
        const size_t bytes_need = zero_pad + ff_bytes + ex_words * 4 + 16 + nrec * 8 + 64;
        uint8_t* s = static_cast<uint8_t*>(scratch(ctx, bytes_need));
        if (!s) return set_error(ctx, CDX_ECUDA, "canon_intern: scratch allocation failed");
        auto* hkey = reinterpret_cast<unsigned long long*>(s);
        auto* bitmap = reinterpret_cast<uint32_t*>(hkey + cap);
        auto* counters = bitmap + words;
        auto* round_done = counters + 8;
        auto* round_cnt = round_done + rounds;
        auto* flags = round_cnt + rounds;
        auto* canon = reinterpret_cast<unsigned long long*>(s + zero_pad);
        auto* first = reinterpret_cast<uint32_t*>(canon + cap);
        auto* excl = first + cap;
        auto* rec = reinterpret_cast<uint64_t*>(reinterpret_cast<uintptr_t>(excl + ex_words + 3) & ~uintptr_t(7));
        auto* total = rec + nrec;
        cudaMemsetAsync(s, 0, zero_bytes, ctx->stream);
        cudaMemsetAsync(canon, 0xff, ff_bytes, ctx->stream);
        WsParams p{};
        p.arena = arena;
        p.off = offsets;
        p.n = n;
        p.tiles = tiles;
        p.hkey = hkey;
        p.first = first;
        p.canon = canon;
        p.cap_mask = cap - 1;
        p.bitmap = bitmap;
        p.round_done = round_done;
        p.round_cnt = round_cnt;
        p.slice_flags = flags;
        p.ids = ids;
        p.hes = hes;
        p.n_keys = counters;
        p.key_limit = static_cast<uint32_t>(std::min<uint64_t>(cap / 2, 0xffffffffull));
        p.status = reinterpret_cast<int*>(counters + 1);
        p.d_err = ctx->d_err;
        static const bool want_stats = std::getenv("CDX_IT_STATS") != nullptr;
        unsigned long long* stats = nullptr;
        if (want_stats) {
            cudaMalloc(&stats, 8 * (8 + 5 * grid));
            cudaMemsetAsync(stats, 0, 8 * (8 + 5 * grid), ctx->stream);
            p.stats = stats;
        }
        intern_ws<<<grid, 32 * (nw + 2), WS_SMEM, ctx->stream>>>(p, mk);
        if (stats) {
            std::vector<unsigned long long> hs(8 + 5 * grid);
            cudaMemcpyAsync(hs.data(), stats, 8 * hs.size(), cudaMemcpyDeviceToHost, ctx->stream);
            cudaStreamSynchronize(ctx->stream);
            unsigned long long t0 = ~0ull, s_lo = ~0ull, s_hi = 0, e_lo = ~0ull, e_hi = 0;
            for (unsigned c = 0; c < grid; ++c) t0 = std::min(t0, hs[8 + 2 * c]);
            for (unsigned c = 0; c < grid; ++c) {
                s_lo = std::min(s_lo, hs[8 + 2 * c] - t0), s_hi = std::max(s_hi, hs[8 + 2 * c] - t0);
                e_lo = std::min(e_lo, hs[9 + 2 * c] - t0), e_hi = std::max(e_hi, hs[9 + 2 * c] - t0);
            }
            fprintf(stderr, "intern_ws: CTA start %llu..%llu ns, end %llu..%llu ns\n", s_lo, s_hi, e_lo, e_hi);
            for (unsigned c = 0; c < grid; c += 8) {
                fprintf(stderr, "  cta %3u: end %7llu ns misses %7llu rc_inserts %5llu lt %3llu\n", c, hs[9 + 2 * c] - t0,
                        hs[8 + 2 * grid + 3 * c], hs[8 + 2 * grid + 3 * c + 1], hs[8 + 2 * grid + 3 * c + 2]);
            }
            fprintf(stderr, "intern_ws: chunks %llu provisional %llu missed answers %llu chunks with atomics %llu\n", hs[0],
                    hs[1], hs[2], hs[3]);
            cudaFree(stats);
        }
        CDX_CHECK_LAUNCH(ctx, "canon_intern(intern)");
        // dense ids: first-occurrence counts per 1024-bit chunk, their exclusive scan (the
        // total is the distinct count), then a rank per occupied slot; flagged slices remapped
        const uint64_t chunks = (words + 31) / 32;
        auto* csum = excl;
        auto* cexcl = excl + chunks;
        const unsigned g1 = static_cast<unsigned>(std::min<uint64_t>((chunks + 255) / 256, ctx->sm_count * 8ull));
        intern_chunk_popc<<<g1, 256, 0, ctx->stream>>>(bitmap, words, csum, chunks, p.status);
        CDX_CHECK_LAUNCH(ctx, "canon_intern(popc)");
        if (int st = scan::scan_excl(ctx, LoadU32Arr{csum}, chunks, cexcl, false, rec, total)) return st;
        auto* rank = reinterpret_cast<uint32_t*>(canon);  // canonical packs are no longer needed
        const unsigned g2 = static_cast<unsigned>(std::min<uint64_t>((cap + 255) / 256, ctx->sm_count * 16ull));
        intern_rank<<<g2, 256, 0, ctx->stream>>>(first, cap, bitmap, cexcl, rank,
                                                 reinterpret_cast<unsigned long long*>(first_index), p.status);
        CDX_CHECK_LAUNCH(ctx, "canon_intern(rank)");
        intern_remap<<<static_cast<unsigned>((fwords * 32 + 255) / 256), 256, 0, ctx->stream>>>(ids, n, rank, flags, fwords,
                                                                                                p.status);
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

namespace cdx {
int canon_intern_direct(cdx_ctx* ctx, const char* bytes, const uint64_t* offsets, uint64_t n, uint32_t* ids,
                        uint64_t* first_index, uint64_t* n_unique) {
    CDX_NVTX("canon_intern_direct");
    if (!offsets || !ids || !n_unique) return set_error(ctx, CDX_EINVAL, "canon_intern: null pointer");
    if (n >= 0xffffffffull) return set_error(ctx, CDX_EINVAL, "canon_intern: at most 2^32-2 answers per call");
    *n_unique = 0;
    if (n == 0) return CDX_OK;
    if (!bytes) return set_error(ctx, CDX_EINVAL, "canon_intern: null pointer");
    uint64_t cap = 1024;
    while (cap < 2 * n) cap <<= 1;
    const uint64_t nrec = (n + scan::SL_TILE - 1) / scan::SL_TILE + 2;  // scan tile records + ticket
    const size_t bytes_need = cap * 8 + cap * 4 + n * 4 * 2 + 16 + nrec * 8 + 16;
    uint8_t* s = static_cast<uint8_t*>(scratch(ctx, bytes_need));
    if (!s) return set_error(ctx, CDX_ECUDA, "canon_intern: scratch allocation failed");
    auto* keys = reinterpret_cast<unsigned long long*>(s);
    auto* first = reinterpret_cast<uint32_t*>(s + cap * 8);
    auto* slot_of = first + cap;
    auto* flags = slot_of + n;
    auto* rec = reinterpret_cast<uint64_t*>(reinterpret_cast<uintptr_t>(flags + n + 3) & ~static_cast<uintptr_t>(7));
    auto* total = rec + nrec;
    cudaMemsetAsync(keys, 0, cap * 8, ctx->stream);
    cudaMemsetAsync(first, 0xff, cap * 4, ctx->stream);
    const unsigned grid = static_cast<unsigned>(std::min<uint64_t>((n + 255) / 256, ctx->sm_count * 16ull));
    const uint8_t* arena = reinterpret_cast<const uint8_t*>(bytes);
    intern_direct_insert<<<grid, 256, 0, ctx->stream>>>(arena, offsets, n, keys, first, slot_of, cap - 1, ctx->d_err);
    CDX_CHECK_LAUNCH(ctx, "canon_intern(direct insert)");
    intern_direct_verify<<<grid, 256, 0, ctx->stream>>>(arena, offsets, n, first, slot_of, flags, ctx->d_err);
    CDX_CHECK_LAUNCH(ctx, "canon_intern(direct verify)");
    // first-occurrence flags -> exclusive prefix in place = dense first-seen ids
    if (int st = scan::scan_excl(ctx, scan::LoadU32{flags}, n, flags, false, rec, total)) return st;
    intern_direct_finish<<<grid, 256, 0, ctx->stream>>>(n, flags, first, slot_of, ids,
                                                         reinterpret_cast<unsigned long long*>(first_index));
    CDX_CHECK_LAUNCH(ctx, "canon_intern(direct finish)");
    uint64_t* h_total = reinterpret_cast<uint64_t*>(ctx->h_small);
    cudaError_t e = cudaMemcpyAsync(h_total, total, 8, cudaMemcpyDeviceToHost, ctx->stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize(ctx->stream);
    if (e != cudaSuccess) return cuda_fail(ctx, e, "canon_intern");
    *n_unique = *h_total;
    return CDX_OK;
}
}  // namespace cdx
