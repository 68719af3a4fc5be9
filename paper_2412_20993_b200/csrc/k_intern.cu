// k_intern.cu — K1: answer canonicalisation, interning and hesitation flags.
//
// Replaces metrics::trim + the unordered_map<string_view> key of cluster_exact (metrics.cpp:
// 12-37) — every comparison of answers in the reference goes through trimmed exact bytes —
// and probe::flag_hesitation (probe.cpp:36-44).  Output ids are DENSE and in first-seen
// order of the trimmed bytes (exactly the cluster order cluster_exact would produce over
// the whole arena), so every downstream kernel compares u32 ids instead of strings.
//
//   pass 1  one thread per answer: trim (6 ASCII whitespace bytes), 64-bit hash of the
//           trimmed bytes, hesitation scan (ASCII tolower of the raw answer, any non-empty
//           marker as a substring), insert into a global open-addressing table with
//           atomicCAS on the hash and atomicMin on the first arena index.
//   pass 2  byte-verify every answer against its slot's first occurrence (a 64-bit hash
//           collision between distinct answers is reported, never silently merged) and
//           flag first occurrences.
//   pass 3  exclusive scan of the first-occurrence flags -> dense ids in first-seen order.
//   pass 4  ids[i] = dense id of its slot's first occurrence; first_index[id] = arena index.
#include <algorithm>
#include <cstring>
#include <vector>

#include "cdx_internal.cuh"
#include "k_scan.cuh"

namespace cdx {
namespace {

constexpr int MAX_MARKERS = 16;
constexpr int MARKER_BYTES = 1024;

struct Markers {
    uint32_t n;
    uint32_t off[MAX_MARKERS + 1];
    char bytes[MARKER_BYTES];
};

__device__ __forceinline__ bool is_space(uint8_t c) {
    return c == ' ' || c == '\t' || c == '\n' || c == '\r' || c == '\f' || c == '\v';
}

__device__ __forceinline__ uint8_t lower(uint8_t c) { return (c >= 'A' && c <= 'Z') ? c + 32 : c; }

__device__ uint64_t hash_bytes(const uint8_t* s, uint64_t n) {
    uint64_t h = 0xcbf29ce484222325ULL ^ (n * 0x9E3779B97F4A7C15ULL);
    for (uint64_t i = 0; i < n; ++i) h = (h ^ s[i]) * 0x100000001b3ULL;
    h ^= h >> 33;
    h *= 0xff51afd7ed558ccdULL;
    h ^= h >> 33;
    return h ? h : 1;  // 0 marks an empty slot
}

// markers travel by value in the kernel's parameter space (per launch, so concurrent calls
// from different contexts never see each other's markers)
__device__ bool hesitant(const Markers& mk, const uint8_t* s, uint64_t n) {
    for (uint32_t k = 0; k < mk.n; ++k) {
        const uint32_t mb = mk.off[k], ml = mk.off[k + 1] - mb;
        if (ml == 0 || ml > n) continue;  // empty markers never match (probe.cpp:41)
        for (uint64_t i = 0; i + ml <= n; ++i) {
            uint32_t j = 0;
            while (j < ml && lower(s[i + j]) == static_cast<uint8_t>(mk.bytes[mb + j])) ++j;
            if (j == ml) return true;
        }
    }
    return false;
}

struct Trim {
    uint64_t b, e;
};
__device__ __forceinline__ Trim trim(const uint8_t* a, uint64_t b, uint64_t e) {
    while (b < e && is_space(a[b])) ++b;
    while (e > b && is_space(a[e - 1])) --e;
    return {b, e};
}

__global__ void intern_insert(const uint8_t* __restrict__ arena, const uint64_t* __restrict__ off, uint64_t n,
                              unsigned long long* __restrict__ keys, uint32_t* __restrict__ first,
                              uint32_t* __restrict__ slot_of, uint8_t* __restrict__ hes, uint64_t cap_mask,
                              const __grid_constant__ Markers mk, int* d_err) {
    for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
        const uint64_t b0 = off[i], e0 = off[i + 1];
        if (hes) hes[i] = hesitant(mk, arena + b0, e0 - b0) ? 1 : 0;
        const Trim t = trim(arena, b0, e0);
        const unsigned long long h = hash_bytes(arena + t.b, t.e - t.b);
        uint64_t s = h & cap_mask;
        uint64_t probes = 0;
        while (true) {
            const unsigned long long prev = atomicCAS(keys + s, 0ull, h);
            if (prev == 0ull || prev == h) break;
            s = (s + 1) & cap_mask;
            if (++probes > cap_mask) {
                set_dev_err(d_err, DEV_INTERN_FULL);
                break;
            }
        }
        atomicMin(first + s, static_cast<uint32_t>(i));
        slot_of[i] = static_cast<uint32_t>(s);
    }
}

// 8 arena bytes from pos (little-endian; bytes past `end` read as 0): one aligned 16-byte
// window (two loads and a funnel shift) when it lies inside the arena [base, end), byte
// loads otherwise.  Alignment is taken on the absolute address (the arena is the caller's).
__device__ __forceinline__ uint64_t load8(const uint8_t* __restrict__ a, uint64_t pos, uint64_t end) {
    const uintptr_t base = reinterpret_cast<uintptr_t>(a);
    const uintptr_t addr = base + pos, al = addr & ~static_cast<uintptr_t>(7);
    if (al >= base && al + 16 <= base + end && pos + 8 <= end) {
        const uint64_t w0 = *reinterpret_cast<const uint64_t*>(al);
        const uint64_t w1 = *reinterpret_cast<const uint64_t*>(al + 8);
        const uint32_t sh = static_cast<uint32_t>(addr & 7) * 8;
        return sh ? (w0 >> sh) | (w1 << (64 - sh)) : w0;
    }
    uint64_t v = 0;
    for (uint32_t k = 0; k < 8 && pos + k < end; ++k) v |= static_cast<uint64_t>(a[pos + k]) << (8 * k);
    return v;
}

__global__ void intern_verify(const uint8_t* __restrict__ arena, const uint64_t* __restrict__ off, uint64_t n,
                              const uint32_t* __restrict__ first, const uint32_t* __restrict__ slot_of,
                              uint32_t* __restrict__ is_first, int* d_err) {
    for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
        const uint32_t rep = first[slot_of[i]];
        is_first[i] = rep == i ? 1u : 0u;
        if (rep != i) {
            const Trim a = trim(arena, off[i], off[i + 1]);
            const Trim b = trim(arena, off[rep], off[rep + 1]);
            const uint64_t len = a.e - a.b, end = off[n];
            bool same = len == b.e - b.b;
            for (uint64_t k = 0; same && k < len; k += 8) {  // 8 bytes per compare
                const uint64_t m = len - k >= 8 ? ~0ull : (1ull << (8 * (len - k))) - 1ull;
                same = ((load8(arena, a.b + k, end) ^ load8(arena, b.b + k, end)) & m) == 0;
            }
            if (!same) set_dev_err(d_err, DEV_INTERN_COLLISION);
        }
    }
}

// simple three-phase exclusive scan of u32 flags (n < 2^32)
__global__ void intern_finish(uint64_t n, const uint32_t* __restrict__ excl,
                              const uint32_t* __restrict__ first, const uint32_t* __restrict__ slot_of,
                              uint32_t* __restrict__ ids, unsigned long long* __restrict__ first_index) {
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
    *n_unique = 0;
    if (n == 0) return CDX_OK;

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
    intern_insert<<<grid, 256, 0, ctx->stream>>>(arena, offsets, n, keys, first, slot_of, hes, cap - 1, mk, ctx->d_err);
    CDX_CHECK_LAUNCH(ctx, "canon_intern(insert)");
    intern_verify<<<grid, 256, 0, ctx->stream>>>(arena, offsets, n, first, slot_of, flags, ctx->d_err);
    CDX_CHECK_LAUNCH(ctx, "canon_intern(verify)");
    // first-occurrence flags -> exclusive prefix in place = dense first-seen ids
    if (int st = scan::scan_excl(ctx, scan::LoadU32{flags}, n, flags, false, rec, total)) return st;
    intern_finish<<<grid, 256, 0, ctx->stream>>>(n, flags, first, slot_of, ids,
                                                  reinterpret_cast<unsigned long long*>(first_index));
    CDX_CHECK_LAUNCH(ctx, "canon_intern(finish)");
    uint64_t h_total = 0;
    cudaError_t e = cudaMemcpyAsync(&h_total, total, 8, cudaMemcpyDeviceToHost, ctx->stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize(ctx->stream);
    if (e != cudaSuccess) return cuda_fail(ctx, e, "canon_intern");
    *n_unique = h_total;
    return CDX_OK;
}
