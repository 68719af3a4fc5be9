#pragma once
// facade_common.hpp — shared plumbing of the C++ host layer (libcdxhost.so): the
// per-thread default context of the scalar API and string-arena interning through K1.

#include <cstdint>
#include <span>
#include <string>
#include <string_view>
#include <vector>

#include "cdx/batch.hpp"

namespace cdx::detail {

// One context per host thread (cdx_c.h: a context is not shared between threads), on the
// device named by $CDX_DEVICE (default 0).  The reference functions are pure and callable
// from any thread; each thread gets its own context and stream.
batch::Context& scalar_ctx();

// Device ids of `strs` interned by K1 (equal id <=> equal trimmed bytes, dense, first-seen
// order), optional hesitation flags against `markers`.
struct Interned {
    batch::DeviceArray<uint32_t> ids;
    batch::DeviceArray<uint8_t> hes;
    std::vector<uint64_t> first_index;  // host: arena index of each id's first occurrence
    uint64_t n_unique = 0;
};

Interned intern(batch::Context& cx, std::span<const std::string_view> strs, std::span<const std::string> markers,
                bool want_hes, bool want_first);

cdx_threshold to_c(const metrics::SignalThreshold& t);

// Answers as one byte arena + offsets[n+1] for the one-round-trip entries (cdx_*_host);
// fits = within their limits (1..2048 answers, at most 1 MiB), else the batched kernels.
struct HostArena {
    std::string bytes;
    std::vector<uint64_t> off;
    bool fits = false;
};
template <class It, class Get>
HostArena host_arena(It begin, It end, Get get) {
    HostArena a;
    a.off.push_back(0);
    for (It it = begin; it != end; ++it) {
        const std::string_view s = get(*it);
        a.bytes.append(s.data(), s.size());
        a.off.push_back(a.bytes.size());
    }
    const size_t n = a.off.size() - 1;
    a.fits = n >= 1 && n <= 2048 && a.bytes.size() <= (1u << 20);
    return a;
}

}  // namespace cdx::detail
