#pragma once
// cdx/rng.hpp — the pure integer mixers of the reference's rng.hpp:25-34 (splitmix64
// finaliser and the seed-derivation tree), header-only.  They define the counter-based
// synthetic traces (cdx_gen_* on the device, cdxo_gen_* in the checker), so host and
// device draw identical values.  The reference's sequential `Rng` (mt19937_64 stream
// state) is not part of the batched path and is not provided.

#include <cstdint>

namespace cdx {

constexpr uint64_t mix64(uint64_t x) {
    x += 0x9e3779b97f4a7c15ULL;
    x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
    x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
    return x ^ (x >> 31);
}

constexpr uint64_t derive_seed(uint64_t master, uint64_t a, uint64_t b = 0) {
    return mix64(mix64(master ^ mix64(a)) ^ mix64(b ^ 0xa5a5a5a5a5a5a5a5ULL));
}

}  // namespace cdx
