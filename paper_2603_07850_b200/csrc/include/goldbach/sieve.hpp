// sieve.hpp -- table and sieve API of the drop-in library, device-backed.
// Same names and semantics as proj/include/goldbach/sieve.hpp:13-47; every
// table here is computed by the sm_100a kernels (K1) on the default GPU and
// copied back only because the reference API returns host vectors.
#pragma once

#include <cstdint>
#include <optional>
#include <vector>

#include "goldbach/oddbits.hpp"

namespace goldbach {

// Odd primes up to sqrt_bound (sieve.hpp:13-16).  cover_limit is the
// argument build_base_primes was called with; the device tables of a worker
// are rebuilt from it on each GPU (the host vector is informational).
struct BasePrimes {
    std::vector<uint32_t> primes;
    uint64_t sqrt_bound = 0;
    uint64_t cover_limit = 0;
};

// Kept for API compatibility (sieve.hpp:20-23).  The device tile size is
// fixed by the kernel geometry; the result is tile-size independent
// (test_sieve.cpp:163-177) so this only validates the value.
struct TileSpec {
    static constexpr uint64_t kDefaultOddsPerTile = 32768;
    uint64_t odds_per_tile = kDefaultOddsPerTile;
};

// Primes <= limit including 2 (sieve.hpp:28-29); ResourceError past the cap.
std::vector<uint64_t> simple_sieve(uint64_t limit, uint64_t mem_cap_bytes = uint64_t(8) << 30);

// Minimal s with s >= cover_limit / s (sieve.cpp:48-52); pure integer math.
uint64_t sqrt_bound_for(uint64_t cover_limit);

// The limit a caller-built BasePrimes covers: its cover_limit, else
// sqrt_bound^2 saturated at 2^64 - 1 (s = 2^32 covers every u64).
inline uint64_t cover_limit_of(const BasePrimes& b) {
    if (b.cover_limit) return b.cover_limit;
    return b.sqrt_bound >= (uint64_t{1} << 32) ? ~uint64_t{0} : b.sqrt_bound * b.sqrt_bound;
}

// K1 on the device (sieve.hpp:34).
BasePrimes build_base_primes(uint64_t cover_limit);

// Same as build_base_primes without copying the primes back: what the CLI
// and run_workers use (each GPU builds its own copy).
BasePrimes base_primes_descriptor(uint64_t cover_limit);

// First odd multiple of p >= max(p^2, tile_lo), as a bit index relative to
// tile_lo, or nullopt past seg_hi (sieve.hpp:40-41).  Integer arithmetic
// only; the device kernels use the same division-free-of-overflow form.
std::optional<uint64_t> first_tile_index(uint64_t p, uint64_t tile_lo, uint64_t seg_hi);

// Odd-prime bitset of [lo, hi] computed by the device sieve (sieve.hpp:46-47).
OddBitset tiled_sieve_segment(uint64_t lo, uint64_t hi, const BasePrimes& base,
                              const TileSpec& tiles = {});

} // namespace goldbach
