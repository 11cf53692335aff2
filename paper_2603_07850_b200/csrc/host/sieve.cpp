// sieve.cpp -- device-backed table/sieve API (sieve.hpp).  All primality
// work is done by the sm_100a kernels; host code sizes buffers and copies.
#include "goldbach/sieve.hpp"

#include <algorithm>
#include <bit>
#include <cmath>
#include <string>

#include "goldbach/device.hpp"
#include "goldbach_b200.h"

namespace goldbach {

namespace {

// a small shared handle for table utilities on device 0
std::shared_ptr<SharedDevice> util_device(uint64_t cover) {
    DeviceConfig c;
    c.device = 0;
    c.cover_limit = cover < 4 ? 4 : cover;
    c.p_small = 3;
    c.max_seg_evens = 1 << 20;
    return SharedDevice::get(c);
}

std::vector<uint32_t> device_odd_primes_upto(uint64_t limit) {
    auto sd = util_device(4);
    return sd->with([&](Device& d) {
        uint64_t n = 0;
        d.check(gb_primes_upto(d.get(), limit, nullptr, 0, &n));
        std::vector<uint32_t> out(n);
        if (n) d.check(gb_primes_upto(d.get(), limit, out.data(), n, &n));
        return out;
    });
}

} // namespace

uint64_t sqrt_bound_for(uint64_t cover) {
    uint64_t s = static_cast<uint64_t>(std::sqrt(static_cast<long double>(cover)));
    if (s == 0) s = 1;
    while (s > 1 && (s - 1) >= cover / (s - 1)) --s;
    while (s < cover / s) ++s;
    return s;
}

std::vector<uint64_t> simple_sieve(uint64_t limit, uint64_t mem_cap_bytes) {
    if (limit < 2) throw ParamError("simple_sieve: limit must be >= 2");
    // host result vector + device bitmap, same order of magnitude as the
    // reference's estimate (sieve.cpp:23-28)
    const double est = limit < 17 ? 8.0 : 1.26 * (double)limit / std::log((double)limit) + 1;
    const uint64_t need = limit / 8 + (uint64_t)est * sizeof(uint64_t) + 4096;
    if (need > mem_cap_bytes)
        throw ResourceError("simple_sieve: working set of " + std::to_string(need) + " bytes exceeds cap of " +
                            std::to_string(mem_cap_bytes) + " bytes");
    std::vector<uint32_t> odd = device_odd_primes_upto(std::min<uint64_t>(limit, 0xFFFFFFFFull));
    std::vector<uint64_t> out;
    out.reserve(limit > 0xFFFFFFFFull ? (size_t)est : odd.size() + 1);
    out.push_back(2);
    for (uint32_t p : odd) out.push_back(p);
    if (limit > 0xFFFFFFFFull) {
        // above 2^32: the device segmented sieve (the fused kernels' K1
        // interval kernel) in windows of 2^30 odd cells; the host only lists
        // the set bits the reference API returns
        auto sd = util_device(limit);
        const uint64_t top = (limit & 1) ? limit : limit - 1; // largest odd <= limit
        const uint64_t span = uint64_t{1} << 31; // integers per window
        std::vector<uint64_t> w;
        for (uint64_t lo = 0x100000001ull; lo <= top;) {
            const uint64_t hi = top - lo >= span - 2 ? lo + span - 2 : top;
            w.assign((((hi - lo) >> 1) + 1 + 63) / 64, 0);
            sd->with([&](Device& d) {
                d.check(gb_sieve_interval(d.get(), lo, hi, w.data(), w.size()));
                return 0;
            });
            for (size_t k = 0; k < w.size(); ++k)
                for (uint64_t b = w[k]; b; b &= b - 1)
                    out.push_back(lo + 2 * ((uint64_t{k} << 6) + (uint64_t)std::countr_zero(b)));
            if (hi == top) break;
            lo = hi + 2;
        }
    }
    return out;
}

BasePrimes base_primes_descriptor(uint64_t cover_limit) {
    if (cover_limit < 1) throw ParamError("build_base_primes: cover_limit must be >= 1");
    BasePrimes b;
    b.sqrt_bound = sqrt_bound_for(cover_limit);
    b.cover_limit = cover_limit;
    return b;
}

BasePrimes build_base_primes(uint64_t cover_limit) {
    BasePrimes b = base_primes_descriptor(cover_limit);
    if (b.sqrt_bound < 3) return b;
    auto sd = util_device(cover_limit);
    b.primes = sd->with([&](Device& d) {
        uint64_t s = 0, n = 0;
        d.check(gb_base_primes(d.get(), &s, &n, nullptr, 0));
        std::vector<uint32_t> v(n);
        if (n) d.check(gb_base_primes(d.get(), nullptr, nullptr, v.data(), n));
        return v;
    });
    return b;
}

std::optional<uint64_t> first_tile_index(uint64_t p, uint64_t tile_lo, uint64_t seg_hi) {
    if (p < 3 || !(p & 1)) throw ParamError("first_tile_index: p must be an odd prime >= 3");
    if (!(tile_lo & 1) || !(seg_hi & 1)) throw ParamError("first_tile_index: bounds must be odd");
    // smallest odd cofactor c >= p with p*c >= tile_lo; range-checked by
    // division before any product is formed
    uint64_t c = tile_lo / p + (tile_lo % p != 0);
    c = c < p ? p : c;
    c |= 1;
    if (c > seg_hi / p) return std::nullopt;
    return (p * c - tile_lo) >> 1;
}

OddBitset tiled_sieve_segment(uint64_t lo, uint64_t hi, const BasePrimes& base, const TileSpec& tiles) {
    if (!(lo & 1) || !(hi & 1)) throw ParamError("tiled_sieve_segment: bounds must be odd");
    if (lo > hi) throw ParamError("tiled_sieve_segment: lo must be <= hi");
    const uint64_t t = tiles.odds_per_tile;
    if (t < 64 || (t & (t - 1)) != 0)
        throw ParamError("tiled_sieve_segment: odds_per_tile must be a power of two >= 64");
    const uint64_t s = base.sqrt_bound;
    if (s == 0 || s < hi / s) throw ParamError("tiled_sieve_segment: base primes insufficient for segment bound");
    OddBitset out = OddBitset::new_filled(lo, hi);
    auto sd = util_device(cover_limit_of(base));
    sd->with([&](Device& d) {
        auto w = out.words();
        d.check(gb_sieve_interval(d.get(), lo, hi, w.data(), w.size()));
        return 0;
    });
    return out;
}

} // namespace goldbach
