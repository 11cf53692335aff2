// primality.cpp -- is_prime_u64 through the device Miller-Rabin kernel.
#include "goldbach/primality.hpp"

#include <memory>

#include "goldbach/device.hpp"

namespace goldbach {

std::vector<bool> is_prime_batch(const std::vector<uint64_t>& values) {
    if (values.empty()) return {};
    DeviceConfig c;
    c.cover_limit = 4;
    c.p_small = 3;
    c.max_seg_evens = 1 << 20;
    auto sd = SharedDevice::get(c);
    std::vector<uint8_t> out(values.size());
    sd->with([&](Device& d) {
        d.check(gb_is_prime_batch(d.get(), values.data(), out.data(), values.size()));
        return 0;
    });
    return std::vector<bool>(out.begin(), out.end());
}

bool is_prime_u64(uint64_t n) { return is_prime_batch({n})[0]; }

uint64_t modpow(uint64_t a, uint64_t e, uint64_t m) {
    if (m == 0) throw ParamError("modpow: modulus must be nonzero");
    uint64_t r = 1 % m;
    a %= m;
    for (; e; e >>= 1) {
        if (e & 1) r = modmul(r, a, m);
        a = modmul(a, a, m);
    }
    return r;
}

} // namespace goldbach
