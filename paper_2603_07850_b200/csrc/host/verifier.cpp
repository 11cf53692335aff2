// verifier.cpp -- verify_segment (the drop-in boundary) and its helpers,
// implemented over the C-ABI of the B200 kernels.
#include "goldbach/verifier.hpp"

#include <algorithm>
#include <bit>

#include "goldbach/device.hpp"
#include "goldbach/errors.hpp"

namespace goldbach {

// set by run_workers for the calling worker thread: its open GPU handle
thread_local Device* tl_worker_device = nullptr;

namespace {

void check_job(const SegmentJob& job) {
    if ((job.a & 1) || (job.b & 1)) throw ParamError("segment bounds must be even");
    if (job.a < 4 || job.a > job.b) throw ParamError("segment must satisfy 4 <= a <= b");
}

DeviceConfig config_of(const VerifyContext& ctx, uint64_t max_seg_evens) {
    DeviceConfig c;
    c.device = ctx.devices.empty() ? 0 : ctx.devices.front();
    c.cover_limit = cover_limit_of(*ctx.base);
    c.p_small = ctx.small->p_small;
    c.inject_fail = ctx.inject_fail;
    c.max_seg_evens = max_seg_evens;
    return c;
}

} // namespace

SmallPrimeTable SmallPrimeTable::build(uint64_t p_small) {
    if (p_small < 3) throw ParamError("SmallPrimeTable: p_small must be >= 3");
    return {simple_sieve(p_small), p_small};
}

SmallPrimeTable SmallPrimeTable::descriptor(uint64_t p_small) {
    if (p_small < 3) throw ParamError("SmallPrimeTable: p_small must be >= 3");
    SmallPrimeTable t;
    t.p_small = p_small;
    return t;
}

Phase2Table Phase2Table::build(uint64_t limit) {
    if (limit < 2) return {};
    return {simple_sieve(limit), limit};
}

OddRange sieve_range_for(const SegmentJob& job, uint64_t p_small) {
    check_job(job);
    // q = n - p for odd p <= p_small: lowest odd >= max(3, a - p_small), top b - 3
    uint64_t lo = job.a > p_small ? job.a - p_small : 0;
    lo = std::max<uint64_t>(lo, 3) | 1;
    uint64_t hi = std::max(job.b - 3, lo);
    return {lo, hi};
}

SegmentReport report_from_record(const gb_seg_record& r) {
    SegmentReport rep;
    rep.evens_checked = r.evens_checked;
    if (r.unverified_p1 > UINT32_MAX) throw InternalError("count_unverified: count does not fit 32 bits");
    rep.unverified_after_phase1 = (uint32_t)r.unverified_p1;
    rep.phase2_resolved = r.phase2_resolved;
    const uint64_t kept = std::min<uint64_t>(r.n_counterexamples, GB_REC_MAX_CE);
    rep.counterexamples.assign(r.counterexamples, r.counterexamples + kept);
    rep.min_prime.p = r.max_p;
    rep.min_prime.n = r.max_n;
    rep.elapsed_seconds = r.elapsed_seconds;
    rep.pmin_sum = r.pmin_sum;
    rep.pmin_hash = r.pmin_hash;
    return rep;
}

SegmentReport verify_segment(const SegmentJob& job, const VerifyContext& ctx) {
    if (!ctx.small || !ctx.phase2 || !ctx.base) throw ParamError("verify_segment: context tables must be set");
    check_job(job);
    if (tl_worker_device) return report_from_record(tl_worker_device->verify(job.a, job.b));
    const uint64_t evens = ((job.b - job.a) >> 1) + 1;
    auto sd = SharedDevice::get(config_of(ctx, std::max<uint64_t>(evens, 200'000'000)));
    return report_from_record(sd->with([&](Device& d) { return d.verify(job.a, job.b); }));
}

std::vector<uint64_t> phase1_min_primes(const SegmentJob& job, uint64_t p_small, uint64_t cover_limit, int device) {
    check_job(job);
    DeviceConfig c;
    c.device = device;
    c.cover_limit = cover_limit;
    c.p_small = p_small;
    c.max_seg_evens = 1 << 20;
    auto sd = SharedDevice::get(c);
    std::vector<uint64_t> out(((job.b - job.a) >> 1) + 1);
    sd->with([&](Device& d) {
        d.check(gb_phase1_pmin(d.get(), job.a, job.b, out.data(), out.size()));
        return 0;
    });
    return out;
}

Phase1Result phase1_verify(const SegmentJob& job, const SmallPrimeTable& small, const OddBitset& qbits,
                           uint64_t batch_size, std::vector<uint64_t>* min_primes_out) {
    check_job(job);
    if (batch_size == 0) throw ParamError("phase1_verify: batch_size must be >= 1");
    if (small.primes.empty() || small.primes.front() != 2)
        throw ParamError("phase1_verify: malformed small-prime table");
    const OddRange need = sieve_range_for(job, small.p_small);
    if (qbits.lo() > need.lo || qbits.hi() < need.hi)
        throw InternalError("phase1_verify: sieved range does not cover the q lookups");
    const uint64_t n = ((job.b - job.a) >> 1) + 1;
    Phase1Result res{PackedBits(n, false), {}};
    if (min_primes_out) min_primes_out->assign(n, 0);
    // device pieces of at most 2^20 - 16 evens (gb_phase1_pmin's limit)
    const uint64_t piece = (uint64_t{1} << 20) - 16;
    std::vector<uint64_t> part;
    for (uint64_t i0 = 0; i0 < n; i0 += piece) {
        const uint64_t m = std::min(piece, n - i0);
        const SegmentJob sub{job.a + 2 * i0, job.a + 2 * (i0 + m - 1), job.index};
        part = phase1_min_primes(sub, small.p_small, std::max<uint64_t>(job.b, 4));
        for (uint64_t k = 0; k < m; ++k) {
            const uint64_t p = part[k];
            if (!p) continue;
            res.verified.set(i0 + k);
            res.min_prime.observe(p, sub.a + 2 * k);
            if (min_primes_out) (*min_primes_out)[i0 + k] = p;
        }
    }
    return res;
}

UnverifiedSet count_unverified(const PackedBits& verified, uint64_t a) {
    if (a & 1) throw ParamError("count_unverified: a must be even");
    const uint64_t zeros = verified.size() - verified.popcount();
    if (zeros > UINT32_MAX) throw InternalError("count_unverified: count does not fit 32 bits");
    UnverifiedSet out;
    out.count = (uint32_t)zeros;
    out.values.reserve(zeros);
    const auto w = verified.words();
    for (size_t k = 0; k < w.size(); ++k) {
        uint64_t z = ~w[k];
        if (k + 1 == w.size() && (verified.size() & 63)) z &= (uint64_t{1} << (verified.size() & 63)) - 1;
        for (; z; z &= z - 1) out.values.push_back(a + 2 * ((uint64_t{k} << 6) + (uint64_t)std::countr_zero(z)));
    }
    return out;
}

std::optional<GoldbachPair> phase2_resolve(uint64_t n, const SmallPrimeTable& small, const Phase2Table&) {
    if (n < 4 || (n & 1)) throw ParamError("phase2_resolve: n must be even and >= 4");
    if (small.p_small < 3) throw ParamError("phase2_resolve: malformed small-prime table");
    DeviceConfig c;
    c.cover_limit = 4;
    c.p_small = small.p_small;
    c.max_seg_evens = 1 << 20;
    auto sd = SharedDevice::get(c);
    uint64_t p = sd->with([&](Device& d) {
        uint64_t r = 0;
        d.check(gb_phase2_resolve(d.get(), n, &r));
        return r;
    });
    if (!p) return std::nullopt;
    return GoldbachPair{p, n - p};
}

} // namespace goldbach
