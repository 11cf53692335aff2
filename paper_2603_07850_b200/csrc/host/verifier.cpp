// verifier.cpp -- verify_segment (the drop-in boundary) and its helpers,
// implemented over the C-ABI of the B200 kernels.
#include "goldbach/verifier.hpp"

#include <algorithm>

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
