// ref_shim.cpp -- C entry points over the UNMODIFIED reference library
// (/root/reference/proj/src, compiled in place by oracle/build_ref.sh into
// oracle/_ref/libref.so).  TEST INFRASTRUCTURE ONLY: used to generate the
// golden vectors under tests/golden and to pin oracle/oracle.c.
//
// The per-segment record follows verify_segment (verifier.cpp:167-206);
// the checksum is taken from phase1_verify(..., min_primes_out)
// (verifier.hpp:74-79) plus the Phase 2 observations, i.e. one term per
// MinPrimeMax::observe call, exactly the definition in include/goldbach_b200.h.
#include <cstdint>
#include <cstring>
#include <vector>

#include "goldbach/primality.hpp"
#include "goldbach/sieve.hpp"
#include "goldbach/verifier.hpp"
#include "../include/goldbach_b200.h"

using namespace goldbach;

namespace {
struct Tables {
    uint64_t cover = 0, p_small = 0;
    BasePrimes base;
    SmallPrimeTable small;
    Phase2Table phase2; // disabled: result-invariant
};
Tables& tables(uint64_t cover, uint64_t p_small) {
    static thread_local Tables t;
    if (t.cover != cover || t.p_small != p_small || t.small.primes.empty()) {
        t.base = build_base_primes(cover);
        t.small = SmallPrimeTable::build(p_small);
        t.cover = cover;
        t.p_small = p_small;
    }
    return t;
}
void observe(gb_seg_record* r, uint64_t p, uint64_t n) {
    r->pmin_sum += p;
    r->pmin_hash += p * (n >> 1);
    if (p > r->max_p || (p == r->max_p && r->max_p != 0 && n < r->max_n)) {
        r->max_p = p;
        r->max_n = n;
    }
}
} // namespace

extern "C" {

int ref_is_prime(uint64_t n) { return is_prime_u64(n) ? 1 : 0; }

int64_t ref_base_primes(uint64_t cover, uint32_t* out, uint64_t cap, uint64_t* s) {
    try {
        BasePrimes b = build_base_primes(cover);
        *s = b.sqrt_bound;
        if (out)
            for (size_t i = 0; i < b.primes.size() && i < cap; ++i) out[i] = b.primes[i];
        return (int64_t)b.primes.size();
    } catch (...) {
        return -1;
    }
}

int ref_sieve(uint64_t lo, uint64_t hi, uint64_t cover, uint64_t tile, uint64_t* words) {
    try {
        BasePrimes b = build_base_primes(cover);
        TileSpec t;
        t.odds_per_tile = tile;
        OddBitset bits = tiled_sieve_segment(lo, hi, b, t);
        // export through the public test() API so no layout is assumed
        uint64_t n = ((hi - lo) >> 1) + 1;
        std::memset(words, 0, ((n + 63) / 64) * 8);
        for (uint64_t i = 0; i < n; ++i)
            if (bits.test_unchecked(lo + 2 * i)) words[i >> 6] |= 1ULL << (i & 63);
        return 0;
    } catch (...) {
        return -1;
    }
}

int ref_phase1_pmin(uint64_t a, uint64_t b, uint64_t cover, uint64_t p_small, uint64_t* out) {
    try {
        Tables& t = tables(cover, p_small);
        SegmentJob job{a, b, 0};
        OddRange r = sieve_range_for(job, p_small);
        OddBitset q = tiled_sieve_segment(r.lo, r.hi, t.base);
        std::vector<uint64_t> mp;
        phase1_verify(job, t.small, q, 2'000'000, &mp);
        std::memcpy(out, mp.data(), mp.size() * 8);
        return 0;
    } catch (...) {
        return -1;
    }
}

int ref_phase2_resolve(uint64_t n, uint64_t p_small, uint64_t* p) {
    try {
        Tables& t = tables(4, p_small);
        auto hit = phase2_resolve(n, t.small, t.phase2);
        *p = hit ? hit->p : 0;
        return 0;
    } catch (...) {
        return -1;
    }
}

// One segment: the reference's own verify_segment report + the checksum.
int ref_segment_record(uint64_t a, uint64_t b, uint64_t cover, uint64_t p_small,
                       uint64_t inject, gb_seg_record* rec) {
    try {
        Tables& t = tables(cover, p_small);
        std::memset(rec, 0, sizeof(*rec));
        rec->a = a;
        rec->b = b;
        VerifyContext ctx;
        ctx.small = &t.small;
        ctx.phase2 = &t.phase2;
        ctx.base = &t.base;
        ctx.inject_fail = inject;
        SegmentReport rep = verify_segment({a, b, 0}, ctx);
        rec->evens_checked = rep.evens_checked;
        rec->unverified_p1 = rep.unverified_after_phase1;
        rec->phase2_resolved = rep.phase2_resolved;
        rec->n_counterexamples = rep.counterexamples.size();
        for (size_t i = 0; i < rep.counterexamples.size() && i < GB_REC_MAX_CE; ++i)
            rec->counterexamples[i] = rep.counterexamples[i];
        // checksum: Phase 1 observations (per-n vector) + Phase 2 observations
        SegmentJob job{a, b, 0};
        OddRange r = sieve_range_for(job, p_small);
        OddBitset q = tiled_sieve_segment(r.lo, r.hi, t.base);
        std::vector<uint64_t> mp;
        phase1_verify(job, t.small, q, 2'000'000, &mp);
        gb_seg_record chk{};
        for (size_t i = 0; i < mp.size(); ++i)
            if (mp[i]) observe(&chk, mp[i], a + 2 * i);
        bool inj = inject >= a && inject <= b && (inject & 1) == 0;
        for (size_t i = 0; i < mp.size(); ++i) {
            uint64_t n = a + 2 * i;
            if (mp[i] && !(inj && n == inject)) continue;
            if (n == inject) continue;
            auto hit = phase2_resolve(n, t.small, t.phase2);
            if (hit) observe(&chk, hit->p, n);
        }
        rec->pmin_sum = chk.pmin_sum;
        rec->pmin_hash = chk.pmin_hash;
        rec->max_p = rep.min_prime.p;
        rec->max_n = rep.min_prime.n;
        // the reference's MinPrimeMax and the checksum walk must agree
        if (chk.max_p != rep.min_prime.p || chk.max_n != rep.min_prime.n) return -3;
        return 0;
    } catch (...) {
        return -1;
    }
}

// Single-pass form of ref_segment_record for the large golden sets (C4/C5).
// Composes the same reference functions in the same order as verify_segment
// (verifier.cpp:172-200): sieve_range_for -> tiled_sieve_segment ->
// phase1_verify (with min_primes_out, so the checksum needs no second pass)
// -> inject clear -> count_unverified -> phase2_resolve per leftover.
// Cross-checked against ref_segment_record (which calls verify_segment
// itself) by make_big_goldens.py --selfcheck.
int ref_segment_record1(uint64_t a, uint64_t b, uint64_t cover, uint64_t p_small,
                        uint64_t inject, gb_seg_record* rec) {
    try {
        Tables& t = tables(cover, p_small);
        std::memset(rec, 0, sizeof(*rec));
        rec->a = a;
        rec->b = b;
        SegmentJob job{a, b, 0};
        OddRange r = sieve_range_for(job, p_small);
        OddBitset q = tiled_sieve_segment(r.lo, r.hi, t.base);
        std::vector<uint64_t> mp;
        Phase1Result p1 = phase1_verify(job, t.small, q, 2'000'000, &mp);
        MinPrimeMax mpm = p1.min_prime;
        rec->evens_checked = p1.verified.size();
        gb_seg_record chk{};
        for (size_t i = 0; i < mp.size(); ++i)
            if (mp[i]) observe(&chk, mp[i], a + 2 * i);
        if (inject >= a && inject <= b && (inject & 1) == 0)
            p1.verified.clear((inject - a) >> 1);
        UnverifiedSet left = count_unverified(p1.verified, a);
        rec->unverified_p1 = left.count;
        std::vector<uint64_t> ces;
        for (uint64_t n : left.values) {
            if (n == inject) { ces.push_back(n); continue; }
            auto hit = phase2_resolve(n, t.small, t.phase2);
            if (!hit) { ces.push_back(n); continue; }
            ++rec->phase2_resolved;
            mpm.observe(hit->p, n);
            observe(&chk, hit->p, n);
        }
        rec->n_counterexamples = ces.size();
        for (size_t i = 0; i < ces.size() && i < GB_REC_MAX_CE; ++i)
            rec->counterexamples[i] = ces[i];
        rec->pmin_sum = chk.pmin_sum;
        rec->pmin_hash = chk.pmin_hash;
        rec->max_p = mpm.p;
        rec->max_n = mpm.n;
        if (chk.max_p != mpm.p || chk.max_n != mpm.n) return -3;
        return 0;
    } catch (...) {
        return -1;
    }
}

} // extern "C"
