// ref_api_conformance.cpp -- every public symbol of the reference's headers
// (proj/include/goldbach/{cli,errors,oddbits,pool,primality,sieve,verifier}.hpp)
// used with the reference's exact signature against this library's headers.
// If this translation unit compiles and links, a reference consumer compiles
// and links against the drop-in unchanged.  Run without arguments it also
// checks the host-only entry points against the reference's known answers
// (no GPU needed); with --gpu it exercises the device-backed ones too.
#include <cassert>
#include <cstdio>
#include <cstring>
#include <iostream>
#include <sstream>
#include <type_traits>

#include "goldbach/cli.hpp"
#include "goldbach/errors.hpp"
#include "goldbach/oddbits.hpp"
#include "goldbach/pool.hpp"
#include "goldbach/primality.hpp"
#include "goldbach/sieve.hpp"
#include "goldbach/verifier.hpp"

using namespace goldbach;

// ---- functions: pointer types of the reference declarations
#define SIG(fn, type) static_assert(std::is_convertible_v<decltype(&fn), type>, #fn " signature")
// verifier.hpp
SIG(sieve_range_for, OddRange (*)(const SegmentJob&, uint64_t));                          // :44
SIG(phase1_verify, Phase1Result (*)(const SegmentJob&, const SmallPrimeTable&, const OddBitset&, uint64_t,
                                    std::vector<uint64_t>*));                               // :77-79
SIG(count_unverified, UnverifiedSet (*)(const PackedBits&, uint64_t));                     // :86
SIG(phase2_resolve, std::optional<GoldbachPair> (*)(uint64_t, const SmallPrimeTable&, const Phase2Table&)); // :91-93
SIG(verify_segment, SegmentReport (*)(const SegmentJob&, const VerifyContext&));           // :118
SIG(SmallPrimeTable::build, SmallPrimeTable (*)(uint64_t));                                // :26
SIG(Phase2Table::build, Phase2Table (*)(uint64_t));                                        // :35
// primality.hpp
SIG(modmul, uint64_t (*)(uint64_t, uint64_t, uint64_t));                                   // :15
SIG(modpow, uint64_t (*)(uint64_t, uint64_t, uint64_t));                                   // :21
SIG(is_prime_u64, bool (*)(uint64_t));                                                     // :24
static_assert(kMillerRabinWitnesses.size() == 12 && kMillerRabinWitnesses[11] == 37, "witnesses");
// sieve.hpp
SIG(simple_sieve, std::vector<uint64_t> (*)(uint64_t, uint64_t));                          // :28-29
SIG(build_base_primes, BasePrimes (*)(uint64_t));                                          // :34
SIG(first_tile_index, std::optional<uint64_t> (*)(uint64_t, uint64_t, uint64_t));          // :40-41
SIG(tiled_sieve_segment, OddBitset (*)(uint64_t, uint64_t, const BasePrimes&, const TileSpec&)); // :46-47
static_assert(TileSpec::kDefaultOddsPerTile == 32768, "TileSpec default");
// cli.hpp
SIG(parse_args, Config (*)(const std::vector<std::string>&, std::ostream&));                // :35
SIG(usage_text, std::string (*)());                                                        // :37
SIG(resolve_workers, unsigned (*)(int64_t));                                               // :40
SIG(validate_resources, MemoryEstimate (*)(const Config&));                                 // :52
SIG(efficiency, double (*)(double, unsigned, double));                                     // :55
SIG(run, int (*)(const Config&, std::ostream&, std::ostream&));                             // :61
// pool.hpp
SIG(progress_snapshot, ProgressSnapshot (*)(const ProgressCounters&, uint64_t, double));   // :99-101
SIG(format_progress_line, std::string (*)(const ProgressSnapshot&));                       // :105
SIG(run_workers, RunResult (*)(WorkPool&, const VerifyContext&, const RunOptions&, Logger&)); // :128-129
static_assert(std::is_convertible_v<decltype(&WorkPool::claim_next), std::optional<SegmentJob> (WorkPool::*)()>,
              "claim_next");
static_assert(std::is_constructible_v<WorkPool, uint64_t, uint64_t, uint64_t>, "WorkPool ctor");
static_assert(std::is_constructible_v<Logger, std::ostream&>, "Logger ctor");
static_assert(std::is_constructible_v<ProgressCounters, unsigned>, "ProgressCounters ctor");
// errors.hpp: the taxonomy
static_assert(std::is_base_of_v<std::invalid_argument, ParamError>, "ParamError");
static_assert(std::is_base_of_v<std::runtime_error, ResourceError>, "ResourceError");
static_assert(std::is_base_of_v<std::logic_error, InternalError>, "InternalError");
static_assert(std::is_base_of_v<ParamError, UsageError>, "UsageError");

// ---- data members with the reference's types
#define MEM(T, m, type) static_assert(std::is_same_v<decltype(T::m), type>, #T "::" #m)
MEM(SegmentJob, a, uint64_t); MEM(SegmentJob, b, uint64_t); MEM(SegmentJob, index, uint64_t);
MEM(SmallPrimeTable, primes, std::vector<uint64_t>); MEM(SmallPrimeTable, p_small, uint64_t);
MEM(Phase2Table, primes, std::vector<uint64_t>); MEM(Phase2Table, limit, uint64_t);
MEM(OddRange, lo, uint64_t); MEM(OddRange, hi, uint64_t);
MEM(GoldbachPair, p, uint64_t); MEM(GoldbachPair, q, uint64_t);
MEM(MinPrimeMax, p, uint64_t); MEM(MinPrimeMax, n, uint64_t);
MEM(Phase1Result, verified, PackedBits); MEM(Phase1Result, min_prime, MinPrimeMax);
MEM(UnverifiedSet, count, uint32_t); MEM(UnverifiedSet, values, std::vector<uint64_t>);
MEM(VerifyContext, small, const SmallPrimeTable*); MEM(VerifyContext, phase2, const Phase2Table*);
MEM(VerifyContext, base, const BasePrimes*); MEM(VerifyContext, tiles, TileSpec);
MEM(VerifyContext, batch_size, uint64_t); MEM(VerifyContext, inject_fail, uint64_t);
MEM(SegmentReport, evens_checked, uint64_t); MEM(SegmentReport, unverified_after_phase1, uint32_t);
MEM(SegmentReport, phase2_resolved, uint64_t); MEM(SegmentReport, counterexamples, std::vector<uint64_t>);
MEM(SegmentReport, min_prime, MinPrimeMax); MEM(SegmentReport, elapsed_seconds, double);
MEM(BasePrimes, primes, std::vector<uint32_t>); MEM(BasePrimes, sqrt_bound, uint64_t);
MEM(TileSpec, odds_per_tile, uint64_t);
MEM(Config, limit, uint64_t); MEM(Config, start, uint64_t); MEM(Config, workers, int64_t);
MEM(Config, seg_size, uint64_t); MEM(Config, p_small, uint64_t); MEM(Config, batch_size, uint64_t);
MEM(Config, phase2_limit, uint64_t); MEM(Config, progress, bool); MEM(Config, json, bool);
MEM(Config, mem_cap, std::optional<uint64_t>); MEM(Config, inject_fail, uint64_t); MEM(Config, help, bool);
MEM(MemoryEstimate, per_worker_bytes, uint64_t); MEM(MemoryEstimate, shared_bytes, uint64_t);
MEM(MemoryEstimate, total_bytes, uint64_t); MEM(MemoryEstimate, workers, unsigned);
MEM(ProgressSnapshot, evens_done, uint64_t); MEM(ProgressSnapshot, throughput, double);
MEM(ProgressSnapshot, eta_seconds, std::optional<double>);
MEM(ProgressSnapshot, per_worker_segments, std::vector<uint64_t>);
MEM(RunOptions, workers, unsigned); MEM(RunOptions, progress, bool);
MEM(RunOptions, progress_interval, std::chrono::milliseconds);
MEM(RunResult, evens_checked, uint64_t); MEM(RunResult, unverified_total, uint64_t);
MEM(RunResult, phase2_total, uint64_t); MEM(RunResult, counterexamples, std::vector<uint64_t>);
MEM(RunResult, min_prime, MinPrimeMax); MEM(RunResult, segments, uint64_t);
MEM(RunResult, per_worker_segments, std::vector<uint64_t>); MEM(RunResult, wall_seconds, double);

static int fails = 0;
#define CHECK(c)                                                        \
    do {                                                                \
        if (!(c)) {                                                     \
            std::fprintf(stderr, "FAIL %s:%d: %s\n", __FILE__, __LINE__, #c); \
            ++fails;                                                    \
        }                                                               \
    } while (0)

// Host-only entry points, the reference tests' known answers.
static void host_checks() {
    // test_primality.cpp: modmul / modpow at full width
    CHECK(modmul(~0ull, ~0ull, ~0ull - 58) == 3364);        // 58 * 58 mod (2^64 - 59)
    CHECK(modpow(2, 10, 1000) == 24);
    CHECK(modpow(3, 0, 7) == 1 && modpow(5, 3, 1) == 0);
    CHECK(modpow(2, 64, ~0ull) == 1);                       // 2^64 = 1 mod 2^64 - 1
    bool threw = false;
    try { modmul(1, 1, 0); } catch (const ParamError&) { threw = true; }
    CHECK(threw);
    threw = false;
    try { modpow(1, 1, 0); } catch (const ParamError&) { threw = true; }
    CHECK(threw);
    // count_unverified (verifier.cpp:106-127): zero bits as even values
    PackedBits v(70, true);
    v.clear(0);
    v.clear(63);
    v.clear(69);
    const UnverifiedSet u = count_unverified(v, 100);
    CHECK(u.count == 3 && u.values.size() == 3);
    CHECK(u.values[0] == 100 && u.values[1] == 226 && u.values[2] == 238);
    threw = false;
    try { count_unverified(v, 101); } catch (const ParamError&) { threw = true; }
    CHECK(threw);
    // sieve_range_for fixed points (test_verifier.cpp:23-37)
    const OddRange r = sieve_range_for({4, 4, 0}, 1'000'000);
    CHECK(r.lo == 3 && r.hi == 3);
    const OddRange r2 = sieve_range_for({2'000'000, 2'000'010, 0}, 1'000'000);
    CHECK(r2.lo == 1'000'001 && r2.hi == 2'000'007);
    // MinPrimeMax tie rule (verifier.hpp:53-66)
    MinPrimeMax m;
    m.observe(5, 12);
    m.observe(5, 10);
    m.observe(3, 8);
    CHECK(m.p == 5 && m.n == 10);
    // WorkPool claim rule (pool.cpp:24-31)
    WorkPool pool(4, 20, 3);
    auto j0 = pool.claim_next(), j1 = pool.claim_next(), j2 = pool.claim_next(), j3 = pool.claim_next();
    CHECK(j0 && j0->a == 4 && j0->b == 8 && j0->index == 0);
    CHECK(j1 && j1->a == 10 && j1->b == 14);
    CHECK(j2 && j2->a == 16 && j2->b == 20);
    CHECK(!j3);
    // CLI surface (cli.hpp)
    std::ostringstream warn;
    const Config c = parse_args({"1000", "--workers=2"}, warn);
    CHECK(c.limit == 1000 && c.workers == 2 && c.start == 4);
    CHECK(!usage_text().empty());
    CHECK(resolve_workers(3) == 3 && resolve_workers(-1) >= 1);
    CHECK(efficiency(10.0, 2, 5.0) == 1.0);
    // progress line (pool.hpp:105)
    ProgressCounters pc(2);
    pc.add_evens(1000);
    pc.add_segment(1);
    const ProgressSnapshot snap = progress_snapshot(pc, 4000, 2.0);
    CHECK(snap.evens_done == 1000 && snap.per_worker_segments.size() == 2);
    CHECK(format_progress_line(snap).rfind("progress: ", 0) == 0);
    Logger log(std::cerr);
    (void)log;
}

// Device-backed entry points through the reference signatures.
static void gpu_checks() {
    CHECK(is_prime_u64(2) && !is_prime_u64(1) && is_prime_u64(18446744073709551557ull));
    const BasePrimes base = build_base_primes(100'000'000);
    CHECK(base.sqrt_bound == 10'000 && base.primes.size() == 1228);
    const SmallPrimeTable small = SmallPrimeTable::build(1'000'000);
    const Phase2Table p2 = Phase2Table::build(0);
    // phase1_verify on [4, 1e4] (test_verifier.cpp:265-282): max 173 @ 7426
    const SegmentJob job{4, 10'000, 0};
    const OddRange need = sieve_range_for(job, small.p_small);
    const OddBitset q = tiled_sieve_segment(need.lo, need.hi, build_base_primes(10'000));
    std::vector<uint64_t> mp;
    const Phase1Result p1 = phase1_verify(job, small, q, 2'000'000, &mp);
    CHECK(p1.min_prime.p == 173 && p1.min_prime.n == 7426);
    CHECK(p1.verified.popcount() == 4999 && mp.size() == 4999 && mp[0] == 2 && mp[4] == 5);
    CHECK(count_unverified(p1.verified, job.a).count == 0);
    VerifyContext ctx;
    ctx.small = &small;
    ctx.phase2 = &p2;
    const BasePrimes b4 = build_base_primes(10'000);
    ctx.base = &b4;
    const SegmentReport rep = verify_segment(job, ctx);
    CHECK(rep.evens_checked == 4999 && rep.min_prime.p == 173 && rep.min_prime.n == 7426);
    const auto hit = phase2_resolve(18446744073709551614ull, small, p2);
    CHECK(hit && hit->p == 277);
    // simple_sieve past 2^32 (the reference is bounded only by its memory cap,
    // sieve.cpp:22-42): pi(2^32) = 203,280,221, then 56 primes to 2^32 + 1000
    const std::vector<uint64_t> big = simple_sieve((uint64_t{1} << 32) + 1000);
    CHECK(big.size() == 203'280'221ull + 56 && big[203'280'221] == 4294967311ull && big.back() == 4294968289ull);
    bool threw = false;
    try {
        const OddBitset small_q = tiled_sieve_segment(need.lo + 200, need.hi, build_base_primes(10'000));
        phase1_verify(job, small, small_q, 2'000'000);
    } catch (const InternalError&) {
        threw = true;
    }
    CHECK(threw);
}

int main(int argc, char** argv) {
    host_checks();
    if (argc > 1 && std::strcmp(argv[1], "--gpu") == 0) gpu_checks();
    std::printf("%s (%d failures)\n", fails ? "FAILED" : "conformance ok", fails);
    return fails ? 1 : 0;
}
