// test_host.cpp -- unit tests of the C++ host layer (no GPU needed for the
// default group; `test_host --gpu` adds the device-backed cases).  Mirrors
// the reference suites test_pool.cpp / test_cli.cpp / test_verifier.cpp /
// test_sieve.cpp case by case where the behaviour is host-side.
#include <algorithm>
#include <atomic>
#include <cstring>
#include <iostream>
#include <set>
#include <sstream>
#include <thread>

#include "goldbach/cli.hpp"
#include "goldbach/pool.hpp"
#include "goldbach/sieve.hpp"
#include "goldbach/verifier.hpp"

using namespace goldbach;

static int g_fail = 0, g_pass = 0;
#define CHECK(c)                                                                          \
    do {                                                                                  \
        if (c) {                                                                          \
            ++g_pass;                                                                     \
        } else {                                                                          \
            ++g_fail;                                                                     \
            std::cerr << __FILE__ << ":" << __LINE__ << ": CHECK failed: " #c "\n";      \
        }                                                                                 \
    } while (0)
#define CHECK_THROWS_AS(expr, T)                                                          \
    do {                                                                                  \
        bool thrown = false;                                                              \
        try {                                                                             \
            (void)(expr);                                                                 \
        } catch (const T&) {                                                              \
            thrown = true;                                                                \
        } catch (...) {                                                                   \
        }                                                                                 \
        CHECK(thrown);                                                                    \
    } while (0)

static Config parse(std::vector<std::string> a) {
    std::ostringstream w;
    return parse_args(a, w);
}

// ---- pool (test_pool.cpp:15-161)
static void test_pool() {
    {
        WorkPool p(4, 40, 10);
        auto j0 = p.claim_next();
        CHECK(j0 && j0->a == 4 && j0->b == 22 && j0->index == 0);
        auto j1 = p.claim_next();
        CHECK(j1 && j1->a == 24 && j1->b == 40 && j1->index == 1);
        CHECK(!p.claim_next());
        CHECK(!p.claim_next());
    }
    {
        WorkPool p(4, 4, 1);
        auto j = p.claim_next();
        CHECK(j && j->a == 4 && j->b == 4);
        CHECK(!p.claim_next());
        CHECK(p.total_evens() == 1);
    }
    {
        WorkPool p(4, 50, 10);
        std::vector<SegmentJob> jobs;
        while (auto j = p.claim_next()) jobs.push_back(*j);
        CHECK(jobs.size() == 3 && jobs.back().a == 44 && jobs.back().b == 50);
        uint64_t ev = 0;
        for (auto& j : jobs) ev += ((j.b - j.a) >> 1) + 1;
        CHECK(ev == p.total_evens());
    }
    CHECK_THROWS_AS(WorkPool(5, 40, 10), ParamError);
    CHECK_THROWS_AS(WorkPool(4, 41, 10), ParamError);
    CHECK_THROWS_AS(WorkPool(2, 40, 10), ParamError);
    CHECK_THROWS_AS(WorkPool(44, 40, 10), ParamError);
    CHECK_THROWS_AS(WorkPool(4, 40, 0), ParamError);
    CHECK_THROWS_AS(WorkPool(4, 40, uint64_t{1} << 32), ParamError);
    // exactly-once claiming under 8-thread contention, 100 repetitions
    for (int rep = 0; rep < 100; ++rep) {
        const uint64_t segs = 10000;
        WorkPool p(4, 4 + 2 * (segs - 1), 1);
        std::vector<std::vector<uint64_t>> logs(8);
        std::vector<std::thread> th;
        for (int t = 0; t < 8; ++t)
            th.emplace_back([&, t] {
                while (auto j = p.claim_next()) logs[t].push_back(j->a);
            });
        for (auto& t : th) t.join();
        std::vector<uint64_t> all;
        for (auto& l : logs) all.insert(all.end(), l.begin(), l.end());
        std::sort(all.begin(), all.end());
        bool ok = all.size() == segs;
        for (uint64_t i = 0; ok && i < segs; ++i) ok = all[i] == 4 + 2 * i;
        CHECK(ok);
    }
    {   // no wrap near 2^64 (test_pool.cpp:84-97)
        const uint64_t limit = ~uint64_t{0} - 1, start = limit - 199'998;
        WorkPool p(start, limit, 25'000);
        std::vector<SegmentJob> jobs;
        while (auto j = p.claim_next()) jobs.push_back(*j);
        CHECK(jobs.size() == 4 && jobs.front().a == start && jobs.back().b == limit);
        for (size_t i = 1; i < jobs.size(); ++i) CHECK(jobs[i].a == jobs[i - 1].b + 2);
        for (int i = 0; i < 10; ++i) CHECK(!p.claim_next());
    }
    {   // shared external cursor: two pools, one counter
        std::atomic<uint64_t> cur{4};
        WorkPool a(4, 40, 10, &cur), b(4, 40, 10, &cur);
        auto ja = a.claim_next(), jb = b.claim_next();
        CHECK(ja && jb && ja->a == 4 && jb->a == 24 && !a.claim_next() && !b.claim_next());
    }
    {   // shared stop word: a stop requested through one pool ends claims on both
        std::atomic<uint64_t> cur{4};
        std::atomic<uint32_t> workers{2}, stop{0};
        WorkPool a(4, 400, 10, &cur, &workers, &stop), b(4, 400, 10, &cur, &workers, &stop);
        CHECK(a.claim_next() && b.claim_next() && !a.stop_requested());
        a.request_stop();
        CHECK(b.stop_requested() && !b.claim_next() && !a.claim_next());
        CHECK(cur.load() == 44); // no claim advanced the cursor after the stop
    }
    {
        std::ostringstream sink;
        Logger log(sink);
        log.log("hello");
        log.log("");
        log.logf("n = ", 42, " ok");
        CHECK(sink.str() == "hello\n\nn = 42 ok\n");
    }
    {
        std::ostringstream sink;
        Logger log(sink);
        std::vector<std::thread> th;
        for (int t = 0; t < 8; ++t)
            th.emplace_back([&, t] {
                for (int i = 0; i < 1000; ++i) log.logf("worker ", t, " line ", i, " tail");
            });
        for (auto& t : th) t.join();
        std::istringstream in(sink.str());
        std::string line;
        std::set<std::string> seen;
        int n = 0;
        bool ok = true;
        while (std::getline(in, line)) {
            ++n;
            ok &= line.rfind("worker ", 0) == 0 && line.size() >= 4 && line.substr(line.size() - 4) == "tail";
            ok &= seen.insert(line).second;
        }
        CHECK(ok && n == 8000);
    }
    {
        ProgressCounters c(2);
        auto s = progress_snapshot(c, 1000, 0.0);
        CHECK(s.evens_done == 0 && s.throughput == 0.0 && !s.eta_seconds);
        CHECK(s.per_worker_segments == std::vector<uint64_t>({0, 0}));
        CHECK(format_progress_line(s) == "progress: 0 evens, 0/s, eta --:--");
        ProgressCounters c1(1);
        c1.add_evens(500);
        c1.add_segment(0);
        auto s1 = progress_snapshot(c1, 1'000'000, 2.0);
        CHECK(s1.evens_done == 500 && s1.throughput == 250.0 && s1.eta_seconds &&
              *s1.eta_seconds == (1'000'000 - 500) / 250.0);
        ProgressSnapshot f;
        f.evens_done = 500;
        f.throughput = 250.0;
        f.eta_seconds = 3661.0;
        CHECK(format_progress_line(f) == "progress: 500 evens, 250/s, eta 01:01:01");
    }
    {   // merge rules (pool.cpp:159-174)
        RunResult t, a, b;
        a.evens_checked = 3;
        a.min_prime = {7, 100};
        a.counterexamples = {30};
        a.pmin_sum = 5;
        b.evens_checked = 4;
        b.min_prime = {7, 90};
        b.counterexamples = {10};
        b.pmin_sum = ~uint64_t{0};
        merge_into(t, a);
        merge_into(t, b);
        CHECK(t.evens_checked == 7 && t.min_prime.p == 7 && t.min_prime.n == 90);
        CHECK(t.counterexamples == std::vector<uint64_t>({10, 30}));
        CHECK(t.pmin_sum == 4); // wraps mod 2^64
    }
    {   // exact counterexample counts past the stored GB_REC_MAX_CE values:
        // a record with 20 counterexamples keeps 16 values and the count 20
        gb_seg_record r{};
        r.a = 4;
        r.b = 1000;
        r.evens_checked = 499;
        r.unverified_p1 = 20;
        r.n_counterexamples = 20;
        for (int i = 0; i < GB_REC_MAX_CE; ++i) r.counterexamples[i] = 10 + 2 * i;
        const SegmentReport rep = report_from_record(r);
        CHECK(rep.counterexamples.size() == GB_REC_MAX_CE && rep.unverified_after_phase1 == 20);
        RunResult t, a;
        a.counterexamples = rep.counterexamples;
        a.counterexample_count = r.n_counterexamples;
        merge_into(t, a);
        merge_into(t, a);
        CHECK(t.counterexample_count == 40 && t.counterexamples.size() == 2 * GB_REC_MAX_CE);
    }
}

// ---- verifier host pieces (test_verifier.cpp:23-37, 239-263)
static void test_verifier_host() {
    CHECK(sieve_range_for({4, 20, 0}, 1'000'000).lo == 3);
    CHECK(sieve_range_for({4, 20, 0}, 1'000'000).hi == 17);
    auto big = sieve_range_for({1'000'000'000'000ull, 1'000'000'000'400ull, 0}, 1'000'000);
    CHECK(big.lo == 999'999'000'001ull && big.hi == 1'000'000'000'397ull);
    auto tiny = sieve_range_for({4, 4, 0}, 1'000'000);
    CHECK(tiny.lo == 3 && tiny.hi == 3);
    CHECK_THROWS_AS(sieve_range_for({5, 20, 0}, 100), ParamError);
    CHECK_THROWS_AS(sieve_range_for({4, 21, 0}, 100), ParamError);
    CHECK_THROWS_AS(sieve_range_for({2, 20, 0}, 100), ParamError);
    CHECK_THROWS_AS(sieve_range_for({20, 4, 0}, 100), ParamError);
    MinPrimeMax t;
    t.observe(3, 10);
    t.observe(5, 18);
    t.observe(5, 12);
    t.observe(5, 30);
    t.observe(3, 2);
    CHECK(t.p == 5 && t.n == 12);
    MinPrimeMax a, b, e;
    a.observe(7, 100);
    b.merge(a);
    b.merge(e);
    CHECK(b.p == 7 && b.n == 100);
    VerifyContext empty;
    CHECK_THROWS_AS(verify_segment({4, 10, 0}, empty), ParamError);
    // first_tile_index (test_sieve.cpp:77-105)
    CHECK(first_tile_index(5, 3, 101) == 11u);
    CHECK(first_tile_index(3, 31, 101) == 1u);
    CHECK(first_tile_index(11, 3, 101) == std::nullopt);
    CHECK(first_tile_index(7, 101, 201) == 2u);
    CHECK_THROWS_AS(first_tile_index(2, 3, 9), ParamError);
    CHECK_THROWS_AS(first_tile_index(3, 4, 9), ParamError);
    const uint64_t hi = ~uint64_t{0}, lo = hi - 199'998;
    auto idx = first_tile_index(4'294'967'311ull, lo, hi);
    if (idx) CHECK((lo + 2 * *idx) % 4'294'967'311ull == 0);
    auto i3 = first_tile_index(3, lo, hi);
    CHECK(i3 && (lo + 2 * *i3) % 3 == 0 && lo + 2 * *i3 >= lo);
    // sqrt_bound (test_sieve.cpp:48-62)
    CHECK(sqrt_bound_for(1) == 1 && sqrt_bound_for(4) == 2 && sqrt_bound_for(11) == 3 && sqrt_bound_for(12) == 4);
    CHECK(sqrt_bound_for(~uint64_t{0} - 1) == (uint64_t{1} << 32));
    // a caller-built BasePrimes without cover_limit: s^2 saturates at s = 2^32
    BasePrimes top;
    top.sqrt_bound = uint64_t{1} << 32;
    CHECK(cover_limit_of(top) == ~uint64_t{0});
    CHECK(sqrt_bound_for(cover_limit_of(top)) == top.sqrt_bound);
    top.sqrt_bound = 1000;
    CHECK(cover_limit_of(top) == 1'000'000);
    top.cover_limit = 999'999;
    CHECK(cover_limit_of(top) == 999'999);
}

// ---- cli (test_cli.cpp:24-155)
static void test_cli() {
    auto c = parse({"10000000000000", "--seg-size=200000000", "--p-small=1000000", "--batch-size=2000000", "--gpus=4"});
    CHECK(c.limit == 10'000'000'000'000ull && c.seg_size == 200'000'000 && c.p_small == 1'000'000 &&
          c.batch_size == 2'000'000 && c.workers == 4 && c.start == 4 && c.phase2_limit == 100'000'000 &&
          !c.progress && !c.json && !c.mem_cap);
    auto d = parse({"100"});
    CHECK(d.limit == 100 && d.start == 4 && d.workers == 1 && d.seg_size == 200'000'000);
    CHECK_THROWS_AS(parse({"--start=50", "40"}), UsageError);
    {
        std::ostringstream w;
        auto r = parse_args({"101", "--start=7"}, w);
        CHECK(r.limit == 100 && r.start == 6);
        CHECK(w.str().find("odd limit 101") != std::string::npos);
        CHECK(w.str().find("odd start 7") != std::string::npos);
    }
    CHECK_THROWS_AS(parse({"18446744073709551616"}), UsageError);
    CHECK_THROWS_AS(parse({"99999999999999999999"}), UsageError);
    CHECK(parse({"18446744073709551615"}).limit == 18'446'744'073'709'551'614ull);
    CHECK_THROWS_AS(parse({}), UsageError);
    CHECK_THROWS_AS(parse({"12x"}), UsageError);
    CHECK_THROWS_AS(parse({"100", "200"}), UsageError);
    CHECK_THROWS_AS(parse({"--frobnicate", "100"}), UsageError);
    CHECK_THROWS_AS(parse({"100", "--start"}), UsageError);
    CHECK_THROWS_AS(parse({"100", "--progress=1"}), UsageError);
    CHECK_THROWS_AS(parse({"100", "--workers=0"}), UsageError);
    CHECK_THROWS_AS(parse({"100", "--workers=-2"}), UsageError);
    CHECK_THROWS_AS(parse({"100", "--seg-size=0"}), UsageError);
    CHECK_THROWS_AS(parse({"100", "--seg-size=4294967296"}), UsageError);
    CHECK_THROWS_AS(parse({"100", "--p-small=2"}), UsageError);
    CHECK_THROWS_AS(parse({"100", "--batch-size=0"}), UsageError);
    CHECK_THROWS_AS(parse({"100", "--mem-cap=0"}), UsageError);
    CHECK_THROWS_AS(parse({"2"}), UsageError);
    CHECK(parse({"100", "--seg-size=4294967295"}).seg_size == 4'294'967'295ull);
    auto v = parse({"--seg-size", "1000", "--workers", "-1", "5000"});
    CHECK(v.seg_size == 1000 && v.workers == -1 && v.limit == 5000);
    CHECK(parse({"--help"}).help && parse({"-h"}).help);
    CHECK(usage_text().find("--seg-size") != std::string::npos);
    CHECK(usage_text().find("exit codes") != std::string::npos);
    CHECK(resolve_workers(1) == 1 && resolve_workers(16) == 16);
    CHECK_THROWS_AS(resolve_workers(0), UsageError);
    CHECK_THROWS_AS(resolve_workers(-3), UsageError);
    CHECK(std::abs(efficiency(80.865, 2, 40.545) - 0.9972) < 1e-3);
    CHECK(std::abs(efficiency(80.865, 4, 20.506) - 0.9859) < 1e-3);
    CHECK(efficiency(12.5, 1, 12.5) == 1.0);
    CHECK_THROWS_AS(efficiency(1.0, 0, 1.0), ParamError);
    CHECK_THROWS_AS(efficiency(1.0, 2, 0.0), ParamError);
    CHECK_THROWS_AS(efficiency(1.0, 2, -3.0), ParamError);
    // a tight --mem-cap is rejected before any device work
    auto m = parse({"1000000000", "--mem-cap=1048576"});
    CHECK_THROWS_AS(validate_resources(m), ResourceError);
    std::ostringstream out, err;
    CHECK_THROWS_AS(run(m, out, err), ResourceError);
    CHECK(out.str().empty());
}

int main(int argc, char** argv) {
    (void)argc;
    (void)argv;
    test_pool();
    test_verifier_host();
    test_cli();
    std::cout << "test_host: " << g_pass << " passed, " << g_fail << " failed\n";
    return g_fail ? 1 : 0;
}
