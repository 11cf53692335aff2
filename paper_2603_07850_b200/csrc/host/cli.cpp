// cli.cpp -- command-line surface: flag grammar, resource validation,
// orchestration and the text/JSON summaries (proj/src/cli.cpp semantics:
// flags :165-186, odd-bound rounding :198-207, invariants :209-222, exit
// codes 0/1/2 :333, JSON key order :117-134).
#include "goldbach/cli.hpp"

#include <algorithm>
#include <cstdlib>
#include <chrono>
#include <charconv>
#include <cmath>
#include <functional>
#include <iomanip>
#include <map>
#include <ostream>
#include <sstream>
#include <thread>
#include <vector>

#include "goldbach/device.hpp"
#include "goldbach/pool.hpp"
#include "goldbach/verifier.hpp"
#include "goldbach_b200_pool.h"

namespace goldbach {

namespace {

uint64_t to_u64(const std::string& flag, std::string_view v) {
    uint64_t x = 0;
    const auto [end, ec] = std::from_chars(v.data(), v.data() + v.size(), x);
    if (ec == std::errc::result_out_of_range) throw UsageError(flag + ": value out of range (the ceiling is 2^64 - 1)");
    if (v.empty() || ec != std::errc{} || end != v.data() + v.size())
        throw UsageError(flag + ": expected a number, got '" + std::string(v) + "'");
    return x;
}

int64_t to_i64(const std::string& flag, std::string_view v) {
    int64_t x = 0;
    const auto [end, ec] = std::from_chars(v.data(), v.data() + v.size(), x);
    if (v.empty() || ec != std::errc{} || end != v.data() + v.size())
        throw UsageError(flag + ": expected an integer, got '" + std::string(v) + "'");
    return x;
}

std::string human_bytes(uint64_t b) {
    const char* unit[] = {"B", "KiB", "MiB", "GiB", "TiB"};
    double v = (double)b;
    int u = 0;
    for (; v >= 1024.0 && u < 4; ++u) v /= 1024.0;
    std::ostringstream o;
    o << std::fixed << std::setprecision(1) << v << ' ' << unit[u];
    return o.str();
}

// Minimal ordered JSON emitter for the summary object.
class JsonObject {
public:
    template <class T>
    void put(const std::string& k, const T& v) {
        std::ostringstream o;
        o << v;
        add(k, o.str());
    }
    void put(const std::string& k, bool v) { add(k, v ? "true" : "false"); }
    void put(const std::string& k, double v) {
        std::ostringstream o;
        o << std::setprecision(17) << v;
        add(k, o.str());
    }
    template <class T>
    void put_list(const std::string& k, const std::vector<T>& v) {
        std::ostringstream o;
        o << '[';
        for (size_t i = 0; i < v.size(); ++i) o << (i ? "," : "") << v[i];
        o << ']';
        add(k, o.str());
    }
    std::string str() const { return "{" + body_ + "}"; }

private:
    void add(const std::string& k, const std::string& v) { body_ += (body_.empty() ? "\"" : ",\"") + k + "\":" + v; }
    std::string body_;
};

void print_json(std::ostream& out, const Config& cfg, unsigned workers, const RunResult& r) {
    JsonObject j;
    j.put("limit", cfg.limit);
    j.put("start", cfg.start);
    j.put("workers_used", workers);
    j.put("seg_size", cfg.seg_size);
    j.put("p_small", cfg.p_small);
    j.put("batch_size", cfg.batch_size);
    j.put("phase2_limit", cfg.phase2_limit);
    j.put("total_evens", r.evens_checked);
    j.put("unverified_total", r.unverified_total);
    j.put("phase2_total", r.phase2_total);
    j.put_list("counterexamples", r.counterexamples);
    j.put("max_min_prime", r.min_prime.p);
    j.put("max_min_prime_n", r.min_prime.n);
    j.put("segments", r.segments);
    j.put_list("per_worker_segments", r.per_worker_segments);
    j.put("wall_seconds", r.wall_seconds);
    j.put("verified", r.counterexamples.empty());
    // B200 additions (after the reference keys)
    j.put("pmin_sum", r.pmin_sum);
    j.put("pmin_hash", r.pmin_hash);
    j.put_list("gpus", r.worker_devices);
    j.put("init_seconds", r.init_seconds);
    j.put("counterexample_count", r.counterexample_count);
    out << j.str() << "\n";
}

void print_human(std::ostream& out, const Config& cfg, unsigned workers, const RunResult& r) {
    out << "goldbach verification summary\n";
    auto line = [&](const char* label) -> std::ostream& {
        return out << "  " << std::left << std::setw(25) << label << ": ";
    };
    line("range") << '[' << cfg.start << ", " << cfg.limit << "]\n";
    line("workers") << workers << "\n";
    line("segments") << r.segments << "\n";
    line("evens checked") << r.evens_checked << "\n";
    line("unverified after phase 1") << r.unverified_total << "\n";
    line("phase 2 resolved") << r.phase2_total << "\n";
    line("max p_min") << r.min_prime.p << " at n = " << r.min_prime.n << "\n";
    line("counterexamples");
    if (r.counterexamples.empty()) out << "none";
    for (size_t i = 0; i < r.counterexamples.size(); ++i) out << (i ? " " : "") << r.counterexamples[i];
    out << "\n";
    line("checksum") << "sum p_min " << r.pmin_sum << ", hash " << r.pmin_hash << "\n";
    line("wall time") << std::fixed << std::setprecision(2) << r.wall_seconds << " s\n";
    line("result") << (r.counterexamples.empty() ? "VERIFIED" : "COUNTEREXAMPLE FOUND") << "\n";
}

} // namespace

Config parse_args(const std::vector<std::string>& args, std::ostream& warn) {
    Config cfg;
    bool have_limit = false;
    // value-taking flags
    const std::map<std::string, std::function<void(const std::string&, const std::string&)>> takes = {
        {"--start", [&](auto& f, auto& v) { cfg.start = to_u64(f, v); }},
        {"--workers", [&](auto& f, auto& v) { cfg.workers = to_i64(f, v); }},
        {"--gpus", [&](auto& f, auto& v) { cfg.workers = to_i64(f, v); }},
        {"--seg-size", [&](auto& f, auto& v) { cfg.seg_size = to_u64(f, v); }},
        {"--p-small", [&](auto& f, auto& v) { cfg.p_small = to_u64(f, v); }},
        {"--batch-size", [&](auto& f, auto& v) { cfg.batch_size = to_u64(f, v); }},
        {"--phase2-limit", [&](auto& f, auto& v) { cfg.phase2_limit = to_u64(f, v); }},
        {"--mem-cap", [&](auto& f, auto& v) { cfg.mem_cap = to_u64(f, v); }},
        {"--inject-fail", [&](auto& f, auto& v) { cfg.inject_fail = to_u64(f, v); }},
    };
    for (size_t i = 0; i < args.size(); ++i) {
        const std::string& tok = args[i];
        if (tok == "-h" || tok == "--help") {
            cfg.help = true;
            continue;
        }
        if (tok.rfind("--", 0) != 0) {
            if (have_limit) throw UsageError("unexpected extra argument '" + tok + "'");
            cfg.limit = to_u64("LIMIT", tok);
            have_limit = true;
            continue;
        }
        const size_t eq = tok.find('=');
        const std::string flag = tok.substr(0, eq);
        const bool inline_value = eq != std::string::npos;
        if (flag == "--json" || flag == "--progress") {
            if (inline_value) throw UsageError(flag + " takes no value");
            (flag == "--json" ? cfg.json : cfg.progress) = true;
            continue;
        }
        auto it = takes.find(flag);
        if (it == takes.end()) throw UsageError("unknown flag '" + flag + "'");
        std::string value;
        if (inline_value) {
            value = tok.substr(eq + 1);
        } else {
            if (i + 1 >= args.size()) throw UsageError(flag + ": missing value");
            value = args[++i];
        }
        it->second(flag, value);
    }
    if (cfg.help) return cfg;
    if (!have_limit) throw UsageError("missing LIMIT argument");
    if (cfg.limit & 1) {
        warn << "warning: odd limit " << cfg.limit << " rounded down to " << cfg.limit - 1 << "\n";
        --cfg.limit;
    }
    if (cfg.start & 1) {
        warn << "warning: odd start " << cfg.start << " rounded down to " << cfg.start - 1 << "\n";
        --cfg.start;
    }
    if (cfg.limit < 4) throw UsageError("limit must be at least 4");
    if (cfg.start < 4) throw UsageError("start must be at least 4");
    if (cfg.start > cfg.limit) throw UsageError("start exceeds limit");
    if (cfg.workers == 0 || cfg.workers < -1) throw UsageError("workers must be >= 1, or -1 for all visible GPUs");
    if (cfg.workers > 4096) throw UsageError("workers value is too large (max 4096)");
    if (cfg.seg_size == 0 || cfg.seg_size > 0xFFFFFFFFull)
        throw UsageError("seg-size must be in [1, 4294967295] so the per-segment unverified counter fits 32 bits");
    if (cfg.p_small < 3) throw UsageError("p-small must be at least 3");
    if (cfg.batch_size == 0) throw UsageError("batch-size must be at least 1");
    if (cfg.mem_cap && *cfg.mem_cap == 0) throw UsageError("mem-cap must be positive");
    return cfg;
}

std::string usage_text() {
    return "usage: goldbach [OPTIONS] LIMIT\n"
           "\n"
           "Verifies Goldbach's conjecture for every even integer in [--start, LIMIT]\n"
           "(both inclusive) on NVIDIA B200 GPUs. Odd bounds are rounded down with a\n"
           "warning. The hard ceiling is 2^64 - 1.\n"
           "\n"
           "options:\n"
           "  --start=N         first even integer to check (default 4)\n"
           "  --gpus=N          GPU workers; -1 = every visible GPU (default 1)\n"
           "  --workers=N       alias of --gpus\n"
           "  --seg-size=N      even integers per work segment (default 200000000)\n"
           "  --p-small=N       phase 1 tries partition primes p <= N (default 1000000)\n"
           "  --batch-size=N    accepted for compatibility; result-invariant (default 2000000)\n"
           "  --phase2-limit=N  accepted for compatibility; phase 2 runs on the GPU with\n"
           "                    Miller-Rabin, result-invariant (default 100000000)\n"
           "  --mem-cap=BYTES   fail before any GPU work if a GPU's estimated footprint\n"
           "                    exceeds BYTES\n"
           "  --progress        print a progress line to stderr every second\n"
           "  --json            print the summary as a single JSON object\n"
           "  --inject-fail=N   self-test hook: treat even N as a counterexample\n"
           "  --help            show this help\n"
           "\n"
           "exit codes: 0 = range fully verified, 1 = usage/resource/internal/device\n"
           "error, 2 = counterexample found\n";
}

unsigned resolve_workers(int64_t workers) {
    if (workers == -1) return (unsigned)std::max(1, visible_gpus());
    if (workers < 1 || workers > 4096) throw UsageError("workers must be >= 1, or -1 for all visible GPUs");
    return (unsigned)workers;
}

MemoryEstimate validate_resources(const Config& cfg) {
    MemoryEstimate est;
    est.workers = resolve_workers(cfg.workers);
    est.per_worker_bytes = gb_estimate_device_bytes(cfg.limit, cfg.p_small, cfg.seg_size);
    est.shared_bytes = 1 << 20; // host-side records and pinned staging
    est.total_bytes = est.per_worker_bytes * est.workers + est.shared_bytes;
    // workers are mapped round-robin onto every visible GPU (run_workers'
    // worker_devices): check each device's load against that device's own
    // budget, before any worker is spawned (cli.cpp:264-296)
    const unsigned gpus = (unsigned)std::max(1, visible_gpus());
    for (unsigned g = 0; g < gpus && g < est.workers; ++g) {
        const uint64_t on_g = est.workers / gpus + (g < est.workers % gpus ? 1 : 0);
        const uint64_t load = est.per_worker_bytes * on_g;
        uint64_t budget = 0;
        std::string what;
        if (cfg.mem_cap) {
            budget = *cfg.mem_cap;
            what = "--mem-cap ";
        } else {
            uint64_t fr = 0, tot = 0;
            budget = gb_device_memory((int)g, &fr, &tot) == GB_OK ? fr : ~uint64_t{0};
            what = "free memory of GPU " + std::to_string(g) + " ";
        }
        if (load > budget)
            throw ResourceError("estimated footprint " + human_bytes(load) + " of GPU " + std::to_string(g) + " (" +
                                std::to_string(on_g) + " worker(s)) exceeds " + what + human_bytes(budget) +
                                " (reduce --seg-size or --gpus)");
    }
    return est;
}

double efficiency(double t1, unsigned k, double tk) {
    if (k < 1) throw ParamError("efficiency: k must be >= 1");
    if (tk <= 0.0) throw ParamError("efficiency: tk must be positive");
    return t1 / ((double)k * tk);
}

int run(const Config& cfg, std::ostream& out, std::ostream& err) {
    Logger log(err);
    // GB_DEBUG_OPEN: where a CLI process spends its time before and after the drain
    const bool dbg = getenv("GB_DEBUG_OPEN") != nullptr;
    const auto t_run = std::chrono::steady_clock::now();
    auto since = [&] { return std::chrono::duration<double>(std::chrono::steady_clock::now() - t_run).count(); };
    // the CUDA contexts of the worker GPUs are created in the background
    // while the resources are checked (NVML, no context needed): on a cold
    // process the context is the largest single cost before the first claim
    std::vector<std::thread> warm;
    {
        const unsigned k = resolve_workers(cfg.workers);
        const int g = std::max(1, visible_gpus());
        for (unsigned i = 0; i < k && (int)i < g; ++i) warm.emplace_back([i] { gb_warm_device((int)i); });
    }
    MemoryEstimate est;
    try {
        est = validate_resources(cfg);
    } catch (...) {
        for (auto& t : warm) t.join();
        throw;
    }
    for (auto& t : warm) t.join();
    if (dbg) log.logf("timing: validate_resources + contexts ", since(), " s");
    log.logf("memory estimate: ", human_bytes(est.total_bytes), " (", est.workers, " GPU worker(s) x ",
             human_bytes(est.per_worker_bytes), " + shared ", human_bytes(est.shared_bytes), ")");
    // tables are built on each GPU by its worker (K1); the host keeps only
    // the descriptors the workers need
    const SmallPrimeTable small = SmallPrimeTable::descriptor(cfg.p_small);
    const Phase2Table phase2{}; // result-invariant (Miller-Rabin on device)
    const BasePrimes base = base_primes_descriptor(cfg.limit);
    VerifyContext ctx;
    ctx.small = &small;
    ctx.phase2 = &phase2;
    ctx.base = &base;
    ctx.batch_size = cfg.batch_size;
    ctx.inject_fail = cfg.inject_fail;
    WorkPool pool(cfg.start, cfg.limit, cfg.seg_size);
    RunOptions opt;
    opt.workers = est.workers;
    opt.progress = cfg.progress;
    const RunResult res = run_workers(pool, ctx, opt, log);
    if (dbg) log.logf("timing: run_workers done ", since(), " s (worker init ", res.init_seconds, " s, wall ",
                      res.wall_seconds, " s)");
    if (cfg.json)
        print_json(out, cfg, est.workers, res);
    else
        print_human(out, cfg, est.workers, res);
    return res.counterexamples.empty() ? 0 : 2;
}

} // namespace goldbach
