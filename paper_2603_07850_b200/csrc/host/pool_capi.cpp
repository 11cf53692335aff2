// pool_capi.cpp -- extern "C" entry points of include/goldbach_b200_pool.h
// over the C++ pool/runner (pool.cpp).  Shared-memory cursors let one
// process per GPU (torchrun) steal segments from one counter.
#include <fcntl.h>
#include <sys/mman.h>
#include <unistd.h>

#include <algorithm>
#include <cstring>
#include <iostream>
#include <new>
#include <sstream>
#include <string>

#include "goldbach/device.hpp"
#include "goldbach/errors.hpp"
#include "goldbach/pool.hpp"
#include "goldbach_b200_pool.h"

namespace goldbach {
extern thread_local Device* tl_worker_device;
}

using namespace goldbach;

namespace {

thread_local std::string t_pool_err;

struct ShmHeader {
    uint64_t magic;
    uint64_t start, limit, span;
    std::atomic<uint64_t> cursor;
    std::atomic<uint32_t> attached; // processes on this cursor (the tail-limit hint)
    std::atomic<uint32_t> stop;     // cooperative stop of every attached rank (pool.cpp:104-111)
};
constexpr uint64_t kMagic = 0x474f4c4442414332ull; // "GOLDBAC2" (layout with the stop word)

int map_exception(const std::exception& e) {
    t_pool_err = e.what();
    if (dynamic_cast<const ParamError*>(&e)) return GB_ERR_PARAM;
    if (dynamic_cast<const ResourceError*>(&e)) return GB_ERR_RESOURCE;
    if (dynamic_cast<const InternalError*>(&e)) return GB_ERR_INTERNAL;
    return GB_ERR_CUDA;
}

void to_c(const RunResult& r, gb_run_result* o) {
    std::memset(o, 0, sizeof(*o));
    o->evens_checked = r.evens_checked;
    o->unverified_total = r.unverified_total;
    o->phase2_total = r.phase2_total;
    o->pmin_sum = r.pmin_sum;
    o->pmin_hash = r.pmin_hash;
    o->max_p = r.min_prime.p;
    o->max_n = r.min_prime.n;
    o->segments = r.segments;
    o->n_counterexamples = std::max<uint64_t>(r.counterexample_count, r.counterexamples.size());
    for (size_t i = 0; i < r.counterexamples.size() && i < GB_REC_MAX_CE; ++i) o->counterexamples[i] = r.counterexamples[i];
    o->wall_seconds = r.wall_seconds;
}

} // namespace

struct gb_pool {
    std::unique_ptr<WorkPool> pool;
    ShmHeader* shm = nullptr;
    std::string name;
};

extern "C" {

const char* gb_pool_last_error(void) { return t_pool_err.c_str(); }

int gb_pool_create(uint64_t start, uint64_t limit, uint64_t seg_size, const char* shm_name, int create,
                   gb_pool** out) {
    *out = nullptr;
    try {
        auto p = std::make_unique<gb_pool>();
        if (!shm_name) {
            p->pool = std::make_unique<WorkPool>(start, limit, seg_size);
        } else {
            WorkPool probe(start, limit, seg_size); // validates arguments first
            (void)probe;
            p->name = shm_name[0] == '/' ? shm_name : std::string("/") + shm_name;
            int fd = shm_open(p->name.c_str(), create ? (O_CREAT | O_RDWR) : O_RDWR, 0600);
            if (fd < 0) throw ResourceError("gb_pool_create: shm_open(" + p->name + ") failed");
            if (create && ftruncate(fd, sizeof(ShmHeader)) != 0) {
                close(fd);
                throw ResourceError("gb_pool_create: ftruncate failed");
            }
            void* m = mmap(nullptr, sizeof(ShmHeader), PROT_READ | PROT_WRITE, MAP_SHARED, fd, 0);
            close(fd);
            if (m == MAP_FAILED) throw ResourceError("gb_pool_create: mmap failed");
            p->shm = static_cast<ShmHeader*>(m);
            if (create) {
                p->shm->start = start;
                p->shm->limit = limit;
                p->shm->span = 2 * seg_size;
                new (&p->shm->cursor) std::atomic<uint64_t>(start);
                new (&p->shm->attached) std::atomic<uint32_t>(0);
                new (&p->shm->stop) std::atomic<uint32_t>(0);
                std::atomic_thread_fence(std::memory_order_release);
                p->shm->magic = kMagic;
            } else if (p->shm->magic != kMagic || p->shm->start != start || p->shm->limit != limit ||
                       p->shm->span != 2 * seg_size) {
                munmap(m, sizeof(ShmHeader));
                throw ParamError("gb_pool_create: shared pool " + p->name + " does not match these bounds");
            }
            p->shm->attached.fetch_add(1, std::memory_order_relaxed);
            p->pool = std::make_unique<WorkPool>(start, limit, seg_size, &p->shm->cursor, &p->shm->attached,
                                                 &p->shm->stop);
        }
        *out = p.release();
        return GB_OK;
    } catch (const std::exception& e) {
        return map_exception(e);
    }
}

int gb_pool_claim(gb_pool* p, uint64_t* a, uint64_t* b, uint64_t* index) {
    if (!p) return -GB_ERR_PARAM;
    auto j = p->pool->claim_next();
    if (!j) return 0;
    *a = j->a;
    *b = j->b;
    *index = j->index;
    return 1;
}

int gb_pool_request_stop(gb_pool* p) {
    if (!p) return GB_ERR_PARAM;
    p->pool->request_stop();
    return GB_OK;
}

int gb_pool_stop_requested(const gb_pool* p) { return p && p->pool->stop_requested() ? 1 : 0; }

int gb_pool_destroy(gb_pool* p, int unlink) {
    if (!p) return GB_OK;
    if (p->shm) {
        munmap(p->shm, sizeof(ShmHeader));
        if (unlink) shm_unlink(p->name.c_str());
    }
    delete p;
    return GB_OK;
}

int gb_drain_pool(gb_dev* dev, gb_pool* pool, int max_inflight, gb_run_result* out) {
    if (!dev || !pool || !out) return GB_ERR_PARAM;
    const auto t0 = std::chrono::steady_clock::now();
    RunResult mine;
    int cap = max_inflight;
    if (cap <= 0 && gb_max_inflight(dev, &cap) != GB_OK) cap = 1;
    int depth = 1, inflight = 0;
    bool exhausted = false, stop = false;
    for (;;) {
        while (!exhausted && !stop && inflight < std::min(depth, pool->pool->tail_limit(cap))) {
            auto job = pool->pool->claim_next();
            if (!job) {
                exhausted = true;
                break;
            }
            int rc = gb_submit_segment(dev, job->a, job->b, job->index);
            if (rc) return rc;
            ++inflight;
        }
        if (inflight == 0) break;
        gb_seg_record r{};
        int rc = gb_wait_segment(dev, &r, nullptr);
        if (rc) return rc;
        --inflight;
        mine.evens_checked += r.evens_checked;
        mine.unverified_total += r.unverified_p1;
        mine.phase2_total += r.phase2_resolved;
        mine.pmin_sum += r.pmin_sum;
        mine.pmin_hash += r.pmin_hash;
        mine.segments += 1;
        mine.min_prime.merge(MinPrimeMax{r.max_p, r.max_n});
        for (uint64_t i = 0; i < r.n_counterexamples && i < GB_REC_MAX_CE; ++i)
            mine.counterexamples.push_back(r.counterexamples[i]);
        mine.counterexample_count += r.n_counterexamples;
        if (r.n_counterexamples) {
            stop = true;
            pool->pool->request_stop(); // reaches every rank on a shared cursor
        }
        depth = std::min(cap, depth * 2);
    }
    std::sort(mine.counterexamples.begin(), mine.counterexamples.end());
    mine.wall_seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    to_c(mine, out);
    return GB_OK;
}

int gb_run_range(uint64_t start, uint64_t limit, uint64_t seg_size, uint64_t p_small, uint64_t inject_fail,
                 const int* devices, int n_devices, int n_workers, int progress, gb_run_result* out,
                 uint64_t* per_worker_segments) {
    try {
        const SmallPrimeTable small = SmallPrimeTable::descriptor(p_small);
        const Phase2Table phase2{};
        const BasePrimes base = base_primes_descriptor(limit);
        VerifyContext ctx;
        ctx.small = &small;
        ctx.phase2 = &phase2;
        ctx.base = &base;
        ctx.inject_fail = inject_fail;
        WorkPool pool(start, limit, seg_size);
        RunOptions opt;
        opt.workers = (unsigned)(n_workers > 0 ? n_workers : std::max(1, n_devices));
        opt.progress = progress != 0;
        for (int i = 0; i < n_devices; ++i) opt.devices.push_back(devices[i]);
        std::ostringstream sink;
        std::ostream& err = progress ? static_cast<std::ostream&>(std::cerr) : sink;
        Logger log(err);
        RunResult r = run_workers(pool, ctx, opt, log);
        to_c(r, out);
        if (per_worker_segments)
            for (size_t w = 0; w < r.per_worker_segments.size(); ++w) per_worker_segments[w] = r.per_worker_segments[w];
        return GB_OK;
    } catch (const std::exception& e) {
        return map_exception(e);
    }
}

} // extern "C"
