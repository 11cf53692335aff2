// device.hpp -- B200 addition to the drop-in API: RAII ownership of one GPU
// worker handle (gb_dev, include/goldbach_b200.h).  The reference has no
// device; its per-worker state is the std::thread in run_workers
// (proj/src/pool.cpp:90-120).  One Device per GPU per host thread.
#pragma once

#include <cstdint>
#include <memory>
#include <mutex>
#include <vector>

#include "goldbach_b200.h"

namespace goldbach {

struct DeviceConfig {
    int device = 0;
    uint64_t cover_limit = 0;
    uint64_t p_small = 1'000'000;
    uint64_t inject_fail = 0;
    uint64_t max_seg_evens = 200'000'000;
};

class Device {
public:
    explicit Device(const DeviceConfig& cfg);
    ~Device();
    Device(Device&& o) noexcept : h_(o.h_), cfg_(o.cfg_) { o.h_ = nullptr; }
    Device(const Device&) = delete;
    Device& operator=(const Device&) = delete;

    gb_dev* get() const { return h_; }
    const DeviceConfig& config() const { return cfg_; }

    gb_seg_record verify(uint64_t a, uint64_t b);  // synchronous segment
    void submit(uint64_t a, uint64_t b, uint64_t tag);
    gb_seg_record wait(uint64_t* tag);
    int max_inflight() const;
    void set_inject_fail(uint64_t n);

    // throws the mapped exception for a non-zero status of this handle
    void check(int status) const;

private:
    gb_dev* h_ = nullptr;
    DeviceConfig cfg_;
};

// Number of CUDA devices visible to this process.
int visible_gpus();

// Process-wide handle used by verify_segment() calls made outside
// run_workers (one per (device, tables, inject) key, serialised by a mutex).
class SharedDevice {
public:
    static std::shared_ptr<SharedDevice> get(const DeviceConfig& cfg);
    explicit SharedDevice(const DeviceConfig& cfg) : dev_(cfg) {}

    // runs f(Device&) with the handle locked
    template <class F>
    auto with(F&& f) {
        std::lock_guard<std::mutex> lock(mu_);
        return f(dev_);
    }

private:
    std::mutex mu_;
    Device dev_;
};

} // namespace goldbach
