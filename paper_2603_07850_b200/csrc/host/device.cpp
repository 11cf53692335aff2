// device.cpp -- status mapping, the Device RAII handle and the shared
// per-process handles used by verify_segment outside run_workers.
#include "goldbach/device.hpp"

#include <map>
#include <mutex>
#include <tuple>

#include "goldbach/errors.hpp"

namespace goldbach {

void raise_status(int status, const std::string& message) {
    switch (status) {
    case GB_ERR_PARAM: throw ParamError(message);
    case GB_ERR_RESOURCE: throw ResourceError(message);
    case GB_ERR_INTERNAL: throw InternalError(message);
    default: throw DeviceError(message.empty() ? std::string("device error") : message);
    }
}

Device::Device(const DeviceConfig& cfg) : cfg_(cfg) {
    gb_params prm{};
    prm.cover_limit = cfg.cover_limit;
    prm.p_small = cfg.p_small;
    prm.phase2_limit = 0;
    prm.batch_size = 0;
    prm.inject_fail = cfg.inject_fail;
    prm.max_seg_evens = cfg.max_seg_evens;
    int rc = gb_open(cfg.device, &prm, &h_);
    if (rc != GB_OK) raise_status(rc, gb_last_error(nullptr));
}

Device::~Device() {
    if (h_) gb_close(h_);
}

void Device::check(int status) const {
    if (status != GB_OK) raise_status(status, gb_last_error(h_));
}

gb_seg_record Device::verify(uint64_t a, uint64_t b) {
    gb_seg_record r{};
    check(gb_verify_segment(h_, a, b, &r));
    return r;
}

void Device::submit(uint64_t a, uint64_t b, uint64_t tag) { check(gb_submit_segment(h_, a, b, tag)); }

gb_seg_record Device::wait(uint64_t* tag) {
    gb_seg_record r{};
    check(gb_wait_segment(h_, &r, tag));
    return r;
}

int Device::max_inflight() const {
    int d = 1;
    check(gb_max_inflight(h_, &d));
    return d;
}

void Device::set_inject_fail(uint64_t n) {
    check(gb_set_inject_fail(h_, n));
    cfg_.inject_fail = n;
}

int visible_gpus() {
    int n = 0;
    gb_device_count(&n);
    return n;
}

std::shared_ptr<SharedDevice> SharedDevice::get(const DeviceConfig& cfg) {
    using Key = std::tuple<int, uint64_t, uint64_t, uint64_t>;
    static std::mutex mu;
    static std::map<Key, std::shared_ptr<SharedDevice>> cache;
    Key key{cfg.device, cfg.cover_limit, cfg.p_small, cfg.inject_fail};
    std::lock_guard<std::mutex> lock(mu);
    auto it = cache.find(key);
    if (it != cache.end()) return it->second;
    auto sd = std::make_shared<SharedDevice>(cfg);
    cache.emplace(key, sd);
    return sd;
}

} // namespace goldbach
