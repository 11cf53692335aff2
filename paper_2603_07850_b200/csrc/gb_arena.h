// gb_arena.h -- process-wide caching allocator for device and pinned host
// buffers of the verifier.  gb_open/gb_close (one per run_workers call,
// cli.cpp:312-321 builds the tables per run) would otherwise pay
// cudaMalloc/cudaFree and cudaMallocHost/cudaFreeHost for ~150 MB of batch
// buffers every time; freed blocks are kept on per-device free lists and
// handed out again (best fit, at most 2x the request + 1 MiB).  On an
// allocation failure the device's cached blocks are released and the
// allocation is retried.
#pragma once

#include <cuda_runtime.h>

#include <cstddef>
#include <map>
#include <mutex>
#include <unordered_map>

namespace gbk {

class Arena {
public:
    static Arena& get() {
        static Arena* a = new Arena(); // process lifetime: never torn down
        return *a;
    }

    cudaError_t dev_alloc(int device, void** p, size_t bytes) {
        bytes = round(bytes);
        if (void* q = take(free_dev_[slot(device)], bytes)) {
            *p = q;
            return cudaSuccess;
        }
        cudaError_t e = cudaMalloc(p, bytes);
        if (e != cudaSuccess) {
            (void)cudaGetLastError();
            release_device(device);
            e = cudaMalloc(p, bytes);
        }
        if (e == cudaSuccess) remember(*p, bytes);
        return e;
    }

    void dev_free(int device, void* p) {
        if (!p) return;
        std::lock_guard<std::mutex> g(mu_);
        auto it = size_.find(p);
        if (it == size_.end()) {
            cudaFree(p);
            return;
        }
        free_dev_[slot(device)].emplace(it->second, p);
    }

    cudaError_t host_alloc(void** p, size_t bytes) {
        bytes = round(bytes);
        if (void* q = take(free_host_, bytes)) {
            *p = q;
            return cudaSuccess;
        }
        cudaError_t e = cudaMallocHost(p, bytes);
        if (e == cudaSuccess) remember(*p, bytes);
        return e;
    }

    void host_free(void* p) {
        if (!p) return;
        std::lock_guard<std::mutex> g(mu_);
        auto it = size_.find(p);
        if (it == size_.end()) {
            cudaFreeHost(p);
            return;
        }
        free_host_.emplace(it->second, p);
    }

    // Returns every cached (free) block of `device` to the driver.
    void release_device(int device) {
        std::lock_guard<std::mutex> g(mu_);
        auto& fl = free_dev_[slot(device)];
        int prev = 0;
        cudaGetDevice(&prev);
        cudaSetDevice(device);
        for (auto& kv : fl) {
            cudaFree(kv.second);
            size_.erase(kv.second);
        }
        fl.clear();
        cudaSetDevice(prev);
    }

private:
    static constexpr int kMaxDevices = 64;
    static size_t round(size_t b) { return ((b ? b : 1) + 255) & ~size_t(255); }
    static int slot(int device) { return device >= 0 && device < kMaxDevices ? device : 0; }

    void* take(std::multimap<size_t, void*>& fl, size_t bytes) {
        std::lock_guard<std::mutex> g(mu_);
        auto it = fl.lower_bound(bytes);
        if (it == fl.end() || it->first > 2 * bytes + (size_t(1) << 20)) return nullptr;
        void* p = it->second;
        fl.erase(it);
        return p;
    }

    void remember(void* p, size_t bytes) {
        std::lock_guard<std::mutex> g(mu_);
        size_[p] = bytes;
    }

    std::mutex mu_;
    std::multimap<size_t, void*> free_dev_[kMaxDevices];
    std::multimap<size_t, void*> free_host_;
    std::unordered_map<void*, size_t> size_;
};

template <class T>
inline cudaError_t dmalloc(int device, T** p, size_t bytes) {
    return Arena::get().dev_alloc(device, reinterpret_cast<void**>(p), bytes);
}
inline void dfree(int device, void* p) { Arena::get().dev_free(device, p); }
template <class T>
inline cudaError_t hmalloc(T** p, size_t bytes) {
    return Arena::get().host_alloc(reinterpret_cast<void**>(p), bytes);
}
inline void hfree(void* p) { Arena::get().host_free(p); }

} // namespace gbk
