// paper_1903_00227_b200/csrc/alloc.cpp -- a caching device allocator for the
// library's large buffers (weights, tables, build and draw scratch).
//
// cudaMalloc / cudaFree of multi-GB buffers cost milliseconds and cudaFree
// synchronises the device; a caller that builds, draws and frees samplers in
// a loop (the reference's usage, and the e2e benchmark) would pay that every
// time.  Freed blocks are kept per (device, size) and handed out again for an
// allocation of exactly that size.  A block is cached only after the device
// is idle (cudaDeviceSynchronize), so no in-flight work can still touch it --
// unless the caller holds an armed SyncedFrees (engine.h): it has synchronised
// every stream that used the block, and the device-wide wait would only stall
// this thread behind other threads' work.
// Cached bytes are capped (WRS_B200_CACHE_MB, default 8 GB per process);
// an allocation that fails for lack of memory returns every cached block of
// its device and retries, and wrs_b200_release_cache() hands every cached
// block back to the driver (e.g. before a co-resident framework allocates).
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdlib>
#include <map>
#include <mutex>
#include <unordered_map>
#include <utility>

#include "engine.h"

namespace wrsb {

namespace {

struct Cache {
    std::mutex mu;
    std::multimap<std::pair<int, size_t>, void*> free_blocks;
    std::unordered_map<void*, std::pair<int, size_t>> live;
    size_t cached = 0;
    const size_t limit = [] {
        const char* e = std::getenv("WRS_B200_CACHE_MB");
        return e ? static_cast<size_t>(std::strtoull(e, nullptr, 10)) << 20 : size_t{8} << 30;
    }();

    // dev < 0: every device
    void release_device(int dev) {
        for (auto it = free_blocks.begin(); it != free_blocks.end();) {
            if (dev < 0 || it->first.first == dev) {
                cudaFree(it->second);
                cached -= it->first.second;
                it = free_blocks.erase(it);
            } else {
                ++it;
            }
        }
    }
};

Cache& cache() {
    static Cache* c = new Cache;  // never destroyed: blocks may outlive static teardown
    return *c;
}

}  // namespace

cudaError_t dev_malloc(void** p, size_t bytes) {
    if (bytes == 0) bytes = 16;
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    Cache& c = cache();
    std::lock_guard<std::mutex> g(c.mu);
    auto it = c.free_blocks.find({dev, bytes});
    if (it != c.free_blocks.end()) {
        *p = it->second;
        c.free_blocks.erase(it);
        c.cached -= bytes;
        c.live[*p] = {dev, bytes};
        return cudaSuccess;
    }
    e = cudaMalloc(p, bytes);
    if (e == cudaErrorMemoryAllocation) {
        cudaGetLastError();
        c.release_device(dev);
        e = cudaMalloc(p, bytes);
    }
    if (e == cudaSuccess) c.live[*p] = {dev, bytes};
    return e;
}

namespace {
thread_local int t_synced_frees = 0;
}

void SyncedFrees::arm() {
    if (!armed) {
        armed = true;
        ++t_synced_frees;
    }
}

SyncedFrees::~SyncedFrees() {
    if (armed) --t_synced_frees;
}

void dev_free(void* p) {
    if (!p) return;
    Cache& c = cache();
    std::lock_guard<std::mutex> g(c.mu);
    auto it = c.live.find(p);
    if (it == c.live.end()) {
        cudaFree(p);
        return;
    }
    const auto key = it->second;
    c.live.erase(it);
    int cur = 0;
    cudaGetDevice(&cur);
    if (cur != key.first) cudaSetDevice(key.first);
    if (c.cached + key.second <= c.limit &&
        (t_synced_frees > 0 || cudaDeviceSynchronize() == cudaSuccess)) {
        c.free_blocks.insert({key, p});
        c.cached += key.second;
    } else {
        cudaFree(p);
    }
    if (cur != key.first) cudaSetDevice(cur);
}

size_t release_cache() {
    Cache& c = cache();
    std::lock_guard<std::mutex> g(c.mu);
    const size_t had = c.cached;
    int cur = 0;
    cudaGetDevice(&cur);
    c.release_device(-1);
    cudaSetDevice(cur);
    return had;
}

}  // namespace wrsb
