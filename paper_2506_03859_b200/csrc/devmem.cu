// devmem.cu -- a cache of large device blocks (Q, B', U, V, the Ozaki slices, A copies).
//
// The stream-ordered pool (cudaMallocAsync) is fine for the many small per-block
// buffers, but a multi-GB request from it costs milliseconds even when the pool already
// holds the memory, and now and then several hundred (measured on the C4 step: 3-8 ms per
// 1-2 GB request, outliers of 185 and 508 ms -- the run-to-run jitter of the bench).  So
// blocks of >= 16 MB come from plain cudaMalloc once and are kept per device: a freed
// block goes back to the cache with an event recorded on the stream that last used it, a
// request takes the smallest cached block that fits (at most 1.5x the request) after a
// stream wait on that event.  Results handed to the caller (Q, B', U, V on the device)
// return here through fqb_result_free.  At most FQB_DEVICE_CACHE_MB (default: half the
// device's memory) stays cached; a failed cudaMalloc empties the cache and retries once.
#include <cuda_runtime.h>

#include <cstdlib>
#include <map>
#include <mutex>
#include <unordered_map>

#include "engine.hpp"

namespace farqb {
namespace {

struct Block {
    void* ptr;
    cudaEvent_t ready;   // the last use of the block has completed once this fires
};

struct DevCache {
    std::mutex mu;
    std::multimap<size_t, Block> free_blocks[64];         // per device: size -> block
    std::unordered_map<void*, std::pair<int, size_t>> live;   // block -> (device, size)
    std::unordered_map<void*, cudaEvent_t> events;             // one event per block, reused
    size_t cached[64] = {};
};
DevCache& cache() {
    static DevCache* c = new DevCache();   // never destroyed (blocks may be freed during teardown)
    return *c;
}

size_t cache_cap(int dev) {
    static size_t cap[64] = {};
    if (!cap[dev]) {
        const char* e = std::getenv("FQB_DEVICE_CACHE_MB");
        if (e && *e) {
            cap[dev] = size_t(std::max(0LL, std::atoll(e))) << 20;
        } else {
            size_t fr = 0, tot = 0;
            cudaMemGetInfo(&fr, &tot);
            cap[dev] = tot / 2;
        }
        if (!cap[dev]) cap[dev] = 1;
    }
    return cap[dev];
}

int current_device() {
    int d = 0;
    cudaGetDevice(&d);
    return (d >= 0 && d < 64) ? d : 0;
}

size_t trim_device(DevCache& c, int dev) {
    size_t freed = 0;
    for (auto& kv : c.free_blocks[dev]) {
        cudaEventSynchronize(kv.second.ready);
        cudaFree(kv.second.ptr);
        freed += kv.first;
        auto ev = c.events.find(kv.second.ptr);
        if (ev != c.events.end()) {
            cudaEventDestroy(ev->second);
            c.events.erase(ev);
        }
    }
    c.free_blocks[dev].clear();
    c.cached[dev] = 0;
    return freed;
}

}  // namespace

void* device_alloc_large(size_t bytes, cudaStream_t s) {
    DevCache& c = cache();
    const int dev = current_device();
    {
        std::lock_guard<std::mutex> lk(c.mu);
        auto it = c.free_blocks[dev].lower_bound(bytes);
        if (it != c.free_blocks[dev].end() && it->first <= bytes + bytes / 2) {
            Block b = it->second;
            const size_t sz = it->first;
            c.free_blocks[dev].erase(it);
            c.cached[dev] -= sz;
            c.live[b.ptr] = {dev, sz};
            FQB_CUDA(cudaStreamWaitEvent(s, b.ready, 0));
            return b.ptr;
        }
    }
    void* p = nullptr;
    cudaError_t e = cudaMalloc(&p, bytes);
    if (e != cudaSuccess) {
        cudaGetLastError();
        {
            std::lock_guard<std::mutex> lk(c.mu);
            trim_device(c, dev);
        }
        e = cudaMalloc(&p, bytes);
    }
    cuda_check(e, "cudaMalloc");
    std::lock_guard<std::mutex> lk(c.mu);
    c.live[p] = {dev, bytes};
    return p;
}

bool device_free_large(void* p, cudaStream_t s) {
    if (!p) return true;
    DevCache& c = cache();
    std::lock_guard<std::mutex> lk(c.mu);
    auto it = c.live.find(p);
    if (it == c.live.end()) return false;   // not one of ours
    const int dev = it->second.first;
    const size_t sz = it->second.second;
    c.live.erase(it);
    cudaEvent_t& ev = c.events[p];
    if (!ev) cudaEventCreateWithFlags(&ev, cudaEventDisableTiming);
    cudaEventRecord(ev, s);   // s = nullptr: the legacy stream (callers freeing from the host sync first)
    if (c.cached[dev] + sz > cache_cap(dev)) {
        cudaEventSynchronize(ev);
        cudaEventDestroy(ev);
        c.events.erase(p);
        cudaFree(p);
        return true;
    }
    c.free_blocks[dev].emplace(sz, Block{p, ev});
    c.cached[dev] += sz;
    return true;
}

size_t device_cache_trim() {
    DevCache& c = cache();
    std::lock_guard<std::mutex> lk(c.mu);
    size_t freed = 0;
    int cur = 0;
    cudaGetDevice(&cur);
    for (int d = 0; d < 64; ++d) {
        if (c.free_blocks[d].empty()) continue;
        cudaSetDevice(d);
        freed += trim_device(c, d);
    }
    cudaSetDevice(cur);
    return freed;
}

}  // namespace farqb
