// hostmem.cu -- pinned host memory for results returned on the host.
//
// Q, B', U and V come back through cudaMemcpy into library-allocated host arrays.
// Fresh malloc() pages cost a page fault per 4 KB on first touch (the C2 outputs,
// 51 MB, took ~24 ms that way against ~1 ms into pinned memory), so host results
// live in page-locked blocks from a process-wide pool: cudaMallocHost once, reused
// after fqb_result_free / fqb_host_free.  Blocks not from the pool (never, unless
// pinning failed) are plain malloc/free.  At most FQB_HOST_POOL_MB (default 4096) MB
// of free blocks stay cached; fqb_host_pool_trim() returns them all to the OS, and
// so does destroying the last handle.
#include <cuda_runtime.h>

#include <cstdlib>
#include <map>
#include <mutex>
#include <unordered_map>

#include "engine.hpp"

namespace farqb {
namespace {

struct Pool {
    std::mutex mu;
    std::multimap<size_t, void*> free_blocks;   // size -> block
    std::unordered_map<void*, size_t> live;     // pooled block -> size
    size_t cached = 0;
};
Pool& pool() {
    static Pool* p = new Pool();   // never destroyed: blocks may be freed during static teardown
    return *p;
}
size_t max_cached() {
    static const size_t cap = [] {
        const char* e = std::getenv("FQB_HOST_POOL_MB");
        const long long mb = e ? std::atoll(e) : 4096;
        return size_t(mb < 0 ? 0 : mb) << 20;
    }();
    return cap;
}

}  // namespace

void* host_alloc(size_t bytes) {
    bytes = std::max<size_t>(bytes, 64);
    Pool& p = pool();
    {
        std::lock_guard<std::mutex> lk(p.mu);
        auto it = p.free_blocks.lower_bound(bytes);
        if (it != p.free_blocks.end() && it->first <= 2 * bytes + (size_t(1) << 20)) {
            void* ptr = it->second;
            p.live[ptr] = it->first;
            p.cached -= it->first;
            p.free_blocks.erase(it);
            return ptr;
        }
    }
    void* ptr = nullptr;
    if (cudaMallocHost(&ptr, bytes) != cudaSuccess) {
        cudaGetLastError();
        return std::malloc(bytes);   // not pooled
    }
    std::lock_guard<std::mutex> lk(p.mu);
    p.live[ptr] = bytes;
    return ptr;
}

void host_free(void* ptr) {
    if (!ptr) return;
    Pool& p = pool();
    std::lock_guard<std::mutex> lk(p.mu);
    auto it = p.live.find(ptr);
    if (it == p.live.end()) {
        std::free(ptr);
        return;
    }
    const size_t bytes = it->second;
    p.live.erase(it);
    if (p.cached + bytes > max_cached()) {
        cudaFreeHost(ptr);
        return;
    }
    p.free_blocks.emplace(bytes, ptr);
    p.cached += bytes;
}

void host_release(void* ptr) {
    if (!ptr) return;
    Pool& p = pool();
    std::lock_guard<std::mutex> lk(p.mu);
    auto it = p.live.find(ptr);
    if (it == p.live.end()) {
        std::free(ptr);
        return;
    }
    p.live.erase(it);
    cudaFreeHost(ptr);
}

size_t host_pool_trim() {
    Pool& p = pool();
    std::lock_guard<std::mutex> lk(p.mu);
    size_t freed = 0;
    for (auto& kv : p.free_blocks) {
        cudaFreeHost(kv.second);
        freed += kv.first;
    }
    p.free_blocks.clear();
    p.cached = 0;
    return freed;
}

}  // namespace farqb
