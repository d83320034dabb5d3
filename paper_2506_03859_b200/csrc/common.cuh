// common.cuh -- shared helpers for the farqb sm_100a kernels and host engine.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

namespace farqb {

// Thrown inside the library, converted to fqb_status at the C-ABI (capi.cpp).
struct Error : std::runtime_error {
    int status;
    Error(int s, const std::string& msg) : std::runtime_error(msg), status(s) {}
};

constexpr int kStatusConfig = 1;
constexpr int kStatusDimension = 2;
constexpr int kStatusDegenerate = 3;
constexpr int kStatusTolerance = 4;
constexpr int kStatusCuda = 5;
constexpr int kStatusNccl = 6;
constexpr int kStatusInvalid = 7;
constexpr int kStatusConvergence = 8;
constexpr int kStatusCallback = 9;
constexpr int kStatusAlloc = 10;
constexpr int kStatusFormat = 11;

inline void cuda_check(cudaError_t e, const char* what) {
    if (e != cudaSuccess)
        throw Error(e == cudaErrorMemoryAllocation ? kStatusAlloc : kStatusCuda,
                    std::string(what) + ": " + cudaGetErrorString(e));
}

#define FQB_CUDA(call) ::farqb::cuda_check((call), #call)
#define FQB_LAUNCHED(ctx) ::farqb::cuda_check(cudaGetLastError(), "kernel launch")

inline int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }
inline int64_t round_up(int64_t a, int64_t b) { return ceil_div(a, b) * b; }

constexpr int kNumSMs = 148;  // B200; the engine queries the device and uses the real count

// Programmatic dependent launch (PDL).  Every kernel starts with FQB_PDL_ENTRY():
// it lets the next kernel in the stream begin launching (its CTAs become resident
// as soon as all of ours have started) and then waits until the previous kernel
// has completed and its writes are visible -- so reading inputs after the entry
// is exactly as safe as with plain stream order, and the ~2-3 us launch gap
// between the many short kernels of a block is overlapped.  FQB_PDL=0 turns the
// launch attribute off (the instructions are then no-ops).
#define FQB_PDL_ENTRY()                                                                      \
    do {                                                                                     \
        if (FQB_PDL_EARLY) asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory"); \
        asm volatile("griddepcontrol.wait;\n" ::: "memory");                                 \
    } while (0)
#ifndef FQB_PDL_EARLY
#define FQB_PDL_EARLY 0
#endif

bool pdl_enabled();

// kernel<<<grid, block, smem, stream>>>(args...) with the PDL launch attribute
template <typename... KArgs, typename... Args>
inline void launch_k(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t stream,
                     Args&&... args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = stream;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = pdl_enabled() ? 1 : 0;
    cuda_check(cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...), "kernel launch");
}

// Per-handle launch accounting: every kernel the engine enqueues bumps this.
struct LaunchCounter {
    int64_t total = 0;
    void bump(int n = 1) { total += n; }
};

// CUDA-event brackets around the A-pass products (k_ozaki + its fixup) of a handle's
// runs, read back by fqb_pass_timing: the dominant kernel timed live inside a caller's
// timed region, on the stream it runs on (ozaki.cu records, engine.cu arms it)
struct LaunchTimer {
    bool on = false;
    std::vector<cudaEvent_t> ev;   // pairs
    size_t used = 0;               // events recorded since the last reset
    double bytes = 0.0;            // algorithmic FP64 bytes 8 (MK + KN + MN) of the timed launches
};

}  // namespace farqb
