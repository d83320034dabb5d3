// common.cuh -- shared helpers for the farqb sm_100a kernels and host engine.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <stdexcept>
#include <string>

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

// Per-handle launch accounting: every kernel the engine enqueues bumps this.
struct LaunchCounter {
    int64_t total = 0;
    void bump(int n = 1) { total += n; }
};

}  // namespace farqb
