// reduce.cu -- deterministic reductions over A and the B blocks.
//
//  launch_sumsq       ||A||_F^2 (reference frob_norm_sq, matrix_core.cpp:46-48):
//                     fixed grid, per-CTA tree sums, then one fixed-order pass.
//  launch_centering   z = A (p 1_n) (reference centering_column, driver.cpp:
//                     178-183): one thread per row, columns in order with one
//                     fma each -- the reference's axpy sequence, so z (and the
//                     centered sketch Y = A S - z) match it bit for bit.
//  launch_colsum      column sums of B' for the centered deflation term.
#include <algorithm>
#include <cstdint>
#include <type_traits>

#include "kernels.hpp"

namespace farqb {
namespace {

// rows per segment: long segments for A (streaming), short ones for the n x b
// blocks so their few segments still spread over many CTAs.  A function of the
// shape only, so the summation order (and result) is reproducible.
__host__ __device__ __forceinline__ int64_t seg_rows(int64_t m, int64_t n) { return m * n >= (int64_t(1) << 26) ? 4096 : 512; }

__device__ __forceinline__ double block_sum(double v, double* sh) {
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) v += __shfl_down_sync(0xffffffffu, v, off);
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if (lane == 0) sh[warp] = v;
    __syncthreads();
    const int nw = blockDim.x >> 5;
    v = threadIdx.x < nw ? sh[threadIdx.x] : 0.0;
    if (warp == 0) {
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) v += __shfl_down_sync(0xffffffffu, v, off);
    }
    return v;  // valid in thread 0
}

template <typename T>   // double, or float A (FP32 input mode; squares summed in FP64)
__global__ void __launch_bounds__(256) k_sumsq_partial(const T* __restrict__ a, int64_t m,
                                                       int64_t n, int64_t lda, double* partial) {
    FQB_PDL_ENTRY();
    __shared__ double sh[32];
    const int64_t seg = seg_rows(m, n);
    const int64_t segs_per_col = (m + seg - 1) / seg;
    const int64_t total = segs_per_col * n;
    // four independent loads / accumulators per thread step (memory-level
    // parallelism), combined in a fixed order: deterministic for a given shape
    double acc[4] = {0.0, 0.0, 0.0, 0.0};
    const int bd = blockDim.x;
    for (int64_t sgi = blockIdx.x; sgi < total; sgi += gridDim.x) {
        const int64_t col = sgi / segs_per_col;
        const int64_t r0 = (sgi - col * segs_per_col) * seg;
        const int64_t r1 = r0 + seg < m ? r0 + seg : m;
        const T* c = a + col * lda;
        int64_t r = r0 + threadIdx.x;
        for (; r + 3 * bd < r1; r += 4 * bd) {
            double v[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) v[u] = double(__ldcs(c + r + u * bd));   // streaming: read once
#pragma unroll
            for (int u = 0; u < 4; ++u) acc[u] = fma(v[u], v[u], acc[u]);
        }
        for (; r < r1; r += bd) {
            const double v = double(__ldg(c + r));
            acc[0] = fma(v, v, acc[0]);
        }
    }
    const double s = block_sum((acc[0] + acc[1]) + (acc[2] + acc[3]), sh);
    if (threadIdx.x == 0) partial[blockIdx.x] = s;
}

// Contiguous A (lda == m): the m*n values as one array, CTA c sums the fixed chunk
// [c*len/P, (c+1)*len/P) with 16-byte loads -- deterministic for a given shape.
template <typename T>
__global__ void __launch_bounds__(256) k_sumsq_flat(const T* __restrict__ a, int64_t len, double* partial) {
    FQB_PDL_ENTRY();
    __shared__ double sh[32];
    const int64_t c0 = len * blockIdx.x / gridDim.x, c1 = len * (blockIdx.x + 1) / gridDim.x;
    double acc[4] = {0.0, 0.0, 0.0, 0.0};
    constexpr int VEC = 16 / sizeof(T);   // elements per 16-byte load
    // head up to 16-byte alignment, then vector body, then tail
    int64_t i = c0;
    const int64_t mis = (reinterpret_cast<uintptr_t>(a + c0) & 15) / sizeof(T);
    const int64_t head = mis ? std::min<int64_t>(c1 - c0, VEC - mis) : 0;
    if (threadIdx.x < head) {
        const double v = double(a[c0 + threadIdx.x]);
        acc[0] = fma(v, v, acc[0]);
    }
    i = c0 + head;
    const int64_t nvec = (c1 - i) / VEC;
    const T* base = a + i;
    using V = typename std::conditional<sizeof(T) == 8, double2, float4>::type;
    const V* vb = reinterpret_cast<const V*>(base);
    auto sq = [](const V& v) -> double {
        if constexpr (sizeof(T) == 8) {
            return fma(v.x, v.x, v.y * v.y);
        } else {
            double s2 = fma(double(v.x), double(v.x), double(v.y) * double(v.y));
            s2 = fma(double(v.z), double(v.z), s2);
            return fma(double(v.w), double(v.w), s2);
        }
    };
    const int64_t bd = blockDim.x;
    int64_t k = threadIdx.x;
    for (; k + 3 * bd < nvec; k += 4 * bd) {   // four 16-byte loads in flight per thread
        V v[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) v[u] = __ldcs(vb + k + u * bd);
#pragma unroll
        for (int u = 0; u < 4; ++u) acc[u] += sq(v[u]);
    }
    for (; k < nvec; k += bd) acc[0] += sq(__ldcs(vb + k));
    for (int64_t k = i + nvec * VEC + threadIdx.x; k < c1; k += blockDim.x) {
        const double v = double(a[k]);
        acc[1] = fma(v, v, acc[1]);
    }
    const double s = block_sum((acc[0] + acc[1]) + (acc[2] + acc[3]), sh);
    if (threadIdx.x == 0) partial[blockIdx.x] = s;
}

__global__ void k_sum_partials(const double* partial, int count, double* out) {
    FQB_PDL_ENTRY();
    __shared__ double sh[32];
    double acc = 0.0;
    for (int i = threadIdx.x; i < count; i += blockDim.x) acc += partial[i];
    const double s = block_sum(acc, sh);
    if (threadIdx.x == 0) *out = s;
}

template <typename T>
__global__ void __launch_bounds__(128) k_centering(const T* __restrict__ a, int64_t m, int64_t n,
                                                   int64_t lda, double p, double* __restrict__ z) {
    FQB_PDL_ENTRY();
    const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= m) return;
    const T* r = a + i;
    double acc = 0.0;
    int64_t c = 0;
    for (; c + 8 <= n; c += 8) {
        double v[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) v[u] = double(__ldg(r + (c + u) * lda));
#pragma unroll
        for (int u = 0; u < 8; ++u) acc = fma(p, v[u], acc);
    }
    for (; c < n; ++c) acc = fma(p, double(__ldg(r + c * lda)), acc);
    z[i] = acc;
}

__global__ void __launch_bounds__(256) k_colsum(const double* __restrict__ x, int64_t rows,
                                                int64_t ld, double* colsum) {
    FQB_PDL_ENTRY();
    __shared__ double sh[32];
    const double* c = x + int64_t(blockIdx.x) * ld;
    double acc = 0.0;
    for (int64_t r = threadIdx.x; r < rows; r += blockDim.x) acc += c[r];
    const double s = block_sum(acc, sh);
    if (threadIdx.x == 0) colsum[blockIdx.x] = s;
}

}  // namespace

template <typename T>
static void sumsq_impl(const T* a, int64_t m, int64_t n, int64_t lda, double* partial, double* out, cudaStream_t s,
                       LaunchCounter& lc) {
    if (lda == m && m * n >= (int64_t(1) << 22))   // big contiguous A: 16-byte streaming loads (C2: 141 -> 84 us)
        launch_k(k_sumsq_flat<T>, kReducePartials, 256, 0, s, a, m * n, partial);
    else launch_k(k_sumsq_partial<T>, kReducePartials, 256, 0, s, a, m, n, lda, partial);
    FQB_LAUNCHED();
    launch_k(k_sum_partials, 1, 1024, 0, s, partial, kReducePartials, out);
    FQB_LAUNCHED();
    lc.bump(2);
}
void launch_sumsq(const double* a, int64_t m, int64_t n, int64_t lda, double* partial, double* out,
                  cudaStream_t s, LaunchCounter& lc) {
    sumsq_impl(a, m, n, lda, partial, out, s, lc);
}
void launch_sumsq(const float* a, int64_t m, int64_t n, int64_t lda, double* partial, double* out,
                  cudaStream_t s, LaunchCounter& lc) {
    sumsq_impl(a, m, n, lda, partial, out, s, lc);
}

template <typename T>
static void centering_impl(const T* a, int64_t m, int64_t n, int64_t lda, double p, double* z, cudaStream_t s,
                           LaunchCounter& lc) {
    launch_k(k_centering<T>, unsigned(ceil_div(m, 128)), 128, 0, s, a, m, n, lda, p, z);
    FQB_LAUNCHED();
    lc.bump();
}
void launch_centering(const double* a, int64_t m, int64_t n, int64_t lda, double p, double* z,
                      cudaStream_t s, LaunchCounter& lc) {
    centering_impl(a, m, n, lda, p, z, s, lc);
}
void launch_centering(const float* a, int64_t m, int64_t n, int64_t lda, double p, double* z,
                      cudaStream_t s, LaunchCounter& lc) {
    centering_impl(a, m, n, lda, p, z, s, lc);
}

// FP32 A -> FP64 copy (FP32 input mode when the A passes run on DMMA)
__global__ void k_widen(const float* __restrict__ a, int64_t m, int64_t lda, double* __restrict__ out,
                        int64_t ldo) {
    FQB_PDL_ENTRY();
    const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    const int64_t c = blockIdx.y;
    if (i < m) out[c * ldo + i] = double(a[c * lda + i]);
}
void launch_widen(const float* a, int64_t m, int64_t n, int64_t lda, double* out, int64_t ldo, cudaStream_t s,
                  LaunchCounter& lc) {
    if (m <= 0 || n <= 0) return;
    for (int64_t c0 = 0; c0 < n; c0 += 65535) {
        const int64_t cols = std::min<int64_t>(65535, n - c0);
        launch_k(k_widen, dim3(unsigned(ceil_div(m, 256)), unsigned(cols)), 256, 0, s, a + c0 * lda, m, lda, out + c0 * ldo,
                                                                                ldo);
        FQB_LAUNCHED();
        lc.bump();
    }
}

void launch_colsum(const double* x, int64_t rows, int k, int64_t ld, double* colsum, cudaStream_t s,
                   LaunchCounter& lc) {
    if (k <= 0) return;
    launch_k(k_colsum, unsigned(k), 256, 0, s, x, rows, ld, colsum);
    FQB_LAUNCHED();
    lc.bump();
}

void launch_sumsq_small(const double* x, int64_t rows, int64_t cols, int64_t ld, double* partial,
                        double* out, cudaStream_t s, LaunchCounter& lc) {
    launch_sumsq(x, rows, cols, ld, partial, out, s, lc);
}

}  // namespace farqb
