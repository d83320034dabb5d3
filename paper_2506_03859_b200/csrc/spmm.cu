// spmm.cu -- gather products with a sparse test block.
//
//  launch_gather_spmm:  Y = A * S [- z]      (reference: sparse_dense_mul,
//      centered_product, /root/reference/proj/src/sketch.cpp:104-140).  Each
//      output column gathers the zeta columns of A that its nonzeros name.  A
//      warp owns 64 consecutive rows (one 16-byte load per lane per nonzero),
//      so every A column segment is read once, fully coalesced, and the
//      nonzeros are accumulated in CSC order with one fma each -- the same
//      operation sequence as the reference's axpy loop (kernels_avx2.cpp:
//      220-231), hence bitwise-identical output.
//  launch_gather_tmul:  T = Wt' * S [- shift * colsum(Wt)]  (reference:
//      dense_sparse_tmul + the centering in tmul_block, sketch.cpp:116-130,
//      driver.cpp:30-45); the deflation product B * Omega with Wt = B'.
#include <cstdint>

#include "kernels.hpp"

namespace farqb {
namespace {

constexpr int kRowsPerWarp = 64;
constexpr int kWarpsPerCta = 8;
constexpr int kUnroll = 8;

template <bool VEC2>
__global__ void __launch_bounds__(256) k_gather_spmm(const double* __restrict__ a, int64_t m,
                                                     int64_t lda, const int* __restrict__ col_ptr,
                                                     const int* __restrict__ row_idx,
                                                     const double* __restrict__ values,
                                                     const double* __restrict__ z,
                                                     double* __restrict__ c, int64_t ldc) {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int j = blockIdx.y;
    const int64_t r0 = (int64_t(blockIdx.x) * kWarpsPerCta + warp) * kRowsPerWarp + 2 * lane;
    if (r0 >= m) return;
    const bool two = r0 + 1 < m;
    const int beg = col_ptr[j], end = col_ptr[j + 1];
    double acc0 = 0.0, acc1 = 0.0;
    int idx = beg;
    for (; idx + kUnroll <= end; idx += kUnroll) {
        double2 av[kUnroll];
        double vv[kUnroll];
#pragma unroll
        for (int u = 0; u < kUnroll; ++u) {
            const double* col = a + int64_t(row_idx[idx + u]) * lda + r0;
            vv[u] = values[idx + u];
            if (VEC2 && two) {
                av[u] = __ldg(reinterpret_cast<const double2*>(col));
            } else {
                av[u].x = __ldg(col);
                av[u].y = two ? __ldg(col + 1) : 0.0;
            }
        }
#pragma unroll
        for (int u = 0; u < kUnroll; ++u) {
            acc0 = fma(vv[u], av[u].x, acc0);
            acc1 = fma(vv[u], av[u].y, acc1);
        }
    }
    for (; idx < end; ++idx) {
        const double* col = a + int64_t(row_idx[idx]) * lda + r0;
        const double v = values[idx];
        acc0 = fma(v, __ldg(col), acc0);
        if (two) acc1 = fma(v, __ldg(col + 1), acc1);
    }
    if (z) {
        acc0 -= z[r0];
        if (two) acc1 -= z[r0 + 1];
    }
    double* out = c + int64_t(j) * ldc + r0;
    if (VEC2 && two) {
        *reinterpret_cast<double2*>(out) = make_double2(acc0, acc1);
    } else {
        out[0] = acc0;
        if (two) out[1] = acc1;
    }
}

// T[i, j] = sum_{idx in col j} v * Wt[r_idx, i]  (- shift * colsum[i])
__global__ void __launch_bounds__(256) k_gather_tmul(const double* __restrict__ wt, int64_t ldw, int k,
                                                     const int* __restrict__ col_ptr,
                                                     const int* __restrict__ row_idx,
                                                     const double* __restrict__ values,
                                                     const double* __restrict__ colsum, double shift,
                                                     double* __restrict__ t, int64_t ldt) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    const int j = blockIdx.y;
    if (i >= k) return;
    const double* col = wt + int64_t(i) * ldw;
    double acc = 0.0;
    for (int idx = col_ptr[j]; idx < col_ptr[j + 1]; ++idx)
        acc = fma(values[idx], __ldg(col + row_idx[idx]), acc);
    if (colsum) acc -= shift * colsum[i];
    t[int64_t(j) * ldt + i] = acc;
}

}  // namespace

void launch_gather_spmm(const double* a, int64_t m, int64_t lda, const int* col_ptr,
                        const int* row_idx, const double* values, int l, const double* z,
                        double* c, int64_t ldc, cudaStream_t s, LaunchCounter& lc) {
    if (m <= 0 || l <= 0) return;
    const bool vec2 = (lda % 2 == 0) && (ldc % 2 == 0) && (reinterpret_cast<uintptr_t>(a) % 16 == 0) &&
                      (reinterpret_cast<uintptr_t>(c) % 16 == 0);
    dim3 grid(unsigned(ceil_div(m, int64_t(kRowsPerWarp) * kWarpsPerCta)), unsigned(l));
    if (vec2)
        k_gather_spmm<true><<<grid, 256, 0, s>>>(a, m, lda, col_ptr, row_idx, values, z, c, ldc);
    else
        k_gather_spmm<false><<<grid, 256, 0, s>>>(a, m, lda, col_ptr, row_idx, values, z, c, ldc);
    FQB_LAUNCHED();
    lc.bump();
}

void launch_gather_tmul(const double* wt, int64_t n, int64_t ldw, int k, const int* col_ptr,
                        const int* row_idx, const double* values, int l, const double* colsum,
                        double shift, double* t, int64_t ldt, cudaStream_t s, LaunchCounter& lc) {
    (void)n;
    if (k <= 0 || l <= 0) return;
    dim3 grid(unsigned(ceil_div(k, 256)), unsigned(l));
    k_gather_tmul<<<grid, 256, 0, s>>>(wt, ldw, k, col_ptr, row_idx, values, colsum, shift, t, ldt);
    FQB_LAUNCHED();
    lc.bump();
}

}  // namespace farqb
