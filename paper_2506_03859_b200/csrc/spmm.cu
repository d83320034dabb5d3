// spmm.cu -- gather products with a sparse test block.
//
//  launch_gather_spmm:  Y = A * S [- z]      (reference: sparse_dense_mul,
//      centered_product, /root/reference/proj/src/sketch.cpp:104-140).  Each
//      output column gathers the zeta columns of A that its nonzeros name.  A
//      warp owns 64*VPL consecutive rows (VPL 16-byte loads per lane per
//      nonzero), so every A column segment is read once, fully coalesced, and the
//      nonzeros are accumulated in CSC order with one fma each -- the same
//      operation sequence as the reference's axpy loop (kernels_avx2.cpp:
//      220-231), hence bitwise-identical output.
//  launch_gather_tmul:  T = Wt' * S [- shift * colsum(Wt)]  (reference:
//      dense_sparse_tmul + the centering in tmul_block, sketch.cpp:116-130,
//      driver.cpp:30-45); the deflation product B * Omega with Wt = B'.
#include <algorithm>
#include <cstdint>
#include <cstdlib>

#include "kernels.hpp"

namespace farqb {
namespace {

constexpr int kWarpsPerCta = 8;
constexpr int kUnroll = 8;

template <typename T> struct Vec2;
template <> struct Vec2<double> { using type = double2; };
template <> struct Vec2<float> { using type = float2; };

// VPL 2-vectors per lane: a warp owns 64*VPL consecutive rows, so every gathered
// column of A is read as one contiguous run.  T = float is the FP32 input mode
// (values widened exactly, accumulation in FP64 as for double A).
template <typename T, bool VEC2, int VPL>
__global__ void __launch_bounds__(256) k_gather_spmm(const T* __restrict__ a, int64_t m,
                                                     int64_t lda, const int* __restrict__ col_ptr,
                                                     const int* __restrict__ row_idx,
                                                     const double* __restrict__ values,
                                                     const double* __restrict__ z,
                                                     double* __restrict__ c, int64_t ldc) {
    FQB_PDL_ENTRY();
    constexpr int ROWS = 64 * VPL;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int j = blockIdx.y;
    const int64_t base = (int64_t(blockIdx.x) * kWarpsPerCta + warp) * ROWS + 2 * lane;
    if (base >= m) return;
    const int beg = col_ptr[j], end = col_ptr[j + 1];
    double acc[VPL][2];
#pragma unroll
    for (int v = 0; v < VPL; ++v) acc[v][0] = acc[v][1] = 0.0;
    int idx = beg;
    constexpr int U = kUnroll / VPL > 0 ? kUnroll / VPL : 1;
    using V2 = typename Vec2<T>::type;
    for (; idx + U <= end; idx += U) {
        V2 av[U][VPL];
        double vv[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const T* col = a + int64_t(row_idx[idx + u]) * lda;
            vv[u] = values[idx + u];
#pragma unroll
            for (int v = 0; v < VPL; ++v) {
                const int64_t r = base + 64 * v;
                if (VEC2 && r + 1 < m) {
                    av[u][v] = __ldg(reinterpret_cast<const V2*>(col + r));
                } else {
                    av[u][v].x = r < m ? __ldg(col + r) : T(0);
                    av[u][v].y = r + 1 < m ? __ldg(col + r + 1) : T(0);
                }
            }
        }
#pragma unroll
        for (int u = 0; u < U; ++u)
#pragma unroll
            for (int v = 0; v < VPL; ++v) {
                acc[v][0] = fma(vv[u], double(av[u][v].x), acc[v][0]);
                acc[v][1] = fma(vv[u], double(av[u][v].y), acc[v][1]);
            }
    }
    for (; idx < end; ++idx) {
        const T* col = a + int64_t(row_idx[idx]) * lda;
        const double vv = values[idx];
#pragma unroll
        for (int v = 0; v < VPL; ++v) {
            const int64_t r = base + 64 * v;
            if (r < m) acc[v][0] = fma(vv, double(__ldg(col + r)), acc[v][0]);
            if (r + 1 < m) acc[v][1] = fma(vv, double(__ldg(col + r + 1)), acc[v][1]);
        }
    }
#pragma unroll
    for (int v = 0; v < VPL; ++v) {
        const int64_t r = base + 64 * v;
        if (r >= m) continue;
        double y0 = acc[v][0], y1 = acc[v][1];
        if (z) {
            y0 -= z[r];
            if (r + 1 < m) y1 -= z[r + 1];
        }
        double* out = c + int64_t(j) * ldc + r;
        if (VEC2 && r + 1 < m) {
            *reinterpret_cast<double2*>(out) = make_double2(y0, y1);
        } else {
            out[0] = y0;
            if (r + 1 < m) out[1] = y1;
        }
    }
}

// T[i, j] = sum_{idx in col j} v * Wt[r_idx, i]  (- shift * colsum[i])
__global__ void __launch_bounds__(256) k_gather_tmul(const double* __restrict__ wt, int64_t ldw, int k,
                                                     const int* __restrict__ col_ptr,
                                                     const int* __restrict__ row_idx,
                                                     const double* __restrict__ values,
                                                     const double* __restrict__ colsum, double shift,
                                                     double* __restrict__ t, int64_t ldt) {
    FQB_PDL_ENTRY();
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

template <typename T>
static void gather_spmm_impl(const T* a, int64_t m, int64_t lda, const int* col_ptr, const int* row_idx,
                             const double* values, int l, const double* z, double* c, int64_t ldc, cudaStream_t s,
                             LaunchCounter& lc) {
    if (m <= 0 || l <= 0) return;
    const bool vec2 = (lda % 2 == 0) && (ldc % 2 == 0) && (reinterpret_cast<uintptr_t>(a) % 16 == 0) &&
                      (reinterpret_cast<uintptr_t>(c) % 16 == 0);
    static int vpl_env = [] {
        const char* e = std::getenv("FQB_SPMM_VPL");
        return e ? std::atoi(e) : 0;
    }();
    // 1 KB runs per gathered column (VPL = 2) once that still leaves >= 4 CTAs per
    // SM; measured on the C3 sketch (20000^2, b = 64, zeta = 8): VPL 1/2/4 ->
    // 4376 / 4932 / 4816 GB/s (profiles/sketch_sweep_r01.txt)
    int vpl = vpl_env ? vpl_env : (ceil_div(m, 1024) * l >= 4 * 148 ? 2 : 1);
    if (vpl != 1 && vpl != 2 && vpl != 4) vpl = 1;
    dim3 grid(unsigned(ceil_div(m, int64_t(64 * vpl) * kWarpsPerCta)), unsigned(l));
    if (vec2) {
        if (vpl == 4) launch_k(k_gather_spmm<T, true, 4>, grid, 256, 0, s, a, m, lda, col_ptr, row_idx, values, z, c, ldc);
        else if (vpl == 2)
            launch_k(k_gather_spmm<T, true, 2>, grid, 256, 0, s, a, m, lda, col_ptr, row_idx, values, z, c, ldc);
        else launch_k(k_gather_spmm<T, true, 1>, grid, 256, 0, s, a, m, lda, col_ptr, row_idx, values, z, c, ldc);
    } else {
        launch_k(k_gather_spmm<T, false, 1>, grid, 256, 0, s, a, m, lda, col_ptr, row_idx, values, z, c, ldc);
    }
    FQB_LAUNCHED();
    lc.bump();
}

void launch_gather_spmm(const double* a, int64_t m, int64_t lda, const int* col_ptr, const int* row_idx,
                        const double* values, int l, const double* z, double* c, int64_t ldc, cudaStream_t s,
                        LaunchCounter& lc) {
    gather_spmm_impl(a, m, lda, col_ptr, row_idx, values, l, z, c, ldc, s, lc);
}
void launch_gather_spmm(const float* a, int64_t m, int64_t lda, const int* col_ptr, const int* row_idx,
                        const double* values, int l, const double* z, double* c, int64_t ldc, cudaStream_t s,
                        LaunchCounter& lc) {
    gather_spmm_impl(a, m, lda, col_ptr, row_idx, values, l, z, c, ldc, s, lc);
}

void launch_gather_tmul(const double* wt, int64_t n, int64_t ldw, int k, const int* col_ptr,
                        const int* row_idx, const double* values, int l, const double* colsum,
                        double shift, double* t, int64_t ldt, cudaStream_t s, LaunchCounter& lc) {
    (void)n;
    if (k <= 0 || l <= 0) return;
    dim3 grid(unsigned(ceil_div(k, 256)), unsigned(l));
    launch_k(k_gather_tmul, grid, 256, 0, s, wt, ldw, k, col_ptr, row_idx, values, colsum, shift, t, ldt);
    FQB_LAUNCHED();
    lc.bump();
}

}  // namespace farqb
