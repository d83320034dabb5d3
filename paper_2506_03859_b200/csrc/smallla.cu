// smallla.cu -- b x b dense linear algebra, one CTA per factorization.
//
//  launch_chol_upper_inv: Cholesky of an SPD Gram block with the reference's
//      relative pivot floor (matrix_core.cpp:117-140; the bordered diag_ref of
//      driver.cpp:270-275), returning both the upper factor R = L' and R^{-1}
//      for the CholeskyQR steps.  Implemented as symmetric Gaussian elimination
//      carried out on an identity augment stored in place: after step j the
//      trailing block holds the Schur complement (so pivot j is exactly the
//      reference's l(j,j)^2), the strictly lower part holds the unit-lower M with
//      M S = U, and
//          R = D^{-1/2} U,   R^{-1} = M' D^{-1/2},   D = diag(U).
//  launch_sym_eig: cyclic-by-rounds (round-robin) Jacobi with the reference's
//      thresholds (matrix_core.cpp:50-115): 1e-14 ||S||_F stop, 30 sweeps,
//      ascending output.  Disjoint rotations of a round are applied in parallel.
//  launch_eigsvd_scale: eigSVD tail (matrix_core.cpp:193-215).
#include <cstdint>
#include <cstdlib>
#include <utility>

#include "kernels.hpp"

namespace farqb {
namespace {

constexpr int kCholThreads = 1024;
constexpr int kSmemMaxB = 128;

__device__ __forceinline__ double block_reduce_max(double v, double* sh) {
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) v = fmax(v, __shfl_down_sync(0xffffffffu, v, off));
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    __syncthreads();
    if (lane == 0) sh[warp] = v;
    __syncthreads();
    if (threadIdx.x == 0) {
        double m = sh[0];
        for (int w = 1; w < int(blockDim.x >> 5); ++w) m = fmax(m, sh[w]);
        sh[0] = m;
    }
    __syncthreads();
    const double r = sh[0];
    __syncthreads();
    return r;
}

__device__ __forceinline__ double block_reduce_sum(double v, double* sh) {
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) v += __shfl_down_sync(0xffffffffu, v, off);
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    __syncthreads();
    if (lane == 0) sh[warp] = v;
    __syncthreads();
    if (threadIdx.x == 0) {
        double m = 0.0;
        for (int w = 0; w < int(blockDim.x >> 5); ++w) m += sh[w];
        sh[0] = m;
    }
    __syncthreads();
    const double r = sh[0];
    __syncthreads();
    return r;
}

// M is b x b row-major with pitch ld (shared memory for b <= 128, else global
// scratch).  Warp w eliminates rows i = j+1+w, j+1+w+nwarps, ... of step j, lanes
// sweep the columns, so a step needs a single __syncthreads (row j+1 must be
// final before it becomes the next pivot row).
__global__ void __launch_bounds__(1024) k_chol_inv(const double* __restrict__ S, int b, int64_t lds,
                                                   double tol, double diag_ref,
                                                   const double* __restrict__ dref_extra,
                                                   int64_t ld_extra, double* __restrict__ R,
                                                   double* __restrict__ Rinv,
                                                   double* __restrict__ max_diag_out,
                                                   unsigned* status, unsigned fail_bit,
                                                   double* gscratch) {
    FQB_PDL_ENTRY();
    extern __shared__ double smem[];
    __shared__ double red[32];
    __shared__ double sd[1024];
    const int ld = b + 1;
    double* M = b <= kSmemMaxB ? smem : gscratch;
    const int tid = threadIdx.x, nt = blockDim.x;
    const int warp = tid >> 5, lane = tid & 31, nwarps = nt >> 5;
    for (int e = tid; e < b * b; e += nt) {
        const int c = e / b, i = e - c * b;
        M[i * ld + c] = S[int64_t(c) * lds + i];
    }
    // pivot reference (matrix_core.cpp:121-123, driver.cpp:270-275)
    double local = 0.0;
    if (dref_extra) {
        for (int i = tid; i < b; i += nt) local = fmax(local, dref_extra[int64_t(i) * ld_extra + i]);
    } else if (!(diag_ref > 0.0)) {
        for (int i = tid; i < b; i += nt) local = fmax(local, S[int64_t(i) * lds + i]);
    }
    double max_diag = block_reduce_max(local, red);  // contains __syncthreads
    if (dref_extra) max_diag = fmax(max_diag, diag_ref);
    else if (diag_ref > 0.0) max_diag = diag_ref;
    const double thresh = tol * max_diag;
    if (tid == 0 && max_diag_out) *max_diag_out = max_diag;

    bool failed = false;
    for (int j = 0; j < b; ++j) {
        __syncthreads();
        const double d = M[j * ld + j];
        if (!(d > thresh)) {  // uniform: every thread reads the same pivot
            failed = true;
            break;
        }
        const double invd = 1.0 / d;
        const double* pivot_row = M + j * ld;
        for (int i = j + 1 + warp; i < b; i += nwarps) {
            double* row = M + i * ld;
            const double f = row[j] * invd;
            __syncwarp();
            for (int c = lane; c < b; c += 32) row[c] = c == j ? -f : fma(-f, pivot_row[c], row[c]);
        }
    }
    __syncthreads();
    if (failed) {
        if (tid == 0) atomicOr(status, fail_bit);
        for (int e = tid; e < b * b; e += nt) {
            const int r = e % b, c = e / b;
            R[e] = r == c ? 1.0 : 0.0;
            Rinv[e] = r == c ? 1.0 : 0.0;
        }
        return;
    }
    for (int i = tid; i < b; i += nt) sd[i] = sqrt(M[i * ld + i]);
    __syncthreads();
    // R[r, c] = U[r][c] / sqrt(d_r) (c >= r);  Rinv[k, j] = M[j][k] / sqrt(d_j) (k < j)
    for (int e = tid; e < b * b; e += nt) {
        const int r = e % b, c = e / b;
        R[e] = c >= r ? M[r * ld + c] / sd[r] : 0.0;
        Rinv[e] = r < c ? M[c * ld + r] / sd[c] : (r == c ? 1.0 / sd[c] : 0.0);
    }
}

// Register-resident variant for b <= 128: thread t owns column c = t % b and
// rows rg, rg + 8, rg + 16, ... (rg = t / b), held in registers (slot s = row
// rg + 8 s).  At step j the owners of row j publish it to shared memory (by
// symmetry of the trailing Schur complement it is also pivot column j), one
// barrier, then every thread updates its rows: M[i][c] -= (M[j][i] / d) M[j][c]
// (c != j), M[i][j] = -f.  The published rows are double buffered, so a step
// costs one barrier.
//
// Steps run in groups of 8 (j = 8Q .. 8Q+7) instantiated per Q: in group Q the
// pivot row lives in slot Q and every slot below Q is finished, so the slot range
// is a compile-time constant -- no per-slot predicates, no jump table for the
// publication, the loads of a step issued together -- and the pivot column's
// "store -f" is folded into the FMA (v keep + (-f) pc with keep = 0, pc = 1
// there).  b = 50: 34.8 -> 18.3 us per call, b = 100: 125 -> 86 us
// (tools/microbench/chol_bench.cu); a two-columns-per-thread form was slower.  Since
// then two pivots per barrier (below).
// Two pivots per barrier: the owners of rows j and j + 1 publish both (row j + 1 as it
// is before step j), and every thread forms row j + 1 after step j itself,
//     f = M[j+1][j] / d_j,  M'[j+1][c] = M[j+1][c] - f M[j][c]  (-f at c = j),
//     d_{j+1} = M'[j+1][j+1],
// then applies steps j and j + 1 to its rows i > j + 1 (M[i][j] = M[j][i] and
// M'[i][j+1] = M'[j+1][i] by the symmetry of the trailing Schur complements), and the
// owner of row j + 1 stores M'[j+1][*].  The same pivots and the same pivot floor as one
// step at a time; the published rows are double buffered per pair: a barrier per two
// columns.
template <int MAXS, int Q>
__device__ __forceinline__ bool chol_group(double (&v)[MAXS], int b, double thresh, int rg, int c, bool active,
                                           double (*prow)[kSmemMaxB]) {
#pragma unroll 1
    for (int r = 0; r < 8; r += 2) {
        const int j = 8 * Q + r;
        if (j >= b) return true;
        const bool two = j + 1 < b;
        double* p0 = prow[((j >> 1) & 1) * 2];
        double* p1 = prow[((j >> 1) & 1) * 2 + 1];
        if (active && rg == r) p0[c] = v[Q];
        if (two && active && rg == r + 1) p1[c] = v[Q];
#ifdef FQB_CHOL_PROBE
        if (threadIdx.x == FQB_CHOL_PROBE) chol_probe_stamp(2 * j);
#endif
        __syncthreads();
#ifdef FQB_CHOL_PROBE
        if (threadIdx.x == FQB_CHOL_PROBE) chol_probe_stamp(2 * j + 1);
#endif
        const double d0 = p0[j];
        if (!(d0 > thresh)) return false;   // uniform: every thread reads the same pivot
        const double inv0 = 1.0 / d0;
        const double p0c = p0[c];
        if (!two) {   // the last column of an odd b: one step
            const bool piv = c == j;
            const double pc = piv ? 1.0 : p0c;
            const double keep = piv ? 0.0 : 1.0;
#pragma unroll
            for (int s = Q; s < MAXS; ++s) {
                const double nv = fma(-(p0[min(rg + 8 * s, b - 1)] * inv0), pc, v[s] * keep);
                if (s == Q) v[s] = rg > r ? nv : v[s];
                else v[s] = nv;
            }
            return true;
        }
        const double f1 = p1[j] * inv0;
        const double d1 = fma(-f1, p0[j + 1], p1[j + 1]);
        if (!(d1 > thresh)) return false;
        const double inv1 = 1.0 / d1;
        const double p1c = c == j ? -f1 : fma(-f1, p0c, p1[c]);   // row j + 1 after step j, column c
#pragma unroll
        for (int s = Q; s < MAXS; ++s) {
            const int i = min(rg + 8 * s, b - 1);
            const double a0 = p0[i], a1 = p1[i];
            const double g0 = a0 * inv0;
            const double g1 = fma(-f1, a0, a1) * inv1;
            double x = c == j ? -g0 : fma(-g0, p0c, v[s]);
            x = c == j + 1 ? -g1 : fma(-g1, p1c, x);
            // slots past row b - 1 collect garbage that is never published or stored
            if (s == Q) v[s] = rg > r + 1 ? x : (rg == r + 1 ? p1c : v[s]);
            else v[s] = x;
        }
    }
    return true;
}

template <int MAXS, int... Qs>
__device__ __forceinline__ bool chol_groups(double (&v)[MAXS], int b, double thresh, int rg, int c, bool active,
                                            double (*prow)[kSmemMaxB], std::integer_sequence<int, Qs...>) {
    return (chol_group<MAXS, Qs>(v, b, thresh, rg, c, active, prow) && ...);
}

template <int MAXS>
__global__ void __launch_bounds__(1024) k_chol_inv_reg(const double* __restrict__ S, int b, int64_t lds,
                                                       double tol, double diag_ref,
                                                       const double* __restrict__ dref_extra, int64_t ld_extra,
                                                       double* __restrict__ R, double* __restrict__ Rinv,
                                                       double* __restrict__ max_diag_out, unsigned* status,
                                                       unsigned fail_bit) {
    FQB_PDL_ENTRY();
    extern __shared__ double smem[];        // final M, b x (b+1), row-major
    __shared__ double prow[4][kSmemMaxB];
    __shared__ double red[32];
    __shared__ double isd[kSmemMaxB];
    constexpr int RG = 8;
    const int tid = threadIdx.x, nt = blockDim.x;
    const int c = tid % b, rg = tid / b;
    const bool active = tid < RG * b;
    double v[MAXS];
#pragma unroll
    for (int s = 0; s < MAXS; ++s) {
        const int i = rg + s * RG;
        v[s] = (active && i < b) ? S[int64_t(c) * lds + i] : 0.0;   // M[i][c] = S[i][c]
    }
    double local = 0.0;
    if (dref_extra) {
        for (int i = tid; i < b; i += nt) local = fmax(local, dref_extra[int64_t(i) * ld_extra + i]);
    } else if (!(diag_ref > 0.0)) {
        for (int i = tid; i < b; i += nt) local = fmax(local, S[int64_t(i) * lds + i]);
    }
    double max_diag = block_reduce_max(local, red);
    if (dref_extra) max_diag = fmax(max_diag, diag_ref);
    else if (diag_ref > 0.0) max_diag = diag_ref;
    const double thresh = tol * max_diag;
    if (tid == 0 && max_diag_out) *max_diag_out = max_diag;

    const bool ok = chol_groups<MAXS>(v, b, thresh, rg, c, active, prow, std::make_integer_sequence<int, MAXS>{});
    if (!ok) {
        if (tid == 0) atomicOr(status, fail_bit);
        for (int e = tid; e < b * b; e += nt) {
            const int r = e % b, cc = e / b;
            R[e] = r == cc ? 1.0 : 0.0;
            Rinv[e] = r == cc ? 1.0 : 0.0;
        }
        return;
    }
    const int ld = b + 1;
    if (active) {
#pragma unroll
        for (int s = 0; s < MAXS; ++s) {
            const int i = rg + s * RG;
            if (i < b) smem[i * ld + c] = v[s];
        }
    }
    __syncthreads();
    for (int i = tid; i < b; i += nt) isd[i] = 1.0 / sqrt(smem[i * ld + i]);
    __syncthreads();
    // R[r, c] = U[r][c] / sqrt(d_r) (c >= r);  Rinv[k, j] = M[j][k] / sqrt(d_j) (k < j)
    for (int e = tid; e < b * b; e += nt) {
        const int cc = e / b, r = e - cc * b;
        R[e] = cc >= r ? smem[r * ld + cc] * isd[r] : 0.0;
        Rinv[e] = r < cc ? smem[cc * ld + r] * isd[cc] : (r == cc ? isd[cc] : 0.0);
    }
}

// Round-robin Jacobi; A in smem (b <= 128) row-major pitch b+1; V global col-major ld b.
__global__ void __launch_bounds__(1024) k_sym_eig(const double* __restrict__ S, int b, int64_t lds,
                                                  double* __restrict__ values,
                                                  double* __restrict__ vectors, double* __restrict__ vtmp,
                                                  unsigned* status, unsigned fail_bit) {
    FQB_PDL_ENTRY();
    extern __shared__ double A[];
    __shared__ double cs[64], sn[64];
    __shared__ int pp[64], qq[64];
    __shared__ double red[32];
    __shared__ double diag[128];
    const int ld = b + 1, tid = threadIdx.x, nt = blockDim.x;
    double* V = vtmp;
    for (int e = tid; e < b * b; e += nt) {
        const int i = e / b, c = e - i * b;
        A[i * ld + c] = S[int64_t(c) * lds + i];
        if (V) V[e] = (e % b) == (e / b) ? 1.0 : 0.0;
    }
    __syncthreads();
    double loc = 0.0;
    for (int e = tid; e < b * b; e += nt) {
        const double v = A[(e / b) * ld + e % b];
        loc = fma(v, v, loc);
    }
    const double fro = sqrt(block_reduce_sum(loc, red));
    const double stop = 1e-14 * fro;
    const double skip = stop / (double(b) * b);
    const int np = (b + 1) & ~1;  // players incl. a dummy when b is odd
    const int pairs = np / 2;
    int sweep = 0;
    bool converged = b <= 1;
    for (; sweep < 30 && !converged; ++sweep) {
        double off = 0.0;
        for (int e = tid; e < b * b; e += nt) {
            const int i = e / b, c = e % b;
            if (c > i) off = fma(A[i * ld + c], A[i * ld + c], off);
        }
        if (sqrt(2.0 * block_reduce_sum(off, red)) <= stop) {
            converged = true;
            break;
        }
        for (int r = 0; r < np - 1; ++r) {
            if (tid < pairs) {
                const int k = tid;
                int p, q;
                if (k == 0) {
                    p = r;
                    q = np - 1;
                } else {
                    p = (r + k) % (np - 1);
                    q = (r - k + (np - 1)) % (np - 1);
                }
                if (p > q) { const int x = p; p = q; q = x; }
                double c = 1.0, s = 0.0;
                if (q < b) {
                    const double apq = A[p * ld + q];
                    if (fabs(apq) > skip) {
                        const double app = A[p * ld + p], aqq = A[q * ld + q];
                        const double tau = (aqq - app) / (2.0 * apq);
                        const double t = (tau >= 0.0 ? 1.0 : -1.0) / (fabs(tau) + sqrt(1.0 + tau * tau));
                        c = 1.0 / sqrt(1.0 + t * t);
                        s = t * c;
                    } else {
                        q = b;  // no rotation
                    }
                }
                pp[k] = p;
                qq[k] = q;
                cs[k] = c;
                sn[k] = s;
            }
            __syncthreads();
            // columns: A <- A J
            for (int e = tid; e < pairs * b; e += nt) {
                const int k = e / b, i = e % b;
                const int p = pp[k], q = qq[k];
                if (q >= b) continue;
                const double x = A[i * ld + p], y = A[i * ld + q];
                A[i * ld + p] = cs[k] * x - sn[k] * y;
                A[i * ld + q] = sn[k] * x + cs[k] * y;
                if (V) {
                    const double vx = V[int64_t(p) * b + i], vy = V[int64_t(q) * b + i];
                    V[int64_t(p) * b + i] = cs[k] * vx - sn[k] * vy;
                    V[int64_t(q) * b + i] = sn[k] * vx + cs[k] * vy;
                }
            }
            __syncthreads();
            // rows: A <- J' A
            for (int e = tid; e < pairs * b; e += nt) {
                const int k = e / b, i = e % b;
                const int p = pp[k], q = qq[k];
                if (q >= b) continue;
                const double x = A[p * ld + i], y = A[q * ld + i];
                A[p * ld + i] = cs[k] * x - sn[k] * y;
                A[q * ld + i] = sn[k] * x + cs[k] * y;
            }
            __syncthreads();
            if (tid < pairs && qq[tid] < b) {
                A[pp[tid] * ld + qq[tid]] = 0.0;
                A[qq[tid] * ld + pp[tid]] = 0.0;
            }
            __syncthreads();
        }
    }
    if (!converged) {
        double off = 0.0;
        for (int e = tid; e < b * b; e += nt) {
            const int i = e / b, c = e % b;
            if (c > i) off = fma(A[i * ld + c], A[i * ld + c], off);
        }
        if (sqrt(2.0 * block_reduce_sum(off, red)) > stop && tid == 0) atomicOr(status, fail_bit);
    }
    for (int i = tid; i < b; i += nt) diag[i] = A[i * ld + i];
    __syncthreads();
    // rank sort (ascending, ties by index)
    for (int i = tid; i < b; i += nt) {
        const double di = diag[i];
        int rank = 0;
        for (int j = 0; j < b; ++j) rank += (diag[j] < di) || (diag[j] == di && j < i);
        values[rank] = di;
        if (vectors)
            for (int r = 0; r < b; ++r) vectors[int64_t(rank) * b + r] = V[int64_t(i) * b + r];
    }
}

__global__ void k_eigsvd_scale(const double* values, const double* vectors, int b, double* vs,
                               double* sigma, unsigned* status, unsigned fail_bit) {
    FQB_PDL_ENTRY();
    const double lmax = values[b - 1];
    if (!(lmax > 0.0)) {
        if (threadIdx.x == 0) atomicOr(status, fail_bit);
    }
    const double fl = lmax * 1e-31;
    for (int j = threadIdx.x; j < b; j += blockDim.x) sigma[j] = sqrt(fmax(values[j], fl));
    __syncthreads();
    for (int e = threadIdx.x; e < b * b; e += blockDim.x) {
        const int c = e / b;
        const double sg = sqrt(fmax(values[c], fl));
        vs[e] = vectors[e] / sg;
    }
}

__global__ void k_axpy_cols(double alpha, const double* x, int64_t ldx, double* y, int64_t ldy,
                            int64_t rows, int cols) {
    FQB_PDL_ENTRY();
    const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    const int c = blockIdx.y;
    if (i < rows && c < cols) y[int64_t(c) * ldy + i] = fma(-alpha, x[int64_t(c) * ldx + i], y[int64_t(c) * ldy + i]);
}

// reference halving rule (driver.cpp:216-221) on the eigSVD sigma (floored like
// matrix_core.cpp:203-206); alpha lives on the device so no host sync is needed.
__global__ void k_shift_update(const double* values, int b, int conv, double* alpha) {
    FQB_PDL_ENTRY();
    const double lmax = values[b - 1];
    const double fl = lmax * 1e-31;
    const double v = conv == 0 ? values[b - 1] : values[0];
    const double shat = sqrt(fmax(v, fl));
    if (*alpha < shat) *alpha = 0.5 * (shat + *alpha);
}

__global__ void k_axpy_cols_dev(const double* alpha, const double* x, int64_t ldx, double* y, int64_t ldy,
                                int64_t rows, int cols) {
    FQB_PDL_ENTRY();
    const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    const int c = blockIdx.y;
    const double a = *alpha;
    if (a != 0.0 && i < rows && c < cols)
        y[int64_t(c) * ldy + i] = fma(-a, x[int64_t(c) * ldx + i], y[int64_t(c) * ldy + i]);
}

}  // namespace

void launch_shift_update(const double* values, int b, int conv, double* alpha, cudaStream_t s,
                         LaunchCounter& lc) {
    launch_k(k_shift_update, 1, 1, 0, s, values, b, conv, alpha);
    FQB_LAUNCHED();
    lc.bump();
}

void launch_axpy_cols_dev(const double* alpha, const double* x, int64_t ldx, double* y, int64_t ldy,
                          int64_t rows, int cols, cudaStream_t s, LaunchCounter& lc) {
    if (rows <= 0 || cols <= 0) return;
    dim3 grid(unsigned(ceil_div(rows, 256)), unsigned(cols));
    launch_k(k_axpy_cols_dev, grid, 256, 0, s, alpha, x, ldx, y, ldy, rows, cols);
    FQB_LAUNCHED();
    lc.bump();
}

void launch_chol_upper_inv(const double* S, int b, int64_t lds, double tol, double diag_ref,
                           const double* dref_extra, int64_t ld_extra, double* R, double* Rinv,
                           double* max_diag_out, double* scratch, unsigned* status, unsigned fail_bit,
                           cudaStream_t s, LaunchCounter& lc) {
    if (b > 1024) throw Error(kStatusConfig, "block size above 1024 is not supported");
    size_t smem = 0;
    if (b <= kSmemMaxB) {
        smem = size_t(b) * (b + 1) * sizeof(double);
        static bool configured[64] = {};
        int dev = 0;
        FQB_CUDA(cudaGetDevice(&dev));
        if (dev < 0 || dev >= 64 || !configured[dev]) {
            const int bytes = int(size_t(kSmemMaxB) * (kSmemMaxB + 1) * sizeof(double));
            FQB_CUDA(cudaFuncSetAttribute(k_chol_inv, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes));
            FQB_CUDA(cudaFuncSetAttribute(k_chol_inv_reg<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes));
            FQB_CUDA(cudaFuncSetAttribute(k_chol_inv_reg<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes));
            FQB_CUDA(cudaFuncSetAttribute(k_chol_inv_reg<16>, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes));
            if (dev >= 0 && dev < 64) configured[dev] = true;
        }
    }
    if (b <= kSmemMaxB) {
        const int threads = int(ceil_div(8 * b, 32) * 32);
        if (b <= 32)
            launch_k(k_chol_inv_reg<4>, 1, threads, smem, s, S, b, lds, tol, diag_ref, dref_extra, ld_extra, R, Rinv,
                                                      max_diag_out, status, fail_bit);
        else if (b <= 64)
            launch_k(k_chol_inv_reg<8>, 1, threads, smem, s, S, b, lds, tol, diag_ref, dref_extra, ld_extra, R, Rinv,
                                                      max_diag_out, status, fail_bit);
        else
            launch_k(k_chol_inv_reg<16>, 1, threads, smem, s, S, b, lds, tol, diag_ref, dref_extra, ld_extra, R, Rinv,
                                                       max_diag_out, status, fail_bit);
        FQB_LAUNCHED();
        lc.bump();
        return;
    }
    const int threads = 1024;
    launch_k(k_chol_inv, 1, threads, smem, s, S, b, lds, tol, diag_ref, dref_extra, ld_extra, R, Rinv,
                                             max_diag_out, status, fail_bit, scratch);
    FQB_LAUNCHED();
    lc.bump();
}

void launch_sym_eig(const double* S, int b, int64_t lds, double* values, double* vectors,
                    double* vtmp, unsigned* status, unsigned fail_bit, cudaStream_t s,
                    LaunchCounter& lc) {
    if (b > kSmemMaxB) throw Error(kStatusConfig, "eigensolver supports block size <= 128");
    const size_t smem = size_t(b) * (b + 1) * sizeof(double);
    static bool configured[64] = {};
    int dev = 0;
    FQB_CUDA(cudaGetDevice(&dev));
    if (dev < 0 || dev >= 64 || !configured[dev]) {
        FQB_CUDA(cudaFuncSetAttribute(k_sym_eig, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      int(size_t(kSmemMaxB) * (kSmemMaxB + 1) * sizeof(double))));
        if (dev >= 0 && dev < 64) configured[dev] = true;
    }
    launch_k(k_sym_eig, 1, 1024, smem, s, S, b, lds, values, vectors, vectors ? vtmp : nullptr, status, fail_bit);
    FQB_LAUNCHED();
    lc.bump();
}

void launch_eigsvd_scale(const double* values, const double* vectors, int b, double* vs,
                         double* sigma, unsigned* status, unsigned fail_bit, cudaStream_t s,
                         LaunchCounter& lc) {
    launch_k(k_eigsvd_scale, 1, 1024, 0, s, values, vectors, b, vs, sigma, status, fail_bit);
    FQB_LAUNCHED();
    lc.bump();
}

void launch_axpy_cols(double alpha, const double* x, int64_t ldx, double* y, int64_t ldy,
                      int64_t rows, int cols, cudaStream_t s, LaunchCounter& lc) {
    if (rows <= 0 || cols <= 0) return;
    dim3 grid(unsigned(ceil_div(rows, 256)), unsigned(cols));
    launch_k(k_axpy_cols, grid, 256, 0, s, alpha, x, ldx, y, ldy, rows, cols);
    FQB_LAUNCHED();
    lc.bump();
}

}  // namespace farqb
