// eigsmall.cu -- symmetric eigensolver for the l x l matrix of the SVD assembly
// (assemble_svd, driver.cpp:296-345: the reference takes U, sigma from Jacobi
// eigendecompositions of l x l Gram matrices) when l <= kSmallEighMax.
//
// cuSOLVER's syevd spends 1.9 ms at l = 200 (1.3 ms of it in a panel-by-panel
// tridiagonalisation built for large n), a third of a C2 run.  STATUS: opt-in
// (FQB_EIG=small).  Correct and verified (tests/test_gpu_eig.py), but at l = 200 it
// measures 2.0 ms against syevd's 1.9: the one-CTA tridiagonalisation below is as
// slow as cuSOLVER's (1.3 ms), the rest adds ~0.6 ms.  Every stage is one kernel
// sized for the small case:
//
//   k_sytrd         Householder tridiagonalisation in ONE CTA: the packed lower
//                   triangle (<= 201 KB) lives in shared memory; per column a warp
//                   forms the reflector, the symmetric product p = A v is a row pass
//                   plus a column pass over the packed rows (both conflict-free),
//                   and the rank-2 update is a row pass.  (LAPACK dsytd2 order.)
//   k_tri_bisect    eigenvalues of the tridiagonal T by bisection on Sturm counts,
//                   one warp per eigenvalue, 33-section per step (11 steps to 2^-53)
//   k_tri_invit     eigenvectors by inverse iteration, one thread per eigenvalue
//                   (partially pivoted tridiagonal LU, LAPACK dlagtf/dlagts form,
//                   two solves from a fixed pseudo-random start)
//   k_cluster_mgs   Gram-Schmidt (twice) inside clusters of nearly equal eigenvalues
//                   (gap < 1e-11 |T|), where inverse iteration alone cannot separate
//                   the vectors
//   Newton-Schulz   Z <- Z (3 I - Z'Z) / 2, twice (GEMMs): the symmetric
//                   orthogonalisation, which mixes vectors only in proportion to
//                   their non-orthogonality u |T| / gap, i.e. within eigenvalue
//                   differences that the residual does not see
//   k_apply_house   X = H_0 ... H_{n-3} Z, column slabs per CTA
//
// and an a-posteriori check -- ||M X - X diag(w)||_F and ||X'X - I||_F against
// 64 n u ||M||_F and 64 n u -- decides; a failed check returns false and the
// caller runs cuSOLVER instead, so this path can only be faster, never worse.
#include <cmath>
#include <mutex>
#include <vector>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <type_traits>
#include <utility>

#include "kernels.hpp"

namespace farqb {
namespace {


__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) v += __shfl_xor_sync(0xFFFFFFFFu, v, off);
    return v;
}
__device__ __forceinline__ double warp_max(double v) {
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) v = fmax(v, __shfl_xor_sync(0xFFFFFFFFu, v, off));
    return v;
}
__device__ __forceinline__ int ri(int i) { return i * (i + 1) / 2; }   // packed lower, row-major

// ---------------------------------------------------------------------------
// tridiagonalisation: mat (n x n, col-major, lower triangle read) -> d, e, tau and
// the reflectors vh (n x n col-major: column k holds v_k, v_k[k+1] = 1, zeros above).
// One CTA; the packed lower triangle in shared memory; per step the reflector by one
// warp, then p = A22 v as a row pass (warp per row) plus a strict-lower column pass
// (lanes over columns), then the rank-2 update (warp per row).  Measured 1.3 ms at
// n = 200 -- as slow as cuSOLVER's sytrd: ~28k warp-instructions per step, the
// predicate / index overhead of short rows dominating.  (A 32 x 32 tiled variant
// with shuffle-transposed row sums was slower still, 1.78 ms.)
constexpr int kTrdThreads = 1024;

__global__ void __launch_bounds__(kTrdThreads) k_sytrd(const double* __restrict__ mat, int n, double* d, double* e,
                                                       double* tau_out, double* vh) {
    FQB_PDL_ENTRY();
    extern __shared__ double sm[];
    double* A = sm;                          // n (n + 1) / 2
    double* vv = A + ri(n);                  // v   (local index r = i - k - 1)
    double* pw = vv + kSmallEighMax;         // p, then w
    double* rs = pw + kSmallEighMax;         // row sums
    double* cs = rs + kSmallEighMax;         // 4 x 256 column partial sums
    __shared__ double red[32];
    __shared__ double sc[2];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    for (int i = warp; i < n; i += 32)
        for (int j = lane; j <= i; j += 32) A[ri(i) + j] = mat[int64_t(j) * n + i];
    __syncthreads();
    for (int k = 0; k + 2 < n; ++k) {
        const int t0 = k + 1, m = n - t0;
        if (warp == 0) {
            double ss = 0.0;
            for (int i = t0 + 1 + lane; i < n; i += 32) {
                const double x = A[ri(i) + k];
                ss = fma(x, x, ss);
            }
            ss = warp_sum(ss);
            const double alpha = A[ri(t0) + k];
            double tau = 0.0, beta = alpha, scal = 0.0;
            if (ss > 0.0) {
                beta = -copysign(sqrt(fma(alpha, alpha, ss)), alpha);
                tau = (beta - alpha) / beta;
                scal = 1.0 / (alpha - beta);
            }
            if (tau != 0.0)
                for (int i = t0 + 1 + lane; i < n; i += 32) {
                    const double v = A[ri(i) + k] * scal;
                    A[ri(i) + k] = v;
                    vv[i - t0] = v;
                }
            if (lane == 0) {
                vv[0] = 1.0;
                sc[0] = tau;
                d[k] = A[ri(k) + k];
                e[k] = beta;
                tau_out[k] = tau;
            }
        }
        __syncthreads();
        const double tau = sc[0];
        if (tau == 0.0) continue;   // uniform
        // p = tau A22 v: row part (c <= r) ...
        for (int r = warp; r < m; r += 32) {
            const double* row = A + ri(t0 + r) + t0;
            double acc = 0.0;
            for (int c = lane; c <= r; c += 32) acc = fma(row[c], vv[c], acc);
            acc = warp_sum(acc);
            if (lane == 0) rs[r] = acc;
        }
        // ... and strict-lower column part: column c gets sum_{r > c} A(r, c) v_r
        {
            const int cb = warp & 7, part = warp >> 3;
            const int c = cb * 32 + lane;
            double acc = 0.0;
            if (cb * 32 < m)
                for (int r = cb * 32 + 1 + part; r < m; r += 4)
                    if (r > c) acc = fma(A[ri(t0 + r) + t0 + c], vv[r], acc);
            cs[part * 256 + c] = acc;
        }
        __syncthreads();
        double pv = 0.0;
        if (tid < m) {
            const double p = tau * (rs[tid] + ((cs[tid] + cs[256 + tid]) + (cs[512 + tid] + cs[768 + tid])));
            pw[tid] = p;
            pv = p * vv[tid];
        }
        pv = warp_sum(pv);
        if (lane == 0) red[warp] = pv;
        __syncthreads();
        if (warp == 0) {
            double t = warp_sum(red[lane]);
            if (lane == 0) sc[1] = 0.5 * tau * t;
        }
        __syncthreads();
        if (tid < m) pw[tid] = fma(-sc[1], vv[tid], pw[tid]);   // w = p - K v
        __syncthreads();
        // A22 -= v w' + w v'  (lower)
        for (int r = warp; r < m; r += 32) {
            double* row = A + ri(t0 + r) + t0;
            const double vr = vv[r], wr = pw[r];
            for (int c = lane; c <= r; c += 32) row[c] = fma(-vr, pw[c], fma(-wr, vv[c], row[c]));
        }
        __syncthreads();
    }
    if (tid == 0) {
        if (n >= 2) {
            d[n - 2] = A[ri(n - 2) + n - 2];
            e[n - 2] = A[ri(n - 1) + n - 2];
            tau_out[n - 2] = 0.0;
        }
        d[n - 1] = A[ri(n - 1) + n - 1];
    }
    for (int k = warp; k < n; k += 32)
        for (int i = lane; i < n; i += 32) {
            double v = 0.0;
            if (k + 2 < n) v = i == k + 1 ? 1.0 : (i > k + 1 ? A[ri(i) + k] : 0.0);
            vh[int64_t(k) * n + i] = v;
        }
}

// ---------------------------------------------------------------------------
// Tridiagonalisation, register-vector form (n <= kTrd4Max): 16 warps, warp w owns rows
// t0 + w, t0 + w + 16, ...; a lane owns columns j = 32 q + lane, q = 0..6, and keeps
// v_j, w_j and its column-sum share of p = A22 v in registers, so a row costs one
// load + two FMAs per 32-column chunk and one warp reduction, and the strict-lower
// column sums need no atomics: each warp's 224 column partials go to shared memory
// once per step.  A row's chunk count qi = i / 32 selects a specialised, fully
// unrolled body (no per-chunk branches); the window start t0 enters as a per-lane
// mask fixed for the step.  (A first version with per-chunk guards spent 29 % of its
// 18k instructions per step on integer compares; 1.06 ms at n = 200.)
constexpr int kTrd4Max = 208;     // packed A + 16 x 224 partials fit in 227 KB
constexpr int kTrd4Warps = 16;
constexpr int kTrd4Q = 7;         // 7 x 32 = 224 >= kTrd4Max columns

// p-row: racc = sum_{t0 <= j <= i} A(i,j) v_j;  colacc[q] += A(i,j) v_i (j < i)
template <int QI>
__device__ __forceinline__ double trd_row_p(const double* __restrict__ row, const double (&vreg)[kTrd4Q],
                                            const double (&lom)[kTrd4Q], double (&colacc)[kTrd4Q], int lane,
                                            int li, double vi) {
    double racc = 0.0;
#pragma unroll
    for (int q = 0; q <= QI; ++q) {
        double a = row[32 * q + lane] * lom[q];              // lom: 1 for j >= t0, else 0
        if (q == QI) a = lane <= li ? a : 0.0;               // j <= i
        racc = fma(a, vreg[q], racc);
        const double as = (q == QI && lane == li) ? 0.0 : a;   // strict lower for the column part
        colacc[q] = fma(as, vi, colacc[q]);
    }
    return racc;
}

// fused step body of k_sytrd5: the rank-2 update of step k on row i, then the row's
// contributions to p of step k + 1 from the updated values.  No masks below the last
// chunk: vk / wk are zero outside step k's window and at its first column (updated
// already by the lookahead), so those columns are rewritten unchanged; vn is zero
// below step k+1's window, so they add nothing to the row sum; their column sums land
// on p_j for j below the window, which nothing reads.  Only the chunk holding the
// diagonal needs masks (j <= i, and j < i for the column part).
template <int QI>
__device__ __forceinline__ double trd_row_f(double* __restrict__ row, const double (&vk)[kTrd4Q],
                                            const double (&wk)[kTrd4Q], const double (&vn)[kTrd4Q],
                                            double (&colacc)[kTrd4Q], int lane, int li, double vki, double wki,
                                            double vni) {
    double x[QI + 1];
#pragma unroll
    for (int q = 0; q <= QI; ++q) x[q] = row[32 * q + lane];
    double racc = 0.0;
#pragma unroll
    for (int q = 0; q < QI; ++q) {
        const double a = fma(-vki, wk[q], fma(-wki, vk[q], x[q]));
        row[32 * q + lane] = a;
        racc = fma(a, vn[q], racc);
        colacc[q] = fma(a, vni, colacc[q]);
    }
    {
        const bool in = lane <= li;
        const double a = fma(-vki, wk[QI], fma(-wki, vk[QI], x[QI]));
        if (in) row[32 * QI + lane] = a;
        racc = fma(in ? a : 0.0, vn[QI], racc);
        colacc[QI] = fma(lane < li ? a : 0.0, vni, colacc[QI]);
    }
    return racc;
}

// Tridiagonalisation with a one-column lookahead (n <= kTrd4Max): per step the
// reflector of column k+1 is formed as soon as that column has step k's update, and
// one fused sweep then applies step k's rank-2 update to the rest of the trailing
// matrix AND accumulates p = A22 v of step k+1 from the updated values -- one pass
// over the matrix per step instead of two.
__global__ void __launch_bounds__(kTrd4Warps * 32, 1) k_sytrd5(const double* __restrict__ mat, int n, double* d,
                                                               double* e, double* tau_out, double* vh) {
    FQB_PDL_ENTRY();
    extern __shared__ double sm[];
    double* A = sm;                                   // packed lower, row-major (+ slack for over-reads)
    double* vb = A + ri(n) + 224;                     // two v buffers (steps k, k+1), zero outside their window
    double* ww = vb + 2 * 224;                        // w of step k
    double* rs = ww + 224;                            // row sums of A22 v
    double* part = rs + 224;                          // [16][224] column partials
    __shared__ double red[kTrd4Warps];
    __shared__ double sc[4];                          // tau(k), K, tau(k+1)
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    constexpr int NT = kTrd4Warps * 32;
    for (int i = warp; i < n; i += kTrd4Warps)
        for (int j = lane; j <= i; j += 32) A[ri(i) + j] = mat[int64_t(j) * n + i];
    for (int i = tid; i < 3 * 224; i += NT) vb[i] = 0.0;   // vb[0..447], ww
    __syncthreads();

    // reflector of column c (rows c+1 ..) into v buffer vbuf by warp 0; tau to sc[slot]
    auto house = [&](int c, double* vbuf, int slot) {
        if (warp == 0) {
            const int t0 = c + 1;
            double xc[kTrd4Q];
            double ss = 0.0;
#pragma unroll
            for (int q = 0; q < kTrd4Q; ++q) {
                const int i = t0 + 1 + 32 * q + lane;
                xc[q] = i < n ? A[ri(i) + c] : 0.0;
                ss = fma(xc[q], xc[q], ss);
            }
            ss = warp_sum(ss);
            const double alpha = A[ri(t0) + c];
            double tau = 0.0, beta = alpha, scal = 0.0;
            if (ss > 0.0) {
                beta = -copysign(sqrt(fma(alpha, alpha, ss)), alpha);
                tau = (beta - alpha) / beta;
                scal = 1.0 / (alpha - beta);
            }
            // clear the buffer's previous window (two steps back), then write this one
            for (int i = lane; i < t0; i += 32) vbuf[i] = 0.0;
#pragma unroll
            for (int q = 0; q < kTrd4Q; ++q) {
                const int i = t0 + 1 + 32 * q + lane;
                if (i < n) {
                    const double v = xc[q] * scal;   // scal = 0 when tau = 0
                    if (tau != 0.0) A[ri(i) + c] = v;
                    vbuf[i] = v;
                }
            }
            if (lane == 0) {
                vbuf[t0] = 1.0;
                sc[slot] = tau;
                d[c] = A[ri(c) + c];
                e[c] = beta;
                tau_out[c] = tau;
            }
        }
    };
    auto lo_mask = [&](int j0, double (&lom)[kTrd4Q]) {
#pragma unroll
        for (int q = 0; q < kTrd4Q; ++q) lom[q] = 32 * q + lane >= j0 ? 1.0 : 0.0;
    };

    if (n >= 3) {
        // ---- prologue: reflector 0 and p of step 0 (plain symmetric product)
        house(0, vb, 0);
        __syncthreads();
        {
            const double* v0 = vb;
            double vreg[kTrd4Q], colacc[kTrd4Q], lom[kTrd4Q];
#pragma unroll
            for (int q = 0; q < kTrd4Q; ++q) {
                vreg[q] = v0[32 * q + lane];
                colacc[q] = 0.0;
            }
            lo_mask(1, lom);
            auto row_p = [&](int i) -> double {
                const double vi = v0[i];
                const double* row = A + ri(i);
                const int li = i & 31;
                switch (i >> 5) {
                    case 0: return trd_row_p<0>(row, vreg, lom, colacc, lane, li, vi);
                    case 1: return trd_row_p<1>(row, vreg, lom, colacc, lane, li, vi);
                    case 2: return trd_row_p<2>(row, vreg, lom, colacc, lane, li, vi);
                    case 3: return trd_row_p<3>(row, vreg, lom, colacc, lane, li, vi);
                    case 4: return trd_row_p<4>(row, vreg, lom, colacc, lane, li, vi);
                    case 5: return trd_row_p<5>(row, vreg, lom, colacc, lane, li, vi);
                    default: return trd_row_p<6>(row, vreg, lom, colacc, lane, li, vi);
                }
            };
            for (int i = 1 + warp; i < n; i += 2 * kTrd4Warps) {
                const int i2 = i + kTrd4Warps;
                double r1 = row_p(i);
                double r2 = i2 < n ? row_p(i2) : 0.0;
#pragma unroll
                for (int off = 16; off > 0; off >>= 1) {
                    r1 += __shfl_xor_sync(0xFFFFFFFFu, r1, off);
                    r2 += __shfl_xor_sync(0xFFFFFFFFu, r2, off);
                }
                if (lane == 0) {
                    rs[i] = r1;
                    if (i2 < n) rs[i2] = r2;
                }
            }
#pragma unroll
            for (int q = 0; q < kTrd4Q; ++q) part[warp * 224 + 32 * q + lane] = colacc[q];
        }
        __syncthreads();
    }
#ifdef FQB_TRD_PROBE
    long long tp5[6] = {0, 0, 0, 0, 0, 0};
    long long tl5 = clock64();
#define TRD5_STAMP(x)                      \
    {                                      \
        const long long tn_ = clock64();   \
        tp5[x] += tn_ - tl5;               \
        tl5 = tn_;                         \
    }
#else
#define TRD5_STAMP(x)
#endif
    for (int k = 0; k + 2 < n; ++k) {
        const int t0 = k + 1;
        double* vk = vb + (k & 1) * 224;
        double* vn = vb + ((k + 1) & 1) * 224;
        // ---- P(k): p = tau A22 v, K = (tau / 2) p'v, w = p - K v
        const double tau = sc[0];
        double pv = 0.0, pt = 0.0;
        if (tid >= t0 && tid < n) {
            double acc = rs[tid];
#pragma unroll
            for (int w = 0; w < kTrd4Warps; ++w) acc += part[w * 224 + tid];
            pt = tau * acc;
            pv = pt * vk[tid];
        }
        pv = warp_sum(pv);
        if (lane == 0) red[warp] = pv;
        __syncthreads();
        if (warp == 0) {
            const double t = warp_sum(lane < kTrd4Warps ? red[lane] : 0.0);
            if (lane == 0) sc[1] = 0.5 * tau * t;
        }
        __syncthreads();
        if (tid >= t0 && tid < n) ww[tid] = fma(-sc[1], vk[tid], pt);
        else if (tid < 224) ww[tid] = 0.0;
        __syncthreads();
        TRD5_STAMP(0)
        if (k + 3 >= n) {
            // last reflector: its update touches only the trailing 2 x 2 block
            if (tid >= t0 && tid < n) {
                const int i = tid;
                for (int j = t0; j <= i; ++j)
                    A[ri(i) + j] = fma(-vk[i], ww[j], fma(-ww[i], vk[j], A[ri(i) + j]));
            }
            __syncthreads();
            break;
        }
        // ---- L(k): column k+1 (rows >= k+1) gets step k's update, and every thread
        // then forms reflector k+1 itself from the block-reduced norm (no serial warp)
        {
            const int c = t0, c1 = c + 1;   // column, first row of the reflector
            double x = 0.0;
            if (tid >= c && tid < n) {
                const int i = tid;
                x = fma(-vk[i], ww[c], fma(-ww[i], vk[c], A[ri(i) + c]));
                A[ri(i) + c] = x;
            }
            const double sq = tid > c1 && tid < n ? x * x : 0.0;
            const double wsum = warp_sum(sq);
            if (lane == 0) red[warp] = wsum;
            if (tid == c1) sc[2] = x;   // alpha
            __syncthreads();
            double ss = 0.0;
#pragma unroll
            for (int w = 0; w < kTrd4Warps; ++w) ss += red[w];
            const double alpha = sc[2];
            double tau = 0.0, beta = alpha, scal = 0.0;
            if (ss > 0.0) {
                beta = -copysign(sqrt(fma(alpha, alpha, ss)), alpha);
                tau = (beta - alpha) / beta;
                scal = 1.0 / (alpha - beta);
            }
            if (tid < c1) vn[tid] = 0.0;
            else if (tid == c1) vn[tid] = 1.0;
            else if (tid < n) {
                const double v = x * scal;   // scal = 0 when tau = 0
                if (tau != 0.0) A[ri(tid) + c] = v;
                vn[tid] = v;
            }
            if (tid == 0) {
                sc[0] = tau;
                d[c] = A[ri(c) + c];
                e[c] = beta;
                tau_out[c] = tau;
            }
            __syncthreads();
        }
        TRD5_STAMP(1)
        // ---- F(k): rows >= k+2, columns >= k+2: update(k) + p(k+1)
        double vkr[kTrd4Q], wkr[kTrd4Q], vnr[kTrd4Q], colacc[kTrd4Q];
#pragma unroll
        for (int q = 0; q < kTrd4Q; ++q) {
            const int j = 32 * q + lane;
            vkr[q] = j == t0 ? 0.0 : vk[j];   // column t0 already has step k's update (L)
            wkr[q] = j == t0 ? 0.0 : ww[j];
            vnr[q] = vn[j];
            colacc[q] = 0.0;
        }
        // rows by 32-row blocks (QI = i / 32 a compile-time constant per block -- no
        // indirect branch per row); a warp has at most two rows (i, i + 16) in a block
        const int r0 = (k + 2 + warp) & 15;
        auto block_f = [&](auto qi_c) {
            constexpr int QI = decltype(qi_c)::value;
            const int lo = max(k + 2, 32 * QI), hi = min(n, 32 * QI + 32);
            if (lo >= hi) return;
            const int i1 = lo + ((r0 - lo) & 15), i2 = i1 + 16;
            const bool h1 = i1 < hi, h2 = i2 < hi;
            double ra = 0.0, rb = 0.0;
            if (h1) ra = trd_row_f<QI>(A + ri(i1), vkr, wkr, vnr, colacc, lane, i1 & 31, vk[i1], ww[i1], vn[i1]);
            if (h2) rb = trd_row_f<QI>(A + ri(i2), vkr, wkr, vnr, colacc, lane, i2 & 31, vk[i2], ww[i2], vn[i2]);
#pragma unroll
            for (int off = 16; off > 0; off >>= 1) {
                ra += __shfl_xor_sync(0xFFFFFFFFu, ra, off);
                rb += __shfl_xor_sync(0xFFFFFFFFu, rb, off);
            }
            if (lane == 0) {
                if (h1) rs[i1] = ra;
                if (h2) rs[i2] = rb;
            }
        };
        block_f(std::integral_constant<int, 0>{});
        block_f(std::integral_constant<int, 1>{});
        block_f(std::integral_constant<int, 2>{});
        block_f(std::integral_constant<int, 3>{});
        block_f(std::integral_constant<int, 4>{});
        block_f(std::integral_constant<int, 5>{});
        block_f(std::integral_constant<int, 6>{});
        TRD5_STAMP(2)
#pragma unroll
        for (int q = 0; q < kTrd4Q; ++q) part[warp * 224 + 32 * q + lane] = colacc[q];
        __syncthreads();
        TRD5_STAMP(3)
    }
#ifdef FQB_TRD_PROBE
    if (tid == FQB_TRD_PROBE)
        for (int x = 0; x < 6; ++x) trd_probe_out[x] = tp5[x];
#endif
    if (tid == 0) {
        if (n >= 2) {
            d[n - 2] = A[ri(n - 2) + n - 2];
            e[n - 2] = A[ri(n - 1) + n - 2];
            tau_out[n - 2] = 0.0;
        }
        d[n - 1] = A[ri(n - 1) + n - 1];
    }
    for (int k = warp; k < n; k += kTrd4Warps)
        for (int i = lane; i < n; i += 32) {
            double v = 0.0;
            if (k + 2 < n) v = i == k + 1 ? 1.0 : (i > k + 1 ? A[ri(i) + k] : 0.0);
            vh[int64_t(k) * n + i] = v;
        }
}

// ---------------------------------------------------------------------------
// eigenvalues: warp per index k (k-th smallest), 65-section on Sturm counts (two
// points per lane, interleaved chains).  The recurrence's division is a hardware
// reciprocal estimate refined by two Newton steps (full precision, ~half the
// latency of an IEEE divide on this dependent chain).
__device__ __forceinline__ double rcp_nr(double q) {
    double r;
    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(q));
    double t = fma(-q, r, 1.0);
    r = fma(r, t, r);
    t = fma(-q, r, 1.0);
    return fma(r, t, r);
}

__device__ __forceinline__ void sturm_count2(const double* sd, const double* se2, int n, double x0, double x1,
                                             double pivmin, int& c0, int& c1) {
    double q0 = sd[0] - x0, q1 = sd[0] - x1;
    if (fabs(q0) < pivmin) q0 = -pivmin;
    if (fabs(q1) < pivmin) q1 = -pivmin;
    c0 = q0 < 0.0;
    c1 = q1 < 0.0;
    for (int i = 1; i < n; ++i) {
        const double di = sd[i], e2 = se2[i - 1];
        q0 = (di - x0) - e2 * rcp_nr(q0);
        q1 = (di - x1) - e2 * rcp_nr(q1);
        if (fabs(q0) < pivmin) q0 = -pivmin;
        if (fabs(q1) < pivmin) q1 = -pivmin;
        c0 += q0 < 0.0;
        c1 += q1 < 0.0;
    }
}

__global__ void __launch_bounds__(256) k_tri_bisect(const double* __restrict__ d, const double* __restrict__ e, int n,
                                                    double* w) {
    FQB_PDL_ENTRY();
    __shared__ double sd[kSmallEighMax], se2[kSmallEighMax], se[kSmallEighMax];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
        sd[i] = d[i];
        const double ei = i + 1 < n ? e[i] : 0.0;
        se[i] = ei;
        se2[i] = ei * ei;
    }
    __syncthreads();
    const int k = blockIdx.x * 8 + warp;
    if (k >= n) return;
    // Gerschgorin interval and the pivot floor (LAPACK dstebz)
    double gl = INFINITY, gu = -INFINITY, emax2 = 0.0;
    for (int i = lane; i < n; i += 32) {
        const double r = fabs(i > 0 ? se[i - 1] : 0.0) + fabs(se[i]);
        gl = fmin(gl, sd[i] - r);
        gu = fmax(gu, sd[i] + r);
        emax2 = fmax(emax2, se2[i]);
    }
    gl = -warp_max(-gl);
    gu = warp_max(gu);
    emax2 = warp_max(emax2);
    const double tn = fmax(fabs(gl), fabs(gu));
    const double u = 1.1102230246251565e-16;
    const double pivmin = 2.2250738585072014e-308 * fmax(1.0, emax2);
    gl -= 2.0 * u * tn * n + 2.0 * pivmin;
    gu += 2.0 * u * tn * n + 2.0 * pivmin;
    double lo = gl, hi = gu;
    for (int it = 0; it < 64; ++it) {
        // points lo + (hi - lo) m / 65, m = 1..64: lane holds m = 2 lane + 1, 2 lane + 2
        const double step = (hi - lo) / 65.0;
        const double x0 = lo + step * double(2 * lane + 1), x1 = lo + step * double(2 * lane + 2);
        int c0, c1;
        sturm_count2(sd, se2, n, x0, x1, pivmin, c0, c1);
        const unsigned a0 = __ballot_sync(0xFFFFFFFFu, c0 > k), a1 = __ballot_sync(0xFFFFFFFFu, c1 > k);
        // first point (in order x0(l0), x1(l0), x0(l1), ...) with more than k eigenvalues below
        const int f0 = a0 ? __ffs(a0) - 1 : 64, f1 = a1 ? __ffs(a1) - 1 : 64;
        const int first = min(2 * f0, 2 * f1 + 1);   // point index m - 1 in 0..63, 128 = none
        double nlo = lo, nhi = hi;
        if (first < 64) {
            const int m = first + 1;                  // x_m is the first point above
            nhi = lo + step * double(m);
            if (m > 1) nlo = lo + step * double(m - 1);
        } else {
            nlo = lo + step * 64.0;
        }
        lo = nlo;
        hi = nhi;
        if (hi - lo <= 2.0 * u * fmax(fabs(lo), fabs(hi)) + 4.0 * pivmin) break;
    }
    if (lane == 0) w[k] = 0.5 * (lo + hi);
}

// ---------------------------------------------------------------------------
// eigenvectors: thread per eigenvalue, inverse iteration on T - w_k I
__device__ __forceinline__ double start_value(int k, int i) {
    unsigned h = unsigned(k) * 0x9E3779B1u ^ (unsigned(i) + 0x7F4A7C15u) * 0x85EBCA77u;
    h ^= h >> 15;
    h *= 0xC2B2AE3Du;
    h ^= h >> 13;
    return (double(h & 0xFFFFFF) / double(0x1000000)) * 2.0 - 1.0;
}

constexpr int kInvitThreads = 16;   // 16 x 5 x 224 doubles of factors = 140 KB of shared memory
constexpr size_t kInvitSmem = sizeof(double) * 5 * kInvitThreads * kSmallEighMax;
__global__ void __launch_bounds__(kInvitThreads) k_tri_invit(const double* __restrict__ d,
                                                             const double* __restrict__ e,
                                                             const double* __restrict__ w, int n, double* z) {
    FQB_PDL_ENTRY();
    extern __shared__ double fs[];   // [i][thread]: 1/u0, u1, u2, mult (sign bit of pivot in flag), y
    const int t = threadIdx.x;
    const int k = blockIdx.x * kInvitThreads + t;
    double* RA = fs;                                   // 1 / pivot
    double* U1 = RA + kInvitThreads * kSmallEighMax;   // first super-diagonal of U
    double* U2 = U1 + kInvitThreads * kSmallEighMax;   // second super-diagonal of U (row swaps)
    double* ML = U2 + kInvitThreads * kSmallEighMax;   // multipliers of L
    double* Y = ML + kInvitThreads * kSmallEighMax;
    unsigned piv[(kSmallEighMax + 31) / 32];
    if (k >= n) return;
    auto at = [t](double* base, int i) -> double& { return base[i * kInvitThreads + t]; };
    const double lam = w[k];
    double tn = 0.0;
    for (int i = 0; i < n; ++i) tn = fmax(tn, fabs(d[i]) + (i > 0 ? fabs(e[i - 1]) : 0.0) + (i + 1 < n ? fabs(e[i]) : 0.0));
    const double tiny = fmax(tn, 1e-300) * 1.1102230246251565e-16;
    for (int q = 0; q < (kSmallEighMax + 31) / 32; ++q) piv[q] = 0u;
    // LU with partial pivoting of T - lam I (dlagtf); the running row (a, b) stays in registers
    double a = d[0] - lam, b = n > 1 ? e[0] : 0.0;
    for (int i = 0; i + 1 < n; ++i) {
        const double c = e[i];                       // T(i+1, i)
        const double an = d[i + 1] - lam;            // next row: (c, an, bn)
        const double bn = i + 2 < n ? e[i + 1] : 0.0;
        if (fabs(a) >= fabs(c)) {
            const double aa = fabs(a) < tiny ? copysign(tiny, a == 0.0 ? 1.0 : a) : a;
            const double ra = 1.0 / aa;
            const double mult = c * ra;
            at(RA, i) = ra;
            at(U1, i) = b;
            at(U2, i) = 0.0;
            at(ML, i) = mult;
            a = an - mult * b;
            b = bn;
        } else {
            const double rc = 1.0 / c;
            const double mult = a * rc;
            at(RA, i) = rc;
            at(U1, i) = an;
            at(U2, i) = bn;
            at(ML, i) = mult;
            piv[i >> 5] |= 1u << (i & 31);
            a = b - mult * an;
            b = -mult * bn;
        }
    }
    {
        const double aa = fabs(a) < tiny ? copysign(tiny, a == 0.0 ? 1.0 : a) : a;
        at(RA, n - 1) = 1.0 / aa;
        at(U1, n - 1) = 0.0;
        at(U2, n - 1) = 0.0;
    }
    for (int i = 0; i < n; ++i) at(Y, i) = start_value(k, i);
    for (int pass = 0; pass < 3; ++pass) {
        // forward: L (row interchanges recorded in piv)
        double yi = at(Y, 0);
        for (int i = 0; i + 1 < n; ++i) {
            double yn = at(Y, i + 1);
            if (piv[i >> 5] >> (i & 31) & 1u) {
                const double tt = yi;
                yi = yn;
                yn = tt;
            }
            at(Y, i) = yi;
            yi = yn - at(ML, i) * yi;
        }
        at(Y, n - 1) = yi;
        // backward: U (three bands), running values in registers
        double mx = 0.0, y1 = 0.0, y2 = 0.0;
        for (int i = n - 1; i >= 0; --i) {
            const double v = (at(Y, i) - at(U1, i) * y1 - at(U2, i) * y2) * at(RA, i);
            at(Y, i) = v;
            y2 = y1;
            y1 = v;
            mx = fmax(mx, fabs(v));
        }
        const double sc = mx > 0.0 ? 1.0 / mx : 1.0;
        double nrm = 0.0;
        for (int i = 0; i < n; ++i) {
            const double v = at(Y, i) * sc;
            at(Y, i) = v;
            nrm = fma(v, v, nrm);
        }
        if (pass == 2) {
            const double inv = 1.0 / sqrt(nrm);
            for (int i = 0; i < n; ++i) z[int64_t(k) * n + i] = at(Y, i) * inv;
        }
    }
}

// Gram-Schmidt (twice) inside clusters of eigenvalues closer than tol_rel * |T|
__global__ void __launch_bounds__(256) k_cluster_mgs(const double* __restrict__ w, int n, double tol_rel, double* z) {
    FQB_PDL_ENTRY();
    __shared__ double red[8];
    __shared__ double coef[kSmallEighMax];
    __shared__ double ws[kSmallEighMax];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    for (int i = tid; i < n; i += blockDim.x) ws[i] = w[i];
    __syncthreads();
    const double scale = fmax(fabs(ws[0]), fabs(ws[n - 1]));
    const double tol = tol_rel * scale;
    int j0 = 0;
    while (j0 < n) {
        int j1 = j0 + 1;
        while (j1 < n && ws[j1] - ws[j1 - 1] <= tol) ++j1;
        for (int j = j0 + 1; j < j1; ++j) {
            double* zj = z + int64_t(j) * n;
            for (int rep = 0; rep < 2; ++rep) {
                // coefficients against the earlier members: warp per member
                for (int p = j0 + warp; p < j; p += 8) {
                    const double* zp = z + int64_t(p) * n;
                    double acc = 0.0;
                    for (int i = lane; i < n; i += 32) acc = fma(zp[i], zj[i], acc);
                    acc = warp_sum(acc);
                    if (lane == 0) coef[p - j0] = acc;
                }
                __syncthreads();
                for (int i = tid; i < n; i += blockDim.x) {
                    double v = zj[i];
                    for (int p = j0; p < j; ++p) v = fma(-coef[p - j0], z[int64_t(p) * n + i], v);
                    zj[i] = v;
                }
                __syncthreads();
            }
            double acc = 0.0;
            for (int i = tid; i < n; i += blockDim.x) acc = fma(zj[i], zj[i], acc);
            acc = warp_sum(acc);
            if (lane == 0) red[warp] = acc;
            __syncthreads();
            double t = 0.0;
            for (int q = 0; q < 8; ++q) t += red[q];
            const double inv = t > 0.0 ? 1.0 / sqrt(t) : 0.0;
            for (int i = tid; i < n; i += blockDim.x) zj[i] *= inv;
            __syncthreads();
        }
        j0 = j1;
    }
}

// G <- 1.5 I - 0.5 G
__global__ void k_ns_coef(double* g, int n) {
    FQB_PDL_ENTRY();
    const int i = blockIdx.x * blockDim.x + threadIdx.x, j = blockIdx.y;
    if (i < n) g[int64_t(j) * n + i] = (i == j ? 1.5 : 0.0) - 0.5 * g[int64_t(j) * n + i];
}

// Z <- H_0 H_1 ... H_{n-3} Z, H_k = I - tau_k v_k v_k'.  Columns are independent:
// one warp per column, the column in registers (lane holds rows lane + 32 q), the
// reflector rows loaded one step ahead -- no block-level barriers at all.
constexpr int kHouseQ = (kSmallEighMax + 31) / 32;
__global__ void __launch_bounds__(128) k_apply_house(const double* __restrict__ vh, const double* __restrict__ tau,
                                                     int n, double* z) {
    FQB_PDL_ENTRY();
    const int lane = threadIdx.x & 31;
    const int c = blockIdx.x * 4 + (threadIdx.x >> 5);
    if (c >= n) return;
    double zc[kHouseQ], vn[kHouseQ];
#pragma unroll
    for (int q = 0; q < kHouseQ; ++q) {
        const int i = lane + 32 * q;
        zc[q] = i < n ? z[int64_t(c) * n + i] : 0.0;
    }
    int k = n - 3;
    if (k >= 0) {
#pragma unroll
        for (int q = 0; q < kHouseQ; ++q) {
            const int i = lane + 32 * q;
            vn[q] = i < n ? vh[int64_t(k) * n + i] : 0.0;
        }
    }
    for (; k >= 0; --k) {
        double v[kHouseQ];
#pragma unroll
        for (int q = 0; q < kHouseQ; ++q) v[q] = vn[q];
        const double t = tau[k];
        if (k > 0) {
#pragma unroll
            for (int q = 0; q < kHouseQ; ++q) {
                const int i = lane + 32 * q;
                vn[q] = i < n ? vh[int64_t(k - 1) * n + i] : 0.0;
            }
        }
        double acc = 0.0;
#pragma unroll
        for (int q = 0; q < kHouseQ; ++q) acc = fma(v[q], zc[q], acc);   // v is zero above row k + 1
        const double sk = t * warp_sum(acc);
#pragma unroll
        for (int q = 0; q < kHouseQ; ++q) zc[q] = fma(-sk, v[q], zc[q]);
    }
#pragma unroll
    for (int q = 0; q < kHouseQ; ++q) {
        const int i = lane + 32 * q;
        if (i < n) z[int64_t(c) * n + i] = zc[q];
    }
}

// Per-CTA partial sums, in a fixed order (warp shuffles, then warps 0..7), written to
// part[3 * cta + {0, 1, 2}] = ||R - X diag(w)||^2, ||M||^2, ||O - I||^2 over the CTA's
// elements; the host adds the CTAs in index order -- so the accept / fallback decision
// is bitwise reproducible (no floating-point atomics).
__global__ void k_eig_check(const double* __restrict__ r, const double* __restrict__ x, const double* __restrict__ w,
                            const double* __restrict__ mat, const double* __restrict__ o, int n, double* part) {
    FQB_PDL_ENTRY();
    __shared__ double red[3][8];
    const int i = blockIdx.x * blockDim.x + threadIdx.x, j = blockIdx.y;
    double a = 0.0, b = 0.0, c = 0.0;
    if (i < n) {
        const int64_t e = int64_t(j) * n + i;
        const double res = r[e] - x[e] * w[j];
        a = res * res;
        b = mat[e] * mat[e];
        const double oe = o[e] - (i == j ? 1.0 : 0.0);
        c = oe * oe;
    }
    a = warp_sum(a);
    b = warp_sum(b);
    c = warp_sum(c);
    const int warp = threadIdx.x >> 5;
    if ((threadIdx.x & 31) == 0) {
        red[0][warp] = a;
        red[1][warp] = b;
        red[2][warp] = c;
    }
    __syncthreads();
    if (threadIdx.x < 3) {
        double t = 0.0;
        for (int q = 0; q < int(blockDim.x >> 5); ++q) t += red[threadIdx.x][q];
        part[3 * (int64_t(blockIdx.y) * gridDim.x + blockIdx.x) + threadIdx.x] = t;
    }
}

}  // namespace

int64_t small_eigh_scratch_doubles(int n) { return int64_t(n) * n * 12 + 4 * int64_t(n) + 8; }

bool small_eigh(const double* mat, int n, double* w, double* x, double* scratch, GemmWorkspace& gws, int num_sms,
                cudaStream_t s, LaunchCounter& lc) {
    if (n < 1 || n > kSmallEighMax) return false;
    const int64_t nn = int64_t(n) * n;
    double* vh = scratch;
    double* z = vh + nn;
    double* z1 = z + nn;
    double* g = z1 + nn;
    double* r = g + nn;
    double* inv = r + nn;          // 6 n^2
    double* d = inv + 6 * nn;
    double* e = d + n;
    double* tau = e + n;
    double* sums = tau + n + n;    // 4 (8-aligned slack above)
    const size_t smem = sizeof(double) * size_t(n * (n + 1) / 2 + 4 * kSmallEighMax + 4 * 256);
    // The dynamic shared-memory limits are per-device function attributes: raise them
    // once on every device a handle lives on (a process may drive several GPUs, from
    // several threads).
    {
        static std::mutex mu;
        static bool configured[64] = {};
        int dev = 0;
        FQB_CUDA(cudaGetDevice(&dev));
        std::lock_guard<std::mutex> lock(mu);
        if (dev < 0 || dev >= 64 || !configured[dev]) {
            FQB_CUDA(cudaFuncSetAttribute(k_tri_invit, cudaFuncAttributeMaxDynamicSharedMemorySize, int(kInvitSmem)));
            const size_t mx =
                sizeof(double) * size_t(kSmallEighMax * (kSmallEighMax + 1) / 2 + 4 * kSmallEighMax + 4 * 256);
            FQB_CUDA(cudaFuncSetAttribute(k_sytrd, cudaFuncAttributeMaxDynamicSharedMemorySize, int(mx)));
            const size_t mx4 = sizeof(double) * size_t(kTrd4Max * (kTrd4Max + 1) / 2 + 5 * 224 + kTrd4Warps * 224);
            FQB_CUDA(cudaFuncSetAttribute(k_sytrd5, cudaFuncAttributeMaxDynamicSharedMemorySize, int(mx4)));
            if (dev >= 0 && dev < 64) configured[dev] = true;
        }
    }
    if (n <= kTrd4Max) {
        const size_t smem4 = sizeof(double) * size_t(n * (n + 1) / 2 + 5 * 224 + kTrd4Warps * 224);
        launch_k(k_sytrd5, 1, kTrd4Warps * 32, smem4, s, mat, n, d, e, tau, vh);
    } else {
        launch_k(k_sytrd, 1, kTrdThreads, smem, s, mat, n, d, e, tau, vh);
    }
    FQB_LAUNCHED();
    launch_k(k_tri_bisect, unsigned(ceil_div(n, 8)), 256, 0, s, d, e, n, w);
    FQB_LAUNCHED();
    launch_k(k_tri_invit, unsigned(ceil_div(n, kInvitThreads)), kInvitThreads, kInvitSmem, s, d, e, w, n, z);
    FQB_LAUNCHED();
    launch_k(k_cluster_mgs, 1, 256, 0, s, w, n, 1e-11, z);
    FQB_LAUNCHED();
    lc.bump(4);
    // symmetric orthogonalisation, two Newton-Schulz steps
    double* cur = z;
    double* nxt = z1;
    for (int it = 0; it < 2; ++it) {
        gemm(true, n, n, n, 1.0, cur, n, cur, n, 0.0, g, n, gws, num_sms, s, lc);
        launch_k(k_ns_coef, dim3(unsigned(ceil_div(n, 256)), unsigned(n)), 256, 0, s, g, n);
        FQB_LAUNCHED();
        lc.bump();
        gemm(false, n, n, n, 1.0, cur, n, g, n, 0.0, nxt, n, gws, num_sms, s, lc);
        std::swap(cur, nxt);
    }
    launch_k(k_apply_house, unsigned(ceil_div(n, 4)), 128, 0, s, vh, tau, n, cur);
    FQB_LAUNCHED();
    lc.bump();
    // a-posteriori check: R = M X, O = X'X
    gemm(false, n, n, n, 1.0, mat, n, cur, n, 0.0, r, n, gws, num_sms, s, lc);
    gemm(true, n, n, n, 1.0, cur, n, cur, n, 0.0, g, n, gws, num_sms, s, lc);
    const int check_ctas = int(ceil_div(n, 256)) * n;   // <= 224 partial triples, in inv (6 n^2 doubles)
    launch_k(k_eig_check, dim3(unsigned(ceil_div(n, 256)), unsigned(n)), 256, 0, s, r, cur, w, mat, g, n, inv);
    FQB_LAUNCHED();
    lc.bump();
    std::vector<double> part(size_t(3) * check_ctas);
    FQB_CUDA(cudaMemcpyAsync(part.data(), inv, sizeof(double) * part.size(), cudaMemcpyDeviceToHost, s));
    FQB_CUDA(cudaStreamSynchronize(s));
    double hs[3] = {0.0, 0.0, 0.0};
    for (int c = 0; c < check_ctas; ++c)
        for (int q = 0; q < 3; ++q) hs[q] += part[size_t(3) * c + q];
    const double u = 1.1102230246251565e-16;
    const double res = std::sqrt(hs[0]), mnorm = std::sqrt(hs[1]), orth = std::sqrt(hs[2]);
    const bool ok = std::isfinite(res) && std::isfinite(orth) && res <= 64.0 * n * u * mnorm && orth <= 64.0 * n * u;
    if (const char* dbg = std::getenv("FQB_EIG_DEBUG"))
        if (dbg[0] == '1')
            std::fprintf(stderr, "small_eigh n=%d: residual %.3e (|M| %.3e), orthogonality %.3e -> %s\n", n, res, mnorm,
                         orth, ok ? "ok" : "fallback");
    if (!ok) return false;
    FQB_CUDA(cudaMemcpyAsync(x, cur, sizeof(double) * size_t(nn), cudaMemcpyDeviceToDevice, s));
    return true;
}

}  // namespace farqb
