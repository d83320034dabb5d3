// eiglarge.cu -- symmetric eigensolver for the SVD assembly's l x l Gram matrix B B'
// when l > kSmallEighMax (configs 3-5: l = 2000 at config 4), the role of the
// reference's sym_eig inside assemble_svd (matrix_core.cpp:50-115, driver.cpp:296-345).
//
// 1. Householder tridiagonalisation, one persistent cooperative kernel over all SMs
//    (k_trd_coop).  The n x n matrix stays in L2 (32 MB at n = 2000).  Column j of the
//    trailing matrix belongs to CTA j % G for the whole run; per step k every CTA
//    (a) rebuilds the Householder vector of column k itself -- column k was left out
//        of step k-1's update, every CTA applies that update on the fly, so no CTA waits
//        for another to publish it --, (b) forms p_j = tau (A22 v)_j for its columns and
//        a partial p'v, then one grid barrier, (c) updates its columns of A22 by
//        -(v w' + w v') with w = p - (tau/2)(p'v) v.  One grid barrier per step.
// 2. Eigenvalues of the tridiagonal: a warp per eigenvalue, 65-section on Sturm counts.
// 3. Eigenvectors: inverse iteration, a thread per eigenvalue (LU factors in global
//    memory, interleaved so a warp's accesses coalesce), Gram-Schmidt twice inside
//    clusters closer than 1e-11 |T|, two Newton-Schulz steps for the rest.
// 4. Back-transformation with the Householder vectors in blocks of 32 (compact WY,
//    T from V'V, DMMA GEMMs).
// An a-posteriori check -- |M X - X diag(w)|_F <= 64 n u |M|_F and |X'X - I|_F <=
// 64 n u -- decides; the caller falls back to cuSOLVER syevd when it fails, so the
// solver can only cost time, never accuracy (same contract as eigsmall.cu).
#include <cooperative_groups.h>

#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <mutex>
#include <vector>

#include "engine.hpp"
#include "kernels.hpp"

namespace cg = cooperative_groups;

namespace farqb {
namespace {

constexpr int kTrdThreads = 512;
constexpr int kLargeEighMax = 8192;   // two n-vectors of the cooperative kernel in shared memory
constexpr int kWyBlock = 32;
constexpr int kMgsMaxCluster = 64;

__device__ __forceinline__ double wsum(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xFFFFFFFFu, v, o);
    return v;
}
__device__ __forceinline__ double wmax(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xFFFFFFFFu, v, o));
    return v;
}
// fixed-order block sum (warp shuffles, then warps 0..nw-1 by one thread): identical bits
// in every CTA for identical inputs
__device__ __forceinline__ double block_sum_fixed(double v, double* red) {
    v = wsum(v);
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    __syncthreads();
    if (lane == 0) red[warp] = v;
    __syncthreads();
    if (threadIdx.x == 0) {
        double t = 0.0;
        for (int w = 0; w < int(blockDim.x >> 5); ++w) t += red[w];
        red[32] = t;
    }
    __syncthreads();
    return red[32];
}

struct TrdArgs {
    double* A;      // n x n, ld n, both triangles (overwritten)
    int n;
    double* d;      // n
    double* e;      // n - 1
    double* tau;    // n - 2
    double* V;      // n x n: column k = v_k (v_k[k+1] = 1, zeros above), k <= n-3
    double* P;      // 2 x n, double-buffered p
    double* S;      // 2 x gridDim, double-buffered partial p'v
};

// 2-barrier fixed-order block sum: every thread adds the warp partials in warp order
__device__ __forceinline__ double block_sum2(double v, double* red) {
    v = wsum(v);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
    __syncthreads();
    double t = 0.0;
    for (int w = 0; w < int(blockDim.x >> 5); ++w) t += red[w];
    return t;
}

__global__ void __launch_bounds__(kTrdThreads, 1) k_trd_coop(const TrdArgs a) {
    cg::grid_group grid = cg::this_grid();
    extern __shared__ double sm[];
    __shared__ double red_a[32], red_b[32], red_c[32];
    __shared__ double tot_s;
    const int n = a.n;
    // x of the current and the previous step, unscaled; v_i = x_i * scale (i >= k+2), v_{k+1} = 1
    double* x = sm;
    double* xp = sm + n;
    const int G = gridDim.x, c = blockIdx.x;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nw = blockDim.x >> 5;
    double cprev = 0.0, scp = 0.0;   // previous step's (tau / 2) p'v and scale
    for (int k = 0; k + 2 < n; ++k) {
        const double* colk = a.A + int64_t(k) * n;
        const double* pp = a.P + ((k + 1) & 1) * int64_t(n);   // previous step's p
        // previous v, from its unscaled x (v_k = 1 at the previous step's k-1 + 1 = k)
        auto vprev = [&](int i) { return i == k ? 1.0 : xp[i] * scp; };
        // (a) column k (rows k .. n-1) with the previous step's update applied on the fly,
        // and the partial |x(k+2..)|^2 in the same pass
        double part = 0.0;
        const double wk = k > 0 ? fma(-cprev, 1.0, pp[k]) : 0.0;   // vprev(k) = 1
        for (int i = k + tid; i < n; i += blockDim.x) {
            double xi = colk[i];
            if (k > 0) {
                const double vi = vprev(i);
                const double wi = fma(-cprev, vi, pp[i]);
                xi -= vi * wk + wi * 1.0;   // same two products, same sum, as in (c)
            }
            x[i] = xi;
            if (i >= k + 2) part = fma(xi, xi, part);
        }
        const double sigma = block_sum2(part, red_a);   // (the barrier also publishes x)
        const double dk = x[k], alpha = x[k + 1];
        double beta = alpha, tau = 0.0, scale = 0.0;
        if (sigma > 0.0) {
            beta = -copysign(sqrt(alpha * alpha + sigma), alpha);
            tau = (beta - alpha) / beta;
            scale = 1.0 / (alpha - beta);
        }
        auto vcur = [&](int i) { return i == k + 1 ? 1.0 : x[i] * scale; };
        if (c == 0) {
            if (tid == 0) {
                a.d[k] = dk;
                a.e[k] = beta;
                a.tau[k] = tau;
            }
            double* vk = a.V + int64_t(k) * n;
            for (int i = tid; i < n; i += blockDim.x) vk[i] = i > k ? vcur(i) : 0.0;
        }
        // (b) p_j = tau (A22 v)_j for the owned columns j >= k + 1, a warp per column
        double* pc = a.P + (k & 1) * int64_t(n);
        double s_local = 0.0;
        const int j_first = k + 1 + ((c - (k + 1)) % G + G) % G;
        int q = 0;
        for (int j = j_first; j < n; j += G, ++q) {
            if (q % nw != warp) continue;
            const double* colj = a.A + int64_t(j) * n;
            double acc = 0.0;
            for (int i = k + 1 + lane; i < n; i += 32) acc = fma(colj[i], vcur(i), acc);
            acc = wsum(acc);   // columns >= k + 1 all carry step k-1's update (only column k skipped it)
            const double pj = tau * acc;
            if (lane == 0) {
                pc[j] = pj;
                s_local = fma(pj, vcur(j), s_local);
            }
        }
        const double s = block_sum2(lane == 0 ? s_local : 0.0, red_b);
        if (tid == 0) a.S[(k & 1) * G + c] = s;
        grid.sync();
        // every CTA sums the G partials in the same fixed order (warp 0, lane-strided, then lanes)
        if (warp == 0) {
            double t = 0.0;
            for (int cc = lane; cc < G; cc += 32) t += a.S[(k & 1) * G + cc];
            red_c[lane] = t;
            __syncwarp();
            if (lane == 0) {
                double u = 0.0;
                for (int l2 = 0; l2 < 32; ++l2) u += red_c[l2];
                tot_s = u;
            }
        }
        __syncthreads();
        const double ck = 0.5 * tau * tot_s;
        // (c) owned columns j >= k + 2: A[i, j] -= v_i w_j + w_i v_j, rows i >= k + 1
        q = 0;
        for (int j = j_first; j < n; j += G, ++q) {
            if (j < k + 2 || q % nw != warp) continue;
            double* colj = a.A + int64_t(j) * n;
            const double vj = vcur(j);
            const double wj = fma(-ck, vj, pc[j]);
            for (int i = k + 1 + lane; i < n; i += 32) {
                const double vi = vcur(i);
                const double wi = fma(-ck, vi, pc[i]);
                colj[i] -= vi * wj + wi * vj;
            }
        }
        cprev = ck;
        scp = scale;
        double* t = x;   // the next step's (a) overwrites the older buffer, last read before this step's barriers
        x = xp;
        xp = t;
    }
    grid.sync();   // the last updates are visible
    if (c == 0 && tid == 0) {
        // trailing 2 x 2: column n-2 still carries the last step's pending update
        if (n >= 3) {
            const int k = n - 3;
            const double* pp = a.P + (k & 1) * int64_t(n);
            const double ck = cprev;
            auto vl = [&](int i) { return i == k + 1 ? 1.0 : xp[i] * scp; };   // the last step's v
            auto corr = [&](int i, int j) {
                const double vi = vl(i), vj = vl(j);
                const double wj = fma(-ck, vj, pp[j]);
                const double wi = fma(-ck, vi, pp[i]);
                return vi * wj + wi * vj;
            };
            const double* c2 = a.A + int64_t(n - 2) * n;
            a.d[n - 2] = c2[n - 2] - corr(n - 2, n - 2);
            a.e[n - 2] = c2[n - 1] - corr(n - 1, n - 2);
            a.d[n - 1] = a.A[int64_t(n - 1) * n + (n - 1)];
        } else if (n == 2) {
            a.d[0] = a.A[0];
            a.e[0] = a.A[1];
            a.d[1] = a.A[3];
        } else {
            a.d[0] = a.A[0];
        }
    }
}

// ---- tridiagonal eigenvalues: warp per eigenvalue, 65-section on Sturm counts ----
__device__ __forceinline__ double rcp_nr(double q) {
    double r;
    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(q));
    double t = fma(-q, r, 1.0);
    r = fma(r, t, r);
    t = fma(-q, r, 1.0);
    return fma(r, t, r);
}

__global__ void __launch_bounds__(256) k_bisect_large(const double* __restrict__ d, const double* __restrict__ e,
                                                      int n, double gl, double gu, double pivmin, double* w) {
    FQB_PDL_ENTRY();
    extern __shared__ double sb[];
    double* sd = sb;
    double* se2 = sb + n;
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
        sd[i] = d[i];
        const double ei = i + 1 < n ? e[i] : 0.0;
        se2[i] = ei * ei;
    }
    __syncthreads();
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int k = blockIdx.x * 8 + warp;
    if (k >= n) return;
    const double u = 1.1102230246251565e-16;
    double lo = gl, hi = gu;
    for (int it = 0; it < 64; ++it) {
        const double step = (hi - lo) / 65.0;
        const double x0 = lo + step * double(2 * lane + 1), x1 = lo + step * double(2 * lane + 2);
        double q0 = sd[0] - x0, q1 = sd[0] - x1;
        if (fabs(q0) < pivmin) q0 = -pivmin;
        if (fabs(q1) < pivmin) q1 = -pivmin;
        int c0 = q0 < 0.0, c1 = q1 < 0.0;
        for (int i = 1; i < n; ++i) {
            const double di = sd[i], e2 = se2[i - 1];
            q0 = (di - x0) - e2 * rcp_nr(q0);
            q1 = (di - x1) - e2 * rcp_nr(q1);
            if (fabs(q0) < pivmin) q0 = -pivmin;
            if (fabs(q1) < pivmin) q1 = -pivmin;
            c0 += q0 < 0.0;
            c1 += q1 < 0.0;
        }
        const unsigned a0 = __ballot_sync(0xFFFFFFFFu, c0 > k), a1 = __ballot_sync(0xFFFFFFFFu, c1 > k);
        const int f0 = a0 ? __ffs(a0) - 1 : 64, f1 = a1 ? __ffs(a1) - 1 : 64;
        const int first = min(2 * f0, 2 * f1 + 1);
        double nlo = lo, nhi = hi;
        if (first < 64) {
            const int m = first + 1;
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

// ---- eigenvectors of the tridiagonal: thread per eigenvalue, inverse iteration ----
__device__ __forceinline__ double start_value(int k, int i) {
    unsigned h = unsigned(k) * 0x9E3779B1u ^ (unsigned(i) + 0x7F4A7C15u) * 0x85EBCA77u;
    h ^= h >> 15;
    h *= 0xC2B2AE3Du;
    h ^= h >> 13;
    return (double(h & 0xFFFFFF) / double(0x1000000)) * 2.0 - 1.0;
}

// scratch: 5 n x nt doubles, element i of thread t at [i * nt + t] (coalesced across a warp)
__global__ void __launch_bounds__(128) k_invit_large(const double* __restrict__ d, const double* __restrict__ e,
                                                     const double* __restrict__ w, int n, double tn,
                                                     double* __restrict__ scratch, unsigned* __restrict__ pivbits,
                                                     double* __restrict__ z) {
    FQB_PDL_ENTRY();
    const int k = blockIdx.x * blockDim.x + threadIdx.x;
    const int nt = gridDim.x * blockDim.x;
    if (k >= n) return;
    double* RA = scratch;
    double* U1 = RA + int64_t(n) * nt;
    double* U2 = U1 + int64_t(n) * nt;
    double* ML = U2 + int64_t(n) * nt;
    double* Y = ML + int64_t(n) * nt;
    auto at = [&](double* base, int i) -> double& { return base[int64_t(i) * nt + k]; };
    unsigned* piv = pivbits + int64_t(k) * ((n + 31) / 32);
    const double lam = w[k];
    const double tiny = fmax(tn, 1e-300) * 1.1102230246251565e-16;
    for (int q = 0; q < (n + 31) / 32; ++q) piv[q] = 0u;
    double a = d[0] - lam, b = n > 1 ? e[0] : 0.0;
    for (int i = 0; i + 1 < n; ++i) {
        const double c = e[i];
        const double an = d[i + 1] - lam;
        const double bn = i + 2 < n ? e[i + 1] : 0.0;
        if (fabs(a) >= fabs(c)) {
            const double aa = fabs(a) < tiny ? copysign(tiny, a == 0.0 ? 1.0 : a) : a;
            const double ra = 1.0 / aa;
            at(RA, i) = ra;
            at(U1, i) = b;
            at(U2, i) = 0.0;
            at(ML, i) = c * ra;
            a = an - c * ra * b;
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
        double yi = at(Y, 0);
        for (int i = 0; i + 1 < n; ++i) {
            double yn = at(Y, i + 1);
            if (piv[i >> 5] >> (i & 31) & 1u) {
                const double t = yi;
                yi = yn;
                yn = t;
            }
            at(Y, i) = yi;
            yi = yn - at(ML, i) * yi;
        }
        at(Y, n - 1) = yi;
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

// Gram-Schmidt twice inside each cluster of eigenvalues closer than tol (a CTA per
// cluster start; clusters are found by the CTA whose index starts one)
__global__ void __launch_bounds__(256) k_cluster_mgs_large(const double* __restrict__ w, int n, double tol,
                                                           double* z) {
    FQB_PDL_ENTRY();
    __shared__ double red[33];
    __shared__ double coef[256];
    const int j0 = blockIdx.x;
    if (j0 >= n) return;
    if (j0 > 0 && w[j0] - w[j0 - 1] <= tol) return;   // not a cluster start
    int j1 = j0 + 1;
    while (j1 < n && w[j1] - w[j1 - 1] <= tol) ++j1;
    // large near-degenerate groups (near-null spaces) are left to the Newton-Schulz steps and
    // the a-posteriori check (syevd when it fails): one CTA would take O(c^2 n)
    if (j1 - j0 > kMgsMaxCluster) return;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    for (int j = j0 + 1; j < j1; ++j) {
        double* zj = z + int64_t(j) * n;
        for (int rep = 0; rep < 2; ++rep) {
            for (int p = j0 + warp; p < j; p += 8) {
                const double* zp = z + int64_t(p) * n;
                double acc = 0.0;
                for (int i = lane; i < n; i += 32) acc = fma(zp[i], zj[i], acc);
                acc = wsum(acc);
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
        const double t = block_sum_fixed(acc, red);
        const double inv = t > 0.0 ? 1.0 / sqrt(t) : 0.0;
        for (int i = tid; i < n; i += blockDim.x) zj[i] *= inv;
        __syncthreads();
    }
}

// T (nb x nb, upper) of the compact WY form of nb reflectors from G = V'V (dlarft,
// forward, columnwise): T_jj = tau_j, T(0:j, j) = -tau_j T(0:j, 0:j) G(0:j, j)
__global__ void k_wy_t(const double* __restrict__ G, const double* __restrict__ tau, int nb, double* T) {
    FQB_PDL_ENTRY();
    __shared__ double tsm[kWyBlock][kWyBlock];
    const int r = threadIdx.x;   // one thread per row
    for (int c = 0; c < nb; ++c) tsm[r][c] = 0.0;
    __syncthreads();
    for (int j = 0; j < nb; ++j) {
        if (r < j) {
            double acc = 0.0;
            for (int q = r; q < j; ++q) acc = fma(tsm[r][q], G[q + j * nb], acc);
            tsm[r][j] = -tau[j] * acc;
        } else if (r == j) {
            tsm[r][j] = tau[j];
        }
        __syncthreads();
    }
    for (int c = 0; c < nb; ++c) T[r + c * nb] = tsm[r][c];
}

__global__ void k_ns_coef_l(double* g, int n) {
    FQB_PDL_ENTRY();
    const int i = blockIdx.x * blockDim.x + threadIdx.x, j = blockIdx.y;
    if (i < n) g[int64_t(j) * n + i] = (i == j ? 1.5 : 0.0) - 0.5 * g[int64_t(j) * n + i];
}

// per-CTA partials of |R - X diag(w)|^2, |M|^2, |O - I|^2 (fixed order), summed on the host
__global__ void __launch_bounds__(256) k_check_l(const double* __restrict__ r, const double* __restrict__ x,
                                                 const double* __restrict__ w, const double* __restrict__ mat,
                                                 const double* __restrict__ o, int n, double* part) {
    FQB_PDL_ENTRY();
    __shared__ double red[33];
    const int j = blockIdx.y;
    double a = 0.0, b = 0.0, c = 0.0;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        const int64_t e = int64_t(j) * n + i;
        const double res = r[e] - x[e] * w[j];
        a = fma(res, res, a);
        b = fma(mat[e], mat[e], b);
        const double oe = o[e] - (i == j ? 1.0 : 0.0);
        c = fma(oe, oe, c);
    }
    a = block_sum_fixed(a, red);
    b = block_sum_fixed(b, red);
    c = block_sum_fixed(c, red);
    if (threadIdx.x == 0) {
        double* p = part + 3 * (int64_t(j) * gridDim.x + blockIdx.x);
        p[0] = a;
        p[1] = b;
        p[2] = c;
    }
}

}  // namespace

bool large_eigh(Handle& h, const double* mat, int n, double* w, double* x) {
    if (n < 3 || n > kLargeEighMax) return false;
    cudaStream_t s = h.stream;
    ensure_gemm_workspace(h);
    const int G = h.num_sms;
    const size_t nn = size_t(n) * n;
    DeviceArray<double> A, V, P, S, d, e, tau, z, z1, g, r, scr, T, W, W2, part;
    DeviceArray<unsigned> piv;
    A.ensure(nn, s);
    V.ensure(nn, s);
    P.ensure(size_t(2) * n, s);
    S.ensure(size_t(2) * G, s);
    d.ensure(size_t(n), s);
    e.ensure(size_t(n), s);
    tau.ensure(size_t(n), s);
    FQB_CUDA(cudaMemcpyAsync(A.ptr, mat, sizeof(double) * nn, cudaMemcpyDeviceToDevice, s));
    // 1. tridiagonalisation (cooperative: all G CTAs resident, one per SM)
    {
        static std::mutex mu;
        static bool configured[64] = {};
        int dev = 0;
        FQB_CUDA(cudaGetDevice(&dev));
        std::lock_guard<std::mutex> lock(mu);
        if (dev < 0 || dev >= 64 || !configured[dev]) {
            FQB_CUDA(cudaFuncSetAttribute(k_trd_coop, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                          int(sizeof(double) * 2 * kLargeEighMax)));
            if (dev >= 0 && dev < 64) configured[dev] = true;
        }
    }
    TrdArgs ta{A.ptr, n, d.ptr, e.ptr, tau.ptr, V.ptr, P.ptr, S.ptr};
    void* args[] = {&ta};
    FQB_CUDA(cudaLaunchCooperativeKernel(reinterpret_cast<void*>(k_trd_coop), dim3(unsigned(G)),
                                         dim3(kTrdThreads), args, sizeof(double) * 2 * size_t(n), s));
    FQB_LAUNCHED();
    h.lc.bump();
    // 2. eigenvalues: Gerschgorin bounds on the host (d, e are 2n doubles)
    std::vector<double> hd(n), he(n);
    FQB_CUDA(cudaMemcpyAsync(hd.data(), d.ptr, sizeof(double) * n, cudaMemcpyDeviceToHost, s));
    FQB_CUDA(cudaMemcpyAsync(he.data(), e.ptr, sizeof(double) * (n - 1), cudaMemcpyDeviceToHost, s));
    FQB_CUDA(cudaStreamSynchronize(s));
    double gl = INFINITY, gu = -INFINITY, emax2 = 0.0, tn = 0.0;
    for (int i = 0; i < n; ++i) {
        const double el = i > 0 ? std::fabs(he[i - 1]) : 0.0, er = i + 1 < n ? std::fabs(he[i]) : 0.0;
        gl = std::fmin(gl, hd[i] - el - er);
        gu = std::fmax(gu, hd[i] + el + er);
        if (i + 1 < n) emax2 = std::fmax(emax2, he[i] * he[i]);
        tn = std::fmax(tn, std::fabs(hd[i]) + el + er);
    }
    if (!std::isfinite(gl) || !std::isfinite(gu)) return false;
    const double u = 1.1102230246251565e-16;
    const double pivmin = 2.2250738585072014e-308 * std::fmax(1.0, emax2);
    const double span = std::fmax(std::fabs(gl), std::fabs(gu));
    gl -= 2.0 * u * span * n + 2.0 * pivmin;
    gu += 2.0 * u * span * n + 2.0 * pivmin;
    const size_t bsm = sizeof(double) * 2 * size_t(n);
    if (bsm > 48 * 1024) FQB_CUDA(cudaFuncSetAttribute(k_bisect_large, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                      int(bsm)));
    launch_k(k_bisect_large, unsigned(ceil_div(n, 8)), 256, bsm, s, d.ptr, e.ptr, n, gl, gu, pivmin, w);
    FQB_LAUNCHED();
    // 3. eigenvectors of T
    const int it = 128, ib = int(ceil_div(n, it));
    scr.ensure(size_t(5) * n * size_t(ib * it), s);
    piv.ensure(size_t(n) * ((n + 31) / 32), s);
    z.ensure(nn, s);
    launch_k(k_invit_large, unsigned(ib), unsigned(it), 0, s, d.ptr, e.ptr, w, n, tn, scr.ptr, piv.ptr, z.ptr);
    FQB_LAUNCHED();
    launch_k(k_cluster_mgs_large, unsigned(n), 256, 0, s, w, n, 1e-11 * tn, z.ptr);
    FQB_LAUNCHED();
    h.lc.bump(3);
    scr.release();
    piv.release();
    // two Newton-Schulz steps: Z <- Z (1.5 I - 0.5 Z'Z)
    g.ensure(nn, s);
    z1.ensure(nn, s);
    double* cur = z.ptr;
    double* nxt = z1.ptr;
    for (int k = 0; k < 2; ++k) {
        gemm(true, n, n, n, 1.0, cur, n, cur, n, 0.0, g.ptr, n, h.gws, h.num_sms, s, h.lc);
        launch_k(k_ns_coef_l, dim3(unsigned(ceil_div(n, 256)), unsigned(n)), 256, 0, s, g.ptr, n);
        FQB_LAUNCHED();
        h.lc.bump();
        gemm(false, n, n, n, 1.0, cur, n, g.ptr, n, 0.0, nxt, n, h.gws, h.num_sms, s, h.lc);
        std::swap(cur, nxt);
    }
    // 4. X = H_0 ... H_{n-3} Z, blocks of kWyBlock reflectors from the last one back
    const int nref = n - 2;
    T.ensure(size_t(kWyBlock) * kWyBlock, s);
    W.ensure(size_t(kWyBlock) * n, s);
    W2.ensure(size_t(kWyBlock) * n, s);
    DeviceArray<double> Gs;
    Gs.ensure(size_t(kWyBlock) * kWyBlock, s);
    for (int k0 = ((nref - 1) / kWyBlock) * kWyBlock; k0 >= 0; k0 -= kWyBlock) {
        const int nb = std::min(kWyBlock, nref - k0);
        const int r0 = k0 + 1;   // first row any of these reflectors touches
        const int rows = n - r0;
        const double* Vb = V.ptr + int64_t(k0) * n + r0;   // rows r0.. of columns k0 .. k0+nb-1
        gemm(true, nb, nb, rows, 1.0, Vb, n, Vb, n, 0.0, Gs.ptr, nb, h.gws, h.num_sms, s, h.lc);
        launch_k(k_wy_t, 1, unsigned(nb), 0, s, Gs.ptr, tau.ptr + k0, nb, T.ptr);
        FQB_LAUNCHED();
        h.lc.bump();
        // W = V' Z (nb x n), W2 = T W, Z -= V W2
        gemm(true, nb, n, rows, 1.0, Vb, n, cur + r0, n, 0.0, W.ptr, nb, h.gws, h.num_sms, s, h.lc);
        gemm(false, nb, n, nb, 1.0, T.ptr, nb, W.ptr, nb, 0.0, W2.ptr, nb, h.gws, h.num_sms, s, h.lc);
        gemm(false, rows, n, nb, -1.0, Vb, n, W2.ptr, nb, 1.0, cur + r0, n, h.gws, h.num_sms, s, h.lc);
    }
    // a-posteriori check: R = M X, O = X'X
    r.ensure(nn, s);
    gemm(false, n, n, n, 1.0, mat, n, cur, n, 0.0, r.ptr, n, h.gws, h.num_sms, s, h.lc);
    gemm(true, n, n, n, 1.0, cur, n, cur, n, 0.0, g.ptr, n, h.gws, h.num_sms, s, h.lc);
    const int cb = 4;
    part.ensure(size_t(3) * n * cb, s);
    launch_k(k_check_l, dim3(unsigned(cb), unsigned(n)), 256, 0, s, r.ptr, cur, w, mat, g.ptr, n, part.ptr);
    FQB_LAUNCHED();
    h.lc.bump();
    std::vector<double> hp(size_t(3) * n * cb);
    FQB_CUDA(cudaMemcpyAsync(hp.data(), part.ptr, sizeof(double) * hp.size(), cudaMemcpyDeviceToHost, s));
    FQB_CUDA(cudaStreamSynchronize(s));
    double hs[3] = {0.0, 0.0, 0.0};
    for (size_t q = 0; q < hp.size(); q += 3)
        for (int t = 0; t < 3; ++t) hs[t] += hp[q + t];
    const double res = std::sqrt(hs[0]), mnorm = std::sqrt(hs[1]), orth = std::sqrt(hs[2]);
    const bool ok = std::isfinite(res) && std::isfinite(orth) && res <= 64.0 * n * u * mnorm && orth <= 64.0 * n * u;
    if (const char* dbg = std::getenv("FQB_EIG_DEBUG"))
        if (dbg[0] == '1')
            std::fprintf(stderr, "large_eigh n=%d: residual %.3e (|M| %.3e), orthogonality %.3e -> %s\n", n, res, mnorm,
                         orth, ok ? "ok" : "fallback");
    if (!ok) return false;
    FQB_CUDA(cudaMemcpyAsync(x, cur, sizeof(double) * nn, cudaMemcpyDeviceToDevice, s));
    FQB_CUDA(cudaStreamSynchronize(s));   // the temporaries are released on return
    return true;
}

}  // namespace farqb
