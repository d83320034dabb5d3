// detgen.cu -- the deterministic low-rank test-matrix generator (BASELINE configs 3-5).
//
//   A = X diag(sigma) Y' + noise_scale * G,  X = Q(QR(X0)), Y = Q(QR(Y0)),
//   X0 / Y0 / G Philox Gaussians (seed; streams 0xFA000001 / 0xFA000002 / 0xFA000003,
//   keyed by column) through the libm-free Box-Muller of include/farqb/detmath.h.
//
// Bit-identical to its host twin oracle/detgen.c (fqo_det_lowrank): every product
// is an fma chain over k ascending from +0.0, the QR is CholeskyQR with a
// right-looking Cholesky (one fma per trailing element and step) and R^-1 formed
// column by column.  That is what lets the unmodified CPU reference run on the
// same 16 GB matrix the B200 factorizes (tests/golden/c4.json) without shipping
// it: both sides rebuild it from the seed, and fqb_checksum proves they agree.
//
// Rows [row0, row0 + rows) only: a rank of a row-sharded run makes its own slab
// (the factor Grams still run over all rows, so every slab is bit-equal to the
// same rows of the whole).  The products run on the FP64 FMA pipe (34 TFLOP/s),
// not DMMA, whose internal accumulation order is not the sequential chain.
#include <cmath>
#include <vector>

#include "../../include/farqb/detmath.h"
#include "engine.hpp"
#include "kernels.hpp"
#include "philox.cuh"

namespace farqb {
namespace {

constexpr uint32_t kStreamX = 0xFA000001u;
constexpr uint32_t kStreamY = 0xFA000002u;
constexpr uint32_t kStreamNoise = 0xFA000003u;

__device__ __forceinline__ double det_gauss(PhiloxKey key, uint32_t stream, uint32_t col, int64_t i) {
    const uint4 o = philox_block(key, stream, col, uint64_t(i) >> 1);
    double z0, z1;
    fqd_box_muller(unit_from_words(o.x, o.y), unit_from_words(o.z, o.w), &z0, &z1);
    return (i & 1) ? z1 : z0;
}

__global__ void k_det_gauss(PhiloxKey key, uint32_t stream, int64_t len, int r, double* out, int64_t ld) {
    FQB_PDL_ENTRY();
    const int64_t pair = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    const int j = blockIdx.y;
    if (2 * pair >= len || j >= r) return;
    const uint4 o = philox_block(key, stream, uint32_t(j), uint64_t(pair));
    double z0, z1;
    fqd_box_muller(unit_from_words(o.x, o.y), unit_from_words(o.z, o.w), &z0, &z1);
    double* c = out + int64_t(j) * ld;
    c[2 * pair] = z0;
    if (2 * pair + 1 < len) c[2 * pair + 1] = z1;
}

// C (M x N) = sum_k a(i,k) b(k,j), k ascending, one fma per k from +0.0.
// a(i,k) = TA ? A[k + i lda] : A[i + k lda];  b(k,j) = TB ? B[j + k ldb] : B[k + j ldb].
// 64 x 64 tile, 256 threads of 4 x 4, 16-deep k chunks through shared memory.
// Epilogue: C += noise_scale * G(row0 + i, j) when noise_scale != 0.
constexpr int kBM = 64, kBN = 64, kBK = 16;

template <bool TA, bool TB>
__global__ void __launch_bounds__(256) k_det_gemm(int64_t M, int64_t N, int64_t K, const double* __restrict__ A,
                                                  int64_t lda, const double* __restrict__ B, int64_t ldb,
                                                  double* __restrict__ C, int64_t ldc, double noise_scale,
                                                  PhiloxKey key, int64_t row0) {
    FQB_PDL_ENTRY();
    __shared__ __align__(16) double As[kBK][kBM];
    __shared__ __align__(16) double Bs[kBK][kBN];
    const int tid = threadIdx.x;
    const int tr = tid & 15, tc = tid >> 4;
    const int64_t i0 = int64_t(blockIdx.x) * kBM, j0 = int64_t(blockIdx.y) * kBN;
    double acc[4][4];
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int b = 0; b < 4; ++b) acc[a][b] = 0.0;
    for (int64_t k0 = 0; k0 < K; k0 += kBK) {
        const int kc = int(K - k0 < kBK ? K - k0 : kBK);
        // 1024 elements of each tile, 4 per thread, coalesced along the contiguous index
#pragma unroll
        for (int t = 0; t < 4; ++t) {
            const int e = tid + t * 256;
            int ii, kk;
            if (TA) { kk = e & 15; ii = e >> 4; } else { ii = e & 63; kk = e >> 6; }
            const int64_t gi = i0 + ii, gk = k0 + kk;
            double v = 0.0;
            if (gi < M && kk < kc) v = TA ? A[gk + gi * lda] : A[gi + gk * lda];
            As[kk][ii] = v;
            int jj;
            if (TB) { jj = e & 63; kk = e >> 6; } else { kk = e & 15; jj = e >> 4; }
            const int64_t gj = j0 + jj, gk2 = k0 + kk;
            double w = 0.0;
            if (gj < N && kk < kc) w = TB ? B[gj + gk2 * ldb] : B[gk2 + gj * ldb];
            Bs[kk][jj] = w;
        }
        __syncthreads();
        for (int kk = 0; kk < kc; ++kk) {
            const double2 a01 = *reinterpret_cast<const double2*>(&As[kk][tr * 4]);
            const double2 a23 = *reinterpret_cast<const double2*>(&As[kk][tr * 4 + 2]);
            const double2 b01 = *reinterpret_cast<const double2*>(&Bs[kk][tc * 4]);
            const double2 b23 = *reinterpret_cast<const double2*>(&Bs[kk][tc * 4 + 2]);
            const double av[4] = {a01.x, a01.y, a23.x, a23.y};
            const double bv[4] = {b01.x, b01.y, b23.x, b23.y};
#pragma unroll
            for (int a = 0; a < 4; ++a)
#pragma unroll
                for (int b = 0; b < 4; ++b) acc[a][b] = __fma_rn(av[a], bv[b], acc[a][b]);
        }
        __syncthreads();
    }
#pragma unroll
    for (int b = 0; b < 4; ++b) {
        const int64_t j = j0 + tc * 4 + b;
        if (j >= N) continue;
#pragma unroll
        for (int a = 0; a < 4; ++a) {
            const int64_t i = i0 + tr * 4 + a;
            if (i >= M) continue;
            double v = acc[a][b];
            if (noise_scale != 0.0)
                v = __dadd_rn(v, __dmul_rn(noise_scale, det_gauss(key, kStreamNoise, uint32_t(j), row0 + i)));
            C[i + j * ldc] = v;
        }
    }
}

// One right-looking Cholesky step k on the upper triangle of S (r x r):
// S_ij = fma(-R_ki, R_kj, S_ij) for k < i <= j, R_kx = S_kx / sqrt(S_kk).
__global__ void k_det_chol_step(double* S, int r, int k) {
    FQB_PDL_ENTRY();
    const int i = k + 1 + int(blockIdx.x) * 16 + int(threadIdx.x);
    const int j = k + 1 + int(blockIdx.y) * 16 + int(threadIdx.y);
    if (i > j || j >= r) return;
    const double rkk = __dsqrt_rn(S[k + int64_t(k) * r]);
    const double rki = __ddiv_rn(S[k + int64_t(i) * r], rkk);
    const double rkj = __ddiv_rn(S[k + int64_t(j) * r], rkk);
    double* p = S + i + int64_t(j) * r;
    *p = __fma_rn(-rki, rkj, *p);
}

// R (upper, zero below) from the factored S: R_kk = sqrt(S_kk), R_kj = S_kj / R_kk
__global__ void k_det_chol_finish(const double* S, int r, double* R) {
    FQB_PDL_ENTRY();
    const int k = int(blockIdx.x) * 16 + int(threadIdx.x);
    const int j = int(blockIdx.y) * 16 + int(threadIdx.y);
    if (k >= r || j >= r) return;
    double v = 0.0;
    if (k <= j) {
        const double rkk = __dsqrt_rn(S[k + int64_t(k) * r]);
        v = (k == j) ? rkk : __ddiv_rn(S[k + int64_t(j) * r], rkk);
    }
    R[k + int64_t(j) * r] = v;
}

// Ri = R^-1 (upper), one thread per column: Ri_jj = 1 / R_jj, then for i = j-1..0
// Ri_ij = -(sum_{k=i+1..j} R_ik Ri_kj) / R_ii, the sum an fma chain in k.
__global__ void k_det_upper_inv(const double* R, int r, double* Ri) {
    FQB_PDL_ENTRY();
    const int j = int(blockIdx.x) * blockDim.x + int(threadIdx.x);
    if (j >= r) return;
    double* cj = Ri + int64_t(j) * r;
    for (int i = j + 1; i < r; ++i) cj[i] = 0.0;
    cj[j] = __ddiv_rn(1.0, R[j + int64_t(j) * r]);
    for (int i = j - 1; i >= 0; --i) {
        double acc = 0.0;
        for (int k = i + 1; k <= j; ++k) acc = __fma_rn(R[i + int64_t(k) * r], cj[k], acc);
        cj[i] = __ddiv_rn(-acc, R[i + int64_t(i) * r]);
    }
}

__global__ void k_det_scale_cols(double* y, int64_t n, int r, const double* sigma) {
    FQB_PDL_ENTRY();
    const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    const int k = blockIdx.y;
    if (i >= n || k >= r) return;
    y[i + k * n] = __dmul_rn(y[i + k * n], sigma[k]);
}

__device__ __forceinline__ uint64_t mix64(uint64_t z) {
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}

__global__ void k_checksum(const double* a, int64_t rows, int64_t cols, int64_t lda, int64_t row0, int64_t m_total,
                           unsigned long long* out) {
    FQB_PDL_ENTRY();
    uint64_t h = 0;
    const int64_t total = rows * cols;
    for (int64_t e = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; e < total;
         e += int64_t(gridDim.x) * blockDim.x) {
        const int64_t j = e / rows, i = e - j * rows;
        const uint64_t bits = uint64_t(__double_as_longlong(a[i + j * lda]));
        const uint64_t idx = uint64_t(j * m_total + row0 + i);
        h += mix64(bits ^ (idx * 0x9E3779B97F4A7C15ULL));
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) h += __shfl_xor_sync(0xffffffffu, h, off);
    if ((threadIdx.x & 31) == 0) atomicAdd(out, (unsigned long long)h);
}

template <bool TA, bool TB>
void det_gemm(Handle& h, int64_t M, int64_t N, int64_t K, const double* A, int64_t lda, const double* B, int64_t ldb,
              double* C, int64_t ldc, double noise_scale = 0.0, uint64_t seed = 0, int64_t row0 = 0) {
    if (M <= 0 || N <= 0) return;
    const dim3 g(unsigned(ceil_div(M, kBM)), unsigned(ceil_div(N, kBN)));
    launch_k(k_det_gemm<TA, TB>, g, 256, 0, h.stream, M, N, K, A, lda, B, ldb, C, ldc, noise_scale,
             philox_key(seed), row0);
    FQB_LAUNCHED();
    h.lc.bump();
}

// rows [row0, row0 + rows) of Q(QR(F0)), F0 the len x r Gaussian of (seed, stream)
void det_factor(Handle& h, int64_t len, int r, uint64_t seed, uint32_t stream, int64_t row0, int64_t rows,
                double* out, int64_t ldo) {
    cudaStream_t s = h.stream;
    DeviceArray<double> f0, g, R, Ri;
    f0.ensure(size_t(len) * r, s);
    g.ensure(size_t(r) * r, s);
    R.ensure(size_t(r) * r, s);
    Ri.ensure(size_t(r) * r, s);
    launch_k(k_det_gauss, dim3(unsigned(ceil_div((len + 1) / 2, 256)), unsigned(r)), 256, 0, s, philox_key(seed),
             stream, len, r, f0.ptr, len);
    FQB_LAUNCHED();
    det_gemm<true, false>(h, r, r, len, f0.ptr, len, f0.ptr, len, g.ptr, r);
    for (int k = 0; k + 1 < r; ++k) {
        const int t = r - k - 1;
        launch_k(k_det_chol_step, dim3(unsigned(ceil_div(t, 16)), unsigned(ceil_div(t, 16))), dim3(16, 16), 0, s,
                 g.ptr, r, k);
        FQB_LAUNCHED();
    }
    launch_k(k_det_chol_finish, dim3(unsigned(ceil_div(r, 16)), unsigned(ceil_div(r, 16))), dim3(16, 16), 0, s,
             g.ptr, r, R.ptr);
    FQB_LAUNCHED();
    launch_k(k_det_upper_inv, dim3(unsigned(ceil_div(r, 32))), 32, 0, s, R.ptr, r, Ri.ptr);
    FQB_LAUNCHED();
    h.lc.bump(r + 3);
    det_gemm<false, false>(h, rows, r, r, f0.ptr + row0, len, Ri.ptr, r, out, ldo);
    // f0 / g / R / Ri are freed stream-ordered when they go out of scope
}

}  // namespace

void gen_lowrank_det_dev(Handle& h, int64_t m, int64_t n, int r, const double* sigma_host, uint64_t seed,
                         double noise_scale, int64_t row0, int64_t rows, double* a, int64_t lda) {
    if (m < 1 || n < 1 || r < 1 || r > m || r > n || row0 < 0 || rows < 0 || row0 + rows > m || lda < rows)
        throw Error(kStatusConfig, "gen_lowrank_det: need 1 <= r <= min(m, n), 0 <= row0 <= row0 + rows <= m, "
                                   "lda >= rows");
    if (rows == 0) return;
    cudaStream_t s = h.stream;
    DeviceArray<double> x, y, sig;
    x.ensure(size_t(rows) * r, s);
    y.ensure(size_t(n) * r, s);
    sig.ensure(size_t(r), s);
    FQB_CUDA(cudaMemcpyAsync(sig.ptr, sigma_host, sizeof(double) * r, cudaMemcpyHostToDevice, s));
    det_factor(h, m, r, seed, kStreamX, row0, rows, x.ptr, rows);
    det_factor(h, n, r, seed, kStreamY, 0, n, y.ptr, n);
    launch_k(k_det_scale_cols, dim3(unsigned(ceil_div(n, 256)), unsigned(r)), 256, 0, s, y.ptr, n, r, sig.ptr);
    FQB_LAUNCHED();
    h.lc.bump();
    det_gemm<false, true>(h, rows, n, r, x.ptr, rows, y.ptr, n, a, lda, noise_scale, seed, row0);
    FQB_CUDA(cudaStreamSynchronize(s));   // sigma_host must outlive the copy
}

uint64_t checksum_dev(Handle& h, const double* a, int64_t rows, int64_t cols, int64_t lda, int64_t row0,
                      int64_t m_total) {
    cudaStream_t s = h.stream;
    DeviceArray<unsigned long long> acc;
    acc.ensure(1, s);
    FQB_CUDA(cudaMemsetAsync(acc.ptr, 0, sizeof(unsigned long long), s));
    if (rows > 0 && cols > 0) {
        launch_k(k_checksum, dim3(unsigned(h.num_sms * 8)), 256, 0, s, a, rows, cols, lda, row0, m_total, acc.ptr);
        FQB_LAUNCHED();
        h.lc.bump();
    }
    unsigned long long out = 0;
    FQB_CUDA(cudaMemcpyAsync(&out, acc.ptr, sizeof out, cudaMemcpyDeviceToHost, s));
    FQB_CUDA(cudaStreamSynchronize(s));
    return out;
}

}  // namespace farqb
