// synthetic.cu -- test matrices generated on the device.
//
//  random_orthonormal (reference: synthetic.cpp:121-126, orthonormalize :56-67,
//      bcgs2_step :36-53): panels of 64 Philox Gaussian columns (stream-keyed:
//      Philox(seed, stream, column), the reference's factor streams 0xFA000001 /
//      0xFA000002), each made orthogonal to the columns before it and to itself by
//      two rounds of block Gram-Schmidt + CholeskyQR -- the same algorithm on the
//      DMMA GEMM and the b x b Cholesky kernel.  Equal to the reference to FP64
//      rounding (the Gaussians themselves to ~4 ulp, CUDA vs glibc libm).
//  gen_synthetic (synthetic.cpp:159-180): A = U diag(sigma) V' with the reference's
//      spectra (1/j^2, e^{-j/20}; sigma < 1e-18 sigma_1 dropped) and block-diagonal
//      V for the stability kind.
//  gen_lowrank: the rectangular low-rank-plus-noise inputs of BASELINE configs 2-5,
//      A = U diag(sigma) V' + noise N(0,1)/sqrt(n), noise on stream 0xFA000003 keyed
//      by column (SURVEY.md section 8(d) seed convention).
#include <cmath>
#include <vector>

#include "engine.hpp"
#include "kernels.hpp"
#include "philox.cuh"

namespace farqb {
namespace {

constexpr uint32_t kStreamU = 0xFA000001u;
constexpr uint32_t kStreamV = 0xFA000002u;
constexpr uint32_t kStreamNoise = 0xFA000003u;
constexpr int kPanel = 64;

// out[:, j] (+)= scale * next_gaussian() sequence of Philox(seed, stream, col0 + j)
__global__ void k_gauss_cols(PhiloxKey key, uint32_t stream, int64_t n, int col0, int w, double scale, int accumulate,
                             double* out, int64_t ld) {
    FQB_PDL_ENTRY();
    const int64_t pairs = (n + 1) >> 1;
    const int64_t idx = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    const int j = blockIdx.y;
    if (idx >= pairs || j >= w) return;
    const uint4 o = philox_block(key, stream, uint32_t(col0 + j), uint64_t(idx));
    double z0, z1;
    box_muller(unit_from_words(o.x, o.y), unit_from_words(o.z, o.w), z0, z1);
    double* c = out + int64_t(j) * ld;
    const int64_t i = 2 * idx;
    if (accumulate) {
        c[i] += scale * z0;
        if (i + 1 < n) c[i + 1] += scale * z1;
    } else {
        c[i] = scale * z0;
        if (i + 1 < n) c[i + 1] = scale * z1;
    }
}

// out (cols x rows, ldo) = (in diag(col_scale))' for in rows x cols (ldi); col_scale may be null
__global__ void k_transpose(const double* __restrict__ in, int64_t ldi, int64_t rows, int64_t cols,
                            const double* __restrict__ col_scale, double* __restrict__ out, int64_t ldo) {
    FQB_PDL_ENTRY();
    __shared__ double t[32][33];
    const int64_t r0 = int64_t(blockIdx.x) * 32, c0 = int64_t(blockIdx.y) * 32;
    for (int k = threadIdx.y; k < 32; k += blockDim.y) {
        const int64_t r = r0 + threadIdx.x, c = c0 + k;
        t[k][threadIdx.x] = (r < rows && c < cols) ? in[c * ldi + r] * (col_scale ? col_scale[c] : 1.0) : 0.0;
    }
    __syncthreads();
    for (int k = threadIdx.y; k < 32; k += blockDim.y) {
        const int64_t c = c0 + threadIdx.x, r = r0 + k;   // out[c][r] = in[r][c]
        if (r < rows && c < cols) out[r * ldo + c] = t[threadIdx.x][k];
    }
}

void gauss_cols(Handle& h, uint64_t seed, uint32_t stream, int64_t n, int col0, int w, double scale, bool acc,
                double* out, int64_t ld) {
    if (n <= 0 || w <= 0) return;
    const dim3 g(unsigned(ceil_div((n + 1) / 2, 256)), unsigned(w));
    launch_k(k_gauss_cols, g, 256, 0, h.stream, philox_key(seed), stream, n, col0, w, scale, acc ? 1 : 0, out, ld);
    h.lc.bump();
}

// dst (cols x rows, ldd) = (src (rows x cols, lds) diag(scale))'
void transpose(Handle& h, const double* src, int64_t lds, int64_t rows, int64_t cols, const double* scale,
               double* dst, int64_t ldd) {
    if (rows <= 0 || cols <= 0) return;
    const dim3 g(unsigned(ceil_div(rows, 32)), unsigned(ceil_div(cols, 32)));
    launch_k(k_transpose, g, dim3(32, 8), 0, h.stream, src, lds, rows, cols, scale, dst, ldd);
    h.lc.bump();
}

}  // namespace

// q (n x r, ld) <- orthonormal basis of the Philox Gaussian panels (bcgs2_step, synthetic.cpp:36-53)
void random_orthonormal_dev(Handle& h, int64_t n, int r, uint64_t seed, uint32_t stream, int first_col, double* q,
                            int64_t ldq) {
    if (r < 1 || n < r) throw Error(kStatusConfig, "random_orthonormal: need 1 <= r <= n");
    cudaStream_t s = h.stream;
    ensure_gemm_workspace(h);
    DeviceArray<double> c, g, R, Ri, t, scratch;
    DeviceArray<unsigned> st;
    c.ensure(size_t(r) * kPanel, s);
    g.ensure(size_t(kPanel) * kPanel, s);
    R.ensure(size_t(kPanel) * kPanel, s);
    Ri.ensure(size_t(kPanel) * kPanel, s);
    t.ensure(size_t(n) * kPanel, s);
    scratch.ensure(size_t(kPanel) * (kPanel + 1), s);
    st.ensure(1, s);
    FQB_CUDA(cudaMemsetAsync(st.ptr, 0, sizeof(unsigned), s));
    for (int s0 = 0; s0 < r; s0 += kPanel) {
        const int w = std::min(kPanel, r - s0);
        double* p = q + int64_t(s0) * ldq;
        gauss_cols(h, seed, stream, n, first_col + s0, w, 1.0, false, p, ldq);
        for (int pass = 0; pass < 2; ++pass) {
            if (s0 > 0) {   // P -= Q (Q' P)
                gemm(true, s0, w, n, 1.0, q, ldq, p, ldq, 0.0, c.ptr, s0, h.gws, h.num_sms, s, h.lc);
                gemm(false, n, w, s0, -1.0, q, ldq, c.ptr, s0, 1.0, p, ldq, h.gws, h.num_sms, s, h.lc);
            }
            // CholeskyQR: P <- P R^-1, R' R = P' P
            gemm(true, w, w, n, 1.0, p, ldq, p, ldq, 0.0, g.ptr, w, h.gws, h.num_sms, s, h.lc);
            launch_chol_upper_inv(g.ptr, w, w, 0.0, 0.0, nullptr, 0, R.ptr, Ri.ptr, nullptr, scratch.ptr, st.ptr, 1u,
                                  s, h.lc);
            gemm(false, n, w, w, 1.0, p, ldq, Ri.ptr, w, 0.0, t.ptr, n, h.gws, h.num_sms, s, h.lc);
            FQB_CUDA(cudaMemcpy2DAsync(p, ldq * sizeof(double), t.ptr, n * sizeof(double), n * sizeof(double), w,
                                       cudaMemcpyDeviceToDevice, s));
        }
    }
    unsigned hst = 0;
    FQB_CUDA(cudaMemcpyAsync(&hst, st.ptr, sizeof(unsigned), cudaMemcpyDeviceToHost, s));
    FQB_CUDA(cudaStreamSynchronize(s));
    if (hst) throw Error(kStatusDegenerate, "random_orthonormal: Gaussian panel lost rank (Cholesky failed)");
}

std::vector<double> synthetic_spectrum(int kind, int n) {
    std::vector<double> sig(size_t(std::max(n, 0)));
    for (int j = 1; j <= n; ++j) sig[size_t(j - 1)] = kind == 1 ? std::exp(-double(j) / 20.0) : 1.0 / (double(j) * j);
    return sig;
}

// A (m x n, lda) = U diag(sigma) V' (+ noise): U m x r, V n x r orthonormal (streams U, V)
static void assemble_lowrank(Handle& h, const double* u, int64_t ldu, const double* sig_host, int r, const double* v,
                             int64_t ldv, int64_t m, int64_t n, double* a, int64_t lda) {
    cudaStream_t s = h.stream;
    DeviceArray<double> sig, vt;
    sig.ensure(size_t(r), s);
    vt.ensure(size_t(r) * n, s);
    FQB_CUDA(cudaMemcpyAsync(sig.ptr, sig_host, sizeof(double) * r, cudaMemcpyHostToDevice, s));
    transpose(h, v, ldv, n, r, sig.ptr, vt.ptr, r);   // vt (r x n) = (V diag(sigma))'
    gemm(false, m, n, r, 1.0, u, ldu, vt.ptr, r, 0.0, a, lda, h.gws, h.num_sms, s, h.lc);
    FQB_CUDA(cudaStreamSynchronize(s));   // sig / vt are host-scoped
}

int gen_synthetic_dev(Handle& h, int kind, int n, int d, uint64_t seed, double* a, int64_t lda) {
    if (n < 1) throw Error(kStatusConfig, "gen_synthetic: n must be positive");
    if (kind < 0 || kind > 2) throw Error(kStatusConfig, "gen_synthetic: unknown kind");
    if (lda < n) throw Error(kStatusDimension, "gen_synthetic: lda < n");
    std::vector<double> sig = synthetic_spectrum(kind, n);
    int r = n;
    while (r > 1 && sig[size_t(r - 1)] < sig[0] * 1e-18) --r;
    sig.resize(size_t(r));
    cudaStream_t s = h.stream;
    DeviceArray<double> u, v;
    u.ensure(size_t(n) * r, s);
    random_orthonormal_dev(h, n, r, seed, kStreamU, 0, u.ptr, n);
    if (kind == 2) {
        // block-diagonal V: d blocks of nb x nb orthonormal Gaussians (stream V, first column bs)
        if (d < 1 || n % d != 0) throw Error(kStatusConfig, "gen_synthetic: d must divide n");
        const int nb = n / d;
        DeviceArray<double> blk, sigd, mt;
        blk.ensure(size_t(nb) * nb, s);
        mt.ensure(size_t(nb) * nb, s);
        sigd.ensure(size_t(n), s);
        FQB_CUDA(cudaMemcpyAsync(sigd.ptr, sig.data(), sizeof(double) * n, cudaMemcpyHostToDevice, s));
        for (int i = 0; i < d; ++i) {
            const int bs = i * nb;
            random_orthonormal_dev(h, nb, nb, seed, kStreamV, bs, blk.ptr, nb);
            // A[:, bs:bs+nb] = U[:, bs:bs+nb] diag(sigma_blk) blk' = U_blk (blk diag(sigma_blk))'
            transpose(h, blk.ptr, nb, nb, nb, sigd.ptr + bs, mt.ptr, nb);
            gemm(false, n, nb, nb, 1.0, u.ptr + int64_t(bs) * n, n, mt.ptr, nb, 0.0, a + int64_t(bs) * lda, lda,
                 h.gws, h.num_sms, s, h.lc);
        }
        FQB_CUDA(cudaStreamSynchronize(s));
        return r;
    }
    v.ensure(size_t(n) * r, s);
    random_orthonormal_dev(h, n, r, seed, kStreamV, 0, v.ptr, n);
    assemble_lowrank(h, u.ptr, n, sig.data(), r, v.ptr, n, n, n, a, lda);
    return r;
}

void gen_lowrank_dev(Handle& h, int64_t m, int64_t n, int r, const double* sigma, uint64_t seed, double noise,
                     double* a, int64_t lda) {
    if (r < 1 || r > std::min(m, n)) throw Error(kStatusConfig, "gen_lowrank: need 1 <= r <= min(m, n)");
    if (lda < m) throw Error(kStatusDimension, "gen_lowrank: lda < m");
    cudaStream_t s = h.stream;
    DeviceArray<double> u, v;
    u.ensure(size_t(m) * r, s);
    v.ensure(size_t(n) * r, s);
    random_orthonormal_dev(h, m, r, seed, kStreamU, 0, u.ptr, m);
    random_orthonormal_dev(h, n, r, seed, kStreamV, 0, v.ptr, n);
    assemble_lowrank(h, u.ptr, m, sigma, r, v.ptr, n, m, n, a, lda);
    if (noise != 0.0) {
        const double scale = noise / std::sqrt(double(n));
        for (int64_t c0 = 0; c0 < n; c0 += 65535) {
            const int w = int(std::min<int64_t>(65535, n - c0));
            gauss_cols(h, seed, kStreamNoise, m, int(c0), w, scale, true, a + c0 * lda, lda);
        }
    }
    FQB_CUDA(cudaStreamSynchronize(s));
}

}  // namespace farqb
