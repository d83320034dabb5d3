/*
 * detgen.c -- host twin of the deterministic low-rank generator
 * (paper_2506_03859_b200/csrc/detgen.cu, fqb_gen_lowrank_det).
 *
 * TEST INFRASTRUCTURE ONLY (see farqb_oracle.h).  It makes the BASELINE
 * config 3/4 matrices on the CPU with the same bits as the GPU makes them, so
 * the unmodified reference (oracle/_ref) can be run on exactly the A the
 * B200 factorizes -- at 100000 x 20000 a 16 GB matrix cannot be shipped
 * between the two machines, but a seed can.  tests/test_gpu_detgen.py checks
 * the GPU output against this file's (checksum and sampled entries).
 *
 *   X0 (m x r), Y0 (n x r): Philox(seed, 0xFA000001 / 0xFA000002, column j)
 *       Gaussians through the libm-free Box-Muller of include/farqb/detmath.h
 *       (element i = z0 (i even) or z1 (i odd) of pair i/2);
 *   X = X0 R_x^-1, R_x = chol(X0' X0)  (CholeskyQR: the Q of QR(X0)), same for Y;
 *   A = X diag(sigma) Y' + noise_scale * G,  G on stream 0xFA000003 keyed by
 *       column like X0.
 *
 * Every product is an fma chain over k = 0, 1, ... in ascending order started
 * from +0.0 -- the order the GPU kernels use -- so blocking, threading and
 * vector width change nothing.  The Cholesky is right-looking (S_ij -= R_ki
 * R_kj at step k, one fma), the inverse of R column by column from the diagonal
 * up.  Build: -ffp-contract=off (no hidden fusing), -mfma (fma() one instruction).
 */
#include <immintrin.h>
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#include "../include/farqb/detmath.h"

#define STREAM_X 0xFA000001u
#define STREAM_Y 0xFA000002u
#define STREAM_NOISE 0xFA000003u

static void philox10(uint32_t c[4], uint32_t k0, uint32_t k1) {
    for (int r = 0; r < 10; ++r) {
        uint64_t p0 = (uint64_t)0xD2511F53u * c[0];
        uint64_t p1 = (uint64_t)0xCD9E8D57u * c[2];
        uint32_t n0 = (uint32_t)(p1 >> 32) ^ c[1] ^ k0;
        uint32_t n1 = (uint32_t)p1;
        uint32_t n2 = (uint32_t)(p0 >> 32) ^ c[3] ^ k1;
        uint32_t n3 = (uint32_t)p0;
        c[0] = n0; c[1] = n1; c[2] = n2; c[3] = n3;
        k0 += 0x9E3779B9u;
        k1 += 0xBB67AE85u;
    }
}

static double unit_from(uint32_t lo, uint32_t hi) {
    uint64_t v = (uint64_t)lo | ((uint64_t)hi << 32);
    return ((double)(v >> 11) + 0.5) * 0x1p-53;
}

/* element i of the Gaussian column (seed, stream, col) */
static double det_gauss(uint64_t seed, uint32_t stream, uint32_t col, int64_t i) {
    uint64_t ctr = (uint64_t)i >> 1;
    uint32_t c[4] = {(uint32_t)ctr, (uint32_t)(ctr >> 32), col, stream};
    philox10(c, (uint32_t)seed, (uint32_t)(seed >> 32));
    double z0, z1;
    fqd_box_muller(unit_from(c[0], c[1]), unit_from(c[2], c[3]), &z0, &z1);
    return (i & 1) ? z1 : z0;
}

double fqo_det_gauss(uint64_t seed, uint32_t stream, uint32_t col, int64_t i) {
    return det_gauss(seed, stream, col, i);
}
double fqo_det_log(double x) { return fqd_log(x); }
void fqo_det_box_muller(double u1, double u2, double* z) { fqd_box_muller(u1, u2, z, z + 1); }

/* ---- the fixed-order GEMM --------------------------------------------------
 * C[i + j ldc] = sum_k a(i,k) b(k,j), k ascending, one fma per k from +0.0
 * (or from the existing C when acc), a(i,k) = ta ? A[k + i lda] : A[i + k lda],
 * b(k,j) = tb ? B[j + k ldb] : B[k + j ldb].  Packed 8 x 4 micro-tiles, AVX2
 * fmadd lanes are independent element chains. */
enum { MR = 8, NR = 4, MC = 128, NC = 128, KC = 256 };

static void micro_8x4(int64_t kc, const double* ap, const double* bp, double* c, int64_t ldc, int mr, int nr,
                      int first) {
    __m256d acc[NR][2];
    double tmp[NR][MR];
    for (int j = 0; j < NR; ++j)
        for (int i = 0; i < MR; ++i) tmp[j][i] = (first || j >= nr || i >= mr) ? 0.0 : c[i + j * ldc];
    for (int j = 0; j < NR; ++j) {
        acc[j][0] = _mm256_loadu_pd(&tmp[j][0]);
        acc[j][1] = _mm256_loadu_pd(&tmp[j][4]);
    }
    for (int64_t k = 0; k < kc; ++k) {
        __m256d a0 = _mm256_loadu_pd(ap + k * MR), a1 = _mm256_loadu_pd(ap + k * MR + 4);
        for (int j = 0; j < NR; ++j) {
            __m256d b = _mm256_broadcast_sd(bp + k * NR + j);
            acc[j][0] = _mm256_fmadd_pd(a0, b, acc[j][0]);
            acc[j][1] = _mm256_fmadd_pd(a1, b, acc[j][1]);
        }
    }
    for (int j = 0; j < NR; ++j) {
        _mm256_storeu_pd(&tmp[j][0], acc[j][0]);
        _mm256_storeu_pd(&tmp[j][4], acc[j][1]);
    }
    for (int j = 0; j < nr; ++j)
        for (int i = 0; i < mr; ++i) c[i + j * ldc] = tmp[j][i];
}

static void det_gemm(int64_t M, int64_t N, int64_t K, const double* A, int64_t lda, int ta, const double* B,
                     int64_t ldb, int tb, double* C, int64_t ldc) {
    const int64_t tiles_m = (M + MC - 1) / MC, tiles_n = (N + NC - 1) / NC;
#pragma omp parallel
    {
        double* ap = (double*)aligned_alloc(64, sizeof(double) * MC * KC);
        double* bp = (double*)aligned_alloc(64, sizeof(double) * NC * KC);
#pragma omp for schedule(dynamic, 1)
        for (int64_t t = 0; t < tiles_m * tiles_n; ++t) {
            const int64_t i0 = (t % tiles_m) * MC, j0 = (t / tiles_m) * NC;
            const int64_t mc = M - i0 < MC ? M - i0 : MC, nc = N - j0 < NC ? N - j0 : NC;
            for (int64_t k0 = 0; k0 < K; k0 += KC) {
                const int64_t kc = K - k0 < KC ? K - k0 : KC;
                /* pack A: panels of MR rows, k-major */
                for (int64_t ib = 0; ib < mc; ib += MR)
                    for (int64_t k = 0; k < kc; ++k)
                        for (int i = 0; i < MR; ++i) {
                            const int64_t gi = i0 + ib + i, gk = k0 + k;
                            ap[ib * kc + k * MR + i] =
                                (ib + i < mc) ? (ta ? A[gk + gi * lda] : A[gi + gk * lda]) : 0.0;
                        }
                for (int64_t jb = 0; jb < nc; jb += NR)
                    for (int64_t k = 0; k < kc; ++k)
                        for (int j = 0; j < NR; ++j) {
                            const int64_t gj = j0 + jb + j, gk = k0 + k;
                            bp[jb * kc + k * NR + j] =
                                (jb + j < nc) ? (tb ? B[gj + gk * ldb] : B[gk + gj * ldb]) : 0.0;
                        }
                for (int64_t jb = 0; jb < nc; jb += NR)
                    for (int64_t ib = 0; ib < mc; ib += MR) {
                        const int mr = (int)(mc - ib < MR ? mc - ib : MR), nr = (int)(nc - jb < NR ? nc - jb : NR);
                        micro_8x4(kc, ap + ib * kc, bp + jb * kc, C + (i0 + ib) + (j0 + jb) * ldc, ldc, mr, nr,
                                  k0 == 0);
                    }
            }
        }
        free(ap);
        free(bp);
    }
}

/* ---- R = chol(G) (upper), right-looking, and R^-1 ---------------------------- */
static void det_chol_upper(double* S, int r, double* R) {
    /* S (r x r col-major, symmetric, upper used) is overwritten. R upper, strictly
     * lower part zero. */
    memset(R, 0, sizeof(double) * (size_t)r * r);
    for (int k = 0; k < r; ++k) {
        const double rkk = FQD_SQRT(S[k + (int64_t)k * r]);
        R[k + (int64_t)k * r] = rkk;
        for (int j = k + 1; j < r; ++j) R[k + (int64_t)j * r] = FQD_DIV(S[k + (int64_t)j * r], rkk);
#pragma omp parallel for schedule(static)
        for (int j = k + 1; j < r; ++j) {
            const double rkj = R[k + (int64_t)j * r];
            double* sj = S + (int64_t)j * r;
            for (int i = k + 1; i <= j; ++i) sj[i] = FQD_FMA(-R[k + (int64_t)i * r], rkj, sj[i]);
        }
    }
}

static void det_upper_inverse(const double* R, int r, double* Ri) {
    memset(Ri, 0, sizeof(double) * (size_t)r * r);
#pragma omp parallel for schedule(dynamic, 8)
    for (int j = 0; j < r; ++j) {
        double* cj = Ri + (int64_t)j * r;
        cj[j] = FQD_DIV(1.0, R[j + (int64_t)j * r]);
        for (int i = j - 1; i >= 0; --i) {
            double acc = 0.0;
            for (int k = i + 1; k <= j; ++k) acc = FQD_FMA(R[i + (int64_t)k * r], cj[k], acc);
            cj[i] = FQD_DIV(-acc, R[i + (int64_t)i * r]);
        }
    }
}

/* Orthonormal factor rows [row0, row0 + rows) of Q(QR(F0)), F0 = Gaussian (len x r) */
static int det_factor(int64_t len, int r, uint64_t seed, uint32_t stream, int64_t row0, int64_t rows, double* out,
                      int64_t ldo) {
    double* f0 = (double*)malloc(sizeof(double) * (size_t)len * r);
    double* g = (double*)malloc(sizeof(double) * (size_t)r * r);
    double* R = (double*)malloc(sizeof(double) * (size_t)r * r);
    double* Ri = (double*)malloc(sizeof(double) * (size_t)r * r);
    if (!f0 || !g || !R || !Ri) {
        free(f0); free(g); free(R); free(Ri);
        return 10;
    }
#pragma omp parallel for schedule(static)
    for (int j = 0; j < r; ++j)
        for (int64_t i = 0; i < len; ++i) f0[i + (int64_t)j * len] = det_gauss(seed, stream, (uint32_t)j, i);
    det_gemm(r, r, len, f0, len, 1, f0, len, 0, g, r);
    det_chol_upper(g, r, R);
    det_upper_inverse(R, r, Ri);
    det_gemm(rows, r, r, f0 + row0, len, 0, Ri, r, 0, out, ldo);
    free(f0); free(g); free(R); free(Ri);
    return 0;
}

/*
 * Rows [row0, row0 + rows) of A = X diag(sigma) Y' + noise_scale * G (m x n).
 * a: rows x n, column-major, leading dimension lda >= rows.  Returns 0, 1 on a
 * bad argument, 10 when out of memory.
 */
int fqo_det_lowrank(int64_t m, int64_t n, int r, const double* sigma, uint64_t seed, double noise_scale,
                    int64_t row0, int64_t rows, double* a, int64_t lda) {
    if (m < 1 || n < 1 || r < 1 || r > m || r > n || row0 < 0 || rows < 0 || row0 + rows > m || lda < rows)
        return 1;
    if (rows == 0) return 0;
    double* x = (double*)malloc(sizeof(double) * (size_t)rows * r);
    double* y = (double*)malloc(sizeof(double) * (size_t)n * r);
    if (!x || !y) {
        free(x); free(y);
        return 10;
    }
    int st = det_factor(m, r, seed, STREAM_X, row0, rows, x, rows);
    if (!st) st = det_factor(n, r, seed, STREAM_Y, 0, n, y, n);
    if (st) {
        free(x); free(y);
        return st;
    }
#pragma omp parallel for schedule(static)
    for (int k = 0; k < r; ++k)
        for (int64_t j = 0; j < n; ++j) y[j + (int64_t)k * n] = FQD_MUL(y[j + (int64_t)k * n], sigma[k]);
    det_gemm(rows, n, r, x, rows, 0, y, n, 1, a, lda);
    if (noise_scale != 0.0) {
#pragma omp parallel for schedule(static)
        for (int64_t j = 0; j < n; ++j)
            for (int64_t i = 0; i < rows; ++i) {
                double* p = a + i + j * lda;
                *p = FQD_ADD(*p, FQD_MUL(noise_scale, det_gauss(seed, STREAM_NOISE, (uint32_t)j, row0 + i)));
            }
    }
    free(x);
    free(y);
    return 0;
}

/* Order-independent 64-bit fingerprint of A's bits: sum over elements of
 * mix(bits ^ (global index * golden)) mod 2^64, global index = j m + row0 + i
 * (so row shards add up to the whole matrix's value). */
static uint64_t mix64(uint64_t z) {
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}

uint64_t fqo_checksum(const double* a, int64_t rows, int64_t cols, int64_t lda, int64_t row0, int64_t m_total) {
    uint64_t h = 0;
#pragma omp parallel for reduction(+ : h) schedule(static)
    for (int64_t j = 0; j < cols; ++j)
        for (int64_t i = 0; i < rows; ++i) {
            uint64_t bits;
            memcpy(&bits, a + i + j * lda, sizeof bits);
            const uint64_t idx = (uint64_t)(j * m_total + row0 + i);
            h += mix64(bits ^ (idx * 0x9E3779B97F4A7C15ULL));
        }
    return h;
}
