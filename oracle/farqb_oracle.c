/*
 * farqb_oracle.c -- plain-C restatement of the reference farPCA QB loop.
 *
 * TEST INFRASTRUCTURE ONLY (see farqb_oracle.h).  Not linked into, loaded by or
 * called from the product path.
 *
 * Citations are relative to /root/reference/proj.  The restatement keeps the
 * reference's numerical recipe (Gram-space bookkeeping with Y, W, Z = Y'Y,
 * T = W'W and the bordered Cholesky factor of Z) so that it is an independent
 * second implementation of the same algorithm; it is pinned against the
 * compiled reference (oracle/_ref) by tests/test_oracle_pin.py.
 */
#include "../include/farqb/detmath.h"
#include "farqb_oracle.h"

#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#define IDX(i, j, ld) ((size_t)(j) * (size_t)(ld) + (size_t)(i))

/* ========================================================================== */
/* Philox4x32-10 -- include/rsvd/rng.hpp:15-88                                */
/* ========================================================================== */

typedef struct {
    uint32_t key[2];
    uint32_t ctr[4];   /* {draw lo, draw hi, column, block_id}  rng.hpp:17-19 */
    uint32_t out[4];
    int pos;
    double spare;
    int have_spare;
} philox_t;

static void philox_init(philox_t* r, uint64_t seed, uint32_t block_id, uint32_t column) {
    r->key[0] = (uint32_t)seed;
    r->key[1] = (uint32_t)(seed >> 32);
    r->ctr[0] = 0;
    r->ctr[1] = 0;
    r->ctr[2] = column;
    r->ctr[3] = block_id;
    r->pos = 4;
    r->spare = 0.0;
    r->have_spare = 0;
}

/* Ten rounds of the Philox4x32 bijection, rng.hpp:64-80. */
static void philox_round10(const uint32_t in[4], uint32_t k0, uint32_t k1, uint32_t out[4]) {
    uint32_t c0 = in[0], c1 = in[1], c2 = in[2], c3 = in[3];
    for (int round = 0; round < 10; ++round) {
        uint64_t p0 = (uint64_t)0xD2511F53u * c0;
        uint64_t p1 = (uint64_t)0xCD9E8D57u * c2;
        uint32_t n0 = (uint32_t)(p1 >> 32) ^ c1 ^ k0;
        uint32_t n1 = (uint32_t)p1;
        uint32_t n2 = (uint32_t)(p0 >> 32) ^ c3 ^ k1;
        uint32_t n3 = (uint32_t)p0;
        c0 = n0; c1 = n1; c2 = n2; c3 = n3;
        k0 += 0x9E3779B9u;
        k1 += 0xBB67AE85u;
    }
    out[0] = c0; out[1] = c1; out[2] = c2; out[3] = c3;
}

static uint32_t philox_next_u32(philox_t* r) {
    if (r->pos == 4) {
        philox_round10(r->ctr, r->key[0], r->key[1], r->out);
        r->pos = 0;
        if (++r->ctr[0] == 0) ++r->ctr[1];
    }
    return r->out[r->pos++];
}

/* rng.hpp:26-35: low word first, then (u64 >> 11 + 0.5) * 2^-53 in (0,1). */
static double philox_next_unit(philox_t* r) {
    uint64_t lo = philox_next_u32(r);
    uint64_t hi = philox_next_u32(r);
    uint64_t v = lo | (hi << 32);
    return ((double)(v >> 11) + 0.5) * 0x1p-53;
}

/* Box-Muller pair with a cached spare; exact zeros redrawn, rng.hpp:39-56. */
/* The same pair logic through the libm-free Box-Muller of include/farqb/detmath.h:
 * the fixed-zeta sparse-Gaussian values (a kind the reference does not have), so
 * the device draws bit-identical Omega values for a seed. */
static double philox_next_gaussian_det(philox_t* r) {
    if (r->have_spare) {
        r->have_spare = 0;
        if (r->spare != 0.0) return r->spare;
    }
    for (;;) {
        double u1 = philox_next_unit(r);
        double u2 = philox_next_unit(r);
        double z0, z1;
        fqd_box_muller(u1, u2, &z0, &z1);
        r->spare = z1;
        r->have_spare = 1;
        if (z0 != 0.0) return z0;
        r->have_spare = 0;
    }
}

static double philox_next_gaussian(philox_t* r) {
    if (r->have_spare) {
        r->have_spare = 0;
        if (r->spare != 0.0) return r->spare;
    }
    for (;;) {
        double u1 = philox_next_unit(r);
        double u2 = philox_next_unit(r);
        double rad = sqrt(-2.0 * log(u1));
        double ang = 6.283185307179586476925286766559 * u2;
        double z0 = rad * cos(ang);
        double z1 = rad * sin(ang);
        r->spare = z1;
        r->have_spare = 1;
        if (z0 != 0.0) return z0;
        r->have_spare = 0;
    }
}

void fqo_philox_u32(uint64_t seed, uint32_t block_id, uint32_t column, int count, uint32_t* out) {
    philox_t r;
    philox_init(&r, seed, block_id, column);
    for (int i = 0; i < count; ++i) out[i] = philox_next_u32(&r);
}

void fqo_philox_units(uint64_t seed, uint32_t block_id, uint32_t column, int count, double* out) {
    philox_t r;
    philox_init(&r, seed, block_id, column);
    for (int i = 0; i < count; ++i) out[i] = philox_next_unit(&r);
}

void fqo_philox_gaussians(uint64_t seed, uint32_t block_id, uint32_t column, int count, double* out) {
    philox_t r;
    philox_init(&r, seed, block_id, column);
    for (int i = 0; i < count; ++i) out[i] = philox_next_gaussian(&r);
}

/* ========================================================================== */
/* Small helpers                                                              */
/* ========================================================================== */

static void* xcalloc(size_t count, size_t size) {
    if (count == 0) count = 1;
    return calloc(count, size);
}

static void set_msg(fqo_result* out, const char* msg) {
    if (!out) return;
    snprintf(out->message, sizeof out->message, "%s", msg);
}

/* ========================================================================== */
/* Dense kernels -- src/kernels_scalar.cpp:13-99                              */
/* ========================================================================== */

/* c (m x n) += a (m x k) * b (k x n); column-oriented axpys, fused multiply-add
 * per element like the reference's axpy path (kernels_avx2.cpp:220-231). */
void fqo_gemm_nn(int m, int n, int k, const double* a, int lda, const double* b,
                 int ldb, double* c, int ldc) {
    for (int j = 0; j < n; ++j) {
        double* cj = c + (size_t)j * ldc;
        for (int p = 0; p < k; ++p) {
            double bv = b[IDX(p, j, ldb)];
            const double* ap = a + (size_t)p * lda;
            for (int i = 0; i < m; ++i) cj[i] = fma(ap[i], bv, cj[i]);
        }
    }
}

/* c (m x n) += a' * b with a stored k x m: one dot product per output entry
 * (kernels_scalar.cpp:29-41), four interleaved partial sums. */
void fqo_gemm_tn(int m, int n, int k, const double* a, int lda, const double* b,
                 int ldb, double* c, int ldc) {
    for (int j = 0; j < n; ++j) {
        const double* bj = b + (size_t)j * ldb;
        for (int i = 0; i < m; ++i) {
            const double* ai = a + (size_t)i * lda;
            double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
            int p = 0;
            for (; p + 4 <= k; p += 4) {
                s0 = fma(ai[p], bj[p], s0);
                s1 = fma(ai[p + 1], bj[p + 1], s1);
                s2 = fma(ai[p + 2], bj[p + 2], s2);
                s3 = fma(ai[p + 3], bj[p + 3], s3);
            }
            double s = (s0 + s1) + (s2 + s3);
            for (; p < k; ++p) s = fma(ai[p], bj[p], s);
            c[IDX(i, j, ldc)] += s;
        }
    }
}

/* matrix_core.cpp:19-44 wrappers: fresh zeroed result. */
static double* mat_nn(const double* a, int m, int k, const double* b, int n) {
    double* c = (double*)xcalloc((size_t)m * n, sizeof(double));
    if (m > 0 && n > 0 && k > 0) fqo_gemm_nn(m, n, k, a, m, b, k, c, m);
    return c;
}

static double* mat_tn(const double* a, int k, int m, const double* b, int n) {
    /* a is k x m, b is k x n, result m x n */
    double* c = (double*)xcalloc((size_t)m * n, sizeof(double));
    if (m > 0 && n > 0 && k > 0) fqo_gemm_tn(m, n, k, a, k, b, k, c, m);
    return c;
}

double fqo_frob_norm_sq(const double* a, int64_t count) {
    /* sum_sq (kernels_scalar.cpp:64-68) */
    double s = 0.0;
    for (int64_t i = 0; i < count; ++i) s = fma(a[i], a[i], s);
    return s;
}

/* Cyclic Jacobi, ascending eigenvalues: matrix_core.cpp:50-115. */
int fqo_sym_eig(const double* mtx, int n, double* values, double* vectors) {
    double* a = (double*)xcalloc((size_t)n * n, sizeof(double));
    double* v = (double*)xcalloc((size_t)n * n, sizeof(double));
    memcpy(a, mtx, sizeof(double) * (size_t)n * n);
    for (int i = 0; i < n; ++i) v[IDX(i, i, n)] = 1.0;
    double fro = sqrt(fqo_frob_norm_sq(mtx, (int64_t)n * n));
    const double stop = 1e-14 * fro;
    int status = FQO_OK;
    if (n > 1) {
        int sweep = 0;
        for (; sweep < 30; ++sweep) {
            double off = 0.0;
            for (int j = 0; j < n; ++j)
                for (int i = j + 1; i < n; ++i) off += a[IDX(i, j, n)] * a[IDX(i, j, n)];
            if (sqrt(2.0 * off) <= stop) break;
            for (int p = 0; p < n - 1; ++p) {
                for (int q = p + 1; q < n; ++q) {
                    double apq = a[IDX(p, q, n)];
                    if (fabs(apq) <= stop / ((double)n * n)) continue;
                    double app = a[IDX(p, p, n)], aqq = a[IDX(q, q, n)];
                    double tau = (aqq - app) / (2.0 * apq);
                    double t = (tau >= 0.0 ? 1.0 : -1.0) / (fabs(tau) + sqrt(1.0 + tau * tau));
                    double c = 1.0 / sqrt(1.0 + t * t);
                    double s = t * c;
                    double* xp = a + (size_t)p * n;
                    double* xq = a + (size_t)q * n;
                    for (int i = 0; i < n; ++i) {
                        double x = xp[i], y = xq[i];
                        xp[i] = c * x - s * y;
                        xq[i] = s * x + c * y;
                    }
                    for (int i = 0; i < n; ++i) {
                        double x = a[IDX(p, i, n)], y = a[IDX(q, i, n)];
                        a[IDX(p, i, n)] = c * x - s * y;
                        a[IDX(q, i, n)] = s * x + c * y;
                    }
                    a[IDX(p, q, n)] = 0.0;
                    a[IDX(q, p, n)] = 0.0;
                    double* vp = v + (size_t)p * n;
                    double* vq = v + (size_t)q * n;
                    for (int i = 0; i < n; ++i) {
                        double x = vp[i], y = vq[i];
                        vp[i] = c * x - s * y;
                        vq[i] = s * x + c * y;
                    }
                }
            }
        }
        if (sweep == 30) {
            double off = 0.0;
            for (int j = 0; j < n; ++j)
                for (int i = j + 1; i < n; ++i) off += a[IDX(i, j, n)] * a[IDX(i, j, n)];
            if (sqrt(2.0 * off) > stop) status = FQO_ERR_CONVERGENCE;
        }
    }
    /* stable ascending order of the diagonal (std::sort on indices) */
    int* order = (int*)xcalloc((size_t)n, sizeof(int));
    for (int i = 0; i < n; ++i) order[i] = i;
    for (int i = 1; i < n; ++i) {
        int key = order[i];
        int j = i - 1;
        while (j >= 0 && a[IDX(order[j], order[j], n)] > a[IDX(key, key, n)]) {
            order[j + 1] = order[j];
            --j;
        }
        order[j + 1] = key;
    }
    for (int j = 0; j < n; ++j) {
        values[j] = a[IDX(order[j], order[j], n)];
        if (vectors) memcpy(vectors + (size_t)j * n, v + (size_t)order[j] * n, sizeof(double) * n);
    }
    free(order);
    free(a);
    free(v);
    return status;
}

/* Right-looking Cholesky with relative pivot floor: matrix_core.cpp:117-140. */
int fqo_chol_factor(const double* z, int n, double pivot_tol, double diag_ref, double* l) {
    memset(l, 0, sizeof(double) * (size_t)n * n);
    double max_diag = diag_ref;
    if (max_diag <= 0.0)
        for (int i = 0; i < n; ++i)
            if (z[IDX(i, i, n)] > max_diag) max_diag = z[IDX(i, i, n)];
    for (int j = 0; j < n; ++j)
        for (int i = j; i < n; ++i) l[IDX(i, j, n)] = z[IDX(i, j, n)];
    for (int j = 0; j < n; ++j) {
        double d = l[IDX(j, j, n)];
        if (d <= pivot_tol * max_diag) return FQO_ERR_BLOCK_DEGENERATE;
        double ljj = sqrt(d);
        l[IDX(j, j, n)] = ljj;
        double inv = 1.0 / ljj;
        for (int i = j + 1; i < n; ++i) l[IDX(i, j, n)] *= inv;
        for (int c = j + 1; c < n; ++c) {
            double f = -l[IDX(c, j, n)];
            for (int i = c; i < n; ++i) l[IDX(i, c, n)] = fma(f, l[IDX(i, j, n)], l[IDX(i, c, n)]);
        }
    }
    return FQO_OK;
}

/* L x = rhs in place (matrix_core.cpp:142-152). */
static void trsm_lower(const double* l, int n, double* x, int ncols) {
    for (int c = 0; c < ncols; ++c) {
        double* xc = x + (size_t)c * n;
        for (int j = 0; j < n; ++j) {
            xc[j] /= l[IDX(j, j, n)];
            double f = -xc[j];
            for (int i = j + 1; i < n; ++i) xc[i] = fma(f, l[IDX(i, j, n)], xc[i]);
        }
    }
}

/* L' x = rhs in place (matrix_core.cpp:154-165). */
static void trsm_lower_trans(const double* l, int n, double* x, int ncols) {
    for (int c = 0; c < ncols; ++c) {
        double* xc = x + (size_t)c * n;
        for (int j = n - 1; j >= 0; --j) {
            double s = 0.0;
            for (int i = j + 1; i < n; ++i) s = fma(l[IDX(i, j, n)], xc[i], s);
            xc[j] = (xc[j] - s) / l[IDX(j, j, n)];
        }
    }
}

/* x <- x L'^{-1}, x is rows x b (matrix_core.cpp:167-179). */
static void trsm_right_lower_trans(const double* l, int b, double* x, int rows) {
    for (int c = 0; c < b; ++c) {
        double* xc = x + (size_t)c * rows;
        for (int p = 0; p < c; ++p) {
            double f = -l[IDX(c, p, b)];
            const double* xp = x + (size_t)p * rows;
            for (int i = 0; i < rows; ++i) xc[i] = fma(f, xp[i], xc[i]);
        }
        double inv = 1.0 / l[IDX(c, c, b)];
        for (int i = 0; i < rows; ++i) xc[i] *= inv;
    }
}

/* eigSVD via the Gram matrix (matrix_core.cpp:193-215).  u is n x b. */
static int eig_svd(const double* w, int n, int b, double eig_tol, double* u, double* sigma) {
    double* g = mat_tn(w, n, b, w, b);
    double* vals = (double*)xcalloc((size_t)b, sizeof(double));
    double* vecs = (double*)xcalloc((size_t)b * b, sizeof(double));
    int st = fqo_sym_eig(g, b, vals, vecs);
    free(g);
    if (st != FQO_OK) { free(vals); free(vecs); return st; }
    double lmax = vals[b - 1];
    if (lmax <= 0.0 || (eig_tol > 0.0 && vals[0] <= eig_tol * lmax)) {
        free(vals); free(vecs);
        return FQO_ERR_BLOCK_DEGENERATE;
    }
    double fl = lmax * 1e-31;
    for (int i = 0; i < b; ++i) sigma[i] = sqrt(vals[i] > fl ? vals[i] : fl);
    for (int j = 0; j < b; ++j) {
        double inv = 1.0 / sigma[j];
        for (int i = 0; i < b; ++i) vecs[IDX(i, j, b)] *= inv;
    }
    memset(u, 0, sizeof(double) * (size_t)n * b);
    fqo_gemm_nn(n, b, b, w, n, vecs, b, u, n);
    free(vals);
    free(vecs);
    return FQO_OK;
}

/* ========================================================================== */
/* Sketch generation and sparse products -- src/sketch.cpp                     */
/* ========================================================================== */

double fqo_default_density(int kind, int n) {   /* driver.cpp:449-455 */
    if (kind == FQO_GAUSSIAN) return 0.0;
    double nn = (double)n;
    double v = kind == FQO_STD_BERNOULLI ? log(nn) / nn : 10.0 / nn;
    return v > 1e-3 ? v : 1e-3;
}

int fqo_default_block(int m, int n) {            /* driver.cpp:457-462 */
    int mn = m < n ? m : n;
    int b = mn / 100;
    if (b < 20) b = 20;
    if (b > 50) b = 50;
    return b < mn ? b : mn;
}

int fqo_default_max_iters(int n, int b) {        /* driver.cpp:464-466 */
    return (n + 2 * b - 1) / (2 * b);
}

void fqo_block_free(fqo_block* blk) {
    if (!blk) return;
    free(blk->dense);
    free(blk->col_ptr);
    free(blk->row_idx);
    free(blk->values);
    memset(blk, 0, sizeof *blk);
}

typedef struct {
    int* rows;
    double* vals;
    int64_t n, cap;
} nzbuf_t;

static int nz_push(nzbuf_t* b, int row, double v) {
    if (b->n == b->cap) {
        int64_t nc = b->cap ? b->cap * 2 : 64;
        int* r = (int*)realloc(b->rows, sizeof(int) * (size_t)nc);
        if (!r) return -1;
        b->rows = r;
        double* x = (double*)realloc(b->vals, sizeof(double) * (size_t)nc);
        if (!x) return -1;
        b->vals = x;
        b->cap = nc;
    }
    b->rows[b->n] = row;
    b->vals[b->n] = v;
    b->n++;
    return 0;
}

/*
 * Test-matrix block, deterministic in (kind, p, seed, zeta, n, l, block_id);
 * column j always draws from Philox(seed, block_id, j)  (sketch.cpp:51-102).
 *
 * zeta == 0: the reference's i.i.d. density-p patterns, walked by geometric
 *   gaps row += 1 + floor(log u / log1p(-p))  (sketch.cpp:35-47, 75-95).
 * zeta  > 0 (sparse sign / sparse Gaussian only; new in this build, the
 *   reference lists it as a non-goal): exactly zeta distinct rows
 *   per column.  Candidates are r = (u32 * n) >> 32 from successive words of
 *   the column stream, duplicates skipped, until zeta rows are held; then one
 *   value per row in draw order -- sign: the next u32's top bit set gives
 *   -1/sqrt(zeta), clear gives +1/sqrt(zeta); Gaussian: next_gaussian() /
 *   sqrt(zeta), next_gaussian through the libm-free Box-Muller of
 *   include/farqb/detmath.h so host and device values are bit-identical -- and
 *   the (row, value) pairs are sorted by row.
 */
int fqo_gen_sketch(int kind, double p, uint64_t seed, int zeta, int n, int l,
                   int block_id, fqo_block* out) {
    memset(out, 0, sizeof *out);
    if (n < 1 || l < 1) return FQO_ERR_CONFIG;
    out->rows = n;
    out->cols = l;
    out->p = p;
    if (kind == FQO_GAUSSIAN) {
        out->is_dense = 1;
        out->dense = (double*)xcalloc((size_t)n * l, sizeof(double));
        if (!out->dense) return FQO_ERR_ALLOC;
        for (int j = 0; j < l; ++j) {
            philox_t r;
            philox_init(&r, seed, (uint32_t)block_id, (uint32_t)j);
            double* col = out->dense + (size_t)j * n;
            for (int i = 0; i < n; ++i) col[i] = philox_next_gaussian(&r);
        }
        return FQO_OK;
    }
    out->col_ptr = (int*)xcalloc((size_t)l + 1, sizeof(int));
    nzbuf_t buf = {0};
    if (zeta > 0) {
        if (kind != FQO_SPARSE_SIGN && kind != FQO_SPARSE_GAUSSIAN) return FQO_ERR_CONFIG;
        if (zeta > n) return FQO_ERR_CONFIG;
        const double scale = 1.0 / sqrt((double)zeta);
        int* rows = (int*)xcalloc((size_t)zeta, sizeof(int));
        double* vals = (double*)xcalloc((size_t)zeta, sizeof(double));
        for (int j = 0; j < l; ++j) {
            philox_t r;
            philox_init(&r, seed, (uint32_t)block_id, (uint32_t)j);
            int have = 0;
            while (have < zeta) {
                uint32_t w = philox_next_u32(&r);
                int row = (int)(((uint64_t)w * (uint64_t)n) >> 32);
                int dup = 0;
                for (int t = 0; t < have; ++t) dup |= rows[t] == row;
                if (!dup) rows[have++] = row;
            }
            for (int t = 0; t < zeta; ++t) {
                if (kind == FQO_SPARSE_SIGN)
                    vals[t] = (philox_next_u32(&r) & 0x80000000u) ? -scale : scale;
                else
                    vals[t] = philox_next_gaussian_det(&r) * scale;
            }
            for (int t = 1; t < zeta; ++t) {   /* insertion sort by row */
                int kr = rows[t];
                double kv = vals[t];
                int s = t - 1;
                while (s >= 0 && rows[s] > kr) {
                    rows[s + 1] = rows[s];
                    vals[s + 1] = vals[s];
                    --s;
                }
                rows[s + 1] = kr;
                vals[s + 1] = kv;
            }
            for (int t = 0; t < zeta; ++t) nz_push(&buf, rows[t], vals[t]);
            out->col_ptr[j + 1] = (int)buf.n;
        }
        free(rows);
        free(vals);
    } else {
        if (!(p > 0.0 && p < 1.0)) { free(out->col_ptr); out->col_ptr = NULL; return FQO_ERR_CONFIG; }
        const double inv_sqrt_p = 1.0 / sqrt(p);
        const double denom = log1p(-p);
        for (int j = 0; j < l; ++j) {
            philox_t r;
            philox_init(&r, seed, (uint32_t)block_id, (uint32_t)j);
            long long row = -1;
            for (;;) {
                double u = philox_next_unit(&r);
                double ratio = log(u) / denom;
                if (ratio >= (double)n) break;
                row += 1 + (long long)ratio;
                if (row >= n) break;
                double v = 1.0;
                if (kind == FQO_SPARSE_SIGN)
                    v = philox_next_unit(&r) < 0.5 ? -inv_sqrt_p : inv_sqrt_p;
                else if (kind == FQO_SPARSE_GAUSSIAN)
                    v = philox_next_gaussian(&r) * inv_sqrt_p;
                nz_push(&buf, (int)row, v);
            }
            out->col_ptr[j + 1] = (int)buf.n;
        }
        if (kind == FQO_STD_BERNOULLI) {
            out->centered = 1;
            out->std_scale = 1.0 / sqrt(p * (1.0 - p));
        }
    }
    out->nnz = buf.n;
    out->row_idx = buf.rows ? buf.rows : (int*)xcalloc(1, sizeof(int));
    out->values = buf.vals ? buf.vals : (double*)xcalloc(1, sizeof(double));
    return FQO_OK;
}

/* c (m x l) = a (m x n) * s: one fused axpy per nonzero in CSC order
 * (sketch.cpp:104-114). */
void fqo_sparse_dense_mul(const double* a, int m, int n, const int* col_ptr,
                          const int* row_idx, const double* values, int l, double* c) {
    (void)n;
    memset(c, 0, sizeof(double) * (size_t)m * l);
    for (int j = 0; j < l; ++j) {
        double* cj = c + (size_t)j * m;
        for (int idx = col_ptr[j]; idx < col_ptr[j + 1]; ++idx) {
            const double v = values[idx];
            const double* ac = a + (size_t)row_idx[idx] * m;
            for (int i = 0; i < m; ++i) cj[i] = fma(v, ac[i], cj[i]);
        }
    }
}

/* c (k x l) = w' s for w n x k (sketch.cpp:116-130). */
void fqo_dense_sparse_tmul(const double* w, int n, int k, const int* col_ptr,
                           const int* row_idx, const double* values, int l, double* c) {
    for (int j = 0; j < l; ++j) {
        for (int i = 0; i < k; ++i) {
            const double* wi = w + (size_t)i * n;
            double acc = 0.0;
            for (int idx = col_ptr[j]; idx < col_ptr[j + 1]; ++idx)
                acc = fma(values[idx], wi[row_idx[idx]], acc);
            c[IDX(i, j, k)] = acc;
        }
    }
}

/* z = A (p 1_n), axpy over columns (driver.cpp:178-183). */
void fqo_centering_column(const double* a, int m, int n, double p, double* z) {
    memset(z, 0, sizeof(double) * (size_t)m);
    for (int c = 0; c < n; ++c) {
        const double* ac = a + (size_t)c * m;
        for (int i = 0; i < m; ++i) z[i] = fma(p, ac[i], z[i]);
    }
}

/* ========================================================================== */
/* Driver -- src/driver.cpp                                                    */
/* ========================================================================== */

typedef struct {
    int m, n, b;
    int l, cap;          /* accumulated columns, allocated columns */
    double* y;           /* m x cap */
    double* w;           /* n x cap */
    double* z;           /* l x l */
    double* t;           /* l x l */
    double* lz;          /* l x l lower */
    double norm_a_sq;
    double trace_acc;
    double alpha;
    int blocks;
} state_t;               /* FactorState, driver.hpp:28-43 */

static double state_residual(const state_t* s) { return s->norm_a_sq - s->trace_acc; }

static void state_free(state_t* s) {
    free(s->y); free(s->w); free(s->z); free(s->t); free(s->lz);
    memset(s, 0, sizeof *s);
}

/* apply_block: A times the raw block, minus z when centered (driver.cpp:21-26). */
static double* apply_block(const double* a, int m, int n, const fqo_block* blk, const double* zc) {
    int b = blk->cols;
    if (blk->is_dense) return mat_nn(a, m, n, blk->dense, b);
    double* c = (double*)xcalloc((size_t)m * b, sizeof(double));
    fqo_sparse_dense_mul(a, m, n, blk->col_ptr, blk->row_idx, blk->values, b, c);
    if (blk->centered)
        for (int j = 0; j < b; ++j)
            for (int i = 0; i < m; ++i) c[IDX(i, j, m)] -= zc[i];
    return c;
}

/* tmul_block: w' times the raw block with the centering correction
 * (driver.cpp:30-45).  w is n x k. */
static double* tmul_block(const double* w, int n, int k, const fqo_block* blk) {
    int b = blk->cols;
    double* r;
    if (blk->is_dense) {
        r = mat_tn(w, n, k, blk->dense, b);
    } else {
        r = (double*)xcalloc((size_t)k * b, sizeof(double));
        fqo_dense_sparse_tmul(w, n, k, blk->col_ptr, blk->row_idx, blk->values, b, r);
    }
    if (blk->centered && k > 0) {
        double* ws = (double*)xcalloc((size_t)k, sizeof(double));
        for (int c = 0; c < k; ++c) {
            double s = 0.0;
            for (int i = 0; i < n; ++i) s += w[IDX(i, c, n)];
            ws[c] = blk->p * s;
        }
        for (int c = 0; c < b; ++c)
            for (int i = 0; i < k; ++i) r[IDX(i, c, k)] -= ws[i];
        free(ws);
    }
    return r;
}

/* c -= a * b (driver.cpp:48-53); a is rows x k, b is k x cols. */
static void sub_product(double* c, int rows, int cols, const double* a, int k, const double* b) {
    double* nb = (double*)xcalloc((size_t)k * cols, sizeof(double));
    for (size_t i = 0; i < (size_t)k * cols; ++i) nb[i] = -b[i];
    fqo_gemm_nn(rows, cols, k, a, rows, nb, k, c, rows);
    free(nb);
}

/* Z^{-1} rhs through the factor (matrix_core.cpp:181-187), in place. */
static void chol_solve_factored(const double* l, int n, double* rhs, int ncols) {
    trsm_lower(l, n, rhs, ncols);
    trsm_lower_trans(l, n, rhs, ncols);
}

/* power_iterate_block (driver.cpp:185-228).  Returns an n x b orthonormal
 * iterate in *gd_out (malloc'd) or a degenerate status. */
static int power_iterate(state_t* st, const double* a, const fqo_block* blk, int power,
                         int conv, const double* zc, double** gd_out) {
    const int m = st->m, n = st->n, b = blk->cols;
    st->alpha = 0.0;
    double* gd = NULL;
    double* sig = (double*)xcalloc((size_t)b, sizeof(double));
    for (int k = 1; k <= power; ++k) {
        double* wj;
        if (k == 1) {
            double* y0 = apply_block(a, m, n, blk, zc);
            wj = mat_tn(a, m, n, y0, b);
            free(y0);
            if (st->blocks > 0) {
                double* x = tmul_block(st->w, n, st->l, blk);
                chol_solve_factored(st->lz, st->l, x, b);
                sub_product(wj, n, b, st->w, st->l, x);
                free(x);
            }
        } else {
            double* y = mat_nn(a, m, n, gd, b);
            wj = mat_tn(a, m, n, y, b);
            free(y);
            if (st->blocks > 0) {
                double* x = mat_tn(st->w, n, st->l, gd, b);
                chol_solve_factored(st->lz, st->l, x, b);
                sub_product(wj, n, b, st->w, st->l, x);
                free(x);
            }
            if (st->alpha != 0.0)
                for (int c = 0; c < b; ++c)
                    for (int i = 0; i < n; ++i)
                        wj[IDX(i, c, n)] = fma(-st->alpha, gd[IDX(i, c, n)], wj[IDX(i, c, n)]);
        }
        double* u = (double*)xcalloc((size_t)n * b, sizeof(double));
        int rc = eig_svd(wj, n, b, 0.0, u, sig);
        free(wj);
        if (rc != FQO_OK) {
            free(u); free(gd); free(sig);
            return rc == FQO_ERR_CONVERGENCE ? rc : FQO_ERR_BLOCK_DEGENERATE;
        }
        free(gd);
        gd = u;
        if (k > 1) {
            double shat = conv == 0 ? sig[b - 1] : sig[0];
            if (st->alpha < shat) st->alpha = 0.5 * (shat + st->alpha);
        }
    }
    free(sig);
    *gd_out = gd;
    return FQO_OK;
}

static int state_reserve(state_t* st, int need) {
    if (need <= st->cap) return 0;
    int nc = st->cap ? st->cap : need;
    while (nc < need) nc *= 2;
    double* y = (double*)realloc(st->y, sizeof(double) * (size_t)st->m * nc);
    if (!y) return -1;
    st->y = y;
    double* w = (double*)realloc(st->w, sizeof(double) * (size_t)st->n * nc);
    if (!w) return -1;
    st->w = w;
    st->cap = nc;
    return 0;
}

/* [[old, off], [off', corner]] (driver.cpp:56-70). */
static double* grow_sym(const double* old, int l, const double* off, const double* corner, int b) {
    int nl = l + b;
    double* z = (double*)xcalloc((size_t)nl * nl, sizeof(double));
    for (int j = 0; j < l; ++j) {
        for (int i = 0; i < l; ++i) z[IDX(i, j, nl)] = old[IDX(i, j, l)];
        for (int i = 0; i < b; ++i) z[IDX(l + i, j, nl)] = off[IDX(j, i, l)];
    }
    for (int j = 0; j < b; ++j) {
        for (int i = 0; i < l; ++i) z[IDX(i, l + j, nl)] = off[IDX(i, j, l)];
        for (int i = 0; i < b; ++i) z[IDX(l + i, l + j, nl)] = corner[IDX(i, j, b)];
    }
    return z;
}

/* [[old, 0], [x', l22]] (driver.cpp:73-83). */
static double* grow_chol(const double* old, int l, const double* x, const double* l22, int b) {
    int nl = l + b;
    double* z = (double*)xcalloc((size_t)nl * nl, sizeof(double));
    for (int j = 0; j < l; ++j) {
        for (int i = 0; i < l; ++i) z[IDX(i, j, nl)] = old[IDX(i, j, l)];
        for (int i = 0; i < b; ++i) z[IDX(l + i, j, nl)] = x[IDX(j, i, l)];
    }
    for (int j = 0; j < b; ++j)
        for (int i = 0; i < b; ++i) z[IDX(l + i, l + j, nl)] = l22[IDX(i, j, b)];
    return z;
}

/* accept_block (driver.cpp:230-294). */
static int accept_block(state_t* st, const double* a, const fqo_block* blk, const double* zc) {
    const int m = st->m, n = st->n, b = blk->cols;
    if (b < 1) return FQO_ERR_DIMENSION;
    double* yj = apply_block(a, m, n, blk, zc);
    double* wj = mat_tn(a, m, n, yj, b);
    const int lold = st->l;
    double* dblk = mat_tn(yj, m, b, yj, b);
    double* tblk = mat_tn(wj, n, b, wj, b);
    double* l22 = (double*)xcalloc((size_t)b * b, sizeof(double));
    int rc = FQO_OK;
    if (lold == 0) {
        rc = fqo_chol_factor(dblk, b, 1e-12, 0.0, l22);
        if (rc != FQO_OK) goto fail;
        double* g = (double*)xcalloc((size_t)n * b, sizeof(double));
        memcpy(g, wj, sizeof(double) * (size_t)n * b);
        trsm_right_lower_trans(l22, b, g, n);
        st->trace_acc += fqo_frob_norm_sq(g, (int64_t)n * b);
        free(g);
        if (state_reserve(st, b)) { rc = FQO_ERR_ALLOC; goto fail; }
        memcpy(st->y, yj, sizeof(double) * (size_t)m * b);
        memcpy(st->w, wj, sizeof(double) * (size_t)n * b);
        st->z = dblk; dblk = NULL;
        st->t = tblk; tblk = NULL;
        st->lz = l22; l22 = NULL;
        st->l = b;
        st->blocks = 1;
        goto done;
    }
    {
        double* c = mat_tn(st->y, m, lold, yj, b);
        double* f = mat_tn(st->w, n, lold, wj, b);
        double* x = (double*)xcalloc((size_t)lold * b, sizeof(double));
        memcpy(x, c, sizeof(double) * (size_t)lold * b);
        trsm_lower(st->lz, lold, x, b);
        double* s = (double*)xcalloc((size_t)b * b, sizeof(double));
        double* xtx = mat_tn(x, lold, b, x, b);
        for (size_t i = 0; i < (size_t)b * b; ++i) s[i] = dblk[i] - xtx[i];
        free(xtx);
        double diag_ref = 0.0;
        for (int i = 0; i < lold; ++i)
            if (st->z[IDX(i, i, lold)] > diag_ref) diag_ref = st->z[IDX(i, i, lold)];
        for (int i = 0; i < b; ++i)
            if (dblk[IDX(i, i, b)] > diag_ref) diag_ref = dblk[IDX(i, i, b)];
        rc = fqo_chol_factor(s, b, 1e-12, diag_ref, l22);
        free(s);
        if (rc != FQO_OK) { free(c); free(f); free(x); goto fail; }
        double* mm = (double*)xcalloc((size_t)lold * b, sizeof(double));
        memcpy(mm, x, sizeof(double) * (size_t)lold * b);
        trsm_lower_trans(st->lz, lold, mm, b);
        double* r = (double*)xcalloc((size_t)n * b, sizeof(double));
        memcpy(r, wj, sizeof(double) * (size_t)n * b);
        sub_product(r, n, b, st->w, lold, mm);
        trsm_right_lower_trans(l22, b, r, n);
        st->trace_acc += fqo_frob_norm_sq(r, (int64_t)n * b);
        free(mm);
        free(r);

        double* nz = grow_sym(st->z, lold, c, dblk, b);
        double* nt = grow_sym(st->t, lold, f, tblk, b);
        double* nl = grow_chol(st->lz, lold, x, l22, b);
        free(st->z); free(st->t); free(st->lz);
        st->z = nz; st->t = nt; st->lz = nl;
        free(c); free(f); free(x);
        if (state_reserve(st, lold + b)) { rc = FQO_ERR_ALLOC; goto fail; }
        memcpy(st->y + (size_t)m * lold, yj, sizeof(double) * (size_t)m * b);
        memcpy(st->w + (size_t)n * lold, wj, sizeof(double) * (size_t)n * b);
        st->l = lold + b;
        st->blocks += 1;
    }
done:
fail:
    free(yj); free(wj); free(dblk); free(tblk); free(l22);
    return rc;
}

/* assemble_svd (driver.cpp:296-345).  sigma ascending; u, v optional. */
static int assemble_svd(const state_t* st, const double* a_unused, fqo_result* out, int want_vectors) {
    (void)a_unused;
    const int l = st->l, m = st->m, n = st->n;
    out->rank = l;
    out->residual_sq = state_residual(st);
    out->norm_a_sq = st->norm_a_sq;
    out->blocks = st->blocks;
    if (l == 0) return FQO_OK;
    double* zval = (double*)xcalloc((size_t)l, sizeof(double));
    double* d = (double*)xcalloc((size_t)l * l, sizeof(double));
    int rc = fqo_sym_eig(st->z, l, zval, d);
    if (rc != FQO_OK) { free(zval); free(d); return rc; }
    double lmax = zval[l - 1] > 0.0 ? zval[l - 1] : 0.0;
    for (int j = 0; j < l; ++j) {
        double lam = zval[j] > lmax * 1e-31 ? zval[j] : lmax * 1e-31;
        double sc = 1.0 / sqrt(lam);
        for (int i = 0; i < l; ++i) d[IDX(i, j, l)] *= sc;
    }
    double* td = mat_nn(st->t, l, l, d, l);
    double* core = mat_tn(d, l, l, td, l);
    free(td);
    for (int j = 0; j < l; ++j)
        for (int i = j + 1; i < l; ++i) {
            double v = 0.5 * (core[IDX(i, j, l)] + core[IDX(j, i, l)]);
            core[IDX(i, j, l)] = v;
            core[IDX(j, i, l)] = v;
        }
    double* cval = (double*)xcalloc((size_t)l, sizeof(double));
    double* cvec = (double*)xcalloc((size_t)l * l, sizeof(double));
    rc = fqo_sym_eig(core, l, cval, cvec);
    free(core);
    if (rc != FQO_OK) { free(zval); free(d); free(cval); free(cvec); return rc; }
    out->sigma = (double*)xcalloc((size_t)l, sizeof(double));
    for (int j = 0; j < l; ++j) out->sigma[j] = sqrt(cval[j] > 0.0 ? cval[j] : 0.0);
    if (want_vectors) {
        double* dv = mat_nn(d, l, l, cvec, l);
        out->u = mat_nn(st->y, m, l, dv, l);
        double smax = out->sigma[l - 1];
        for (int j = 0; j < l; ++j) {
            double sc = out->sigma[j] > 1e-14 * smax ? 1.0 / out->sigma[j] : 0.0;
            for (int i = 0; i < l; ++i) dv[IDX(i, j, l)] *= sc;
        }
        out->v = mat_nn(st->w, n, l, dv, l);
        free(dv);
    }
    free(zval); free(d); free(cval); free(cvec);
    return FQO_OK;
}

typedef struct {
    int kind;
    double p;
    uint64_t seed;
    int zeta;
} default_src_t;

static int default_source(void* user, int n, int b, int block_id, fqo_block* out) {
    default_src_t* d = (default_src_t*)user;
    return fqo_gen_sketch(d->kind, d->p, d->seed, d->zeta, n, b, block_id, out);
}

typedef struct {
    fqo_source_fn fn;
    void* user;
    int owned;          /* default source: blocks are ours to free */
} source_t;

static int push_id(fqo_result* out, int id) {
    int* v = (int*)realloc(out->block_ids, sizeof(int) * (size_t)(out->n_ids + 1));
    if (!v) return -1;
    out->block_ids = v;
    v[out->n_ids++] = id;
    return 0;
}

static int push_residual(fqo_result* out, int index, double e) {
    double* v = (double*)realloc(out->block_residuals, sizeof(double) * (size_t)(index + 1));
    if (!v) return -1;
    out->block_residuals = v;
    v[index] = e;
    return 0;
}

/* process_block: up to 3 redraws with id + 1000 r (driver.cpp:134-160). */
static int process_block(state_t* st, const double* a, const fqo_config* cfg, source_t* src,
                         const double* zc, int index, fqo_result* out) {
    for (int attempt = 0;; ++attempt) {
        int id = index + 1000 * attempt;
        fqo_block raw;
        memset(&raw, 0, sizeof raw);
        push_id(out, id);
        if (src->fn(src->user, st->n, cfg->block, id, &raw) != 0) {
            set_msg(out, "block source failed");
            return FQO_ERR_CALLBACK;
        }
        int rc;
        if (cfg->power >= 1) {
            double* gd = NULL;
            rc = power_iterate(st, a, &raw, cfg->power, cfg->shift_convention, zc, &gd);
            if (rc == FQO_OK) {
                fqo_block it;
                memset(&it, 0, sizeof it);
                it.is_dense = 1;
                it.rows = st->n;
                it.cols = raw.cols;
                it.dense = gd;
                rc = accept_block(st, a, &it, zc);
                free(gd);
            }
        } else {
            st->alpha = 0.0;
            rc = accept_block(st, a, &raw, zc);
        }
        if (src->owned) fqo_block_free(&raw);
        if (rc == FQO_OK) return FQO_OK;
        if (rc != FQO_ERR_BLOCK_DEGENERATE) return rc;
        if (attempt >= 3) {
            set_msg(out, "block degenerate after 3 redraws");
            return FQO_ERR_BLOCK_DEGENERATE;
        }
    }
}

/* resolve (driver.cpp:116-132). */
static int resolve(int m, int n, const fqo_config* in, int fixed_precision, fqo_config* cfg,
                   fqo_result* out) {
    if (m < 1 || n < 1) { set_msg(out, "matrix must be non-empty"); return FQO_ERR_CONFIG; }
    *cfg = *in;
    if (cfg->block == 0) cfg->block = fqo_default_block(m, n);
    if (cfg->block < 1) { set_msg(out, "block size must be at least 1"); return FQO_ERR_CONFIG; }
    if (cfg->block > (m < n ? m : n)) { set_msg(out, "block size exceeds matrix dimensions"); return FQO_ERR_CONFIG; }
    if (cfg->max_iters == 0) cfg->max_iters = fqo_default_max_iters(n, cfg->block);
    if (cfg->max_iters < 1) { set_msg(out, "max_iters must be at least 1"); return FQO_ERR_CONFIG; }
    if (cfg->power < 0) { set_msg(out, "power must be non-negative"); return FQO_ERR_CONFIG; }
    if (cfg->kind != FQO_GAUSSIAN && cfg->p == 0.0) cfg->p = fqo_default_density(cfg->kind, n);
    if (fixed_precision && !(cfg->eps > 0.0)) {
        set_msg(out, "fixed-precision mode needs a positive tolerance");
        return FQO_ERR_CONFIG;
    }
    return FQO_OK;
}

static int run_common(const double* a, int m, int n, int rank, int fixed_precision,
                      const fqo_config* cfg_in, fqo_source_fn fn, void* user,
                      int want_vectors, fqo_result* out) {
    memset(out, 0, sizeof *out);
    out->m = m;
    out->n = n;
    fqo_config cfg;
    int rc = resolve(m, n, cfg_in, fixed_precision, &cfg, out);
    if (rc == FQO_OK && !fixed_precision) {
        if (rank < 1) { set_msg(out, "rank must be at least 1"); rc = FQO_ERR_CONFIG; }
        else if (rank > (m < n ? m : n)) { set_msg(out, "rank exceeds matrix dimensions"); rc = FQO_ERR_CONFIG; }
    }
    if (rc != FQO_OK) { out->status = rc; return rc; }
    out->resolved_block = cfg.block;
    out->resolved_max_iters = cfg.max_iters;
    out->resolved_p = cfg.p;

    default_src_t dflt = {cfg.kind, cfg.p, cfg.seed, cfg.zeta};
    source_t src = {fn, user, 0};
    if (!fn) { src.fn = default_source; src.user = &dflt; src.owned = 1; }

    state_t st;
    memset(&st, 0, sizeof st);
    st.m = m; st.n = n; st.b = cfg.block;
    st.norm_a_sq = fqo_frob_norm_sq(a, (int64_t)m * n);
    double* zc = NULL;
    if (cfg.kind == FQO_STD_BERNOULLI) {
        zc = (double*)xcalloc((size_t)m, sizeof(double));
        fqo_centering_column(a, m, n, cfg.p, zc);
    }
    int converged = 0;
    if (fixed_precision) {
        double norm_a = sqrt(st.norm_a_sq);
        double eps_abs = cfg.relative ? cfg.eps * norm_a : cfg.eps;
        double eps_sq = eps_abs * eps_abs;
        if (state_residual(&st) <= eps_sq) {
            converged = 1;
        } else {
            for (int j = 0; j < cfg.max_iters; ++j) {
                rc = process_block(&st, a, &cfg, &src, zc, j, out);
                if (rc != FQO_OK) break;
                push_residual(out, st.blocks - 1, state_residual(&st));
                if (state_residual(&st) < eps_sq) { converged = 1; break; }
            }
        }
    } else {
        int nblocks = (rank + cfg.block - 1) / cfg.block;
        for (int j = 0; j < nblocks; ++j) {
            rc = process_block(&st, a, &cfg, &src, zc, j, out);
            if (rc != FQO_OK) break;
            push_residual(out, st.blocks - 1, state_residual(&st));
        }
        converged = 1;
    }
    if (rc == FQO_OK) {
        rc = assemble_svd(&st, a, out, want_vectors);
        if (rc == FQO_OK && !fixed_precision) {
            /* drop_smallest (driver.cpp:85-106) */
            int extra = ((rank + cfg.block - 1) / cfg.block) * cfg.block - rank;
            if (extra > 0 && out->rank > extra) {
                double acc = out->residual_sq;
                for (int i = 0; i < extra; ++i) acc += out->sigma[i] * out->sigma[i];
                out->residual_sq = acc;
                int r = out->rank - extra;
                memmove(out->sigma, out->sigma + extra, sizeof(double) * (size_t)r);
                if (out->u) memmove(out->u, out->u + (size_t)m * extra, sizeof(double) * (size_t)m * r);
                if (out->v) memmove(out->v, out->v + (size_t)n * extra, sizeof(double) * (size_t)n * r);
                out->rank = r;
            }
        }
        out->converged = converged;
        if (rc == FQO_OK && fixed_precision && !converged) {
            rc = FQO_ERR_TOLERANCE_NOT_REACHED;
            set_msg(out, "tolerance not reached");
        }
    } else {
        out->blocks = st.blocks;
        out->residual_sq = state_residual(&st);
        out->norm_a_sq = st.norm_a_sq;
    }
    free(zc);
    state_free(&st);
    out->status = rc;
    return rc;
}

int fqo_run_fixed_precision(const double* a, int m, int n, const fqo_config* cfg,
                            fqo_source_fn src, void* user, int want_vectors,
                            fqo_result* out) {
    return run_common(a, m, n, 0, 1, cfg, src, user, want_vectors, out);
}

int fqo_run_fixed_rank(const double* a, int m, int n, int rank, const fqo_config* cfg,
                       fqo_source_fn src, void* user, int want_vectors, fqo_result* out) {
    return run_common(a, m, n, rank, 0, cfg, src, user, want_vectors, out);
}

void fqo_result_free(fqo_result* r) {
    if (!r) return;
    free(r->sigma); free(r->u); free(r->v); free(r->block_residuals); free(r->block_ids);
    r->sigma = NULL; r->u = NULL; r->v = NULL; r->block_residuals = NULL; r->block_ids = NULL;
}
