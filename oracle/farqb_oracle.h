/*
 * farqb_oracle.h -- CPU restatement of the reference farPCA blocked QB loop.
 *
 * TEST INFRASTRUCTURE ONLY.  Nothing in the product path (paper_2506_03859_b200,
 * libfarqb) may include, link or call this.  It is the checker that the CUDA
 * path is compared against: tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline leg are its only users.
 *
 * Each function restates the reference algorithm in plain C and cites the
 * reference file:line it follows (paths relative to /root/reference/proj).
 * The restatement is pinned against the reference itself (oracle/_ref, built
 * from the untouched reference sources by oracle/Makefile) and against the
 * golden vectors in tests/golden/.
 *
 * The shared ABI below (fqo_block / fqo_config / fqo_result / fqo_source_fn)
 * is also exported by oracle/ref_shim.cpp under the ref_ prefix, so a test can
 * run the same case through the restatement and through the reference.
 */
#ifndef FARQB_ORACLE_H
#define FARQB_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Sketch kinds, numbered like rsvd::SketchKind (include/rsvd/sketch.hpp:11). */
enum { FQO_GAUSSIAN = 0, FQO_BERNOULLI = 1, FQO_STD_BERNOULLI = 2,
       FQO_SPARSE_SIGN = 3, FQO_SPARSE_GAUSSIAN = 4 };

/* Status codes, identical to the product C-ABI (include/farqb.h). */
enum { FQO_OK = 0, FQO_ERR_CONFIG = 1, FQO_ERR_DIMENSION = 2,
       FQO_ERR_BLOCK_DEGENERATE = 3, FQO_ERR_TOLERANCE_NOT_REACHED = 4,
       FQO_ERR_CONVERGENCE = 8, FQO_ERR_CALLBACK = 9, FQO_ERR_ALLOC = 10 };

/* One test-matrix block: rsvd::SketchBlock (include/rsvd/sketch.hpp:37-44). */
typedef struct {
    int is_dense;
    int rows, cols;
    double* dense;      /* rows x cols, column-major, when is_dense          */
    int* col_ptr;       /* cols + 1                                          */
    int* row_idx;       /* nnz, strictly increasing within each column        */
    double* values;     /* nnz                                               */
    int64_t nnz;
    int centered;       /* StdBernoulli: consumers apply the centering trick  */
    double p;
    double std_scale;
} fqo_block;

/* rsvd::FarpcaConfig (include/rsvd/driver.hpp:18-26) plus zeta: when > 0 the
 * sparse-sign / sparse-Gaussian kinds draw exactly zeta nonzeros per column
 * (BASELINE configs 3-5), see fqo_gen_sketch. */
typedef struct {
    double eps;
    int power;
    int block;
    int kind;
    double p;
    uint64_t seed;
    int zeta;
    int max_iters;
    int shift_convention; /* 0 LastDiagonal, 1 FirstDiagonal */
    int relative;
} fqo_config;

typedef struct {
    int status;
    int m, n;
    int rank;                 /* number of singular triplets               */
    int blocks;
    int converged;
    double residual_sq;
    double norm_a_sq;
    double* sigma;            /* ascending, length rank                     */
    double* u;                /* m x rank, only with want_vectors           */
    double* v;                /* n x rank, only with want_vectors           */
    double* block_residuals;  /* E after each accepted block, length blocks */
    int* block_ids;           /* ids requested from the source, in order    */
    int n_ids;
    int resolved_block;
    int resolved_max_iters;
    double resolved_p;
    char message[256];
} fqo_result;

/* rsvd::BlockSource::next (include/rsvd/driver.hpp:69-73).  The callee fills
 * *out; its arrays must stay valid until the next call or the end of the run.
 * Return 0 on success. */
typedef int (*fqo_source_fn)(void* user, int n, int b, int block_id, fqo_block* out);

/* ---- Philox4x32-10 (include/rsvd/rng.hpp:15-88) ---------------------------- */
void fqo_philox_u32(uint64_t seed, uint32_t block_id, uint32_t column, int count, uint32_t* out);
void fqo_philox_units(uint64_t seed, uint32_t block_id, uint32_t column, int count, double* out);
void fqo_philox_gaussians(uint64_t seed, uint32_t block_id, uint32_t column, int count, double* out);

/* ---- sketches (src/sketch.cpp:51-148) ------------------------------------- */
int fqo_gen_sketch(int kind, double p, uint64_t seed, int zeta, int n, int l,
                   int block_id, fqo_block* out);
void fqo_block_free(fqo_block* blk);
void fqo_sparse_dense_mul(const double* a, int m, int n, const int* col_ptr,
                          const int* row_idx, const double* values, int l, double* c);
void fqo_dense_sparse_tmul(const double* w, int n, int k, const int* col_ptr,
                           const int* row_idx, const double* values, int l, double* c);
void fqo_centering_column(const double* a, int m, int n, double p, double* z);
double fqo_frob_norm_sq(const double* a, int64_t count);

/* ---- dense kernels (src/kernels_scalar.cpp, src/matrix_core.cpp) --------- */
void fqo_gemm_nn(int m, int n, int k, const double* a, int lda, const double* b,
                 int ldb, double* c, int ldc);
void fqo_gemm_tn(int m, int n, int k, const double* a, int lda, const double* b,
                 int ldb, double* c, int ldc);
int fqo_sym_eig(const double* mtx, int n, double* values, double* vectors);
int fqo_chol_factor(const double* z, int n, double pivot_tol, double diag_ref, double* l);

/* ---- driver (src/driver.cpp) ---------------------------------------------- */
int fqo_run_fixed_precision(const double* a, int m, int n, const fqo_config* cfg,
                            fqo_source_fn src, void* user, int want_vectors,
                            fqo_result* out);
int fqo_run_fixed_rank(const double* a, int m, int n, int rank, const fqo_config* cfg,
                       fqo_source_fn src, void* user, int want_vectors, fqo_result* out);
void fqo_result_free(fqo_result* r);

double fqo_default_density(int kind, int n);
int fqo_default_block(int m, int n);
int fqo_default_max_iters(int n, int b);

#ifdef __cplusplus
}
#endif
#endif
