/*
 * farqb.h -- C-ABI of libfarqb.so, the B200 (sm_100a) farPCA blocked-QB engine.
 *
 * This is the drop-in boundary for the reference's hot path.  The reference is
 * a C++ library with no FFI of its own; the entry points below are what a
 * C/ctypes/cgo/JNI binding of its QB API would bind, one for one:
 *
 *   fqb_qb_fixed_precision  <- rsvd::run_fixed_precision
 *                              (/root/reference/proj/include/rsvd/driver.hpp:98-99,
 *                               src/driver.cpp:347-388)
 *   fqb_qb_fixed_rank       <- rsvd::run_fixed_rank (driver.hpp:101-103, driver.cpp:390-413)
 *   fqb_block_source_fn     <- rsvd::BlockSource::next (driver.hpp:67-73)
 *   fqb_config              <- rsvd::FarpcaConfig (driver.hpp:18-26) + SketchSpec
 *                              (sketch.hpp:18-22), plus `zeta` (fixed nonzeros per
 *                              column, BASELINE configs 3-5)
 *   fqb_qb_result           <- rsvd::ApproxSvd's scalars (driver.hpp:45-58) plus the
 *                              north-star QB outputs Q (m x l) and B' (n x l)
 *   fqb_status              <- the exception taxonomy of errors.hpp:9-46 and
 *                              ToleranceNotReached (driver.hpp:60-65)
 *   fqb_gen_sketch          <- rsvd::gen_sketch (sketch.hpp:46, sketch.cpp:51-102)
 *   fqb_sparse_dense_mul    <- rsvd::sparse_dense_mul / centered_product (sketch.cpp:104-140)
 *   fqb_centering_column    <- rsvd::centering_column (driver.hpp:78, driver.cpp:178-183)
 *   fqb_frob_norm_sq        <- rsvd::frob_norm_sq (matrix_core.hpp:59, matrix_core.cpp:46-48)
 *   fqb_relative_error      <- rsvd::relative_error (experiment.hpp, experiment.cpp:317-342)
 *   fqb_sym_eig             <- rsvd::sym_eig (matrix_core.hpp, matrix_core.cpp:50-115) as used by
 *                              assemble_svd (driver.cpp:296-345) for the l x l Gram matrices
 *   fqb_gemm                <- rsvd::kern::Ops::gemm_nn / gemm_tn (kernels.hpp:9-19)
 *   fqb_chol_factor         <- rsvd::chol_factor (matrix_core.hpp:36-38, matrix_core.cpp:117-140),
 *                              the b x b factorizations of the CholeskyQR steps
 *   fqb_gram                <- rsvd::matmul_tn(y, y) (matrix_core.cpp:28-35) for the b x b Grams
 *                              of accept_block / eig_svd (driver.cpp:230-294, matrix_core.cpp:193-215)
 *   fqb_mul_upper           <- trsm_right_lower_trans (matrix_core.cpp:167-179) given the inverse
 *                              factor: Y R^-1 with R^-1 upper triangular
 *   fqb_philox_u32          <- rsvd::Philox::next_u32 (rng.hpp:21-24)
 *   fqb_random_orthonormal  <- rsvd::random_orthonormal (synthetic.hpp, synthetic.cpp:121-126)
 *   fqb_gen_synthetic       <- rsvd::gen_synthetic (synthetic.hpp, synthetic.cpp:159-180)
 *
 * Beyond the reference: fqb_qb_*_f32 (FP32 input, BASELINE config 5), the INT8
 * tensor-core FP64 emulation of the A passes (fqb_gemm_emulated, fqb_slice_operand /
 * fqb_sliced_gemm), fqb_gen_lowrank (configs 2-5 inputs), row-sharded multi-GPU
 * (fqb_comm_*).
 *
 * Conventions: matrices are column-major doubles with an explicit leading
 * dimension; sizes are int64_t; no C++ types cross this boundary and no
 * exception escapes it.  Every call returns an fqb_status; the message of the
 * last failure on the calling thread is fqb_last_error().  There is no CPU
 * compute path: without a CUDA device every compute entry point fails with
 * FQB_ERR_CUDA.
 */
#ifndef FARQB_H
#define FARQB_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define FARQB_ABI_VERSION 3

typedef enum fqb_status {
    FQB_OK = 0,
    FQB_ERR_CONFIG = 1,                 /* rsvd::ConfigError                     */
    FQB_ERR_DIMENSION = 2,              /* rsvd::DimensionError                  */
    FQB_ERR_BLOCK_DEGENERATE = 3,       /* rsvd::BlockDegenerate (after 3 redraws) */
    FQB_ERR_TOLERANCE_NOT_REACHED = 4,  /* rsvd::ToleranceNotReached; result still filled */
    FQB_ERR_CUDA = 5,                   /* CUDA runtime / no device              */
    FQB_ERR_NCCL = 6,                   /* collective failure                    */
    FQB_ERR_INVALID_ARGUMENT = 7,       /* null pointer, bad handle, bad enum    */
    FQB_ERR_CONVERGENCE = 8,            /* rsvd::ConvergenceFailure              */
    FQB_ERR_CALLBACK = 9,               /* block source returned non-zero        */
    FQB_ERR_ALLOC = 10,                 /* device or host allocation failed      */
    FQB_ERR_FORMAT = 11                 /* rsvd::FormatError (matrix file); byte offset returned */
} fqb_status;

/* rsvd::SketchKind, same numbering (sketch.hpp:11). */
typedef enum fqb_sketch_kind {
    FQB_GAUSSIAN = 0,
    FQB_BERNOULLI = 1,
    FQB_STD_BERNOULLI = 2,
    FQB_SPARSE_SIGN = 3,
    FQB_SPARSE_GAUSSIAN = 4
} fqb_sketch_kind;

typedef struct fqb_sketch_spec {
    int kind;          /* fqb_sketch_kind                                        */
    double p;          /* density; 0 picks default_density (driver.cpp:449-455)  */
    uint64_t seed;
    int zeta;          /* > 0: exactly zeta nonzeros per column (sign/Gaussian)  */
} fqb_sketch_spec;

typedef struct fqb_config {
    double eps;              /* Frobenius tolerance (relative when `relative`)  */
    int power;               /* power-iteration passes P                        */
    int block;               /* block size b; 0 picks default_block             */
    fqb_sketch_spec sketch;
    int max_iters;           /* 0 picks ceil(n / 2b)                            */
    int shift_convention;    /* 0 LastDiagonal, 1 FirstDiagonal (driver.hpp:16) */
    int relative;            /* eps is a fraction of ||A||_F                    */
} fqb_config;

/* One raw test-matrix block handed over by a block source (HOST memory, owned
 * by the source, valid until the source is called again or the run returns).
 * Mirrors rsvd::SketchBlock (sketch.hpp:37-44). */
typedef struct fqb_block {
    int is_dense;
    int rows, cols;
    const double* dense;     /* rows x cols column-major (ld = rows)            */
    const int* col_ptr;      /* cols + 1                                        */
    const int* row_idx;      /* nnz, strictly increasing per column             */
    const double* values;    /* nnz                                             */
    int64_t nnz;
    int centered;            /* StdBernoulli centering trick                    */
    double p;
    double std_scale;
} fqb_block;

/* BlockSource::next.  Return 0 on success, anything else aborts the run with
 * FQB_ERR_CALLBACK.  NULL source = the on-device Philox generator. */
typedef int (*fqb_block_source_fn)(void* user, int n, int b, int block_id, fqb_block* out);

/* Output placement flags for fqb_qb_*. */
#define FQB_OUT_NONE   0u   /* scalars, trace and ids only                       */
#define FQB_OUT_HOST   1u   /* copy Q and B' into malloc'd host arrays           */
#define FQB_OUT_DEVICE 2u   /* keep Q and B' on the device (library-owned)       */
#define FQB_OUT_SVD    4u   /* also assemble U, sigma, V like rsvd::ApproxSvd     */
                            /* (assemble_svd, driver.cpp:296-345); fixed-rank runs */
                            /* drop the overshoot like drop_smallest (:85-106)     */

typedef struct fqb_qb_result {
    int status;              /* same as the call's return value                 */
    int64_t m, n;
    int rank;                /* l = blocks * b                                  */
    int blocks;
    int converged;
    double residual_sq;      /* E = ||A||_F^2 - sum_j ||B_j||_F^2                */
    double norm_a_sq;
    double* q;               /* m x rank, ld = ldq  (host or device, see flags) */
    int64_t ldq;
    double* bt;              /* n x rank = B',  ld = ldbt                        */
    int64_t ldbt;
    int on_device;
    double* block_residuals; /* host, E after each accepted block, `blocks`     */
    int* block_ids;          /* host, every id requested from the source        */
    int n_ids;
    int resolved_block;
    int resolved_max_iters;
    double resolved_p;
    int gpu_launches;        /* kernels this call launched                      */
    double elapsed_ms;       /* device time of the call (CUDA events)           */
    /* ApproxSvd fields (driver.hpp:45-58), filled with FQB_OUT_SVD: */
    int svd_rank;            /* r (fixed rank: the requested rank)               */
    double* sigma;           /* host, ascending, r                               */
    char* v_flagged;         /* host, r                                          */
    double* u;               /* m x r (this rank's rows), placement as q         */
    int64_t ldu;
    double* v;               /* n x r                                            */
    int64_t ldv;
    double svd_residual_sq;  /* residual_sq plus the dropped energy (fixed rank) */
    void* internal;
} fqb_qb_result;

typedef struct fqb_handle_s* fqb_handle;

/* ---- lifecycle ------------------------------------------------------------- */
int fqb_abi_version(void);
fqb_status fqb_create(int device, fqb_handle* out);
fqb_status fqb_destroy(fqb_handle h);
/* Run subsequent work on this cudaStream_t (NULL = the handle's own stream, which
 * is a blocking stream: it waits for work queued on the legacy default stream).
 * Device inputs must be complete in the order of the stream the handle uses. */
fqb_status fqb_set_stream(fqb_handle h, void* cuda_stream);
fqb_status fqb_synchronize(fqb_handle h);
const char* fqb_last_error(void);
const char* fqb_status_name(int status);
/* Kernels launched by this handle since creation (launch accounting). */
int64_t fqb_launch_count(fqb_handle h);
/* Live timing of the dominant kernel: while on, every A-pass k_ozaki launch (with its
 * stream-K fixup) of this handle's runs is bracketed by CUDA events on the handle's
 * stream.  fqb_set_pass_timing synchronizes the stream and resets the record;
 * fqb_pass_timing synchronizes and returns the summed launch time (ms), the number of
 * launches and their algorithmic FP64 bytes 8 (MK + KN + MN) (any pointer may be NULL). */
fqb_status fqb_set_pass_timing(fqb_handle h, int on);
fqb_status fqb_pass_timing(fqb_handle h, double* total_ms, int64_t* launches, double* bytes);

/* ---- the QB loop ----------------------------------------------------------- */
/* A is m x n column-major with leading dimension lda, on the device when
 * a_on_device != 0 (used in place when lda is even and 16-byte aligned,
 * otherwise copied once), else on the host (copied to the device inside the
 * call).  `src` may be NULL.  On FQB_ERR_TOLERANCE_NOT_REACHED the result is
 * the partial factorization, like ToleranceNotReached::partial. */
fqb_status fqb_qb_fixed_precision(fqb_handle h, const double* a, int64_t m, int64_t n,
                                  int64_t lda, int a_on_device, const fqb_config* cfg,
                                  fqb_block_source_fn src, void* user, unsigned flags,
                                  fqb_qb_result* out);
fqb_status fqb_qb_fixed_rank(fqb_handle h, const double* a, int64_t m, int64_t n,
                             int64_t lda, int a_on_device, int rank, const fqb_config* cfg,
                             fqb_block_source_fn src, void* user, unsigned flags,
                             fqb_qb_result* out);
/* FP32 input mode (BASELINE config 5: 400000 x 50000 FP32): A stays in FP32 in
 * HBM (half the bytes of FP64), every product is formed in FP64 from the exactly
 * widened values -- the results are those of the FP64 loop on double(A), within
 * the FP64 parity bounds, which are tighter than the FP32-mode 1e-4.  The A passes
 * slice A straight from FP32 for the INT8 tensor cores; when they run on DMMA
 * instead (b > 64, small A, slices out of memory) one widened FP64 copy is made. */
fqb_status fqb_qb_fixed_precision_f32(fqb_handle h, const float* a, int64_t m, int64_t n,
                                      int64_t lda, int a_on_device, const fqb_config* cfg,
                                      fqb_block_source_fn src, void* user, unsigned flags,
                                      fqb_qb_result* out);
fqb_status fqb_qb_fixed_rank_f32(fqb_handle h, const float* a, int64_t m, int64_t n,
                                 int64_t lda, int a_on_device, int rank, const fqb_config* cfg,
                                 fqb_block_source_fn src, void* user, unsigned flags,
                                 fqb_qb_result* out);
void fqb_result_free(fqb_qb_result* r);
/* Host results (Q, B', U, V) live in pinned, pooled memory (fast D2H, no page
 * faults).  A caller that keeps one of those arrays beyond the result frees it
 * with fqb_host_free and sets the field to NULL before fqb_result_free. */
void fqb_host_free(void* p);
/* Host results live in a process-wide pool of pinned blocks, reused across runs; at most
 * FQB_HOST_POOL_MB (environment, default 4096) MB of free blocks stay cached.  This
 * releases every cached free block now (also done when the last handle is destroyed);
 * returns the bytes released. */
size_t fqb_host_pool_trim(void);
/* Device blocks of >= 16 MB (Q, B', U, V, the A slices, A copies) come from a per-device
 * cache of cudaMalloc'd blocks (a multi-GB cudaMallocAsync costs milliseconds, sometimes
 * hundreds); device results freed with fqb_result_free return to it.  At most
 * FQB_DEVICE_CACHE_MB (default half the device memory) stays cached; this releases every
 * cached block now (also done when the last handle is destroyed); returns the bytes. */
size_t fqb_device_cache_trim(void);

/* ---- row-sharded multi-GPU (one rank per GPU, NCCL over NVLink) ------------- */
/* Rank 0 creates a 128-byte id, the caller distributes it (e.g. with
 * torch.distributed or MPI), every rank attaches.  With a communicator attached,
 * the `a, m, lda` passed to fqb_qb_* are this rank's contiguous row block of A;
 * Q comes back as this rank's rows, B' (and every scalar) is replicated.  The
 * sums over rows (||A||^2, A'Y and the Gram blocks) are NCCL all-reduces. */
fqb_status fqb_comm_unique_id(void* out128);
fqb_status fqb_comm_attach(fqb_handle h, const void* id128, int nranks, int rank);
fqb_status fqb_comm_detach(fqb_handle h);
/* The same row sharding over a host transport: at every reduction point the engine
 * copies the partial sums to pinned host memory and calls fn(user, buf, count), which
 * must sum `count` doubles in place across all ranks (MPI_Allreduce, a gloo all-reduce)
 * and return 0; nonzero fails the run with FQB_ERR_NCCL.  Called on the thread that
 * runs fqb_qb_*.  Slower than NCCL (a device sync per reduction), for hosts that bring
 * their own transport and for multi-rank tests sharing one GPU. */
typedef int (*fqb_host_allreduce_fn)(void* user, double* buf, int64_t count);
fqb_status fqb_comm_attach_host(fqb_handle h, fqb_host_allreduce_fn fn, void* user, int nranks, int rank);
/* ---- RawF64 matrix files (matrix_io.cpp:141-200, rsvd::load_matrix RawF64) ---- */
/* Validates a "SKLR" file exactly like the reference's loader: on a malformed file
 * FQB_ERR_FORMAT, the reference's FormatError message in fqb_last_error() and its byte
 * offset in *err_offset (may be NULL). */
fqb_status fqb_raw_header(const char* path, int64_t* rows, int64_t* cols, int64_t* err_offset);
/* Rows [row0, row0 + rows) of every column (a rank's row shard; all rows: row0 = 0,
 * rows = m) into dst (rows x cols, ld >= rows), device memory when dst_on_device (pinned
 * staging panels, reads overlapped with the uploads on the handle's stream; returns when
 * the data has landed), else host memory (h may then be NULL).  Multi-threaded pread. */
fqb_status fqb_load_raw_rows(fqb_handle h, const char* path, int64_t row0, int64_t rows, double* dst, int64_t ld,
                             int dst_on_device, int64_t* err_offset);

/* collectives issued by this handle since creation */
int64_t fqb_collective_count(fqb_handle h);

/* ---- building blocks (device pointers unless stated) ------------------------ */
/* First `count` u32 words of the Philox stream (seed, block_id, column), into
 * host memory; generated on the device. */
fqb_status fqb_philox_u32(fqb_handle h, uint64_t seed, uint32_t block_id, uint32_t column,
                          int count, uint32_t* host_out);

/* Host copy of a device-generated test block (rsvd::gen_sketch).  Arrays are
 * malloc'd by the library; release with fqb_sketch_free. */
typedef struct fqb_sketch_host {
    int is_dense, rows, cols;
    double* dense;
    int* col_ptr;
    int* row_idx;
    double* values;
    int64_t nnz;
    int centered;
    double p, std_scale;
} fqb_sketch_host;
fqb_status fqb_gen_sketch(fqb_handle h, const fqb_sketch_spec* spec, int n, int l, int block_id,
                          fqb_sketch_host* out);
void fqb_sketch_free(fqb_sketch_host* s);

/* c (m x l, ldc) = a (m x n, lda) * S (CSC, device arrays) [- z broadcast when
 * z != NULL]; one fused multiply-add per nonzero in CSC order. */
fqb_status fqb_sparse_dense_mul(fqb_handle h, const double* a, int64_t m, int64_t n, int64_t lda,
                                const int* col_ptr, const int* row_idx, const double* values,
                                int l, const double* z, double* c, int64_t ldc);
/* z (m) = A (p 1_n) */
fqb_status fqb_centering_column(fqb_handle h, const double* a, int64_t m, int64_t n, int64_t lda,
                                double p, double* z);
/* ||A||_F^2 into *host_out */
fqb_status fqb_frob_norm_sq(fqb_handle h, const double* a, int64_t m, int64_t n, int64_t lda,
                            double* host_out);
/* FP32 input mode (fqb_qb_*_f32): slices per operand of the A passes on the INT8 tensor
 * cores.  Any value >= 7 (the default sentinel is 8): every product FP64-class -- the FP64
 * scheme with fqb_fp64_slices() slices (7 by default) -- and the run equals the FP64 run on
 * the widened A to ~1e-15.  4: FP32-class products (~2^-26 of
 * max|row| max|col|, ten int8 products on 7-bit digits, 4 bytes per element of A);
 * 3: FP32-class on 8-bit digits (8 products, 3 bytes per element, representation 2^-23
 * of the line max) -- both within the FP32-mode parity bar of 1e-4 and about twice as
 * fast as 8.  Applies to runs started after the call. */
fqb_status fqb_set_fp32_slices(fqb_handle h, int slices);
/* int8 slices per element of A in the FP64-class A passes: 7 (8-bit digits, 34 int8
 * products per output; the default) or 8 (7-bit digits, 36 products; environment
 * FQB_OZ_SLICES=8).  Also the bytes per element of A each pass streams from HBM. */
int fqb_fp64_slices(void);

/* Symmetric eigendecomposition (device pointers; both triangles of A read):
 * eigenvalues ascending into w (n), eigenvectors into V (n x n, ldv).  The solver of
 * the SVD assembly: for n <= 224 a one-CTA Householder tridiagonalisation + bisection /
 * inverse-iteration solver verified a posteriori (residual and orthogonality at 64 n u;
 * cuSOLVER syevd when the check fails or FQB_EIG=syevd), cuSOLVER syevd above.
 * *used_small (nullable) = 1 when the former produced the result. */
fqb_status fqb_sym_eig(fqb_handle h, const double* a, int n, int64_t lda, double* w, double* v, int64_t ldv,
                       int* used_small);
/* Exact relative error ||A - U diag(sigma) V'||_F / ||A||_F (experiment.cpp:317-342),
 * one pass over A in column strips on the device.  U is m x r (ldu), V is n x r (ldv);
 * sigma (host, r values) may be NULL for a QB pair (U = Q, V = B').  A and the factors
 * are on the device when the *_on_device flags are set, else copied in.  0 for A = 0,
 * 1 for r = 0, like the reference. */
fqb_status fqb_relative_error(fqb_handle h, const double* a, int64_t m, int64_t n, int64_t lda, int a_on_device,
                              const double* u, int64_t ldu, const double* sigma, const double* v, int64_t ldv,
                              int r, int factors_on_device, double* host_out);
/* Cholesky of a symmetric n x n matrix Z (device pointers; Z must be symmetric), the
 * reference's chol_factor: with max_diag = diag_ref if > 0, else max_i Z(i,i), a pivot
 * (the Schur complement diagonal l(j,j)^2) at or below pivot_tol * max_diag makes
 * *rank_deficient = 1 (the reference's RankDeficient) and R = R^-1 = I; otherwise
 * *rank_deficient = 0, R (n x n, ldr) = L' (upper) and Rinv (ldri) = L'^-1 (upper) --
 * the forms the CholeskyQR steps use.  One CTA, n <= 1024 (registers + one barrier per
 * column for n <= 128, shared / global memory above). */
fqb_status fqb_chol_factor(fqb_handle h, const double* z, int n, int64_t ldz, double pivot_tol, double diag_ref,
                           double* r, int64_t ldr, double* rinv, int64_t ldri, int* rank_deficient);
/* S (b x b, lds) = Y' Y for a tall Y (K x b, ldy), device pointers: for b <= 128 only the
 * 8 x 8 tiles on and above the diagonal are formed and mirrored (S exactly symmetric),
 * rows split over the SMs and the partials summed in a fixed order (deterministic). */
fqb_status fqb_gram(fqb_handle h, const double* y, int64_t k, int b, int64_t ldy, double* s, int64_t lds);
/* Z (M x b, ldz) = Y (M x b, ldy) * R with R (b x b, ldr) upper triangular -- its strictly
 * lower part is not read.  Device pointers; Z must not overlap Y. */
fqb_status fqb_mul_upper(fqb_handle h, const double* y, int64_t m, int b, int64_t ldy, const double* r, int64_t ldr,
                         double* z, int64_t ldz);
/* C (m x n) = alpha * op(A) * B + beta * C, op(A) = A (trans_a = 0, A is m x k)
 * or A' (trans_a = 1, A is k x m); B is k x n.  FP64 on the DMMA tensor pipe. */
fqb_status fqb_gemm(fqb_handle h, int trans_a, int64_t m, int64_t n, int64_t k, double alpha,
                    const double* a, int64_t lda, const double* b, int64_t ldb, double beta,
                    double* c, int64_t ldc);

/* Same contract as fqb_gemm, computed on the INT8 tensor cores (tcgen05
 * kind::i8) by Ozaki slicing: 8 signed 7-bit slices per operand with one
 * power-of-two scale per output row / column, exact int32 slice products, FP64
 * recombination -- the accuracy class of an FP64 GEMM.  Any n (B is sliced in chunks
 * of <= 64 columns, one pass over the slices of A each). */
fqb_status fqb_gemm_emulated(fqb_handle h, int trans_a, int64_t m, int64_t n, int64_t k, double alpha,
                             const double* a, int64_t lda, const double* b, int64_t ldb, double beta,
                             double* c, int64_t ldc);

/* Persistent sliced operand: A (m x n, lda, device memory) cut once into the Ozaki
 * slices of both layouts (16 m n bytes of device memory), then any number of
 *     C = alpha op(A) B + beta C,   op(A) = A' (trans_a: B m x nb, C n x nb)
 *                                   op(A) = A  (B n x nb, C m x nb)
 * (nb > 64 in chunks of <= 64 columns)
 * products on the INT8 tensor cores -- the engine's A-pass path, exposed for
 * callers that apply one matrix many times (and used by bench.py to time it).
 * A must stay unchanged while the slices are in use only in the sense that the
 * slices are a snapshot of it.  Asynchronous on the handle's stream. */
typedef struct fqb_sliced_s* fqb_sliced;
fqb_status fqb_slice_operand(fqb_handle h, const double* a, int64_t m, int64_t n, int64_t lda, fqb_sliced* out);
fqb_status fqb_sliced_gemm(fqb_handle h, fqb_sliced s, int trans_a, int64_t nb, double alpha, const double* b,
                           int64_t ldb, double beta, double* c, int64_t ldc);
/* The last fqb_sliced_gemm on s once more, on the B slices it left behind (its nb <= 128):
 * C = alpha op(A) B + beta C with the same op(A) and B -- only the tensor-core GEMM
 * (k_ozaki, + the stream-K fixup when a tile is split) runs, no slicing of B.  For
 * repeated products with one B, and for timing the GEMM kernel by itself. */
fqb_status fqb_sliced_gemm_again(fqb_handle h, fqb_sliced s, double alpha, double beta, double* c, int64_t ldc);
/* C (m x nb) = alpha A B + beta C (B n x nb) computed from the A'Y-layout slices alone,
 * read MN-major by the kernel (B's rows are first scaled by A's column scales) -- the
 * product the engine's block Gram-Schmidt uses for Y -= Q C on the slices of Q its
 * Q'Y products made.  Same accuracy class as fqb_sliced_gemm(trans_a = 0), different
 * rounding (per-column instead of per-row scales of A). */
fqb_status fqb_sliced_gemm_mn(fqb_handle h, fqb_sliced s, int64_t nb, double alpha, const double* b, int64_t ldb,
                              double beta, double* c, int64_t ldc);
fqb_status fqb_sliced_free(fqb_handle h, fqb_sliced s);

/* ---- test matrices on the device (reference synthetic.cpp) ----- */
/* rsvd::random_orthonormal (synthetic.cpp:121-126): n x r orthonormal columns from
 * Philox(seed, stream, column) Gaussian panels of 64, block Gram-Schmidt + CholeskyQR
 * twice per panel (bcgs2_step, :36-53).  q is device memory (ldq >= n). */
fqb_status fqb_random_orthonormal(fqb_handle h, int64_t n, int r, uint64_t seed, uint32_t stream, double* q,
                                  int64_t ldq);
/* rsvd::gen_synthetic (synthetic.cpp:159-180) into device memory: kind 0 slow decay
 * (1/j^2), 1 fast decay (e^{-j/20}), 2 block-diagonal V with d blocks; *rank_out = the
 * kept rank (sigma < 1e-18 sigma_1 dropped). */
fqb_status fqb_gen_synthetic(fqb_handle h, int kind, int n, int d, uint64_t seed, double* a, int64_t lda,
                             int* rank_out);
/* Rectangular low-rank-plus-noise inputs (BASELINE configs 2-5):
 * A = U diag(sigma) V' + noise N(0,1)/sqrt(n), U m x r on stream 0xFA000001, V n x r on
 * 0xFA000002, noise on 0xFA000003 keyed by column; sigma on the host. */
fqb_status fqb_gen_lowrank(fqb_handle h, int64_t m, int64_t n, int r, const double* sigma, uint64_t seed,
                           double noise, double* a, int64_t lda);
/* Deterministic low-rank inputs (BASELINE configs 3-4 at full size): rows [row0, row0 + rows)
 * of A = X diag(sigma) Y' + noise_scale G, X / Y the Q of CholeskyQR of Philox Gaussians
 * (streams 0xFA000001 / 0xFA000002, G on 0xFA000003, libm-free Box-Muller of
 * include/farqb/detmath.h), every product an fma chain in ascending k on the FP64 pipe.
 * Bit-identical to the host twin oracle/detgen.c (fqo_det_lowrank), so the CPU reference
 * can be run on the same matrix.  a: device, rows x n, lda >= rows; sigma on the host. */
fqb_status fqb_gen_lowrank_det(fqb_handle h, int64_t m, int64_t n, int r, const double* sigma, uint64_t seed,
                               double noise_scale, int64_t row0, int64_t rows, double* a, int64_t lda);
/* Order-independent 64-bit fingerprint of a device matrix's bits (row shard [row0, row0 +
 * rows) of an m_total-row matrix; shards sum mod 2^64 to the whole), = fqo_checksum. */
fqb_status fqb_checksum(fqb_handle h, const double* a, int64_t rows, int64_t cols, int64_t lda, int64_t row0,
                        int64_t m_total, uint64_t* out);

/* ---- defaults (driver.cpp:449-466) ------------------------------------------- */
double fqb_default_density(int kind, int64_t n);
int fqb_default_block(int64_t m, int64_t n);
int fqb_default_max_iters(int64_t n, int b);

#ifdef __cplusplus
}
#endif
#endif
