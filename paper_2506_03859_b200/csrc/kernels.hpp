// kernels.hpp -- host-side launchers for the farqb sm_100a kernels.
//
// Everything here enqueues device work on the given stream and returns
// immediately; nothing falls back to the host.  The engine (engine.cu) and the
// C-ABI building blocks (capi.cpp) are the only callers.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

#include "common.cuh"

namespace farqb {

enum SketchKindId { kGaussian = 0, kBernoulli = 1, kStdBernoulli = 2, kSparseSign = 3, kSparseGaussian = 4 };

// Device status word shared by generator kernels: bit 0 = a Gaussian draw hit
// an exact zero (the reference would redraw, rng.hpp:41-53); bit 1 = CSC
// capacity exceeded.
constexpr unsigned kGenZeroGaussian = 1u;
constexpr unsigned kGenOverflow = 2u;

// ---- sketch.cu ---------------------------------------------------------------
void launch_philox_u32(uint64_t seed, uint32_t block_id, uint32_t column, int count, uint32_t* out,
                       cudaStream_t s, LaunchCounter& lc);
// Dense N(0,1) block, column j from stream (seed, block_id, j); out is n x l (ld).
void launch_gaussian_dense(uint64_t seed, int block_id, int64_t n, int l, double* out, int64_t ld,
                           unsigned* status, cudaStream_t s, LaunchCounter& lc);
// i.i.d. density-p pattern (geometric gap walk, sketch.cpp:35-47, 75-95).
// count pass -> counts[l]; csc pass needs col_ptr; dense pass writes
// (value - shift) at nonzeros and -shift elsewhere into an n x l buffer.
void launch_iid_count(int kind, uint64_t seed, int block_id, int64_t n, int l, double denom,
                      int* counts, cudaStream_t s, LaunchCounter& lc);
void launch_iid_fill_csc(int kind, uint64_t seed, int block_id, int64_t n, int l, double denom,
                         double scale, const int* col_ptr, int* row_idx, double* values,
                         unsigned* status, cudaStream_t s, LaunchCounter& lc);
void launch_iid_fill_dense(int kind, uint64_t seed, int block_id, int64_t n, int l, double denom,
                           double scale, double shift, double* out, int64_t ld, unsigned* status,
                           cudaStream_t s, LaunchCounter& lc);
// Fixed zeta nonzeros per column (sparse sign / sparse Gaussian).
void launch_zeta_fill(int kind, uint64_t seed, int block_id, int64_t n, int l, int zeta,
                      double scale, int* col_ptr, int* row_idx, double* values, unsigned* status,
                      cudaStream_t s, LaunchCounter& lc);
// exclusive scan of counts[l] into col_ptr[l+1] (single CTA)
void launch_exclusive_scan(const int* counts, int l, int* col_ptr, cudaStream_t s, LaunchCounter& lc);
// out (n x l, ld) = dense(S) - shift
void launch_densify(const int* col_ptr, const int* row_idx, const double* values, int64_t n, int l,
                    double shift, double* out, int64_t ld, cudaStream_t s, LaunchCounter& lc);

// ---- spmm.cu -----------------------------------------------------------------
// C (m x l) = A (m x n) * S  [- z]   one fma per nonzero in CSC order.
void launch_gather_spmm(const double* a, int64_t m, int64_t lda, const int* col_ptr,
                        const int* row_idx, const double* values, int l, const double* z,
                        double* c, int64_t ldc, cudaStream_t s, LaunchCounter& lc);
void launch_gather_spmm(const float* a, int64_t m, int64_t lda, const int* col_ptr,
                        const int* row_idx, const double* values, int l, const double* z,
                        double* c, int64_t ldc, cudaStream_t s, LaunchCounter& lc);
// T (k x l) = Wt' * S [- shift * colsum(Wt) broadcast] where Wt is n x k (ld),
// i.e. the row-gather product used by the deflation B * Omega.
void launch_gather_tmul(const double* wt, int64_t n, int64_t ldw, int k, const int* col_ptr,
                        const int* row_idx, const double* values, int l, const double* colsum,
                        double shift, double* t, int64_t ldt, cudaStream_t s, LaunchCounter& lc);

// ---- reduce.cu ---------------------------------------------------------------
// Deterministic two-stage sums.  partial must hold kReducePartials doubles.
constexpr int kReducePartials = 1184;  // 8 x 148
void launch_sumsq(const double* a, int64_t m, int64_t n, int64_t lda, double* partial, double* out,
                  cudaStream_t s, LaunchCounter& lc);
void launch_sumsq(const float* a, int64_t m, int64_t n, int64_t lda, double* partial, double* out,
                  cudaStream_t s, LaunchCounter& lc);
// FP32 input mode: out (ldo) = double(a) when the A passes run on DMMA
void launch_widen(const float* a, int64_t m, int64_t n, int64_t lda, double* out, int64_t ldo, cudaStream_t s,
                  LaunchCounter& lc);
// z[i] = sum_c fma(p, A[i,c], z[i]) in column order (driver.cpp:178-183), bitwise
// the reference's axpy sequence.
void launch_centering(const double* a, int64_t m, int64_t n, int64_t lda, double p, double* z,
                      cudaStream_t s, LaunchCounter& lc);
void launch_centering(const float* a, int64_t m, int64_t n, int64_t lda, double p, double* z,
                      cudaStream_t s, LaunchCounter& lc);
// colsum[j] = sum_i X[i, j] for j < k (X is rows x k, ld)
void launch_colsum(const double* x, int64_t rows, int k, int64_t ld, double* colsum, cudaStream_t s,
                   LaunchCounter& lc);

// ---- gemm.cu -----------------------------------------------------------------
// C (m x n) = alpha op(A) B + beta C, column-major; DMMA (mma.sync f64) tensor
// pipe, deterministic split-K.  `work` must hold gemm_workspace_doubles(...).
// Split-K / stream-K scratch: `work` doubles of partials plus `flags` (num_sms
// unsigned, zero-initialised once) and a per-stream epoch for the stream-K fixup.
struct GemmWorkspace {
    double* work = nullptr;
    int64_t work_doubles = 0;
    unsigned* flags = nullptr;
    unsigned epoch = 0;
    bool use_tma = true;
    unsigned* counters = nullptr;  // split-K tile counters (zero between launches)
    int64_t counter_count = 0;
};
int64_t gemm_workspace_doubles(int64_t m, int64_t n, int64_t k, int num_sms);
void gemm(bool trans_a, int64_t m, int64_t n, int64_t k, double alpha, const double* a, int64_t lda,
          const double* b, int64_t ldb, double beta, double* c, int64_t ldc, GemmWorkspace& ws,
          int num_sms, cudaStream_t s, LaunchCounter& lc);
// gemm_tma.cu: TMA + mbarrier + stream-K variant (used by gemm() when the
// operands have even leading dimensions and 16-byte aligned bases)
int64_t gemm_tma_workspace_doubles(int num_sms);
bool gemm_tma_supported(bool trans_a, int64_t M, int64_t N, int64_t K, int64_t lda, int64_t ldb, const double* A,
                        const double* B, int num_sms);
// a3d_slack: the caller guarantees 16 readable doubles past the end of A
// (engine-owned buffers), so the NN 3-D box may overrun the last row block.
void gemm_tma(bool trans_a, int64_t M, int64_t N, int64_t K, double alpha, const double* A, int64_t lda,
              const double* B, int64_t ldb, double beta, double* C, int64_t ldc, double* work, unsigned* flags,
              unsigned epoch, int num_sms, cudaStream_t s, bool a3d_slack = false);

// ---- tsmm.cu: the b x b Grams of the CholeskyQR steps (b <= 128) ----------------
// S (b x b) = alpha Y'Y + beta S for Y (K x b): upper tiles only, mirrored, deterministic
// (per-CTA partials in work, ts_gram_workspace_doubles, summed in CTA order)
bool ts_enabled();   // FQB_TSMM=0: the general GEMMs instead
int64_t ts_gram_workspace_doubles(int b, int num_sms);
void ts_gram(const double* Y, int64_t K, int b, int64_t ldy, double alpha, double beta, double* S, int64_t lds,
             double* work, int64_t work_doubles, int num_sms, cudaStream_t s, LaunchCounter& lc);
// Z (M x b) = Y R, R upper triangular b x b (its strictly lower part is not read);
// false (nothing launched) when b > 104
bool ts_trmm(const double* Y, int64_t M, int b, int64_t ldy, const double* R, int64_t ldr, double* Z, int64_t ldz,
             int num_sms, cudaStream_t s, LaunchCounter& lc);

// ---- ozaki.cu: FP64 GEMM on the INT8 tensor cores ------------------------------
// Operands are int8 slices with one power-of-two exponent per operand row, stored
// pre-tiled and pre-swizzled (ozaki_x_bytes / ozaki_z_bytes).  C (M x N) =
// alpha X' Z + beta C with X the K x M operand, Z the K x N operand, N <= 64.
// nsl = slices per operand: 7 (FP64-class, 8-bit digits: 7 bytes of slices per element,
// 34 products; the default), 8 (FP64-class, 7-bit digits, 36 products; FQB_OZ_SLICES=8
// makes it the default) or 4 (FP32-class: 10 products; FP32 inputs on request).
int ozaki_fp64_slices();
int ozaki_slices();
int ozaki_max_n();
int ozaki_bn(int64_t n);
int64_t ozaki_x_bytes(int64_t rows, int64_t k, int nsl = ozaki_fp64_slices());
int64_t ozaki_z_bytes(int64_t n, int64_t k, int nsl = ozaki_fp64_slices());
int64_t ozaki_apply_z_bytes(int64_t k, int nsl = ozaki_fp64_slices());
// ozaki_apply's products again on the B slices its last call left in z / ez (N <= 128)
// Y (M x N) = alpha X C + beta Y for an X (M x K) held as its A'Y-layout slices xs_tn
// (column exponents xe, as made by ozaki_slice_a for the A'Y layout): C's rows scaled by
// 2^xe into cs (K x N scratch), sliced per column into z, and multiplied reading the
// slices MN-major (no slices of X in the A G layout are needed)
void ozaki_apply_mn(int64_t M, int64_t N, int64_t K, double alpha, const int8_t* xs_tn, const int* xe,
                    const double* c, int64_t ldc_in, double beta, double* Y, int64_t ldy, double* cs, int8_t* z,
                    int* ez, double* work, int num_sms, cudaStream_t s, LaunchCounter& lc, int nsl,
                    unsigned* zmax);
// while set (per thread), launch_ozaki brackets each k_ozaki (+ fixup) launch with a
// pair of events from this timer
void ozaki_set_timer(LaunchTimer* t);
void ozaki_apply_presliced(int64_t M, int64_t N, int64_t K, double alpha, const int8_t* xs, const int* ex, double beta,
                           double* C, int64_t ldc, const int8_t* z, const int* ez, double* work, int num_sms,
                           cudaStream_t s, LaunchCounter& lc, int nsl = ozaki_fp64_slices());
int ozaki_apply_ez_count();
int64_t ozaki_workspace_doubles(int num_sms);
// Slices of A (m x n, ld) in both layouts from one pass (either may be null):
//   x_tn / e_tn: operand rows = columns of A, K = m   (A' Y)
//   x_nn / e_nn: operand rows = rows of A,    K = n   (A G)
// line_max: ozaki_line_max_words(m, n) words of scratch, zero-filled once when allocated
// (DeviceArray::ensure_zeroed): the maxima are tagged with a per-call generation, so no
// memset is needed between calls.  With norm_out, ||A||_F^2
// comes out of the same read of A (norm_partial: ozaki_norm_partials(m, n) doubles).
int64_t ozaki_line_max_words(int64_t m, int64_t n);
int64_t ozaki_norm_partials(int64_t m, int64_t n);
void ozaki_slice_a(const double* a, int64_t m, int64_t n, int64_t ld, unsigned* line_max, int8_t* x_tn, int* e_tn,
                   int8_t* x_nn, int* e_nn, cudaStream_t s, LaunchCounter& lc, double* norm_partial = nullptr,
                   double* norm_out = nullptr, int nsl = ozaki_fp64_slices());
void ozaki_slice_a(const float* a, int64_t m, int64_t n, int64_t ld, unsigned* line_max, int8_t* x_tn, int* e_tn,
                   int8_t* x_nn, int* e_nn, cudaStream_t s, LaunchCounter& lc, double* norm_partial = nullptr,
                   double* norm_out = nullptr, int nsl = ozaki_fp64_slices());
// Z (k x n, ld)
void ozaki_slice_z(const double* b, int64_t k, int64_t n, int64_t ld, int* e, int8_t* out, cudaStream_t s,
                   LaunchCounter& lc, int nsl = ozaki_fp64_slices());
// C = alpha X' B + beta C for any N: B (K x N, ld, FP64) sliced in chunks of <= 64
// columns into z (ozaki_apply_z_bytes(K)) / ez (ozaki_apply_ez_count()); N > 64
// runs two chunks at a time on CTA pairs sharing the A tiles (FQB_OZ_PAIR=0: off)
// zmax: ozaki_apply_ez_count() words of scratch, zero-filled once when allocated (as
// line_max); lets a long B (K > 16384 rows) take its column maxima in one pass before
// slicing (null: the one-kernel slicer)
void ozaki_apply(int64_t M, int64_t N, int64_t K, double alpha, const int8_t* xs, const int* ex, const double* b,
                 int64_t ldb, double beta, double* C, int64_t ldc, int8_t* z, int* ez, double* work, int num_sms,
                 cudaStream_t s, LaunchCounter& lc, int nsl = ozaki_fp64_slices(), unsigned* zmax = nullptr);
void ozaki_gemm(int64_t M, int64_t N, int64_t K, double alpha, const int8_t* xs, const int* ex, const int8_t* zs,
                const int* ez, double beta, double* C, int64_t ldc, double* work, int num_sms, cudaStream_t s,
                LaunchCounter& lc, int nsl = ozaki_fp64_slices());

// ---- smallla.cu --------------------------------------------------------------
// Cholesky of the b x b SPD matrix S (ld = lds) with the reference pivot rule
// (matrix_core.cpp:117-140): pivot <= tol * max(diag_ref, max diag(S)) fails.
// Writes R = L' (upper) and R^{-1}, both b x b with ld = b; on failure sets
// *status |= fail_bit and writes identities.
// max_diag_out (optional) receives the pivot reference actually used; scratch
// (b x (b+1) doubles) is only touched when b > 128.
void launch_chol_upper_inv(const double* S, int b, int64_t lds, double tol, double diag_ref,
                           const double* dref_extra, int64_t ld_extra, double* R, double* Rinv,
                           double* max_diag_out, double* scratch, unsigned* status, unsigned fail_bit,
                           cudaStream_t s, LaunchCounter& lc);
// eigenvalues (ascending) of a b x b symmetric matrix (cyclic Jacobi,
// matrix_core.cpp:50-115) and optionally eigenvectors (ld = b).
// vtmp: b x b doubles of scratch when vectors are wanted.
// eigsmall.cu: symmetric eigensolver for the SVD assembly's l x l matrix, l <= kSmallEighMax.
// mat: full symmetric n x n (col-major, ld n, left intact); eigenvalues ascending into w,
// eigenvectors into x (n x n, ld n).  false when its a-posteriori residual /
// orthogonality check fails -- the caller then uses cuSOLVER.  Synchronizes s.
constexpr int kSmallEighMax = 224;
int64_t small_eigh_scratch_doubles(int n);
bool small_eigh(const double* mat, int n, double* w, double* x, double* scratch, GemmWorkspace& gws, int num_sms,
                cudaStream_t s, LaunchCounter& lc);
void launch_sym_eig(const double* S, int b, int64_t lds, double* values, double* vectors,
                    double* vtmp, unsigned* status, unsigned fail_bit, cudaStream_t s,
                    LaunchCounter& lc);
// alpha <- (shat + alpha)/2 if alpha < shat (driver.cpp:216-221), on the device
void launch_shift_update(const double* values, int b, int conv, double* alpha, cudaStream_t s,
                         LaunchCounter& lc);
// y[:, c] -= (*alpha) * x[:, c]
void launch_axpy_cols_dev(const double* alpha, const double* x, int64_t ldx, double* y, int64_t ldy,
                          int64_t rows, int cols, cudaStream_t s, LaunchCounter& lc);
// eigSVD tail (matrix_core.cpp:193-215): from ascending eigenvalues/vectors of
// W'W build V Sigma^{-1} (b x b) and sigma; sets fail_bit if lmax <= 0.
void launch_eigsvd_scale(const double* values, const double* vectors, int b, double* vs,
                         double* sigma, unsigned* status, unsigned fail_bit, cudaStream_t s,
                         LaunchCounter& lc);
// out[0] = sum of squares of a column-major x (rows x cols, ld) (two-stage)
void launch_sumsq_small(const double* x, int64_t rows, int64_t cols, int64_t ld, double* partial,
                        double* out, cudaStream_t s, LaunchCounter& lc);
// y[:, c] -= alpha * x[:, c] (rows x cols)
void launch_axpy_cols(double alpha, const double* x, int64_t ldx, double* y, int64_t ldy,
                      int64_t rows, int cols, cudaStream_t s, LaunchCounter& lc);

}  // namespace farqb
