// engine.cu -- the farPCA blocked adaptive QB loop, device resident.
//
// Host-side orchestration of the reference's run_fixed_precision /
// run_fixed_rank (/root/reference/proj/src/driver.cpp:134-160, 185-294,
// 347-413).  All matrix work runs in the sm_100a kernels of this directory on
// one CUDA stream; the host only makes the per-block decisions (converged?
// degenerate -> redraw?) from a handful of scalars read back once per block.
//
// Numerical recipe (explicit Q instead of the reference's Gram-space Y/W/Z/L):
//   sketch     Y_j = A * Omega_j           (gather SpMM or DMMA GEMM)
//   power      W = A' Y - B'(B Omega) [- alpha G],  G = orth(W)   (P passes)
//   accept     Y_j = A G;  W_j = A' Y_j
//              [C1; D] = [Q | Y_j]' Y_j            one TN GEMM
//              Y' = Y_j - Q C1;  R1 = chol(Y''Y')  pivot rule of driver.cpp:265-279
//              Q1 = Y' R1^-1;   C2 = Q' Q1;  Q2 = Q1 - Q C2;  R2 = chol(Q2'Q2)
//              Q_j = Q2 R2^-1,  R = R2 R1,  C = C1 + C2 R1       (CholeskyQR2 + BGS2)
//              B_j' = (W_j - B' C) R^-1                          (no extra pass over A)
//              E  -= ||B_j||_F^2                                 (driver.cpp:280-286)
// Y_j = Q C + Q_j R and W_j = A'Y_j give the B_j identity; the reference's
// r = (w_j - W Z^-1 Y'y_j) L22^-T is the same quantity in Gram form.
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "engine.hpp"
#include "kernels.hpp"

namespace farqb {

namespace {

constexpr unsigned kStAcceptPivot = 1u << 4;
constexpr unsigned kStAcceptChol2 = 1u << 5;
constexpr unsigned kStPowerChol = 1u << 6;
constexpr unsigned kStPowerDegenerate = 1u << 7;
constexpr unsigned kStEigConv = 1u << 8;
constexpr double kDenseThreshold = 1.0 / 32.0;  // density above which Omega is densified

enum ScalarSlot { kNormA = 0, kBNorm = 1, kDMax = 2, kAlpha = 3, kScalarCount = 8 };

}  // namespace

bool pdl_enabled() {
    static const bool on = [] {
        const char* e = std::getenv("FQB_PDL");
        return !(e && e[0] == '0');
    }();
    return on;
}

void ensure_gemm_workspace(Handle& h) {
    const int64_t need = std::max<int64_t>(int64_t(h.num_sms) * 256 * 128 + 16, gemm_tma_workspace_doubles(h.num_sms));
    if (h.ws.splitk.count < size_t(need)) {
        h.ws.splitk.ensure(size_t(need), h.stream);
        h.gws.work = h.ws.splitk.ptr;
        h.gws.work_doubles = need;
    }
    if (!h.ws.gemm_flags.ptr) {
        // [0, num_sms): stream-K partial flags; then 4*num_sms split-K tile counters
        const size_t count = size_t(h.num_sms) * 5 + 16;
        h.ws.gemm_flags.ensure(count, h.stream);
        FQB_CUDA(cudaMemsetAsync(h.ws.gemm_flags.ptr, 0, sizeof(unsigned) * count, h.stream));
        h.gws.flags = h.ws.gemm_flags.ptr;
        h.gws.epoch = 0;
        h.gws.counters = h.ws.gemm_flags.ptr + h.num_sms + 16;
        h.gws.counter_count = int64_t(h.num_sms) * 4;
    }
    const char* env = std::getenv("FQB_GEMM_TMA");
    h.gws.use_tma = !(env && env[0] == '0');
}

double default_density(int kind, int64_t n) {
    if (kind == kGaussian) return 0.0;
    const double nn = double(n);
    return std::max(1e-3, kind == kStdBernoulli ? std::log(nn) / nn : 10.0 / nn);
}

int default_block(int64_t m, int64_t n) {
    const int64_t mn = std::min(m, n);
    return int(std::min<int64_t>(std::min<int64_t>(std::max<int64_t>(20, mn / 100), 50), mn));
}

int default_max_iters(int64_t n, int b) { return int((n + 2 * int64_t(b) - 1) / (2 * int64_t(b))); }

fqb_config resolve_config(int64_t m, int64_t n, const fqb_config& in, bool fixed_precision) {
    if (m < 1 || n < 1) throw Error(kStatusConfig, "matrix must be non-empty");
    if (m > INT32_MAX || n > INT32_MAX) throw Error(kStatusDimension, "dimensions exceed 2^31-1");
    fqb_config cfg = in;
    if (cfg.sketch.kind < kGaussian || cfg.sketch.kind > kSparseGaussian)
        throw Error(kStatusConfig, "unknown sketch kind");
    if (cfg.block == 0) cfg.block = default_block(m, n);
    if (cfg.block < 1) throw Error(kStatusConfig, "block size must be at least 1");
    if (cfg.block > std::min(m, n)) throw Error(kStatusConfig, "block size exceeds matrix dimensions");
    if (cfg.block > 1024) throw Error(kStatusConfig, "block size above 1024 is not supported");
    if (cfg.max_iters == 0) cfg.max_iters = default_max_iters(n, cfg.block);
    if (cfg.max_iters < 1) throw Error(kStatusConfig, "max_iters must be at least 1");
    if (cfg.power < 0) throw Error(kStatusConfig, "power must be non-negative");
    if (cfg.power >= 3 && cfg.block > 128)
        throw Error(kStatusConfig, "shifted power iteration (power >= 3) supports block size <= 128");
    if (cfg.sketch.zeta < 0) throw Error(kStatusConfig, "zeta must be non-negative");
    if (cfg.sketch.zeta > 0) {
        if (cfg.sketch.kind != kSparseSign && cfg.sketch.kind != kSparseGaussian)
            throw Error(kStatusConfig, "zeta applies to the sparse sign / sparse Gaussian kinds only");
        if (cfg.sketch.zeta > n || cfg.sketch.zeta > 256)
            throw Error(kStatusConfig, "zeta must not exceed min(n, 256)");
        if (cfg.sketch.p == 0.0) cfg.sketch.p = double(cfg.sketch.zeta) / double(n);
    } else if (cfg.sketch.kind != kGaussian && cfg.sketch.p == 0.0) {
        cfg.sketch.p = default_density(cfg.sketch.kind, n);
    }
    if (fixed_precision && !(cfg.eps > 0.0))
        throw Error(kStatusConfig, "fixed-precision mode needs a positive tolerance");
    cfg.shift_convention = cfg.shift_convention ? 1 : 0;
    return cfg;
}

namespace {

class QbRun {
  public:
    // exactly one of a (FP64) / af (FP32 input mode) is non-null
    QbRun(Handle& h, const double* a, const float* af, int64_t m, int64_t n, int64_t lda, const fqb_config& cfg,
          fqb_block_source_fn src, void* user)
        : h_(h), s_(h.stream), a_(a), af_(af), m_(m), n_(n), lda_(lda), cfg_(cfg), b_(cfg.block), src_(src),
          user_(user) {
        ldq_ = round_up(m_, 8);
        ldbt_ = round_up(n_, 8);
        ldo_ = round_up(n_, 8);
        Workspace& w = h_.ws;
        const int64_t b = b_;
        w.omega.ensure(size_t(ldo_) * b, s_);
        w.y0.ensure(size_t(ldq_) * b, s_);
        w.ys.ensure(size_t(ldq_) * b, s_);
        w.wp.ensure(size_t(ldbt_) * b, s_);
        w.wraw.ensure(size_t(ldbt_) * b, s_);
        w.g.ensure(size_t(ldbt_) * b, s_);
        w.small.ensure(size_t(12) * b * b + 4 * b, s_);
        w.scalars.ensure(kScalarCount, s_);
        w.partial.ensure(kReducePartials, s_);
        w.status.ensure(4, s_);
        w.scratch.ensure(size_t(b) * (b + 1), s_);
        w.col_ptr.ensure(size_t(b) + 1, s_);
        w.counts.ensure(size_t(b), s_);
        ensure_gemm_workspace(h_);
        oz_on_ = ozaki_default(m_, n_, b_);
        // FP32 input may opt into FP32-class A passes (4 slices: half the bytes)
        oz_nsl_ = (af_ && h_.fp32_slices < 7) ? h_.fp32_slices : ozaki_fp64_slices();
        double* sm = w.small.ptr;
        S_ = sm;
        S2_ = sm + 1 * b * b;
        R1_ = sm + 2 * b * b;
        R1i_ = sm + 3 * b * b;
        R2_ = sm + 4 * b * b;
        R2i_ = sm + 5 * b * b;
        R_ = sm + 6 * b * b;
        Ri_ = sm + 7 * b * b;
        V_ = sm + 8 * b * b;
        VS_ = sm + 9 * b * b;
        VT_ = sm + 10 * b * b;
        eig_ = sm + 12 * b * b;
        sig_ = eig_ + b;
        scal_ = w.scalars.ptr;
        status_ = w.status.ptr;
    }

    // --- setup: ||A||^2 and (StdBernoulli) the centering column -----------------
    void setup() {
        FQB_CUDA(cudaMemsetAsync(scal_, 0, kScalarCount * sizeof(double), s_));
        // With the emulation on, A is sliced now and ||A||^2 comes out of the
        // slicing's line-max pass (one read of A fewer)
        bool norm_done = false;
        if (oz_on_) {
            oz_ready_ = true;
            norm_done = prepare_ozaki(scal_ + kNormA);
            if (!norm_done) oz_on_ = false;
        }
        if (!norm_done) {
            if (af_) launch_sumsq(af_, m_, n_, lda_, h_.ws.partial.ptr, scal_ + kNormA, s_, h_.lc);
            else launch_sumsq(a_, m_, n_, lda_, h_.ws.partial.ptr, scal_ + kNormA, s_, h_.lc);
        }
        comm_allreduce_sum(h_, scal_ + kNormA, 1, s_);
        // z = A (p 1_n) exists when the reference would build it (driver.cpp:364-365);
        // it is only computed once a sparse centered block actually needs it.
        z_allowed_ = cfg_.sketch.kind == kStdBernoulli;
        FQB_CUDA(cudaMemcpyAsync(h_.host_scalars, scal_ + kNormA, sizeof(double), cudaMemcpyDeviceToHost, s_));
        FQB_CUDA(cudaStreamSynchronize(s_));
        norm_a_sq_ = h_.host_scalars[0];
        // non-finite A: DMMA, whose Inf/NaN propagation is the reference's
        if (oz_on_ && !std::isfinite(norm_a_sq_)) oz_on_ = false;
        // Q'X products on the INT8 path when the A passes are there and the rows are many
        q_oz_on_ = oz_on_ && q_oz_default() && m_ >= 4096;
        // B G and B' T likewise (K = n, resp. the l columns of B')
        b_oz_on_ = oz_on_ && b_oz_default() && n_ >= 4096;
    }

    double norm_a_sq() const { return norm_a_sq_; }
    double residual() const { return norm_a_sq_ - trace_; }
    int blocks() const { return blocks_; }
    int rank() const { return int(l_); }
    std::vector<double>& residuals() { return residuals_; }
    std::vector<int>& ids() { return ids_; }

    void reserve_blocks(int nblocks) { grow(int64_t(nblocks) * b_); }

    // Host Q, B' (FQB_OUT_HOST): each committed block's columns leave on the handle's
    // copy stream while the next block runs, so only U, V are copied after the loop.
    // Host capacity: the device's, or the rank the handle's last run of this shape
    // reached; outgrowing it copies the committed columns again from the device.
    void stream_out_host() { stream_out_ = true; }
    bool streamed() const { return hq_ != nullptr; }
    // the host arrays (ld m, n), every committed column queued on the copy stream
    void take_host(double** q, double** bt) {
        *q = hq_;
        *bt = hbt_;
        hq_ = hbt_ = nullptr;
    }
    ~QbRun() {
        // queued copies read q_ / bt_, which are released on s_ below
        if (hcopied_ > 0) cudaStreamSynchronize(h_.copy_stream);
        host_free(hq_);
        host_free(hbt_);
    }

    // process_block (driver.cpp:134-160): up to 3 redraws with id + 1000 r
    void process_block(int index) {
        for (int attempt = 0;; ++attempt) {
            const int id = index + 1000 * attempt;
            ids_.push_back(id);
            const unsigned st = try_block(id);
            if (st == 0) return;
            if (attempt >= 3)
                throw DegenerateError(std::string("block degenerate after 3 redraws (status ") +
                                      std::to_string(st) + ")");
        }
    }

    struct DegenerateError : Error {
        explicit DegenerateError(const std::string& m) : Error(kStatusDegenerate, m) {}
    };

    // Final outputs
    DeviceArray<double>& q() { return q_; }
    DeviceArray<double>& bt() { return bt_; }
    bool ozaki() const { return oz_on_; }
    int64_t ldq() const { return ldq_; }
    int64_t ldbt() const { return ldbt_; }

  private:
    // ---- buffers ------------------------------------------------------------
    void grow(int64_t need_cols) {
        if (need_cols <= cap_) return;
        int64_t nc = std::max<int64_t>(need_cols, cap_ ? 2 * cap_ : int64_t(b_) * 4);
        nc = std::min<int64_t>(std::max(nc, need_cols), std::max<int64_t>(need_cols, int64_t(cfg_.max_iters) * b_));
        if (hcopied_ > 0) {   // host copies of the old Q / B' may still be in flight
            FQB_CUDA(cudaEventRecord(h_.ev_copied, h_.copy_stream));
            FQB_CUDA(cudaStreamWaitEvent(s_, h_.ev_copied, 0));
        }
        auto regrow = [&](DeviceArray<double>& arr, int64_t ld) {
            DeviceArray<double> fresh;
            fresh.ensure(size_t(ld) * nc, s_);
            if (l_ > 0) FQB_CUDA(cudaMemcpyAsync(fresh.ptr, arr.ptr, size_t(ld) * l_ * sizeof(double),
                                                 cudaMemcpyDeviceToDevice, s_));
            arr.release();
            arr.ptr = fresh.detach();
            arr.count = size_t(ld) * nc;
            arr.stream = s_;
        };
        regrow(q_, ldq_);
        regrow(bt_, ldbt_);
        if (z_allowed_) regrow(rowsum_, 1);
        // the slices of the committed Q (B') columns move with Q (B')
        auto regrow_slices = [&](DeviceArray<int8_t>& xs, DeviceArray<int>& xe, int64_t sliced, int64_t k) {
            const int nsl = ozaki_fp64_slices();
            DeviceArray<int8_t> fresh;
            fresh.ensure(size_t(ozaki_x_bytes(nc, k, nsl)), s_);
            if (sliced > 0)
                FQB_CUDA(cudaMemcpyAsync(fresh.ptr, xs.ptr, size_t(ozaki_x_bytes(sliced, k, nsl)),
                                         cudaMemcpyDeviceToDevice, s_));
            xs.release();
            xs.ptr = fresh.detach();
            xs.count = size_t(ozaki_x_bytes(nc, k, nsl));
            xs.stream = s_;
            DeviceArray<int> fe;
            fe.ensure(size_t(nc), s_);
            if (sliced > 0)
                FQB_CUDA(cudaMemcpyAsync(fe.ptr, xe.ptr, sizeof(int) * size_t(sliced), cudaMemcpyDeviceToDevice, s_));
            xe.release();
            xe.ptr = fe.detach();
            xe.count = size_t(nc);
            xe.stream = s_;
        };
        if (q_oz_on_) regrow_slices(h_.ws.oz_q_tn, h_.ws.oz_q_e, q_sliced_, m_);
        if (b_oz_on_) regrow_slices(h_.ws.oz_b_tn, h_.ws.oz_b_e, b_sliced_, n_);
        cap_ = nc;
        Workspace& w = h_.ws;
        w.t.ensure(size_t(nc) * b_, s_);
        w.cd.ensure(size_t(nc + b_) * b_, s_);
        w.c2.ensure(size_t(nc) * b_, s_);
    }

    void push_host() {
        if (l_ > hcap_) {
            // the first run of a shape on this handle copies after the loop (its final
            // size is unknown; growing host blocks would leave odd sizes in the pool)
            const bool hinted = h_.out_hint_m == m_ && h_.out_hint_n == n_ && h_.out_hint_l > 0;
            if (!hinted) {
                stream_out_ = false;
                return;
            }
            const int64_t want = hcap_ == 0 ? std::max(l_, h_.out_hint_l) : std::max(cap_, l_);
            if (hcopied_ > 0) FQB_CUDA(cudaStreamSynchronize(h_.copy_stream));
            host_release(hq_);   // outgrown: unpinned, not cached
            host_release(hbt_);
            hq_ = static_cast<double*>(host_alloc(sizeof(double) * size_t(m_) * size_t(want)));
            hbt_ = static_cast<double*>(host_alloc(sizeof(double) * size_t(n_) * size_t(want)));
            if (!hq_ || !hbt_) throw Error(kStatusAlloc, "host result allocation failed");
            hcap_ = want;
            hcopied_ = 0;
        }
        if (!h_.copy_stream) FQB_CUDA(cudaStreamCreateWithFlags(&h_.copy_stream, cudaStreamNonBlocking));
        if (!h_.ev_qb) FQB_CUDA(cudaEventCreateWithFlags(&h_.ev_qb, cudaEventDisableTiming));
        if (!h_.ev_copied) FQB_CUDA(cudaEventCreateWithFlags(&h_.ev_copied, cudaEventDisableTiming));
        FQB_CUDA(cudaEventRecord(h_.ev_qb, s_));
        FQB_CUDA(cudaStreamWaitEvent(h_.copy_stream, h_.ev_qb, 0));
        const int64_t c0 = hcopied_, nc = l_ - hcopied_;
        FQB_CUDA(cudaMemcpy2DAsync(hq_ + c0 * m_, m_ * sizeof(double), q_.ptr + c0 * ldq_, ldq_ * sizeof(double),
                                   m_ * sizeof(double), nc, cudaMemcpyDeviceToHost, h_.copy_stream));
        FQB_CUDA(cudaMemcpy2DAsync(hbt_ + c0 * n_, n_ * sizeof(double), bt_.ptr + c0 * ldbt_,
                                   ldbt_ * sizeof(double), n_ * sizeof(double), nc, cudaMemcpyDeviceToHost,
                                   h_.copy_stream));
        hcopied_ = l_;
    }

    void gemm_(bool ta, int64_t M, int64_t N, int64_t K, double alpha, const double* A, int64_t lda,
               const double* B, int64_t ldb, double beta, double* C, int64_t ldc) {
        gemm(ta, M, N, K, alpha, A, lda, B, ldb, beta, C, ldc, h_.gws, h_.num_sms, s_, h_.lc);
    }
    // S (b x b) = Y'Y for a tall Y (K x b): the symmetric tall-skinny kernel (tsmm.cu)
    void gram_(const double* Y, int64_t K, int64_t ldy, double* S) {
        if (ts_enabled() && b_ <= 128 &&
            h_.gws.work_doubles >= ts_gram_workspace_doubles(b_, std::min<int>(h_.num_sms, 8))) {
            ts_gram(Y, K, b_, ldy, 1.0, 0.0, S, b_, h_.gws.work, h_.gws.work_doubles, h_.num_sms, s_, h_.lc);
            return;
        }
        gemm_(true, b_, b_, K, 1.0, Y, ldy, Y, ldy, 0.0, S, b_);
    }
    // Z (M x b) = Y R for an upper-triangular b x b R (the R^-1 factors; tsmm.cu)
    void trmm_(const double* Y, int64_t M, int64_t ldy, const double* R, double* Z, int64_t ldz) {
        if (ts_enabled() && ts_trmm(Y, M, b_, ldy, R, b_, Z, ldz, h_.num_sms, s_, h_.lc)) return;
        gemm_(false, M, b_, b_, 1.0, Y, ldy, R, b_, 0.0, Z, ldz);
    }

    // ---- A-pass products ------------------------------------------------------
    // C = A' B (ta) or A B with B of N <= b columns: the passes over A that dominate
    // the run.  With the Ozaki path on, A is sliced once per run per layout into
    // int8 (ozaki.cu) and every pass runs on the tcgen05 INT8 tensor cores; otherwise
    // the FP64 DMMA GEMM.
    static bool ozaki_default(int64_t m, int64_t n, int b) {
        const char* e = std::getenv("FQB_OZAKI");
        if (e && e[0] == '0') return false;
        // b > 64 runs in column chunks of <= 64, each one more pass over the slices:
        // still 1.5-3x ahead of DMMA for b in (64, 128]
        return (e && e[0] == '1') || (double(m) * double(n) >= double(1 << 24) && b >= 16);   // small: DMMA is fine
    }

    // Slice A once per run into the handle's buffers; false (and DMMA from then on)
    // when the two slice layouts do not fit in device memory.
    bool prepare_ozaki(double* norm_out = nullptr) {
        Workspace& w = h_.ws;
        try {
            w.oz_x_nn.ensure(size_t(ozaki_x_bytes(m_, n_, oz_nsl_)), s_);
            w.oz_x_tn.ensure(size_t(ozaki_x_bytes(n_, m_, oz_nsl_)), s_);
        } catch (const Error&) {
            cudaGetLastError();   // clear the allocation failure
            w.oz_x_nn.release();
            w.oz_x_tn.release();
            return false;
        }
        w.oz_e_nn.ensure(size_t(m_), s_);
        w.oz_e_tn.ensure(size_t(n_), s_);
        w.oz_line_max.ensure_zeroed(size_t(ozaki_line_max_words(m_, n_)), s_);
        if (norm_out) w.oz_norm_partial.ensure(size_t(std::max<int64_t>(1, ozaki_norm_partials(m_, n_))), s_);
        double* np = norm_out ? w.oz_norm_partial.ptr : nullptr;
        if (af_)
            ozaki_slice_a(af_, m_, n_, lda_, w.oz_line_max.ptr, w.oz_x_tn.ptr, w.oz_e_tn.ptr, w.oz_x_nn.ptr,
                          w.oz_e_nn.ptr, s_, h_.lc, np, norm_out, oz_nsl_);
        else
            ozaki_slice_a(a_, m_, n_, lda_, w.oz_line_max.ptr, w.oz_x_tn.ptr, w.oz_e_tn.ptr, w.oz_x_nn.ptr,
                          w.oz_e_nn.ptr, s_, h_.lc, np, norm_out, oz_nsl_);
        return true;
    }

    // FP32 input on the DMMA path: one widened FP64 copy of A for the run
    void ensure_fp64_a() {
        if (a_) return;
        const int64_t ld = round_up(m_, 8);
        h_.ws.a_copy.ensure(size_t(ld) * size_t(n_), s_);
        launch_widen(af_, m_, n_, lda_, h_.ws.a_copy.ptr, ld, s_, h_.lc);
        a_ = h_.ws.a_copy.ptr;
        a_ld64_ = ld;
    }

    // the A passes' k_ozaki launches are bracketed by the handle's pass timer when armed
    struct PassTimerScope {
        explicit PassTimerScope(Handle& h) { ozaki_set_timer(h.pass_timer.on ? &h.pass_timer : nullptr); }
        ~PassTimerScope() { ozaki_set_timer(nullptr); }
    };

    void a_gemm(bool ta, int N, const double* B, int64_t ldb, double* C, int64_t ldc) {
        if (!oz_on_) {
            ensure_fp64_a();
            const int64_t lda = a_ld64_ ? a_ld64_ : lda_;
            if (ta) gemm_(true, n_, N, m_, 1.0, a_, lda, B, ldb, 0.0, C, ldc);
            else gemm_(false, m_, N, n_, 1.0, a_, lda, B, ldb, 0.0, C, ldc);
            return;
        }
        const int64_t M = ta ? n_ : m_, K = ta ? m_ : n_;
        if (!oz_ready_) {
            oz_ready_ = true;
            if (!prepare_ozaki()) {
                oz_on_ = false;
                a_gemm(ta, N, B, ldb, C, ldc);
                return;
            }
        }
        Workspace& w = h_.ws;
        w.oz_z.ensure(size_t(ozaki_apply_z_bytes(K, oz_nsl_)), s_);
        w.oz_ez.ensure(size_t(ozaki_apply_ez_count()), s_);
        w.oz_zmax.ensure_zeroed(size_t(ozaki_apply_ez_count()), s_);
        PassTimerScope timed(h_);
        ozaki_apply(M, N, K, 1.0, ta ? w.oz_x_tn.ptr : w.oz_x_nn.ptr, ta ? w.oz_e_tn.ptr : w.oz_e_nn.ptr, B, ldb, 0.0,
                    C, ldc, w.oz_z.ptr, w.oz_ez.ptr, h_.gws.work, h_.num_sms, s_, h_.lc, oz_nsl_, w.oz_zmax.ptr);
    }

    // W (n x N) = sum over ranks of A_g' B (the A'Y passes).  With a NCCL communicator
    // the product runs in two halves of W's rows (A's columns, split on a 128 multiple):
    // the all-reduce of the first half, on a second stream, overlaps the second half's
    // product (16 MB per pass at config 4).  Otherwise product, then sum.
    void a_tn_reduced(int N, const double* B, int64_t ldb, double* C, int64_t ldc) {
        const int64_t n1 = (n_ / 2 / 128) * 128;
        if (!h_.comm || n1 == 0) {
            a_gemm(true, N, B, ldb, C, ldc);
            comm_allreduce_sum(h_, C, size_t(ldc) * N, s_);
            return;
        }
        if (!h_.comm_stream) {
            FQB_CUDA(cudaStreamCreateWithFlags(&h_.comm_stream, cudaStreamNonBlocking));
            FQB_CUDA(cudaEventCreateWithFlags(&h_.ev_half, cudaEventDisableTiming));
            FQB_CUDA(cudaEventCreateWithFlags(&h_.ev_reduced, cudaEventDisableTiming));
        }
        // the halves are C rows [0, n1) and [n1, n) of every column: each is packed into a
        // contiguous buffer for one all-reduce and unpacked after it
        double* buf = h_.ws.w_half.ensure(size_t(n_) * N, s_);
        auto reduce_rows = [&](int64_t r0, int64_t rows, cudaStream_t st) {
            double* pk = buf + r0 * N;
            FQB_CUDA(cudaMemcpy2DAsync(pk, rows * sizeof(double), C + r0, ldc * sizeof(double), rows * sizeof(double),
                                       N, cudaMemcpyDeviceToDevice, st));
            comm_allreduce_sum(h_, pk, size_t(rows) * N, st);
            FQB_CUDA(cudaMemcpy2DAsync(C + r0, ldc * sizeof(double), pk, rows * sizeof(double), rows * sizeof(double),
                                       N, cudaMemcpyDeviceToDevice, st));
        };
        a_gemm_rows(0, n1, N, B, ldb, C, ldc, false);
        FQB_CUDA(cudaEventRecord(h_.ev_half, s_));
        FQB_CUDA(cudaStreamWaitEvent(h_.comm_stream, h_.ev_half, 0));
        reduce_rows(0, n1, h_.comm_stream);
        a_gemm_rows(n1, n_ - n1, N, B, ldb, C, ldc, true);
        FQB_CUDA(cudaEventRecord(h_.ev_half, s_));
        FQB_CUDA(cudaStreamWaitEvent(h_.comm_stream, h_.ev_half, 0));
        reduce_rows(n1, n_ - n1, h_.comm_stream);   // same communicator: issued in order on one stream
        FQB_CUDA(cudaEventRecord(h_.ev_reduced, h_.comm_stream));
        FQB_CUDA(cudaStreamWaitEvent(s_, h_.ev_reduced, 0));
    }
    // rows [r0, r0 + rows) of A' B (A's columns r0..): the Ozaki TN slices start at a
    // 128-row tile boundary; `again` reuses the B slices the first half made
    void a_gemm_rows(int64_t r0, int64_t rows, int N, const double* B, int64_t ldb, double* C, int64_t ldc,
                     bool again) {
        if (!oz_on_) {
            ensure_fp64_a();
            const int64_t lda = a_ld64_ ? a_ld64_ : lda_;
            gemm_(true, rows, N, m_, 1.0, a_ + r0 * lda, lda, B, ldb, 0.0, C + r0, ldc);
            return;
        }
        if (!oz_ready_) {
            oz_ready_ = true;
            if (!prepare_ozaki()) {
                oz_on_ = false;
                a_gemm_rows(r0, rows, N, B, ldb, C, ldc, false);
                return;
            }
        }
        Workspace& w = h_.ws;
        const int8_t* xs = w.oz_x_tn.ptr + (r0 / 128) * ozaki_x_bytes(128, m_, oz_nsl_);
        PassTimerScope timed(h_);
        if (again && N <= 128) {
            ozaki_apply_presliced(rows, N, m_, 1.0, xs, w.oz_e_tn.ptr + r0, 0.0, C + r0, ldc, w.oz_z.ptr, w.oz_ez.ptr,
                                  h_.gws.work, h_.num_sms, s_, h_.lc, oz_nsl_);
            return;
        }
        w.oz_z.ensure(size_t(ozaki_apply_z_bytes(m_, oz_nsl_)), s_);
        w.oz_ez.ensure(size_t(ozaki_apply_ez_count()), s_);
        w.oz_zmax.ensure_zeroed(size_t(ozaki_apply_ez_count()), s_);
        ozaki_apply(rows, N, m_, 1.0, xs, w.oz_e_tn.ptr + r0, B, ldb, 0.0, C + r0, ldc, w.oz_z.ptr, w.oz_ez.ptr,
                    h_.gws.work, h_.num_sms, s_, h_.lc, oz_nsl_, w.oz_zmax.ptr);
    }

    // ---- the block Gram-Schmidt products Q' X on the INT8 tensor cores --------
    // Q's columns are final once committed, so their slices (A'Y layout: one operand row
    // per column of Q, K = m, a power-of-two scale per column) are made once: each block
    // slices from the 128-column tile holding column l through l + b (Y_j / Q_j in place)
    // and [Q|Y]'Y, Q'Y_s become one k_ozaki pass each instead of a DMMA GEMM (2 m l b
    // flops per product; FP64-class like the A passes).  FQB_OZ_Q=0 keeps them on DMMA.
    static bool q_oz_default() {
        const char* e = std::getenv("FQB_OZ_Q");
        return !(e && e[0] == '0');
    }
    bool use_q_oz(int64_t l) const { return q_oz_on_ && l >= kQOzMinCols; }
    // the projections Y -= Q C (K = l) on the INT8 path reading the A'Y-layout slices of Q
    // (the ones slice_q made for Q'Y) MN-major, C's rows scaled by Q's column scales --
    // nothing is re-sliced.  FQB_OZ_QMN=0 keeps them on DMMA.
    bool use_q_mn(int64_t l) const {
        static const bool on = [] {
            const char* e = std::getenv("FQB_OZ_QMN");
            return !(e && e[0] == '0');
        }();
        return on && use_q_oz(l);
    }
    void q_mn_sub(int64_t l, const double* Cm, int64_t ldcm, double* Y) {   // Y (m x b) -= Q(:, :l) Cm
        Workspace& w = h_.ws;
        const int nsl = ozaki_fp64_slices();
        w.oz_z.ensure(size_t(std::max(ozaki_apply_z_bytes(m_, nsl), ozaki_apply_z_bytes(l, nsl))), s_);
        w.oz_ez.ensure(size_t(ozaki_apply_ez_count()), s_);
        w.oz_zmax.ensure_zeroed(size_t(ozaki_apply_ez_count()), s_);
        w.oz_q_cs.ensure(size_t(l) * size_t(b_), s_);
        ozaki_apply_mn(m_, b_, l, -1.0, w.oz_q_tn.ptr, w.oz_q_e.ptr, Cm, ldcm, 1.0, Y, ldq_, w.oz_q_cs.ptr,
                       w.oz_z.ptr, w.oz_ez.ptr, h_.gws.work, h_.num_sms, s_, h_.lc, nsl, w.oz_zmax.ptr);
    }
    // slices of q_ columns [floor(q_sliced_ / 128) * 128, upto): every committed column not
    // sliced yet, the current block's Y_j, and the rest of the 128-column tile they start in
    void slice_q(int64_t upto) {
        Workspace& w = h_.ws;
        const int nsl = ozaki_fp64_slices();
        const int64_t c0 = (std::min(q_sliced_, l_) / 128) * 128;
        const int64_t cols = upto - c0;
        if (cols <= 0) return;
        w.oz_q_line_max.ensure_zeroed(size_t(ozaki_line_max_words(m_, cols)), s_);
        ozaki_slice_a(q_.ptr + c0 * ldq_, m_, cols, ldq_, w.oz_q_line_max.ptr,
                      w.oz_q_tn.ptr + (c0 / 128) * (ozaki_x_bytes(128, m_, nsl)), w.oz_q_e.ptr + c0, nullptr, nullptr,
                      s_, h_.lc, nullptr, nullptr, nsl);
        q_sliced_ = l_;   // committed columns with valid slices (the rest is redone next block)
    }
    void q_tn(int64_t M, const double* B, double* C, int64_t ldc) {   // C (M x b) = Q(:, :M)' B
        Workspace& w = h_.ws;
        const int nsl = ozaki_fp64_slices();
        w.oz_z.ensure(size_t(ozaki_apply_z_bytes(m_, nsl)), s_);
        w.oz_ez.ensure(size_t(ozaki_apply_ez_count()), s_);
        w.oz_zmax.ensure_zeroed(size_t(ozaki_apply_ez_count()), s_);
        ozaki_apply(M, b_, m_, 1.0, w.oz_q_tn.ptr, w.oz_q_e.ptr, B, ldq_, 0.0, C, ldc, w.oz_z.ptr, w.oz_ez.ptr,
                    h_.gws.work, h_.num_sms, s_, h_.lc, nsl, w.oz_zmax.ptr);
    }

    // ---- the B-side products on the INT8 tensor cores ---------------------------
    // T = B G (K = n) and W -= B' T (K = l) for every committed column of B' -- 2 n l b
    // flops each, three to four per block -- read B' from slices made once per committed
    // column like Q's (A'Y layout: one operand row per column of B', a power-of-two scale
    // per column; B' T reads them MN-major with T's rows scaled).  FQB_OZ_B=0: DMMA.
    static bool b_oz_default() {
        const char* e = std::getenv("FQB_OZ_B");
        return !(e && e[0] == '0');
    }
    bool use_b_oz(int64_t l) const { return b_oz_on_ && l >= kQOzMinCols; }
    void slice_b() {   // every committed column of B' not sliced yet (from its 128-column tile)
        Workspace& w = h_.ws;
        const int nsl = ozaki_fp64_slices();
        const int64_t c0 = (std::min(b_sliced_, l_) / 128) * 128;
        const int64_t cols = l_ - c0;
        if (cols <= 0) return;
        w.oz_q_line_max.ensure_zeroed(size_t(ozaki_line_max_words(n_, cols)), s_);
        ozaki_slice_a(bt_.ptr + c0 * ldbt_, n_, cols, ldbt_, w.oz_q_line_max.ptr,
                      w.oz_b_tn.ptr + (c0 / 128) * (ozaki_x_bytes(128, n_, nsl)), w.oz_b_e.ptr + c0, nullptr, nullptr,
                      s_, h_.lc, nullptr, nullptr, nsl);
        b_sliced_ = l_;
    }
    // T (l x b, ldt) = B(:l, :) G   (G: n x b, ldg)
    void b_tn(int64_t l, const double* G, int64_t ldg, double* T, int64_t ldt) {
        if (!use_b_oz(l)) {
            gemm_(true, l, b_, n_, 1.0, bt_.ptr, ldbt_, G, ldg, 0.0, T, ldt);
            return;
        }
        slice_b();
        Workspace& w = h_.ws;
        const int nsl = ozaki_fp64_slices();
        w.oz_z.ensure(size_t(ozaki_apply_z_bytes(n_, nsl)), s_);
        w.oz_ez.ensure(size_t(ozaki_apply_ez_count()), s_);
        w.oz_zmax.ensure_zeroed(size_t(ozaki_apply_ez_count()), s_);
        ozaki_apply(l, b_, n_, 1.0, w.oz_b_tn.ptr, w.oz_b_e.ptr, G, ldg, 0.0, T, ldt, w.oz_z.ptr, w.oz_ez.ptr,
                    h_.gws.work, h_.num_sms, s_, h_.lc, nsl, w.oz_zmax.ptr);
    }
    // W (n x b, ldw) -= B(:l, :)' C   (C: l x b, ldc)
    void b_mn_sub(int64_t l, const double* Cm, int64_t ldcm, double* W, int64_t ldw) {
        if (!use_b_oz(l)) {
            gemm_(false, n_, b_, l, -1.0, bt_.ptr, ldbt_, Cm, ldcm, 1.0, W, ldw);
            return;
        }
        slice_b();
        Workspace& w = h_.ws;
        const int nsl = ozaki_fp64_slices();
        w.oz_z.ensure(size_t(std::max(ozaki_apply_z_bytes(n_, nsl), ozaki_apply_z_bytes(l, nsl))), s_);
        w.oz_ez.ensure(size_t(ozaki_apply_ez_count()), s_);
        w.oz_zmax.ensure_zeroed(size_t(ozaki_apply_ez_count()), s_);
        w.oz_q_cs.ensure(size_t(l) * size_t(b_), s_);
        ozaki_apply_mn(n_, b_, l, -1.0, w.oz_b_tn.ptr, w.oz_b_e.ptr, Cm, ldcm, 1.0, W, ldw, w.oz_q_cs.ptr, w.oz_z.ptr,
                       w.oz_ez.ptr, h_.gws.work, h_.num_sms, s_, h_.lc, nsl, w.oz_zmax.ptr);
    }

    // ---- Omega ----------------------------------------------------------------
    void make_block(int id) {
        Workspace& w = h_.ws;
        const int b = b_;
        om_centered_ = false;
        om_shift_folded_ = false;
        om_p_ = cfg_.sketch.p;
        if (src_) {
            fqb_block blk;
            std::memset(&blk, 0, sizeof blk);
            if (src_(user_, int(n_), b, id, &blk) != 0)
                throw Error(kStatusCallback, "block source returned an error for block " + std::to_string(id));
            if (blk.rows != n_ || blk.cols != b)
                throw Error(kStatusDimension, "block source returned a block of the wrong shape");
            om_centered_ = blk.centered != 0;
            om_p_ = blk.p;
            if (blk.is_dense) {
                if (!blk.dense) throw Error(kStatusInvalid, "dense block without data");
                FQB_CUDA(cudaMemcpy2DAsync(w.omega.ptr, ldo_ * sizeof(double), blk.dense, n_ * sizeof(double),
                                           n_ * sizeof(double), b, cudaMemcpyHostToDevice, s_));
                om_dense_ = true;
                return;
            }
            if (!blk.col_ptr || (blk.nnz > 0 && (!blk.row_idx || !blk.values)))
                throw Error(kStatusInvalid, "sparse block without arrays");
            const int64_t nnz = blk.col_ptr[b];
            w.row_idx.ensure(size_t(std::max<int64_t>(nnz, 1)), s_);
            w.values.ensure(size_t(std::max<int64_t>(nnz, 1)), s_);
            FQB_CUDA(cudaMemcpyAsync(w.col_ptr.ptr, blk.col_ptr, (b + 1) * sizeof(int), cudaMemcpyHostToDevice, s_));
            if (nnz > 0) {
                FQB_CUDA(cudaMemcpyAsync(w.row_idx.ptr, blk.row_idx, nnz * sizeof(int), cudaMemcpyHostToDevice, s_));
                FQB_CUDA(cudaMemcpyAsync(w.values.ptr, blk.values, nnz * sizeof(double), cudaMemcpyHostToDevice, s_));
            }
            FQB_CUDA(cudaStreamSynchronize(s_));  // host arrays may change after the callback returns
            finish_sparse(double(nnz) / (double(n_) * b));
            return;
        }
        const int kind = cfg_.sketch.kind;
        const uint64_t seed = cfg_.sketch.seed;
        if (kind == kGaussian) {
            launch_gaussian_dense(seed, id, n_, b, w.omega.ptr, ldo_, status_, s_, h_.lc);
            om_dense_ = true;
            return;
        }
        om_centered_ = kind == kStdBernoulli;
        if (cfg_.sketch.zeta > 0) {
            const int zeta = cfg_.sketch.zeta;
            const int64_t nnz = int64_t(zeta) * b;
            w.row_idx.ensure(size_t(nnz), s_);
            w.values.ensure(size_t(nnz), s_);
            launch_zeta_fill(kind, seed, id, n_, b, zeta, 1.0 / std::sqrt(double(zeta)), w.col_ptr.ptr,
                             w.row_idx.ptr, w.values.ptr, status_, s_, h_.lc);
            finish_sparse(double(zeta) / double(n_));
            return;
        }
        const double p = cfg_.sketch.p;
        const double denom = std::log1p(-p);  // host libm, like sketch.cpp:38
        const double scale = (kind == kSparseSign || kind == kSparseGaussian) ? 1.0 / std::sqrt(p) : 1.0;
        if (p > kDenseThreshold) {
            // densified directly by the walk, centering folded in: Omega_c = S - p
            launch_iid_fill_dense(kind, seed, id, n_, b, denom, scale, om_centered_ ? p : 0.0, w.omega.ptr,
                                  ldo_, status_, s_, h_.lc);
            om_dense_ = true;
            om_shift_folded_ = true;
            return;
        }
        const int64_t cap = n_ * int64_t(b);  // every row may be a nonzero
        w.row_idx.ensure(size_t(cap), s_);
        w.values.ensure(size_t(cap), s_);
        launch_iid_count(kind, seed, id, n_, b, denom, w.counts.ptr, s_, h_.lc);
        launch_exclusive_scan(w.counts.ptr, b, w.col_ptr.ptr, s_, h_.lc);
        launch_iid_fill_csc(kind, seed, id, n_, b, denom, scale, w.col_ptr.ptr, w.row_idx.ptr, w.values.ptr,
                            status_, s_, h_.lc);
        // sparse (p <= kDenseThreshold): a centered block needs z = p A 1 and B's row sums
        finish_sparse(p);
    }

    void finish_sparse(double density) {
        Workspace& w = h_.ws;
        if (density > kDenseThreshold) {
            launch_densify(w.col_ptr.ptr, w.row_idx.ptr, w.values.ptr, n_, b_, om_centered_ ? om_p_ : 0.0,
                           w.omega.ptr, ldo_, s_, h_.lc);
            om_dense_ = true;
            om_shift_folded_ = true;
        } else {
            om_dense_ = false;
            if (om_centered_) ensure_centering();
        }
    }

    void ensure_centering() {
        if (!z_allowed_) throw Error(kStatusDimension, "centered_product: stale centering column");
        if (!have_z_) {
            h_.ws.zc.ensure(size_t(m_), s_);
            if (af_) launch_centering(af_, m_, n_, lda_, cfg_.sketch.p, h_.ws.zc.ptr, s_, h_.lc);
            else launch_centering(a_, m_, n_, lda_, cfg_.sketch.p, h_.ws.zc.ptr, s_, h_.lc);
            have_z_ = true;
        }
        // B row sums for the centered deflation term, for every accepted column
        if (rowsum_cols_ < l_) {
            launch_colsum(bt_.ptr + rowsum_cols_ * ldbt_, n_, int(l_ - rowsum_cols_), ldbt_, rowsum_.ptr + rowsum_cols_,
                          s_, h_.lc);
            rowsum_cols_ = l_;
        }
        need_rowsum_ = true;
    }

    // Y (m x b, ldy) = A * Omega  [centered]   (apply_block, driver.cpp:21-26)
    void apply_omega(double* y, int64_t ldy) {
        Workspace& w = h_.ws;
        if (om_dense_) {
            a_gemm(false, b_, w.omega.ptr, ldo_, y, ldy);
        } else {
            if (af_)
                launch_gather_spmm(af_, m_, lda_, w.col_ptr.ptr, w.row_idx.ptr, w.values.ptr, b_,
                                   om_centered_ ? w.zc.ptr : nullptr, y, ldy, s_, h_.lc);
            else
                launch_gather_spmm(a_, m_, lda_, w.col_ptr.ptr, w.row_idx.ptr, w.values.ptr, b_,
                                   om_centered_ ? w.zc.ptr : nullptr, y, ldy, s_, h_.lc);
        }
    }

    // T (l x b) = B * Omega_c  (tmul_block, driver.cpp:30-45, with W Z^-1 W' = B'B)
    void tmul_omega(double* t, int64_t ldt) {
        Workspace& w = h_.ws;
        if (om_dense_) {
            b_tn(l_, w.omega.ptr, ldo_, t, ldt);
            if (om_centered_ && !om_shift_folded_) {
                // a dense block flagged centered: subtract p * rowsum(B) like the reference
                throw Error(kStatusConfig, "dense centered blocks are not supported");
            }
        } else {
            launch_gather_tmul(bt_.ptr, n_, ldbt_, int(l_), w.col_ptr.ptr, w.row_idx.ptr, w.values.ptr, b_,
                               om_centered_ ? rowsum_.ptr : nullptr, om_p_, t, ldt, s_, h_.lc);
        }
    }

    // ---- orth(W) -> G (n x b) ---------------------------------------------------
    void orth_power(const double* wsrc, double* gdst, bool eig_mode, bool need_sigma) {
        const int b = b_;
        gram_(wsrc, n_, ldbt_, S_);
        if (need_sigma || eig_mode) {
            launch_sym_eig(S_, b, b, eig_, eig_mode ? V_ : nullptr, VT_, status_, kStEigConv, s_, h_.lc);
        }
        if (eig_mode) {
            // eig_svd (matrix_core.cpp:193-215): G = W V Sigma^-1
            launch_eigsvd_scale(eig_, V_, b, VS_, sig_, status_, kStPowerDegenerate, s_, h_.lc);
            gemm_(false, n_, b, b, 1.0, wsrc, ldbt_, VS_, b, 0.0, gdst, ldbt_);
        } else {
            // one CholeskyQR pass: same span, orthonormal to the same u*cond^2 as eigSVD
            launch_chol_upper_inv(S_, b, b, 0.0, 0.0, nullptr, 0, R1_, R1i_, nullptr, h_.ws.scratch.ptr,
                                  status_, kStPowerChol, s_, h_.lc);
            trmm_(wsrc, n_, ldbt_, R1i_, gdst, ldbt_);
        }
    }

    // power_iterate_block (driver.cpp:185-228); leaves the iterate in ws.g
    void power_iterate(bool eig_mode) {
        Workspace& w = h_.ws;
        const int P = cfg_.power;
        FQB_CUDA(cudaMemsetAsync(scal_ + kAlpha, 0, sizeof(double), s_));
        for (int k = 1; k <= P; ++k) {
            if (k == 1) apply_omega(w.y0.ptr, ldq_);
            else a_gemm(false, b_, w.g.ptr, ldbt_, w.y0.ptr, ldq_);
            a_tn_reduced(b_, w.y0.ptr, ldq_, w.wp.ptr, ldbt_);   // W = sum_g A_g' Y_g
            if (l_ > 0) {
                if (k == 1) tmul_omega(w.t.ptr, l_);
                else b_tn(l_, w.g.ptr, ldbt_, w.t.ptr, l_);
                b_mn_sub(l_, w.t.ptr, l_, w.wp.ptr, ldbt_);
            }
            if (k > 1 && P >= 3)
                launch_axpy_cols_dev(scal_ + kAlpha, w.g.ptr, ldbt_, w.wp.ptr, ldbt_, n_, b_, s_, h_.lc);
            const bool need_sigma = k > 1 && k < P;  // the shift only matters for a later pass
            orth_power(w.wp.ptr, w.g.ptr, eig_mode, need_sigma);
            if (need_sigma) launch_shift_update(eig_, b_, cfg_.shift_convention, scal_ + kAlpha, s_, h_.lc);
        }
    }

    // accept_block (driver.cpp:230-294), explicit-Q form
    void accept(bool from_iterate) {
        Workspace& w = h_.ws;
        const int b = b_;
        const int64_t l = l_;
        double* yj = q_.ptr + l * ldq_;
        double* btj = bt_.ptr + l * ldbt_;
        if (from_iterate) a_gemm(false, b, w.g.ptr, ldbt_, yj, ldq_);
        else apply_omega(yj, ldq_);
        a_tn_reduced(b, yj, ldq_, w.wraw.ptr, ldbt_);
        const int64_t ldcd = l + b;
        double* cd = w.cd.ptr;
        // [C1; D] = [Q_old | Y_j]' Y_j
        if (use_q_oz(l)) {
            slice_q(l + b);
            q_tn(l + b, yj, cd, ldcd);
        } else {
            gemm_(true, l + b, b, m_, 1.0, q_.ptr, ldq_, yj, ldq_, 0.0, cd, ldcd);
        }
        comm_allreduce_sum(h_, cd, size_t(ldcd) * b, s_);
        double* dblk = cd + l;  // rows l..l+b-1, ld = l+b
        if (l == 0) {
            launch_chol_upper_inv(dblk, b, ldcd, 1e-12, 0.0, dblk, ldcd, R1_, R1i_, scal_ + kDMax,
                                  w.scratch.ptr, status_, kStAcceptPivot, s_, h_.lc);
            trmm_(yj, m_, ldq_, R1i_, w.ys.ptr, ldq_);
        } else {
            if (use_q_mn(l)) {
                q_mn_sub(l, cd, ldcd, yj);
            } else {
                gemm_(false, m_, b, l, -1.0, q_.ptr, ldq_, cd, ldcd, 1.0, yj, ldq_);
            }
            gram_(yj, m_, ldq_, S_);
            comm_allreduce_sum(h_, S_, size_t(b) * b, s_);
            launch_chol_upper_inv(S_, b, b, 1e-12, diag_max_, dblk, ldcd, R1_, R1i_, scal_ + kDMax,
                                  w.scratch.ptr, status_, kStAcceptPivot, s_, h_.lc);
            trmm_(yj, m_, ldq_, R1i_, w.ys.ptr, ldq_);
            if (use_q_oz(l)) q_tn(l, w.ys.ptr, w.c2.ptr, l);
            else gemm_(true, l, b, m_, 1.0, q_.ptr, ldq_, w.ys.ptr, ldq_, 0.0, w.c2.ptr, l);
            comm_allreduce_sum(h_, w.c2.ptr, size_t(l) * b, s_);
            if (use_q_mn(l)) q_mn_sub(l, w.c2.ptr, l, w.ys.ptr);
            else gemm_(false, m_, b, l, -1.0, q_.ptr, ldq_, w.c2.ptr, l, 1.0, w.ys.ptr, ldq_);
        }
        gram_(w.ys.ptr, m_, ldq_, S2_);
        comm_allreduce_sum(h_, S2_, size_t(b) * b, s_);
        launch_chol_upper_inv(S2_, b, b, 0.0, 0.0, nullptr, 0, R2_, R2i_, nullptr, w.scratch.ptr, status_,
                              kStAcceptChol2, s_, h_.lc);
        trmm_(w.ys.ptr, m_, ldq_, R2i_, yj, ldq_);  // Q_j
        gemm_(false, b, b, b, 1.0, R1i_, b, R2i_, b, 0.0, Ri_, b);              // R^-1 = R1^-1 R2^-1
        if (l > 0) {
            gemm_(false, l, b, b, 1.0, w.c2.ptr, l, R1_, b, 1.0, cd, ldcd);     // C = C1 + C2 R1
            b_mn_sub(l, cd, ldcd, w.wraw.ptr, ldbt_);
        }
        trmm_(w.wraw.ptr, n_, ldbt_, Ri_, btj, ldbt_);  // B_j'
        launch_sumsq(btj, n_, b, ldbt_, w.partial.ptr, scal_ + kBNorm, s_, h_.lc);
        if (need_rowsum_ && rowsum_cols_ == l) {
            launch_colsum(btj, n_, b, ldbt_, rowsum_.ptr + l, s_, h_.lc);
            pending_rowsum_ = true;
        }
    }

    // One attempt; returns 0 when accepted, the degenerate status bits otherwise.
    unsigned try_block(int id) {
        grow(l_ + b_);
        bool eig_mode = false;
        for (int pass = 0; pass < 2; ++pass) {
            pending_rowsum_ = false;
            FQB_CUDA(cudaMemsetAsync(status_, 0, sizeof(unsigned), s_));
            // the eigSVD retry reuses the block already on the device: the reference asks
            // its source once per attempt (driver.cpp:141-143)
            if (pass == 0) make_block(id);
            if (cfg_.power >= 1) power_iterate(eig_mode);
            accept(cfg_.power >= 1);
            FQB_CUDA(cudaMemcpyAsync(h_.host_status, status_, sizeof(unsigned), cudaMemcpyDeviceToHost, s_));
            FQB_CUDA(cudaMemcpyAsync(h_.host_scalars, scal_, 4 * sizeof(double), cudaMemcpyDeviceToHost, s_));
            const auto tw0 = std::chrono::steady_clock::now();
            FQB_CUDA(cudaStreamSynchronize(s_));
            host_wait_s_ += std::chrono::duration<double>(std::chrono::steady_clock::now() - tw0).count();
            const unsigned st = *h_.host_status;
            if (st & kGenZeroGaussian)
                throw Error(kStatusConvergence, "a Gaussian draw hit an exact zero (reference would redraw)");
            if (st & kStEigConv) throw Error(kStatusConvergence, "sym_eig: jacobi sweeps exhausted");
            if ((st & kStPowerChol) && !eig_mode) {
                eig_mode = true;  // CholeskyQR broke down: redo with eigSVD like the reference
                continue;
            }
            if (st & (kStPowerDegenerate | kStAcceptPivot | kStAcceptChol2 | kStPowerChol)) return st;
            // commit
            trace_ += h_.host_scalars[kBNorm];
            diag_max_ = h_.host_scalars[kDMax];
            l_ += b_;
            if (pending_rowsum_) rowsum_cols_ = l_;
            pending_rowsum_ = false;
            ++blocks_;
            residuals_.push_back(residual());
            if (stream_out_) push_host();
            return 0;
        }
        return kStPowerDegenerate;
    }

    Handle& h_;
    cudaStream_t s_;
    const double* a_;
    const float* af_;          // FP32 input mode (a_ null until a DMMA pass needs the widened copy)
    int64_t a_ld64_ = 0;       // leading dimension of the widened copy
    int64_t m_, n_, lda_;
    fqb_config cfg_;
    int b_;
    fqb_block_source_fn src_;
    void* user_;
    int64_t ldq_, ldbt_, ldo_;
    int64_t cap_ = 0, l_ = 0;
    int blocks_ = 0;
    double norm_a_sq_ = 0.0, trace_ = 0.0, diag_max_ = 0.0;
    bool have_z_ = false, need_rowsum_ = false, z_allowed_ = false, pending_rowsum_ = false;
    int64_t rowsum_cols_ = 0;  // B' columns whose row sums are in rowsum_
    bool stream_out_ = false;  // stream_out_host()
    double *hq_ = nullptr, *hbt_ = nullptr;
    int64_t hcap_ = 0, hcopied_ = 0;
  public:
    double host_wait_s_ = 0.0;  // time the host spent blocked on the device (FQB_HOST_STATS)
    bool om_dense_ = true, om_centered_ = false, om_shift_folded_ = false;
    double om_p_ = 0.0;
    DeviceArray<double> q_, bt_, rowsum_;
    bool oz_on_ = false;              // A-pass products on the INT8 tensor cores (a_gemm)
    int oz_nsl_ = 7;                  // slices per operand of the A passes (7 / 8: FP64-class, 4: FP32-class)
    bool oz_ready_ = false;           // A sliced for this run (buffers live in the handle workspace)
    bool q_oz_on_ = false;            // Q'X products of the accept step on the INT8 tensor cores
    int64_t q_sliced_ = 0;            // columns of Q whose slices in ws.oz_q_tn are valid
    bool b_oz_on_ = false;            // B G and B' T products on the INT8 tensor cores
    int64_t b_sliced_ = 0;            // columns of B' whose slices in ws.oz_b_tn are valid
    static constexpr int64_t kQOzMinCols = 200;
    std::vector<double> residuals_;
    std::vector<int> ids_;
    double *S_, *S2_, *R1_, *R1i_, *R2_, *R2i_, *R_, *Ri_, *V_, *VS_, *VT_, *eig_, *sig_, *scal_;
    unsigned* status_;
};

}  // namespace

int run_qb(Handle& h, const void* a, bool a_f32, int64_t m, int64_t n, int64_t lda, bool a_on_device,
           bool fixed_precision, int rank, const fqb_config& cfg_in, fqb_block_source_fn src, void* user,
           unsigned flags, fqb_qb_result* out, std::string* message_out) {
    std::memset(out, 0, sizeof *out);
    out->m = m;
    out->n = n;
    if (!a && !(sharded(h) && m == 0)) throw Error(kStatusInvalid, "null matrix pointer");
    if (lda < m) throw Error(kStatusDimension, "lda < m");
    // with a communicator, (a, m, lda) is this rank's row block of A
    int64_t m_global = m;
    if (sharded(h)) {
        h.ws.scalars.ensure(8, h.stream);
        const double local = double(m);
        FQB_CUDA(cudaMemcpyAsync(h.ws.scalars.ptr, &local, sizeof(double), cudaMemcpyHostToDevice, h.stream));
        comm_allreduce_sum(h, h.ws.scalars.ptr, 1, h.stream);
        double total = 0.0;
        FQB_CUDA(cudaMemcpyAsync(&total, h.ws.scalars.ptr, sizeof(double), cudaMemcpyDeviceToHost, h.stream));
        FQB_CUDA(cudaStreamSynchronize(h.stream));
        m_global = int64_t(total);
    }
    fqb_config cfg = resolve_config(m_global, n, cfg_in, fixed_precision);
    if (!fixed_precision) {
        if (rank < 1) throw Error(kStatusConfig, "rank must be at least 1");
        if (rank > std::min(m_global, n)) throw Error(kStatusConfig, "rank exceeds matrix dimensions");
    }
    if (!src && cfg.sketch.kind != kGaussian && cfg.sketch.zeta == 0 && !(cfg.sketch.p > 0.0 && cfg.sketch.p < 1.0))
        throw Error(kStatusConfig, "gen_sketch: sparse kinds require p in (0,1)");
    out->resolved_block = cfg.block;
    out->resolved_max_iters = cfg.max_iters;
    out->resolved_p = cfg.sketch.p;
    const int64_t launches0 = h.lc.total;
    cudaStream_t s = h.stream;
    FQB_CUDA(cudaEventRecord(h.ev0, s));

    // A on the device with an even, 16-byte aligned leading dimension (FP64, or
    // FP32 in the FP32 input mode: A kept in FP32, every product in FP64)
    const size_t esz = a_f32 ? sizeof(float) : sizeof(double);
    const void* ad = a;
    int64_t ldad = lda;
    const bool usable = a_on_device && lda % 2 == 0 && reinterpret_cast<uintptr_t>(a) % 16 == 0;
    if (!usable) {
        ldad = round_up(m, 8);
        void* dst;
        if (a_f32) {
            h.ws.a_copy_f32.ensure(size_t(ldad) * n, s);
            dst = h.ws.a_copy_f32.ptr;
        } else {
            h.ws.a_copy.ensure(size_t(ldad) * n, s);
            dst = h.ws.a_copy.ptr;
        }
        FQB_CUDA(cudaMemcpy2DAsync(dst, ldad * esz, a, lda * esz, m * esz, n,
                                   a_on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice, s));
        ad = dst;
    }

    const auto t_host0 = std::chrono::steady_clock::now();
    QbRun run(h, a_f32 ? nullptr : static_cast<const double*>(ad), a_f32 ? static_cast<const float*>(ad) : nullptr, m,
              n, ldad, cfg, src, user);
    if (!(flags & FQB_OUT_DEVICE) && (flags & FQB_OUT_HOST) && !std::getenv("FQB_OUT_TAIL")) run.stream_out_host();
    run.setup();
    int status = 0;
    bool converged = false;
    std::string message;
    try {
        if (fixed_precision) {
            const double norm_a = std::sqrt(run.norm_a_sq());
            const double eps_abs = cfg.relative ? cfg.eps * norm_a : cfg.eps;
            const double eps_sq = eps_abs * eps_abs;
            if (run.residual() <= eps_sq) {
                converged = true;
            } else {
                for (int j = 0; j < cfg.max_iters; ++j) {
                    run.process_block(j);
                    if (run.residual() < eps_sq) {
                        converged = true;
                        break;
                    }
                }
            }
            if (!converged) {
                status = kStatusTolerance;
                message = "tolerance not reached after " + std::to_string(run.blocks()) + " blocks";
            }
        } else {
            const int nblocks = (rank + cfg.block - 1) / cfg.block;
            run.reserve_blocks(nblocks);
            for (int j = 0; j < nblocks; ++j) run.process_block(j);
            converged = true;
        }
    } catch (const Error& e) {
        if (e.status != kStatusDegenerate) throw;
        status = kStatusDegenerate;
        message = e.what();
    }
    // Host Q, B' are final now: copy them out on a second stream while the SVD
    // assembly runs (the assembly only reads them)
    const int l_qb = run.rank();
    double *host_q = nullptr, *host_bt = nullptr;
    struct HostGuard {   // returns the blocks to the pool if the assembly below throws
        double** a;
        double** b;
        cudaStream_t* copies;   // drained first: async copies may still target the blocks
        ~HostGuard() {
            if ((*a || *b) && *copies) cudaStreamSynchronize(*copies);
            if (*a) host_free(*a);
            if (*b) host_free(*b);
        }
    } host_guard{&host_q, &host_bt, &h.copy_stream};
    const bool host_out = l_qb > 0 && !(flags & FQB_OUT_DEVICE) && (flags & FQB_OUT_HOST);
    if (host_out) {   // host capacity for the next run of this shape (QbRun::push_host)
        h.out_hint_m = m;
        h.out_hint_n = n;
        h.out_hint_l = l_qb;
    }
    if (host_out && run.streamed()) {
        run.take_host(&host_q, &host_bt);   // every committed column already queued
    } else if (host_out) {
        host_q = static_cast<double*>(host_alloc(sizeof(double) * size_t(m) * l_qb));
        host_bt = static_cast<double*>(host_alloc(sizeof(double) * size_t(n) * l_qb));
        if (!host_q || !host_bt) throw Error(kStatusAlloc, "host result allocation failed");
        if (!h.copy_stream) {
            FQB_CUDA(cudaStreamCreateWithFlags(&h.copy_stream, cudaStreamNonBlocking));
            FQB_CUDA(cudaEventCreateWithFlags(&h.ev_qb, cudaEventDisableTiming));
        }
        FQB_CUDA(cudaEventRecord(h.ev_qb, s));
        FQB_CUDA(cudaStreamWaitEvent(h.copy_stream, h.ev_qb, 0));
        FQB_CUDA(cudaMemcpy2DAsync(host_q, m * sizeof(double), run.q().ptr, run.ldq() * sizeof(double),
                                   m * sizeof(double), l_qb, cudaMemcpyDeviceToHost, h.copy_stream));
        FQB_CUDA(cudaMemcpy2DAsync(host_bt, n * sizeof(double), run.bt().ptr, run.ldbt() * sizeof(double),
                                   n * sizeof(double), l_qb, cudaMemcpyDeviceToHost, h.copy_stream));
    }

    // ApproxSvd (assemble_svd, driver.cpp:296-345): also for the partial result of
    // ToleranceNotReached; BlockDegenerate carries no factorization (errors.hpp:28-37)
    std::vector<double> sig;
    std::vector<char> flg;
    DeviceArray<double> u_dev, v_dev;
    int svd_r = 0, drop = 0;
    double svd_res = run.residual();
    const int l_final = run.rank();
    // host U / V (FQB_OUT_HOST): allocated up front and filled on the copy stream
    // while the rest of the assembly runs
    double *host_u = nullptr, *host_v = nullptr;
    HostGuard uv_guard{&host_u, &host_v, &h.copy_stream};
    bool uv_to_host = false;
    if ((flags & FQB_OUT_SVD) && status != kStatusDegenerate && l_final > 0) {
        u_dev.ensure(size_t(run.ldq()) * l_final, s);
        v_dev.ensure(size_t(run.ldbt()) * l_final, s);
        if (!fixed_precision) drop = std::max(0, l_final - rank);  // drop_smallest (driver.cpp:85-106)
        svd_r = l_final - drop;
        HostSvdCopy hc{};
        const bool uv_host = svd_r > 0 && !(flags & FQB_OUT_DEVICE) && (flags & FQB_OUT_HOST);
        if (uv_host) {
            host_u = static_cast<double*>(host_alloc(sizeof(double) * size_t(m) * svd_r));
            host_v = static_cast<double*>(host_alloc(sizeof(double) * size_t(n) * svd_r));
            if (!host_u || !host_v) throw Error(kStatusAlloc, "host result allocation failed");
            if (!h.copy_stream) FQB_CUDA(cudaStreamCreateWithFlags(&h.copy_stream, cudaStreamNonBlocking));
            if (!h.ev_u) FQB_CUDA(cudaEventCreateWithFlags(&h.ev_u, cudaEventDisableTiming));
            if (!h.ev_v) FQB_CUDA(cudaEventCreateWithFlags(&h.ev_v, cudaEventDisableTiming));
            hc = HostSvdCopy{h.copy_stream, h.ev_u, h.ev_v, host_u, host_v, drop};
        }
        assemble_svd(h, run.q().ptr, run.ldq(), run.bt().ptr, run.ldbt(), m, n, l_final, u_dev.ptr, run.ldq(),
                     v_dev.ptr, run.ldbt(), sig, flg, uv_host ? &hc : nullptr, run.ozaki() && l_final >= 256);
        uv_to_host = uv_host;
        for (int i = 0; i < drop; ++i) svd_res += sig[i] * sig[i];
    }
    FQB_CUDA(cudaEventRecord(h.ev1, s));

    out->status = status;
    out->rank = run.rank();
    out->blocks = run.blocks();
    out->converged = converged ? 1 : 0;
    out->residual_sq = run.residual();
    out->norm_a_sq = run.norm_a_sq();
    out->ldq = run.ldq();
    out->ldbt = run.ldbt();
    const int l = run.rank();
    if (l > 0 && (flags & FQB_OUT_DEVICE)) {
        out->q = run.q().detach();
        out->bt = run.bt().detach();
        out->on_device = 1;
    } else if (host_out) {
        out->q = host_q;     // copied on the copy stream above
        out->bt = host_bt;
        host_q = host_bt = nullptr;   // owned by the result now
        out->ldq = m;
        out->ldbt = n;
        out->on_device = 0;
    }
    if (flags & FQB_OUT_SVD) {
        out->svd_rank = svd_r;
        out->svd_residual_sq = svd_res;
        out->sigma = static_cast<double*>(std::malloc(sizeof(double) * std::max(svd_r, 1)));
        out->v_flagged = static_cast<char*>(std::malloc(std::max(svd_r, 1)));
        for (int i = 0; i < svd_r; ++i) {
            out->sigma[i] = sig[drop + i];
            out->v_flagged[i] = flg[drop + i];
        }
        if (svd_r > 0 && (flags & FQB_OUT_DEVICE)) {
            // the kept columns are the last svd_r (ascending order): into fresh buffers
            // (source and destination would overlap in place -- undefined for memcpy)
            if (drop > 0) {
                DeviceArray<double> uk, vk;
                uk.ensure(size_t(run.ldq()) * svd_r, s);
                vk.ensure(size_t(run.ldbt()) * svd_r, s);
                FQB_CUDA(cudaMemcpyAsync(uk.ptr, u_dev.ptr + int64_t(drop) * run.ldq(),
                                         sizeof(double) * run.ldq() * svd_r, cudaMemcpyDeviceToDevice, s));
                FQB_CUDA(cudaMemcpyAsync(vk.ptr, v_dev.ptr + int64_t(drop) * run.ldbt(),
                                         sizeof(double) * run.ldbt() * svd_r, cudaMemcpyDeviceToDevice, s));
                u_dev.release();
                v_dev.release();
                u_dev.ptr = uk.detach();
                v_dev.ptr = vk.detach();
            }
            out->u = u_dev.detach();
            out->v = v_dev.detach();
            out->ldu = run.ldq();
            out->ldv = run.ldbt();
        } else if (svd_r > 0 && host_u) {
            out->u = host_u;    // copied on the copy stream during the assembly
            out->v = host_v;
            host_u = host_v = nullptr;   // owned by the result now
            out->ldu = m;
            out->ldv = n;
        }
    }
    FQB_CUDA(cudaStreamSynchronize(s));
    if (host_out || uv_to_host) FQB_CUDA(cudaStreamSynchronize(h.copy_stream));
    float ms = 0.f;
    cudaEventElapsedTime(&ms, h.ev0, h.ev1);
    out->elapsed_ms = ms;
    const auto& res = run.residuals();
    out->block_residuals = static_cast<double*>(std::malloc(sizeof(double) * std::max<size_t>(res.size(), 1)));
    if (!res.empty()) std::memcpy(out->block_residuals, res.data(), sizeof(double) * res.size());
    const auto& ids = run.ids();
    out->block_ids = static_cast<int*>(std::malloc(sizeof(int) * std::max<size_t>(ids.size(), 1)));
    if (!ids.empty()) std::memcpy(out->block_ids, ids.data(), sizeof(int) * ids.size());
    out->n_ids = int(ids.size());
    out->gpu_launches = int(h.lc.total - launches0);
    if (const char* e = std::getenv("FQB_HOST_STATS"); e && e[0] == '1') {
        const double tot = std::chrono::duration<double>(std::chrono::steady_clock::now() - t_host0).count();
        std::fprintf(stderr, "[farqb] host %.3f ms, blocked on device %.3f ms, device %.3f ms, launches %d\n",
                     tot * 1e3, run.host_wait_s_ * 1e3, double(ms), out->gpu_launches);
    }
    if (message_out) *message_out = message;
    return status;
}

}  // namespace farqb
