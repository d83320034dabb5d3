// engine.hpp -- the device-resident farPCA blocked QB loop (C++ host side).
#pragma once

#include <cuda_runtime.h>

#include <chrono>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <string>
#include <vector>

#include "../../include/farqb.h"
#include "common.cuh"
#include "kernels.hpp"

namespace farqb {

// FQB_ALLOC_STATS=1: report slow pool allocations on stderr (diagnostics)
inline bool alloc_stats_enabled() {
    static const bool on = [] {
        const char* e = std::getenv("FQB_ALLOC_STATS");
        return e && e[0] == '1';
    }();
    return on;
}

// devmem.cu: cached large device blocks (>= kLargeBlock bytes), see there
constexpr size_t kLargeBlock = size_t(16) << 20;
void* device_alloc_large(size_t bytes, cudaStream_t s);
bool device_free_large(void* p, cudaStream_t s);   // false: not a cached-path block
size_t device_cache_trim();

// Stream-ordered device allocation, grown on demand: the cudaMallocAsync pool for small
// buffers, the large-block cache (devmem.cu) from kLargeBlock bytes up.
template <typename T>
struct DeviceArray {
    T* ptr = nullptr;
    size_t count = 0;
    cudaStream_t stream = nullptr;
    DeviceArray() = default;
    DeviceArray(const DeviceArray&) = delete;
    DeviceArray& operator=(const DeviceArray&) = delete;
    ~DeviceArray() { release(); }
    void release() {
        if (ptr && !device_free_large(ptr, stream)) cudaFreeAsync(ptr, stream);
        ptr = nullptr;
        count = 0;
    }
    // contents are not preserved
    T* ensure(size_t n, cudaStream_t s) {
        if (n <= count && ptr) return ptr;
        release();
        stream = s;
        const auto t0 = std::chrono::steady_clock::now();
        const size_t bytes = std::max<size_t>(n, 1) * sizeof(T);
        if (bytes >= kLargeBlock)
            ptr = static_cast<T*>(device_alloc_large(bytes, s));
        else
            FQB_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&ptr), bytes, s));
        count = std::max<size_t>(n, 1);
        if (alloc_stats_enabled()) {
            const double ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
            if (ms > 0.2) std::fprintf(stderr, "[farqb] device allocation %.3f GB took %.2f ms\n",
                                       double(count * sizeof(T)) / 1e9, ms);
        }
        return ptr;
    }
    // as ensure, and a new allocation is zero-filled: the generation-tagged line maxima of
    // ozaki.cu rely on never finding a word tagged above the current generation
    T* ensure_zeroed(size_t n, cudaStream_t s) {
        if (n <= count && ptr) return ptr;
        ensure(n, s);
        FQB_CUDA(cudaMemsetAsync(ptr, 0, count * sizeof(T), s));
        return ptr;
    }
    // hand ownership to the caller
    T* detach() {
        T* p = ptr;
        ptr = nullptr;
        count = 0;
        return p;
    }
};

// Per-handle reusable workspace (everything except the Q and B' outputs).
struct Workspace {
    DeviceArray<double> omega, y0, ys, wp, wraw, g, t, cd, c2, small, zc, rowsum_b, splitk, partial,
        scalars, scratch, a_copy, oz_norm_partial, w_half, oz_q_cs;
    DeviceArray<float> a_copy_f32;   // FP32 input mode staging
    DeviceArray<int> col_ptr, row_idx, counts;
    DeviceArray<double> values;
    DeviceArray<unsigned> status;
    DeviceArray<unsigned> gemm_flags;
    // Ozaki slices of A (both layouts), kept across runs so a run does not pay
    // for two large allocations; released with the handle
    DeviceArray<int8_t> oz_x_nn, oz_x_tn, oz_z;
    DeviceArray<int> oz_e_nn, oz_e_tn, oz_ez;
    DeviceArray<unsigned> oz_line_max;
    // Ozaki slices of Q in the A'Y layout (operand rows = columns of Q), grown with Q,
    // for the block Gram-Schmidt products [Q|Y]'Y and Q'Y_s (engine.cu, accept)
    DeviceArray<int8_t> oz_q_tn;   // Q in the A'Y layout (grown with Q; also read MN-major for Y -= Q C)
    DeviceArray<int> oz_q_e;
    DeviceArray<unsigned> oz_q_line_max, oz_zmax;
    // B' (n x l) in the same layout (operand rows = rows of B, K = n), grown with B', for
    // T = B G and W -= B' T (engine.cu, power_iterate / accept)
    DeviceArray<int8_t> oz_b_tn;
    DeviceArray<int> oz_b_e;

    // every member, while the stream the frees are ordered on still exists
    void release_all() {
        for (auto* d : {&omega, &y0, &ys, &wp, &wraw, &g, &t, &cd, &c2, &small, &zc, &rowsum_b, &splitk, &partial,
                        &scalars, &scratch, &a_copy, &values, &oz_norm_partial, &w_half, &oz_q_cs})
            d->release();
        for (auto* d : {&col_ptr, &row_idx, &counts, &oz_e_nn, &oz_e_tn, &oz_ez, &oz_q_e, &oz_b_e}) d->release();
        for (auto* d : {&status, &gemm_flags, &oz_line_max, &oz_q_line_max, &oz_zmax}) d->release();
        a_copy_f32.release();
        for (auto* d : {&oz_x_nn, &oz_x_tn, &oz_z, &oz_q_tn, &oz_b_tn}) d->release();
    }
};

struct Handle {
    int device = 0;
    int num_sms = 148;
    int fp32_slices = 8;              // FP32 input: 8 (FP64-class A passes), 4 or 3 (FP32-class, fqb_set_fp32_slices)
    cudaStream_t own_stream = nullptr;
    cudaStream_t stream = nullptr;
    LaunchCounter lc;
    LaunchTimer pass_timer;           // fqb_set_pass_timing
    Workspace ws;
    GemmWorkspace gws;                // views into ws.splitk / ws.gemm_flags
    unsigned* host_status = nullptr;  // pinned readback slot
    double* host_scalars = nullptr;   // pinned readback slots
    cudaEvent_t ev0 = nullptr, ev1 = nullptr;
    // row-sharded multi-GPU (comm.cu); nullptr = single GPU
    void* comm = nullptr;
    // ... or the host reduction backend (fqb_comm_attach_host): sums staged through
    // pinned host memory and handed to a caller-supplied all-reduce
    fqb_host_allreduce_fn host_ar = nullptr;
    void* host_ar_user = nullptr;
    double* host_ar_buf = nullptr;
    size_t host_ar_cap = 0;
    int nranks = 1, rank = 0;
    int64_t collectives = 0;
    void* cusolver = nullptr;  // svd.cu
    // D2H of host results overlapped with the SVD assembly (created on first use)
    cudaStream_t copy_stream = nullptr;
    // NCCL all-reduce of the first half of W = A'Y overlapped with the second half's product
    cudaStream_t comm_stream = nullptr;
    cudaEvent_t ev_half = nullptr, ev_reduced = nullptr;
    cudaEvent_t ev_qb = nullptr;
    cudaEvent_t ev_copied = nullptr;                // copy stream -> engine stream (QbRun::grow)
    int64_t out_hint_m = -1, out_hint_n = -1, out_hint_l = 0;   // host Q / B' capacity hint (QbRun::push_host)
    cudaEvent_t ev_u = nullptr, ev_v = nullptr;   // host U / V copies of the SVD assembly
};

// eiglarge.cu: l x l symmetric eigensolver for 224 < l <= 8192 (a-posteriori checked; false: use syevd)
bool large_eigh(Handle& h, const double* mat, int n, double* w, double* x);
// svd.cu: U = Q U~, V = Bt U~ Sigma^-1 from eig(B B'); sigma ascending
bool eigh_inplace(Handle& h, double* mat, int l, double* w);
// Host copies of U / V's kept columns (the last l - drop), issued on `stream` right
// after each factor's GEMM (events ev_u / ev_v order them after it); null u / v skip.
struct HostSvdCopy {
    cudaStream_t stream;
    cudaEvent_t ev_u, ev_v;
    double* u;
    double* v;
    int drop;
};
void assemble_svd(Handle& h, const double* q, int64_t ldq, const double* bt, int64_t ldbt, int64_t m, int64_t n,
                  int l, double* u, int64_t ldu, double* v, int64_t ldv, std::vector<double>& sigma,
                  std::vector<char>& flagged, const HostSvdCopy* hc = nullptr, bool emulate = false);
void destroy_cusolver(Handle& h);
// synthetic.cu: test matrices on the device (reference synthetic.cpp)
void random_orthonormal_dev(Handle& h, int64_t n, int r, uint64_t seed, uint32_t stream, int first_col, double* q,
                            int64_t ldq);
int gen_synthetic_dev(Handle& h, int kind, int n, int d, uint64_t seed, double* a, int64_t lda);
void gen_lowrank_dev(Handle& h, int64_t m, int64_t n, int r, const double* sigma, uint64_t seed, double noise,
                     double* a, int64_t lda);
// detgen.cu: the deterministic generator (bit-equal to oracle/detgen.c) and the matrix fingerprint
void gen_lowrank_det_dev(Handle& h, int64_t m, int64_t n, int r, const double* sigma_host, uint64_t seed,
                         double noise_scale, int64_t row0, int64_t rows, double* a, int64_t lda);
uint64_t checksum_dev(Handle& h, const double* a, int64_t rows, int64_t cols, int64_t lda, int64_t row0,
                      int64_t m_total);
// hostmem.cu: pinned, pooled host arrays for results returned on the host
void* host_alloc(size_t bytes);
void host_free(void* ptr);
void host_release(void* ptr);   // like host_free, never cached
size_t host_pool_trim();   // release every cached free block; returns the bytes released
// ||A - U diag(sigma) V'||_F / ||A||_F (sigma host or null = unscaled), strips of A on the device
double relative_error(Handle& h, const double* a, int64_t m, int64_t n, int64_t lda, bool a_on_device,
                      const double* u, int64_t ldu, const double* sigma, const double* v, int64_t ldv, int r,
                      bool factors_on_device);

// rawio.cu: RawF64 files (matrix_io.cpp:141-200); FormatFailure carries the byte offset
struct FormatFailure : Error {
    int64_t offset;
    FormatFailure(const std::string& m, int64_t off) : Error(kStatusFormat, m), offset(off) {}
};
void raw_header(const char* path, int64_t* rows, int64_t* cols);
void load_raw_rows(Handle* h, const char* path, int64_t row0, int64_t rows, double* dst, int64_t ld,
                   bool dst_on_device);

// comm.cu
void comm_unique_id(void* out128);
void comm_attach(Handle& h, const void* id128, int nranks, int rank);
void comm_detach(Handle& h);
void comm_allreduce_sum(Handle& h, double* buf, size_t count, cudaStream_t s);
void comm_attach_host(Handle& h, fqb_host_allreduce_fn fn, void* user, int nranks, int rank);
inline bool sharded(const Handle& h) { return h.comm != nullptr || h.host_ar != nullptr; }

struct ResolvedConfig {
    fqb_config cfg;
    int64_t m, n;
};

// Sizes the GEMM scratch (split-K partials, stream-K flags) on the handle.
void ensure_gemm_workspace(Handle& h);

// Runs the loop; fills `out` (status also returned).  Throws farqb::Error for
// configuration / CUDA failures before any result exists.
int run_qb(Handle& h, const void* a, bool a_f32, int64_t m, int64_t n, int64_t lda, bool a_on_device,
           bool fixed_precision, int rank, const fqb_config& cfg, fqb_block_source_fn src,
           void* user, unsigned flags, fqb_qb_result* out, std::string* message_out);

// Resolution rules of the reference (driver.cpp:116-132) plus zeta checks.
fqb_config resolve_config(int64_t m, int64_t n, const fqb_config& in, bool fixed_precision);

double default_density(int kind, int64_t n);
int default_block(int64_t m, int64_t n);
int default_max_iters(int64_t n, int b);

}  // namespace farqb
