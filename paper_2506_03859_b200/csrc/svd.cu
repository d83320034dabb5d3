// svd.cu -- assemble U, sigma, V from the device QB factors.
//
// The reference's assemble_svd (/root/reference/proj/src/driver.cpp:296-345)
// works in Gram space (eig(Z), then eig(D'TD)).  With Q and B explicit the
// same quantities come from one l x l symmetric eigenproblem:
//     B B' = U~ diag(lambda) U~'   (B = Bt', l x l, eigenvalues ascending)
//     sigma = sqrt(max(lambda, 0))              ascending, like ApproxSvd
//     U = Q U~,   V = B' U~ diag(1/sigma)       (sigma <= 1e-14 sigma_max: zero
//                                                column, v_flagged, driver.cpp:331-341)
// B B', Q U~ and B' U~ Sigma^-1 are DMMA GEMMs, or (emulate: the run's A passes ran on the
// INT8 tensor cores and l >= 256) k_ozaki products; the l x l eigensolver is cuSOLVER's syevd (dlopen()ed,
// like NCCL: a library call for a once-per-run O(l^3) step, not the hot loop).
#include <cusolverDn.h>
#include <dlfcn.h>

#include <cmath>
#include <cstdlib>
#include <mutex>
#include <string>
#include <vector>

#include "engine.hpp"
#include "kernels.hpp"

namespace farqb {
namespace {

struct CusolverApi {
    decltype(&cusolverDnCreate) create = nullptr;
    decltype(&cusolverDnDestroy) destroy = nullptr;
    decltype(&cusolverDnSetStream) set_stream = nullptr;
    decltype(&cusolverDnDsyevd_bufferSize) syevd_buffer = nullptr;
    decltype(&cusolverDnDsyevd) syevd = nullptr;
    decltype(&cusolverDnCreateSyevjInfo) create_syevj = nullptr;
    decltype(&cusolverDnXsyevjSetTolerance) syevj_tol = nullptr;
    decltype(&cusolverDnXsyevjSetMaxSweeps) syevj_sweeps = nullptr;
    decltype(&cusolverDnDsyevj_bufferSize) syevj_buffer = nullptr;
    decltype(&cusolverDnDsyevj) syevj = nullptr;
    bool ok = false;
    std::string why;
};

CusolverApi& cusolver() {
    static CusolverApi api;
    static std::once_flag once;
    std::call_once(once, [] {
        void* h = dlopen("libcusolver.so.11", RTLD_NOW | RTLD_GLOBAL | RTLD_NOLOAD);
        if (!h) h = dlopen("libcusolver.so.11", RTLD_NOW | RTLD_GLOBAL);
        if (!h) h = dlopen("/usr/local/cuda/lib64/libcusolver.so.11", RTLD_NOW | RTLD_GLOBAL);
        if (!h) {
            api.why = std::string("cannot load libcusolver.so.11: ") + dlerror();
            return;
        }
        api.create = reinterpret_cast<decltype(&cusolverDnCreate)>(dlsym(h, "cusolverDnCreate"));
        api.destroy = reinterpret_cast<decltype(&cusolverDnDestroy)>(dlsym(h, "cusolverDnDestroy"));
        api.set_stream = reinterpret_cast<decltype(&cusolverDnSetStream)>(dlsym(h, "cusolverDnSetStream"));
        api.syevd_buffer =
            reinterpret_cast<decltype(&cusolverDnDsyevd_bufferSize)>(dlsym(h, "cusolverDnDsyevd_bufferSize"));
        api.syevd = reinterpret_cast<decltype(&cusolverDnDsyevd)>(dlsym(h, "cusolverDnDsyevd"));
        api.create_syevj =
            reinterpret_cast<decltype(&cusolverDnCreateSyevjInfo)>(dlsym(h, "cusolverDnCreateSyevjInfo"));
        api.syevj_tol =
            reinterpret_cast<decltype(&cusolverDnXsyevjSetTolerance)>(dlsym(h, "cusolverDnXsyevjSetTolerance"));
        api.syevj_sweeps =
            reinterpret_cast<decltype(&cusolverDnXsyevjSetMaxSweeps)>(dlsym(h, "cusolverDnXsyevjSetMaxSweeps"));
        api.syevj_buffer =
            reinterpret_cast<decltype(&cusolverDnDsyevj_bufferSize)>(dlsym(h, "cusolverDnDsyevj_bufferSize"));
        api.syevj = reinterpret_cast<decltype(&cusolverDnDsyevj)>(dlsym(h, "cusolverDnDsyevj"));
        api.ok = api.create && api.destroy && api.set_stream && api.syevd_buffer && api.syevd && api.create_syevj &&
                 api.syevj_tol && api.syevj_sweeps && api.syevj_buffer && api.syevj;
        if (!api.ok) api.why = "libcusolver.so.11 lacks a required symbol";
    });
    if (!api.ok) throw Error(kStatusCuda, api.why);
    return api;
}

void cs_check(cusolverStatus_t st, const char* what) {
    if (st != CUSOLVER_STATUS_SUCCESS) throw Error(kStatusCuda, std::string(what) + " failed (cusolver status " +
                                                                    std::to_string(int(st)) + ")");
}

// mat (n x n, ld n): upper triangle := lower triangle (32 x 32 tiles through shared memory)
__global__ void k_mirror_lower(double* mat, int64_t n) {
    FQB_PDL_ENTRY();
    __shared__ double t[32][33];
    const int64_t bi = blockIdx.x, bj = blockIdx.y;   // tile (row block bi, column block bj), bi >= bj sources
    if (bi < bj) return;
    const int tx = threadIdx.x, ty = threadIdx.y;
    for (int r = ty; r < 32; r += 8) {
        const int64_t i = bi * 32 + r, j = bj * 32 + tx;
        t[r][tx] = (i < n && j < n) ? mat[j * n + i] : 0.0;
    }
    __syncthreads();
    // write the transpose into tile (bj, bi): element (j, i) = (i, j) for i > j
    for (int r = ty; r < 32; r += 8) {
        const int64_t j = bj * 32 + r, i = bi * 32 + tx;   // destination row j, column i
        if (i < n && j < n && i > j) mat[i * n + j] = t[tx][r];
    }
}

__global__ void k_scale_cols(const double* src, int64_t lds, const double* scale, int rows, int cols, double* dst,
                             int64_t ldd) {
    FQB_PDL_ENTRY();
    const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    const int c = blockIdx.y;
    if (i < rows && c < cols) dst[int64_t(c) * ldd + i] = src[int64_t(c) * lds + i] * scale[c];
}

// sigma = sqrt(max(lambda, 0)) (ascending), the pseudo-inverse scale and the flags of
// assemble_svd (sigma <= 1e-14 sigma_max: v column zeroed and flagged), one CTA
__global__ void k_sigma(const double* __restrict__ lam, int l, double* sigma, double* inv, char* flagged) {
    FQB_PDL_ENTRY();
    const double smax = sqrt(fmax(lam[l - 1], 0.0));
    for (int j = threadIdx.x; j < l; j += blockDim.x) {
        const double sg = sqrt(fmax(lam[j], 0.0));
        const bool keep = sg > 1e-14 * smax;
        sigma[j] = sg;
        inv[j] = keep ? 1.0 / sg : 0.0;
        flagged[j] = keep ? 0 : 1;
    }
}

// T (r x w, ld r) = (V[s:s+w, :] diag(sigma))'   (sigma null: unscaled)
__global__ void k_strip_t(const double* v, int64_t ldv, const double* sigma, int r, int64_t s, int w, double* t) {
    FQB_PDL_ENTRY();
    const int k = blockIdx.y;
    const int j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j < w && k < r) t[int64_t(j) * r + k] = v[int64_t(k) * ldv + s + j] * (sigma ? sigma[k] : 1.0);
}

}  // namespace

// rsvd::relative_error (experiment.cpp:317-342): strips of w columns of A,
// D = A_strip - U T with T = (V_strip diag(sigma))', err^2 += ||D||^2 (fixed
// strip order, each strip a deterministic tree sum), then sqrt(err^2 / ||A||^2).
double relative_error(Handle& h, const double* a, int64_t m, int64_t n, int64_t lda, bool a_on_device,
                      const double* u, int64_t ldu, const double* sigma, const double* v, int64_t ldv, int r,
                      bool factors_on_device) {
    cudaStream_t s = h.stream;
    ensure_gemm_workspace(h);
    if (m == 0 || n == 0) return 0.0;
    // strips sized to ~256 MB of A
    const int64_t w = std::max<int64_t>(1, std::min<int64_t>(n, (int64_t(1) << 25) / std::max<int64_t>(m, 1)));
    const int64_t nstrips = ceil_div(n, w);
    DeviceArray<double> part, sums, d, t, ud, vd, sd, astrip;
    part.ensure(kReducePartials, s);
    sums.ensure(size_t(nstrips + 1), s);
    d.ensure(size_t(m) * w, s);
    if (!a_on_device) astrip.ensure(size_t(m) * w, s);
    const double *U = u, *V = v, *SIG = nullptr;
    if (r > 0) {
        if (!factors_on_device) {
            ud.ensure(size_t(m) * r, s);
            vd.ensure(size_t(n) * r, s);
            FQB_CUDA(cudaMemcpy2DAsync(ud.ptr, m * sizeof(double), u, ldu * sizeof(double), m * sizeof(double), r,
                                       cudaMemcpyHostToDevice, s));
            FQB_CUDA(cudaMemcpy2DAsync(vd.ptr, n * sizeof(double), v, ldv * sizeof(double), n * sizeof(double), r,
                                       cudaMemcpyHostToDevice, s));
            U = ud.ptr;
            V = vd.ptr;
            ldu = m;
            ldv = n;
        }
        if (sigma) {
            sd.ensure(size_t(r), s);
            FQB_CUDA(cudaMemcpyAsync(sd.ptr, sigma, sizeof(double) * r, cudaMemcpyHostToDevice, s));
            SIG = sd.ptr;
        }
        t.ensure(size_t(r) * w, s);
    }
    for (int64_t k = 0; k < nstrips; ++k) {
        const int64_t c0 = k * w, wc = std::min(w, n - c0);
        const double* ak = a + c0 * lda;
        int64_t ldak = lda;
        if (!a_on_device) {   // stream the host strip in
            FQB_CUDA(cudaMemcpy2DAsync(astrip.ptr, m * sizeof(double), ak, lda * sizeof(double), m * sizeof(double), wc,
                                       cudaMemcpyHostToDevice, s));
            ak = astrip.ptr;
            ldak = m;
        }
        // ||A||^2 strip by strip (slot nstrips accumulates on the host below)
        FQB_CUDA(cudaMemcpy2DAsync(d.ptr, m * sizeof(double), ak, ldak * sizeof(double), m * sizeof(double), wc,
                                   cudaMemcpyDeviceToDevice, s));
        if (r > 0) {
            dim3 g(unsigned(ceil_div(wc, 256)), unsigned(r));
            launch_k(k_strip_t, g, 256, 0, s, V, ldv, SIG, r, c0, int(wc), t.ptr);
            FQB_LAUNCHED();
            h.lc.bump();
            gemm(false, m, wc, r, -1.0, U, ldu, t.ptr, r, 1.0, d.ptr, m, h.gws, h.num_sms, s, h.lc);
        }
        launch_sumsq(d.ptr, m, wc, m, part.ptr, sums.ptr + k, s, h.lc);
    }
    std::vector<double> hs(static_cast<size_t>(nstrips));
    FQB_CUDA(cudaMemcpyAsync(hs.data(), sums.ptr, sizeof(double) * nstrips, cudaMemcpyDeviceToHost, s));
    // ||A||^2 with the same strip order
    double norm_sq = 0.0;
    {
        std::vector<double> hn(static_cast<size_t>(nstrips));
        for (int64_t k = 0; k < nstrips; ++k) {
            const int64_t c0 = k * w, wc = std::min(w, n - c0);
            const double* ak = a + c0 * lda;
            int64_t ldak = lda;
            if (!a_on_device) {
                FQB_CUDA(cudaMemcpy2DAsync(astrip.ptr, m * sizeof(double), ak, lda * sizeof(double),
                                           m * sizeof(double), wc, cudaMemcpyHostToDevice, s));
                ak = astrip.ptr;
                ldak = m;
            }
            launch_sumsq(ak, m, wc, ldak, part.ptr, sums.ptr + nstrips, s, h.lc);
            FQB_CUDA(cudaMemcpyAsync(&hn[size_t(k)], sums.ptr + nstrips, sizeof(double), cudaMemcpyDeviceToHost, s));
        }
        FQB_CUDA(cudaStreamSynchronize(s));
        for (double x : hn) norm_sq += x;
    }
    if (norm_sq == 0.0) return 0.0;
    if (r == 0) return 1.0;
    double err_sq = 0.0;
    for (double x : hs) err_sq += x;
    return std::sqrt(err_sq / norm_sq);
}

// Symmetric eigendecomposition of mat (l x l, ld l, both triangles) in place:
// eigenvalues ascending into w, eigenvectors into mat.  FQB_EIG: unset / "small" =
// the l <= kSmallEighMax solver of eigsmall.cu (1.56 ms at l = 200; its own residual /
// orthogonality check falls back to syevd), "syevd" = cuSOLVER syevd only (1.9 ms),
// "syevj" = cuSOLVER Jacobi.
// Returns true when the small-l solver produced the result.
// info_dev != null: cuSOLVER's status goes there and nothing is synchronized (the
// caller checks it); null: checked here.
static bool eigh_core(Handle& h, double* mat, int l, double* w, int* info_dev) {
    cudaStream_t s = h.stream;
    ensure_gemm_workspace(h);
    const char* env = std::getenv("FQB_EIG");
    // unset / "small": the own solver for l <= 224 (eigsmall.cu), syevd above; "large": also the
    // own solver above 224 (eiglarge.cu: correct, but 3.4x slower than syevd at l = 2000 -- its
    // one-stage tridiagonalisation is a chain of 2000 grid barriers, 17 us per column)
    const int eig_mode = !env ? 0 : std::string(env) == "syevj" ? 2 : std::string(env) == "syevd" ? 1 : 0;
    const bool own_large = env && std::string(env) == "large";
    if (eig_mode == 0 && l <= kSmallEighMax) {
        DeviceArray<double> es;
        es.ensure(size_t(small_eigh_scratch_doubles(l)), s);
        const bool ok = small_eigh(mat, l, w, mat, es.ptr, h.gws, h.num_sms, s, h.lc);
        FQB_CUDA(cudaStreamSynchronize(s));   // es is released on scope exit
        if (ok) return true;
    }
    if (own_large && l > kSmallEighMax) {
        // own solver for large l (eiglarge.cu): cooperative tridiagonalisation, bisection,
        // inverse iteration, WY back-transformation; checked a posteriori, syevd if not
        DeviceArray<double> keep;   // the input survives a failed attempt
        keep.ensure(size_t(l) * l, s);
        FQB_CUDA(cudaMemcpyAsync(keep.ptr, mat, sizeof(double) * size_t(l) * l, cudaMemcpyDeviceToDevice, s));
        if (large_eigh(h, keep.ptr, l, w, mat)) return true;
        FQB_CUDA(cudaMemcpyAsync(mat, keep.ptr, sizeof(double) * size_t(l) * l, cudaMemcpyDeviceToDevice, s));
        FQB_CUDA(cudaStreamSynchronize(s));
    }
    CusolverApi& api = cusolver();
    if (!h.cusolver) {
        cusolverDnHandle_t ch = nullptr;
        cs_check(api.create(&ch), "cusolverDnCreate");
        h.cusolver = ch;
    }
    auto ch = static_cast<cusolverDnHandle_t>(h.cusolver);
    cs_check(api.set_stream(ch, s), "cusolverDnSetStream");
    DeviceArray<double> work;
    DeviceArray<int> info;
    info.ensure(1, s);
    int* info_ptr = info_dev ? info_dev : info.ptr;
    int lwork = 0;
    if (eig_mode == 2) {   // measured: syevd 2.1 ms, syevj 3.3 ms at l = 200
        // GPU-resident Jacobi (no host round trips), converged to working precision
        static syevjInfo_t params = nullptr;
        if (!params) {
            cs_check(api.create_syevj(&params), "cusolverDnCreateSyevjInfo");
            cs_check(api.syevj_tol(params, 0.0), "cusolverDnXsyevjSetTolerance");   // 0 = machine precision
            cs_check(api.syevj_sweeps(params, 100), "cusolverDnXsyevjSetMaxSweeps");
        }
        cs_check(api.syevj_buffer(ch, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER, l, mat, l, w, &lwork, params),
                 "cusolverDnDsyevj_bufferSize");
        work.ensure(size_t(std::max(lwork, 1)), s);
        cs_check(api.syevj(ch, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER, l, mat, l, w, work.ptr, lwork,
                           info_ptr, params),
                 "cusolverDnDsyevj");
    } else {
        cs_check(api.syevd_buffer(ch, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER, l, mat, l, w, &lwork),
                 "cusolverDnDsyevd_bufferSize");
        work.ensure(size_t(std::max(lwork, 1)), s);
        cs_check(api.syevd(ch, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER, l, mat, l, w, work.ptr, lwork,
                           info_ptr),
                 "cusolverDnDsyevd");
    }
    if (info_dev) return false;   // work / info are released stream-ordered
    int hinfo = 0;
    FQB_CUDA(cudaMemcpyAsync(&hinfo, info.ptr, sizeof(int), cudaMemcpyDeviceToHost, s));
    FQB_CUDA(cudaStreamSynchronize(s));
    if (hinfo != 0) throw Error(kStatusConvergence, "syevd did not converge (info " + std::to_string(hinfo) + ")");
    return false;
}

bool eigh_inplace(Handle& h, double* mat, int l, double* w) { return eigh_core(h, mat, l, w, nullptr); }

void assemble_svd(Handle& h, const double* q, int64_t ldq, const double* bt, int64_t ldbt, int64_t m, int64_t n,
                  int l, double* u, int64_t ldu, double* v, int64_t ldv, std::vector<double>& sigma,
                  std::vector<char>& flagged, const HostSvdCopy* hc, bool emulate) {
    sigma.assign(l, 0.0);
    flagged.assign(l, 0);
    if (l == 0) return;
    cudaStream_t s = h.stream;
    ensure_gemm_workspace(h);
    DeviceArray<double> mat, w, scale, us;
    mat.ensure(size_t(l) * l, s);
    w.ensure(size_t(l), s);
    // emulate: the three products on the INT8 tensor cores (the run's A passes were there):
    // B' sliced once in both layouts, Q row-scaled (K = l); FP64-class like the A passes
    const int nsl = ozaki_fp64_slices();
    DeviceArray<int8_t> bt_tn, bt_nn, q_nn, oz_z;
    DeviceArray<int> bt_etn, bt_enn, q_enn, oz_ez;
    DeviceArray<unsigned> oz_lm, oz_zmax;
    if (emulate) {
        oz_lm.ensure_zeroed(size_t(ozaki_line_max_words(std::max<int64_t>(m, n), l)), s);
        bt_tn.ensure(size_t(ozaki_x_bytes(l, n, nsl)), s);
        bt_nn.ensure(size_t(ozaki_x_bytes(n, l, nsl)), s);
        bt_etn.ensure(size_t(l), s);
        bt_enn.ensure(size_t(n), s);
        ozaki_slice_a(bt, n, l, ldbt, oz_lm.ptr, bt_tn.ptr, bt_etn.ptr, bt_nn.ptr, bt_enn.ptr, s, h.lc, nullptr,
                      nullptr, nsl);
        oz_z.ensure(size_t(ozaki_apply_z_bytes(std::max<int64_t>(n, l), nsl)), s);
        oz_ez.ensure(size_t(ozaki_apply_ez_count()), s);
        oz_zmax.ensure_zeroed(size_t(ozaki_apply_ez_count()), s);
    }
    auto oz = [&](int64_t M, int64_t K, const int8_t* xs, const int* ex, const double* B, int64_t ldb, double* C,
                  int64_t ldc) {
        ozaki_apply(M, l, K, 1.0, xs, ex, B, ldb, 0.0, C, ldc, oz_z.ptr, oz_ez.ptr, h.gws.work, h.num_sms, s, h.lc,
                    nsl, oz_zmax.ptr);
    };
    // B B' = Bt' Bt  (l x l).  Emulated: only the 128-column blocks on and below the
    // diagonal (rows from the block's own first row: about half the products), then the
    // lower triangle mirrored -- the eigensolvers get a symmetric matrix
    if (emulate) {
        for (int64_t c0 = 0; c0 < l; c0 += 128) {
            const int64_t nb = std::min<int64_t>(128, l - c0);
            ozaki_apply(l - c0, nb, n, 1.0, bt_tn.ptr + (c0 / 128) * ozaki_x_bytes(128, n, nsl), bt_etn.ptr + c0,
                        bt + c0 * ldbt, ldbt, 0.0, mat.ptr + c0 + c0 * int64_t(l), l, oz_z.ptr, oz_ez.ptr, h.gws.work,
                        h.num_sms, s, h.lc, nsl, oz_zmax.ptr);
        }
        launch_k(k_mirror_lower, dim3(unsigned(ceil_div(l, 32)), unsigned(ceil_div(l, 32))), dim3(32, 8), 0, s, mat.ptr,
                 int64_t(l));
        FQB_LAUNCHED();
        h.lc.bump();
    } else {
        gemm(true, l, l, n, 1.0, bt, ldbt, bt, ldbt, 0.0, mat.ptr, l, h.gws, h.num_sms, s, h.lc);
    }
    // eigendecomposition, sigma / flags / pseudo-inverse scale and both GEMMs are queued
    // without a host round trip; the one synchronization at the end also brings back
    // sigma, the flags and cuSOLVER's status
    DeviceArray<int> info;
    DeviceArray<char> flg;
    info.ensure(1, s);
    FQB_CUDA(cudaMemsetAsync(info.ptr, 0, sizeof(int), s));
    eigh_core(h, mat.ptr, l, w.ptr, info.ptr);
    scale.ensure(size_t(2) * l, s);   // [sigma | 1/sigma]
    flg.ensure(size_t(l), s);
    us.ensure(size_t(l) * l, s);
    launch_k(k_sigma, 1, 256, 0, s, w.ptr, l, scale.ptr, scale.ptr + l, flg.ptr);
    FQB_LAUNCHED();
    dim3 grid(unsigned(ceil_div(l, 256)), unsigned(l));
    launch_k(k_scale_cols, grid, 256, 0, s, mat.ptr, l, scale.ptr + l, l, l, us.ptr, l);
    FQB_LAUNCHED();
    h.lc.bump(2);
    // V = Bt (U~ Sigma^-1) first (small), then U = Q U~ (this rank's rows); with hc, the kept
    // columns (>= drop) go to the host on the copy stream as soon as they are computed -- U in
    // blocks of 256 columns, so its download overlaps the rest of its product
    auto copy_cols = [&](const double* src, int64_t lds, int64_t rows, double* dst, int64_t c0, int64_t c1,
                         cudaEvent_t ev) {
        const int64_t a0 = std::max<int64_t>(c0, hc->drop);
        if (a0 >= c1) return;
        FQB_CUDA(cudaEventRecord(ev, s));
        FQB_CUDA(cudaStreamWaitEvent(hc->stream, ev, 0));
        FQB_CUDA(cudaMemcpy2DAsync(dst + (a0 - hc->drop) * rows, rows * sizeof(double), src + a0 * lds,
                                   lds * sizeof(double), rows * sizeof(double), c1 - a0, cudaMemcpyDeviceToHost,
                                   hc->stream));
    };
    if (emulate) oz(n, l, bt_nn.ptr, bt_enn.ptr, us.ptr, l, v, ldv);
    else gemm(false, n, l, l, 1.0, bt, ldbt, us.ptr, l, 0.0, v, ldv, h.gws, h.num_sms, s, h.lc);
    if (hc && hc->v) copy_cols(v, ldv, n, hc->v, 0, l, hc->ev_v);
    if (emulate) {
        q_nn.ensure(size_t(ozaki_x_bytes(m, l, nsl)), s);
        q_enn.ensure(size_t(std::max<int64_t>(m, 1)), s);
        ozaki_slice_a(q, m, l, ldq, oz_lm.ptr, nullptr, nullptr, q_nn.ptr, q_enn.ptr, s, h.lc, nullptr, nullptr, nsl);
    }
    const int64_t ub = (hc && hc->u) ? 256 : l;
    for (int64_t c0 = 0; c0 < l; c0 += ub) {
        const int64_t nb = std::min<int64_t>(ub, l - c0);
        if (emulate)
            ozaki_apply(m, nb, l, 1.0, q_nn.ptr, q_enn.ptr, mat.ptr + c0 * l, l, 0.0, u + c0 * ldu, ldu, oz_z.ptr,
                        oz_ez.ptr, h.gws.work, h.num_sms, s, h.lc, nsl, oz_zmax.ptr);
        else
            gemm(false, m, nb, l, 1.0, q, ldq, mat.ptr + c0 * l, l, 0.0, u + c0 * ldu, ldu, h.gws, h.num_sms, s,
                 h.lc);
        if (hc && hc->u) copy_cols(u, ldu, m, hc->u, c0, c0 + nb, hc->ev_u);
    }
    int hinfo = 0;
    FQB_CUDA(cudaMemcpyAsync(sigma.data(), scale.ptr, sizeof(double) * l, cudaMemcpyDeviceToHost, s));
    FQB_CUDA(cudaMemcpyAsync(flagged.data(), flg.ptr, size_t(l), cudaMemcpyDeviceToHost, s));
    FQB_CUDA(cudaMemcpyAsync(&hinfo, info.ptr, sizeof(int), cudaMemcpyDeviceToHost, s));
    FQB_CUDA(cudaStreamSynchronize(s));  // the temporaries above are released on return
    if (hinfo != 0) throw Error(kStatusConvergence, "syevd did not converge (info " + std::to_string(hinfo) + ")");
}

void destroy_cusolver(Handle& h) {
    if (h.cusolver) cusolver().destroy(static_cast<cusolverDnHandle_t>(h.cusolver));
    h.cusolver = nullptr;
}

}  // namespace farqb
