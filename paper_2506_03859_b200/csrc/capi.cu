// capi.cu -- the extern "C" boundary (include/farqb.h).
//
// Every entry point converts farqb::Error / std::exception into an fqb_status
// and a thread-local message; no C++ exception crosses the boundary.  There is
// no host compute path: without a CUDA device every compute call fails with
// FQB_ERR_CUDA.
#include <atomic>
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <new>
#include <string>

#include "../../include/farqb.h"
#include "engine.hpp"
#include "kernels.hpp"

struct fqb_handle_s {
    farqb::Handle h;
};

namespace {

thread_local std::string g_last_error;
std::atomic<int> g_live_handles{0};   // the pinned host pool is trimmed when the last handle goes

fqb_status set_error(int status, const std::string& msg) {
    g_last_error = msg;
    return static_cast<fqb_status>(status);
}

template <typename F>
fqb_status guarded(F&& f) {
    try {
        return f();
    } catch (const farqb::Error& e) {
        return set_error(e.status, e.what());
    } catch (const std::bad_alloc&) {
        return set_error(FQB_ERR_ALLOC, "host allocation failed");
    } catch (const std::exception& e) {
        return set_error(FQB_ERR_INVALID_ARGUMENT, e.what());
    } catch (...) {
        return set_error(FQB_ERR_INVALID_ARGUMENT, "unknown error");
    }
}

void bind(fqb_handle h) {
    if (!h) throw farqb::Error(FQB_ERR_INVALID_ARGUMENT, "null handle");
    FQB_CUDA(cudaSetDevice(h->h.device));
}

}  // namespace

extern "C" {

int fqb_abi_version(void) { return FARQB_ABI_VERSION; }

const char* fqb_last_error(void) { return g_last_error.c_str(); }

size_t fqb_host_pool_trim(void) { return farqb::host_pool_trim(); }

size_t fqb_device_cache_trim(void) { return farqb::device_cache_trim(); }

const char* fqb_status_name(int status) {
    switch (status) {
        case FQB_OK: return "ok";
        case FQB_ERR_CONFIG: return "config";
        case FQB_ERR_DIMENSION: return "dimension";
        case FQB_ERR_BLOCK_DEGENERATE: return "block_degenerate";
        case FQB_ERR_TOLERANCE_NOT_REACHED: return "tolerance_not_reached";
        case FQB_ERR_CUDA: return "cuda";
        case FQB_ERR_NCCL: return "nccl";
        case FQB_ERR_INVALID_ARGUMENT: return "invalid_argument";
        case FQB_ERR_CONVERGENCE: return "convergence";
        case FQB_ERR_CALLBACK: return "callback";
        case FQB_ERR_ALLOC: return "alloc";
        case FQB_ERR_FORMAT: return "format";
        default: return "unknown";
    }
}

fqb_status fqb_create(int device, fqb_handle* out) {
    return guarded([&]() -> fqb_status {
        if (!out) throw farqb::Error(FQB_ERR_INVALID_ARGUMENT, "null output handle");
        *out = nullptr;
        int count = 0;
        const cudaError_t e = cudaGetDeviceCount(&count);
        if (e != cudaSuccess || count == 0)
            throw farqb::Error(FQB_ERR_CUDA, "no CUDA device available (libfarqb has no CPU path)");
        if (device < 0 || device >= count) throw farqb::Error(FQB_ERR_INVALID_ARGUMENT, "bad device ordinal");
        FQB_CUDA(cudaSetDevice(device));
        auto* hs = new fqb_handle_s();
        farqb::Handle& h = hs->h;
        h.device = device;
        FQB_CUDA(cudaDeviceGetAttribute(&h.num_sms, cudaDevAttrMultiProcessorCount, device));
        // A blocking stream: work on it is ordered after work the caller queued on the
        // legacy default stream (e.g. PyTorch producing A), so a device-resident A is
        // always complete when the engine reads it.  Callers on other streams pass
        // their stream with fqb_set_stream.
        FQB_CUDA(cudaStreamCreateWithFlags(&h.own_stream, cudaStreamDefault));
        h.stream = h.own_stream;
        FQB_CUDA(cudaEventCreate(&h.ev0));
        FQB_CUDA(cudaEventCreate(&h.ev1));
        FQB_CUDA(cudaMallocHost(&h.host_status, 64));
        FQB_CUDA(cudaMallocHost(&h.host_scalars, 64 * sizeof(double)));
        cudaMemPool_t pool;
        FQB_CUDA(cudaDeviceGetDefaultMemPool(&pool, device));
        uint64_t threshold = UINT64_MAX;
        FQB_CUDA(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &threshold));
        *out = hs;
        g_live_handles.fetch_add(1);
        return FQB_OK;
    });
}

fqb_status fqb_destroy(fqb_handle h) {
    return guarded([&]() -> fqb_status {
        if (!h) return FQB_OK;
        bind(h);
        cudaStreamSynchronize(h->h.stream);
        farqb::comm_detach(h->h);
        farqb::destroy_cusolver(h->h);
        h->h.ws.release_all();
        cudaStreamSynchronize(h->h.stream);
        cudaFreeHost(h->h.host_status);
        cudaFreeHost(h->h.host_scalars);
        cudaEventDestroy(h->h.ev0);
        cudaEventDestroy(h->h.ev1);
        if (h->h.copy_stream) cudaStreamDestroy(h->h.copy_stream);
        if (h->h.comm_stream) cudaStreamDestroy(h->h.comm_stream);
        if (h->h.ev_half) cudaEventDestroy(h->h.ev_half);
        if (h->h.ev_reduced) cudaEventDestroy(h->h.ev_reduced);
        if (h->h.ev_qb) cudaEventDestroy(h->h.ev_qb);
        if (h->h.ev_copied) cudaEventDestroy(h->h.ev_copied);
        if (h->h.ev_u) cudaEventDestroy(h->h.ev_u);
        if (h->h.ev_v) cudaEventDestroy(h->h.ev_v);
        for (cudaEvent_t e : h->h.pass_timer.ev) cudaEventDestroy(e);
        cudaStreamDestroy(h->h.own_stream);
        delete h;
        if (g_live_handles.fetch_sub(1) == 1) {
            farqb::host_pool_trim();
            farqb::device_cache_trim();
        }
        return FQB_OK;
    });
}

fqb_status fqb_set_stream(fqb_handle h, void* stream) {
    return guarded([&]() -> fqb_status {
        bind(h);
        h->h.stream = stream ? static_cast<cudaStream_t>(stream) : h->h.own_stream;
        return FQB_OK;
    });
}

fqb_status fqb_synchronize(fqb_handle h) {
    return guarded([&]() -> fqb_status {
        bind(h);
        FQB_CUDA(cudaStreamSynchronize(h->h.stream));
        return FQB_OK;
    });
}

int64_t fqb_launch_count(fqb_handle h) { return h ? h->h.lc.total : 0; }

int64_t fqb_collective_count(fqb_handle h) { return h ? h->h.collectives : 0; }

fqb_status fqb_set_pass_timing(fqb_handle h, int on) {
    return guarded([&]() -> fqb_status {
        if (!h) throw farqb::Error(FQB_ERR_INVALID_ARGUMENT, "null handle");
        bind(h);
        FQB_CUDA(cudaStreamSynchronize(h->h.stream));   // no recorded event is still pending
        h->h.pass_timer.on = on != 0;
        h->h.pass_timer.used = 0;
        h->h.pass_timer.bytes = 0.0;
        return FQB_OK;
    });
}

fqb_status fqb_pass_timing(fqb_handle h, double* total_ms, int64_t* launches, double* bytes) {
    return guarded([&]() -> fqb_status {
        if (!h) throw farqb::Error(FQB_ERR_INVALID_ARGUMENT, "null handle");
        bind(h);
        FQB_CUDA(cudaStreamSynchronize(h->h.stream));
        const farqb::LaunchTimer& t = h->h.pass_timer;
        double ms = 0.0;
        for (size_t i = 0; i + 1 < t.used; i += 2) {
            float e = 0.f;
            FQB_CUDA(cudaEventElapsedTime(&e, t.ev[i], t.ev[i + 1]));
            ms += double(e);
        }
        if (total_ms) *total_ms = ms;
        if (launches) *launches = int64_t(t.used / 2);
        if (bytes) *bytes = t.bytes;
        return FQB_OK;
    });
}

fqb_status fqb_comm_unique_id(void* out128) {
    return guarded([&]() -> fqb_status {
        if (!out128) throw farqb::Error(FQB_ERR_INVALID_ARGUMENT, "null id buffer");
        farqb::comm_unique_id(out128);
        return FQB_OK;
    });
}

fqb_status fqb_comm_attach(fqb_handle h, const void* id128, int nranks, int rank) {
    return guarded([&]() -> fqb_status {
        bind(h);
        if (!id128) throw farqb::Error(FQB_ERR_INVALID_ARGUMENT, "null id");
        farqb::comm_attach(h->h, id128, nranks, rank);
        return FQB_OK;
    });
}

fqb_status fqb_comm_attach_host(fqb_handle h, fqb_host_allreduce_fn fn, void* user, int nranks, int rank) {
    return guarded([&]() -> fqb_status {
        bind(h);
        farqb::comm_attach_host(h->h, fn, user, nranks, rank);
        return FQB_OK;
    });
}

fqb_status fqb_comm_detach(fqb_handle h) {
    return guarded([&]() -> fqb_status {
        bind(h);
        farqb::comm_detach(h->h);
        farqb::destroy_cusolver(h->h);
        return FQB_OK;
    });
}

static fqb_status run_common(fqb_handle h, const void* a, bool a_f32, int64_t m, int64_t n, int64_t lda,
                             int a_on_device, bool fixed_precision, int rank, const fqb_config* cfg,
                             fqb_block_source_fn src, void* user, unsigned flags, fqb_qb_result* out) {
    if (out) std::memset(out, 0, sizeof *out);
    return guarded([&]() -> fqb_status {
        bind(h);
        if (!cfg || !out) throw farqb::Error(FQB_ERR_INVALID_ARGUMENT, "null config or result");
        std::string msg;
        const int st = farqb::run_qb(h->h, a, a_f32, m, n, lda, a_on_device != 0, fixed_precision, rank, *cfg,
                                     src, user, flags, out, &msg);
        out->status = st;
        if (st != FQB_OK) g_last_error = msg;
        return static_cast<fqb_status>(st);
    });
}

fqb_status fqb_qb_fixed_precision(fqb_handle h, const double* a, int64_t m, int64_t n, int64_t lda,
                                  int a_on_device, const fqb_config* cfg, fqb_block_source_fn src,
                                  void* user, unsigned flags, fqb_qb_result* out) {
    const fqb_status st = run_common(h, a, false, m, n, lda, a_on_device, true, 0, cfg, src, user, flags, out);
    if (out) out->status = st;
    return st;
}

fqb_status fqb_qb_fixed_precision_f32(fqb_handle h, const float* a, int64_t m, int64_t n, int64_t lda,
                                      int a_on_device, const fqb_config* cfg, fqb_block_source_fn src, void* user,
                                      unsigned flags, fqb_qb_result* out) {
    const fqb_status st = run_common(h, a, true, m, n, lda, a_on_device, true, 0, cfg, src, user, flags, out);
    if (out) out->status = st;
    return st;
}

fqb_status fqb_qb_fixed_rank_f32(fqb_handle h, const float* a, int64_t m, int64_t n, int64_t lda,
                                 int a_on_device, int rank, const fqb_config* cfg, fqb_block_source_fn src,
                                 void* user, unsigned flags, fqb_qb_result* out) {
    const fqb_status st = run_common(h, a, true, m, n, lda, a_on_device, false, rank, cfg, src, user, flags, out);
    if (out) out->status = st;
    return st;
}

fqb_status fqb_qb_fixed_rank(fqb_handle h, const double* a, int64_t m, int64_t n, int64_t lda,
                             int a_on_device, int rank, const fqb_config* cfg, fqb_block_source_fn src,
                             void* user, unsigned flags, fqb_qb_result* out) {
    const fqb_status st = run_common(h, a, false, m, n, lda, a_on_device, false, rank, cfg, src, user, flags, out);
    if (out) out->status = st;
    return st;
}

void fqb_host_free(void* p) { farqb::host_free(p); }

void fqb_result_free(fqb_qb_result* r) {
    if (!r) return;
    if (r->on_device && (r->q || r->bt || r->u || r->v)) {
        // like cudaFree: no work still queued anywhere may use the blocks afterwards
        cudaDeviceSynchronize();
        for (double* p : {r->q, r->bt, r->u, r->v})
            if (p && !farqb::device_free_large(p, nullptr)) cudaFree(p);
    } else if (!r->on_device) {
        farqb::host_free(r->q);
        farqb::host_free(r->bt);
    }
    if (!r->on_device) {
        farqb::host_free(r->u);
        farqb::host_free(r->v);
    }
    std::free(r->sigma);
    std::free(r->v_flagged);
    r->u = r->v = r->sigma = nullptr;
    r->v_flagged = nullptr;
    std::free(r->block_residuals);
    std::free(r->block_ids);
    r->q = r->bt = nullptr;
    r->block_residuals = nullptr;
    r->block_ids = nullptr;
}

// ---- building blocks ----------------------------------------------------------

fqb_status fqb_philox_u32(fqb_handle h, uint64_t seed, uint32_t block_id, uint32_t column, int count,
                          uint32_t* host_out) {
    return guarded([&]() -> fqb_status {
        bind(h);
        if (count < 0 || (count > 0 && !host_out)) throw farqb::Error(FQB_ERR_INVALID_ARGUMENT, "bad output");
        if (count == 0) return FQB_OK;
        cudaStream_t s = h->h.stream;
        farqb::DeviceArray<uint32_t> d;
        d.ensure(size_t(count), s);
        farqb::launch_philox_u32(seed, block_id, column, count, d.ptr, s, h->h.lc);
        FQB_CUDA(cudaMemcpyAsync(host_out, d.ptr, sizeof(uint32_t) * count, cudaMemcpyDeviceToHost, s));
        FQB_CUDA(cudaStreamSynchronize(s));
        return FQB_OK;
    });
}

fqb_status fqb_gen_sketch(fqb_handle h, const fqb_sketch_spec* spec, int n, int l, int block_id,
                          fqb_sketch_host* out) {
    if (out) std::memset(out, 0, sizeof *out);
    return guarded([&]() -> fqb_status {
        bind(h);
        if (!spec || !out) throw farqb::Error(FQB_ERR_INVALID_ARGUMENT, "null spec or output");
        if (n < 1 || l < 1) throw farqb::Error(FQB_ERR_CONFIG, "gen_sketch: dimensions must be positive");
        const int kind = spec->kind;
        if (kind < 0 || kind > 4) throw farqb::Error(FQB_ERR_CONFIG, "unknown sketch kind");
        cudaStream_t s = h->h.stream;
        farqb::LaunchCounter& lc = h->h.lc;
        farqb::DeviceArray<unsigned> status;
        status.ensure(1, s);
        FQB_CUDA(cudaMemsetAsync(status.ptr, 0, sizeof(unsigned), s));
        out->rows = n;
        out->cols = l;
        out->p = spec->p;
        if (kind == FQB_GAUSSIAN) {
            farqb::DeviceArray<double> d;
            d.ensure(size_t(n) * l, s);
            farqb::launch_gaussian_dense(spec->seed, block_id, n, l, d.ptr, n, status.ptr, s, lc);
            out->is_dense = 1;
            out->dense = static_cast<double*>(std::malloc(sizeof(double) * size_t(n) * l));
            FQB_CUDA(cudaMemcpyAsync(out->dense, d.ptr, sizeof(double) * size_t(n) * l, cudaMemcpyDeviceToHost, s));
            FQB_CUDA(cudaStreamSynchronize(s));
            return FQB_OK;
        }
        farqb::DeviceArray<int> cp, ri, counts;
        farqb::DeviceArray<double> va;
        cp.ensure(size_t(l) + 1, s);
        int64_t cap;
        if (spec->zeta > 0) {
            if (kind != FQB_SPARSE_SIGN && kind != FQB_SPARSE_GAUSSIAN)
                throw farqb::Error(FQB_ERR_CONFIG, "zeta applies to the sparse sign / sparse Gaussian kinds only");
            if (spec->zeta > n || spec->zeta > 256) throw farqb::Error(FQB_ERR_CONFIG, "zeta must not exceed min(n, 256)");
            cap = int64_t(spec->zeta) * l;
            ri.ensure(size_t(cap), s);
            va.ensure(size_t(cap), s);
            farqb::launch_zeta_fill(kind, spec->seed, block_id, n, l, spec->zeta, 1.0 / std::sqrt(double(spec->zeta)),
                                    cp.ptr, ri.ptr, va.ptr, status.ptr, s, lc);
        } else {
            const double p = spec->p;
            if (!(p > 0.0 && p < 1.0)) throw farqb::Error(FQB_ERR_CONFIG, "gen_sketch: sparse kinds require p in (0,1)");
            cap = int64_t(n) * l;
            ri.ensure(size_t(cap), s);
            va.ensure(size_t(cap), s);
            counts.ensure(size_t(l), s);
            const double denom = std::log1p(-p);
            const double scale = (kind == FQB_SPARSE_SIGN || kind == FQB_SPARSE_GAUSSIAN) ? 1.0 / std::sqrt(p) : 1.0;
            farqb::launch_iid_count(kind, spec->seed, block_id, n, l, denom, counts.ptr, s, lc);
            farqb::launch_exclusive_scan(counts.ptr, l, cp.ptr, s, lc);
            farqb::launch_iid_fill_csc(kind, spec->seed, block_id, n, l, denom, scale, cp.ptr, ri.ptr, va.ptr,
                                       status.ptr, s, lc);
            if (kind == FQB_STD_BERNOULLI) {
                out->centered = 1;
                out->std_scale = 1.0 / std::sqrt(p * (1.0 - p));
            }
        }
        out->col_ptr = static_cast<int*>(std::malloc(sizeof(int) * (size_t(l) + 1)));
        FQB_CUDA(cudaMemcpyAsync(out->col_ptr, cp.ptr, sizeof(int) * (size_t(l) + 1), cudaMemcpyDeviceToHost, s));
        FQB_CUDA(cudaStreamSynchronize(s));
        const int64_t nnz = out->col_ptr[l];
        out->nnz = nnz;
        out->row_idx = static_cast<int*>(std::malloc(sizeof(int) * size_t(std::max<int64_t>(nnz, 1))));
        out->values = static_cast<double*>(std::malloc(sizeof(double) * size_t(std::max<int64_t>(nnz, 1))));
        if (nnz > 0) {
            FQB_CUDA(cudaMemcpyAsync(out->row_idx, ri.ptr, sizeof(int) * nnz, cudaMemcpyDeviceToHost, s));
            FQB_CUDA(cudaMemcpyAsync(out->values, va.ptr, sizeof(double) * nnz, cudaMemcpyDeviceToHost, s));
        }
        unsigned st = 0;
        FQB_CUDA(cudaMemcpyAsync(&st, status.ptr, sizeof(unsigned), cudaMemcpyDeviceToHost, s));
        FQB_CUDA(cudaStreamSynchronize(s));
        if (st & farqb::kGenZeroGaussian)
            throw farqb::Error(FQB_ERR_CONVERGENCE, "a Gaussian draw hit an exact zero");
        return FQB_OK;
    });
}

void fqb_sketch_free(fqb_sketch_host* s) {
    if (!s) return;
    std::free(s->dense);
    std::free(s->col_ptr);
    std::free(s->row_idx);
    std::free(s->values);
    std::memset(s, 0, sizeof *s);
}

fqb_status fqb_sparse_dense_mul(fqb_handle h, const double* a, int64_t m, int64_t n, int64_t lda,
                                const int* col_ptr, const int* row_idx, const double* values, int l,
                                const double* z, double* c, int64_t ldc) {
    return guarded([&]() -> fqb_status {
        bind(h);
        (void)n;
        if (!a || !col_ptr || !c) throw farqb::Error(FQB_ERR_INVALID_ARGUMENT, "null pointer");
        if (lda < m || ldc < m) throw farqb::Error(FQB_ERR_DIMENSION, "leading dimension too small");
        farqb::launch_gather_spmm(a, m, lda, col_ptr, row_idx, values, l, z, c, ldc, h->h.stream, h->h.lc);
        return FQB_OK;
    });
}

fqb_status fqb_centering_column(fqb_handle h, const double* a, int64_t m, int64_t n, int64_t lda, double p,
                                double* z) {
    return guarded([&]() -> fqb_status {
        bind(h);
        if (!a || !z) throw farqb::Error(FQB_ERR_INVALID_ARGUMENT, "null pointer");
        farqb::launch_centering(a, m, n, lda, p, z, h->h.stream, h->h.lc);
        return FQB_OK;
    });
}

fqb_status fqb_frob_norm_sq(fqb_handle h, const double* a, int64_t m, int64_t n, int64_t lda,
                            double* host_out) {
    return guarded([&]() -> fqb_status {
        bind(h);
        if (!a || !host_out) throw farqb::Error(FQB_ERR_INVALID_ARGUMENT, "null pointer");
        cudaStream_t s = h->h.stream;
        farqb::DeviceArray<double> part;
        part.ensure(farqb::kReducePartials + 1, s);
        farqb::launch_sumsq(a, m, n, lda, part.ptr, part.ptr + farqb::kReducePartials, s, h->h.lc);
        FQB_CUDA(cudaMemcpyAsync(host_out, part.ptr + farqb::kReducePartials, sizeof(double),
                                 cudaMemcpyDeviceToHost, s));
        FQB_CUDA(cudaStreamSynchronize(s));
        return FQB_OK;
    });
}

fqb_status fqb_set_fp32_slices(fqb_handle h, int slices) {
    return guarded([&]() -> fqb_status {
        if (!h) throw farqb::Error(FQB_ERR_INVALID_ARGUMENT, "null handle");
        if (slices != 3 && slices != 4 && slices != 8)
            throw farqb::Error(FQB_ERR_INVALID_ARGUMENT, "slices must be 3, 4 or 8");
        h->h.fp32_slices = slices;
        return FQB_OK;
    });
}

int fqb_fp64_slices(void) { return farqb::ozaki_fp64_slices(); }

fqb_status fqb_sym_eig(fqb_handle h, const double* a, int n, int64_t lda, double* w, double* v, int64_t ldv,
                       int* used_small) {
    return guarded([&]() -> fqb_status {
        bind(h);
        if (!a || !w || !v) throw farqb::Error(FQB_ERR_INVALID_ARGUMENT, "null pointer");
        if (n < 0) throw farqb::Error(FQB_ERR_DIMENSION, "negative dimension");
        if (n > 0 && (lda < n || ldv < n)) throw farqb::Error(FQB_ERR_DIMENSION, "leading dimension below n");
        if (used_small) *used_small = 0;
        if (n == 0) return FQB_OK;
        cudaStream_t s = h->h.stream;
        farqb::DeviceArray<double> mat;
        mat.ensure(size_t(n) * n, s);
        FQB_CUDA(cudaMemcpy2DAsync(mat.ptr, sizeof(double) * n, a, sizeof(double) * lda, sizeof(double) * n, n,
                                   cudaMemcpyDeviceToDevice, s));
        const bool small = farqb::eigh_inplace(h->h, mat.ptr, n, w);
        FQB_CUDA(cudaMemcpy2DAsync(v, sizeof(double) * ldv, mat.ptr, sizeof(double) * n, sizeof(double) * n, n,
                                   cudaMemcpyDeviceToDevice, s));
        FQB_CUDA(cudaStreamSynchronize(s));
        if (used_small) *used_small = small ? 1 : 0;
        return FQB_OK;
    });
}

fqb_status fqb_relative_error(fqb_handle h, const double* a, int64_t m, int64_t n, int64_t lda, int a_on_device,
                              const double* u, int64_t ldu, const double* sigma, const double* v, int64_t ldv,
                              int r, int factors_on_device, double* host_out) {
    return guarded([&]() -> fqb_status {
        bind(h);
        if (!a || !host_out) throw farqb::Error(FQB_ERR_INVALID_ARGUMENT, "null pointer");
        if (m < 0 || n < 0 || r < 0) throw farqb::Error(FQB_ERR_DIMENSION, "negative dimension");
        if (lda < m || (r > 0 && (!u || !v || ldu < m || ldv < n)))
            throw farqb::Error(FQB_ERR_DIMENSION, "relative_error: factor shape mismatch");
        *host_out = farqb::relative_error(h->h, a, m, n, lda, a_on_device != 0, u, ldu, sigma, v, ldv, r,
                                          factors_on_device != 0);
        return FQB_OK;
    });
}

fqb_status fqb_chol_factor(fqb_handle h, const double* z, int n, int64_t ldz, double pivot_tol, double diag_ref,
                           double* r, int64_t ldr, double* rinv, int64_t ldri, int* rank_deficient) {
    return guarded([&]() -> fqb_status {
        bind(h);
        if (!z || !r || !rinv) throw farqb::Error(FQB_ERR_INVALID_ARGUMENT, "null pointer");
        if (n < 0) throw farqb::Error(FQB_ERR_DIMENSION, "negative dimension");
        if (n > 1024) throw farqb::Error(FQB_ERR_CONFIG, "fqb_chol_factor: n above 1024");
        if (n > 0 && (ldz < n || ldr < n || ldri < n))
            throw farqb::Error(FQB_ERR_DIMENSION, "leading dimension below n");
        if (rank_deficient) *rank_deficient = 0;
        if (n == 0) return FQB_OK;
        cudaStream_t s = h->h.stream;
        farqb::DeviceArray<double> rr, ri, scratch;
        farqb::DeviceArray<unsigned> st;
        rr.ensure(size_t(n) * n, s);
        ri.ensure(size_t(n) * n, s);
        scratch.ensure(size_t(n) * (n + 1), s);
        st.ensure(1, s);
        FQB_CUDA(cudaMemsetAsync(st.ptr, 0, sizeof(unsigned), s));
        farqb::launch_chol_upper_inv(z, n, ldz, pivot_tol, diag_ref, nullptr, 0, rr.ptr, ri.ptr, nullptr,
                                     scratch.ptr, st.ptr, 1u, s, h->h.lc);
        FQB_CUDA(cudaMemcpy2DAsync(r, sizeof(double) * ldr, rr.ptr, sizeof(double) * n, sizeof(double) * n, n,
                                   cudaMemcpyDeviceToDevice, s));
        FQB_CUDA(cudaMemcpy2DAsync(rinv, sizeof(double) * ldri, ri.ptr, sizeof(double) * n, sizeof(double) * n, n,
                                   cudaMemcpyDeviceToDevice, s));
        unsigned hs = 0;
        FQB_CUDA(cudaMemcpyAsync(&hs, st.ptr, sizeof(unsigned), cudaMemcpyDeviceToHost, s));
        FQB_CUDA(cudaStreamSynchronize(s));
        if (rank_deficient) *rank_deficient = hs ? 1 : 0;
        return FQB_OK;
    });
}

fqb_status fqb_gram(fqb_handle h, const double* y, int64_t k, int b, int64_t ldy, double* s_out, int64_t lds) {
    return guarded([&]() -> fqb_status {
        bind(h);
        if (!y || !s_out) throw farqb::Error(FQB_ERR_INVALID_ARGUMENT, "null pointer");
        if (k < 0 || b < 0) throw farqb::Error(FQB_ERR_DIMENSION, "negative dimension");
        if (b > 0 && (ldy < std::max<int64_t>(k, 1) || lds < b))
            throw farqb::Error(FQB_ERR_DIMENSION, "leading dimension too small");
        if (b == 0) return FQB_OK;
        cudaStream_t s = h->h.stream;
        farqb::ensure_gemm_workspace(h->h);
        if (b <= 128 && k > 0)
            farqb::ts_gram(y, k, b, ldy, 1.0, 0.0, s_out, lds, h->h.gws.work, h->h.gws.work_doubles, h->h.num_sms, s,
                           h->h.lc);
        else
            farqb::gemm(true, b, b, k, 1.0, y, ldy, y, ldy, 0.0, s_out, lds, h->h.gws, h->h.num_sms, s, h->h.lc);
        return FQB_OK;
    });
}

fqb_status fqb_mul_upper(fqb_handle h, const double* y, int64_t m, int b, int64_t ldy, const double* r, int64_t ldr,
                         double* z, int64_t ldz) {
    return guarded([&]() -> fqb_status {
        bind(h);
        if (!y || !r || !z) throw farqb::Error(FQB_ERR_INVALID_ARGUMENT, "null pointer");
        if (m < 0 || b < 0) throw farqb::Error(FQB_ERR_DIMENSION, "negative dimension");
        if (b > 0 && (ldy < std::max<int64_t>(m, 1) || ldz < std::max<int64_t>(m, 1) || ldr < b))
            throw farqb::Error(FQB_ERR_DIMENSION, "leading dimension too small");
        if (b == 0 || m == 0) return FQB_OK;
        cudaStream_t s = h->h.stream;
        if (farqb::ts_trmm(y, m, b, ldy, r, ldr, z, ldz, h->h.num_sms, s, h->h.lc)) return FQB_OK;
        // b > 104: the general GEMM on a copy of R with its strictly lower part zeroed
        farqb::ensure_gemm_workspace(h->h);
        farqb::DeviceArray<double> ru;
        ru.ensure(size_t(b) * b, s);
        FQB_CUDA(cudaMemcpy2DAsync(ru.ptr, sizeof(double) * b, r, sizeof(double) * ldr, sizeof(double) * b, b,
                                   cudaMemcpyDeviceToDevice, s));
        for (int c = 0; c + 1 < b; ++c)
            FQB_CUDA(cudaMemsetAsync(ru.ptr + int64_t(c) * b + c + 1, 0, sizeof(double) * (b - c - 1), s));
        farqb::gemm(false, m, b, b, 1.0, y, ldy, ru.ptr, b, 0.0, z, ldz, h->h.gws, h->h.num_sms, s, h->h.lc);
        return FQB_OK;
    });
}

fqb_status fqb_gemm(fqb_handle h, int trans_a, int64_t m, int64_t n, int64_t k, double alpha,
                    const double* a, int64_t lda, const double* b, int64_t ldb, double beta, double* c,
                    int64_t ldc) {
    return guarded([&]() -> fqb_status {
        bind(h);
        if (m < 0 || n < 0 || k < 0) throw farqb::Error(FQB_ERR_DIMENSION, "negative dimension");
        if (ldc < m || ldb < k || lda < (trans_a ? k : m)) throw farqb::Error(FQB_ERR_DIMENSION, "leading dimension too small");
        cudaStream_t s = h->h.stream;
        farqb::ensure_gemm_workspace(h->h);
        farqb::gemm(trans_a != 0, m, n, k, alpha, a, lda, b, ldb, beta, c, ldc, h->h.gws, h->h.num_sms, s,
                    h->h.lc);
        return FQB_OK;
    });
}

fqb_status fqb_gemm_emulated(fqb_handle h, int trans_a, int64_t m, int64_t n, int64_t k, double alpha,
                             const double* a, int64_t lda, const double* b, int64_t ldb, double beta, double* c,
                             int64_t ldc) {
    return guarded([&]() -> fqb_status {
        bind(h);
        if (m < 0 || n < 0 || k < 0) throw farqb::Error(FQB_ERR_DIMENSION, "negative dimension");
        if (ldc < m || ldb < k || lda < (trans_a ? k : m))
            throw farqb::Error(FQB_ERR_DIMENSION, "leading dimension too small");
        if (m == 0 || n == 0) return FQB_OK;
        if (k == 0) throw farqb::Error(FQB_ERR_DIMENSION, "fqb_gemm_emulated: k = 0");
        cudaStream_t s = h->h.stream;
        farqb::ensure_gemm_workspace(h->h);
        farqb::DeviceArray<int8_t> xs, zs;
        farqb::DeviceArray<int> ex, ez;
        xs.ensure(size_t(farqb::ozaki_x_bytes(m, k)), s);
        zs.ensure(size_t(farqb::ozaki_apply_z_bytes(k)), s);
        ex.ensure(size_t(m), s);
        ez.ensure(size_t(farqb::ozaki_apply_ez_count()), s);
        farqb::DeviceArray<unsigned> line_max, zmax;
        line_max.ensure_zeroed(size_t(farqb::ozaki_line_max_words(m, k)), s);
        zmax.ensure_zeroed(size_t(farqb::ozaki_apply_ez_count()), s);
        if (trans_a) farqb::ozaki_slice_a(a, k, m, lda, line_max.ptr, xs.ptr, ex.ptr, nullptr, nullptr, s, h->h.lc);
        else farqb::ozaki_slice_a(a, m, k, lda, line_max.ptr, nullptr, nullptr, xs.ptr, ex.ptr, s, h->h.lc);
        farqb::ozaki_apply(m, n, k, alpha, xs.ptr, ex.ptr, b, ldb, beta, c, ldc, zs.ptr, ez.ptr, h->h.gws.work,
                           h->h.num_sms, s, h->h.lc, farqb::ozaki_fp64_slices(), zmax.ptr);
        return FQB_OK;   // temporaries are freed stream-ordered, after the kernels
    });
}

}  // extern "C"

struct fqb_sliced_s {
    int64_t m = 0, n = 0;
    farqb::DeviceArray<int8_t> x_nn, x_tn, z;
    farqb::DeviceArray<int> e_nn, e_tn, ez;
    farqb::DeviceArray<unsigned> zmax;
    farqb::DeviceArray<double> cs;   // fqb_sliced_gemm_mn: B with its rows scaled by A's column scales
    int last_trans = -1;   // the last fqb_sliced_gemm: B slices left in z / ez
    int64_t last_nb = 0;
};

extern "C" {

fqb_status fqb_slice_operand(fqb_handle h, const double* a, int64_t m, int64_t n, int64_t lda, fqb_sliced* out) {
    return guarded([&]() -> fqb_status {
        bind(h);
        if (!out) throw farqb::Error(FQB_ERR_INVALID_ARGUMENT, "null output");
        *out = nullptr;
        if (m <= 0 || n <= 0) throw farqb::Error(FQB_ERR_DIMENSION, "fqb_slice_operand: empty operand");
        if (lda < m) throw farqb::Error(FQB_ERR_DIMENSION, "leading dimension too small");
        if (!a) throw farqb::Error(FQB_ERR_INVALID_ARGUMENT, "null operand");
        cudaStream_t s = h->h.stream;
        auto* sl = new fqb_sliced_s();
        try {
            sl->m = m;
            sl->n = n;
            sl->x_nn.ensure(size_t(farqb::ozaki_x_bytes(m, n)), s);
            sl->x_tn.ensure(size_t(farqb::ozaki_x_bytes(n, m)), s);
            sl->e_nn.ensure(size_t(m), s);
            sl->e_tn.ensure(size_t(n), s);
            sl->ez.ensure(size_t(farqb::ozaki_apply_ez_count()), s);
            farqb::DeviceArray<unsigned> line_max;
            line_max.ensure_zeroed(size_t(farqb::ozaki_line_max_words(m, n)), s);
            farqb::ozaki_slice_a(a, m, n, lda, line_max.ptr, sl->x_tn.ptr, sl->e_tn.ptr, sl->x_nn.ptr, sl->e_nn.ptr, s,
                                 h->h.lc);
        } catch (...) {
            delete sl;
            throw;
        }
        *out = sl;
        return FQB_OK;
    });
}

fqb_status fqb_sliced_gemm(fqb_handle h, fqb_sliced sl, int trans_a, int64_t nb, double alpha, const double* b,
                           int64_t ldb, double beta, double* c, int64_t ldc) {
    return guarded([&]() -> fqb_status {
        bind(h);
        if (!sl) throw farqb::Error(FQB_ERR_INVALID_ARGUMENT, "null sliced operand");
        if (nb < 0) throw farqb::Error(FQB_ERR_DIMENSION, "fqb_sliced_gemm: negative nb");
        const int64_t M = trans_a ? sl->n : sl->m, K = trans_a ? sl->m : sl->n;
        if (ldb < K || ldc < M) throw farqb::Error(FQB_ERR_DIMENSION, "leading dimension too small");
        if (nb == 0) return FQB_OK;
        cudaStream_t s = h->h.stream;
        farqb::ensure_gemm_workspace(h->h);
        sl->z.ensure(size_t(farqb::ozaki_apply_z_bytes(K)), s);
        sl->zmax.ensure_zeroed(size_t(farqb::ozaki_apply_ez_count()), s);
        farqb::ozaki_apply(M, nb, K, alpha, trans_a ? sl->x_tn.ptr : sl->x_nn.ptr,
                           trans_a ? sl->e_tn.ptr : sl->e_nn.ptr, b, ldb, beta, c, ldc, sl->z.ptr, sl->ez.ptr,
                           h->h.gws.work, h->h.num_sms, s, h->h.lc, farqb::ozaki_fp64_slices(), sl->zmax.ptr);
        sl->last_trans = trans_a ? 1 : 0;
        sl->last_nb = nb;
        return FQB_OK;
    });
}

fqb_status fqb_sliced_gemm_mn(fqb_handle h, fqb_sliced sl, int64_t nb, double alpha, const double* b, int64_t ldb,
                              double beta, double* c, int64_t ldc) {
    return guarded([&]() -> fqb_status {
        bind(h);
        if (!sl) throw farqb::Error(FQB_ERR_INVALID_ARGUMENT, "null sliced operand");
        if (nb < 0) throw farqb::Error(FQB_ERR_DIMENSION, "fqb_sliced_gemm_mn: negative nb");
        const int64_t M = sl->m, K = sl->n;
        if (ldb < K || ldc < M) throw farqb::Error(FQB_ERR_DIMENSION, "leading dimension too small");
        if (nb == 0) return FQB_OK;
        cudaStream_t s = h->h.stream;
        farqb::ensure_gemm_workspace(h->h);
        sl->z.ensure(size_t(farqb::ozaki_apply_z_bytes(K)), s);
        sl->zmax.ensure_zeroed(size_t(farqb::ozaki_apply_ez_count()), s);
        sl->cs.ensure(size_t(K) * size_t(nb), s);
        farqb::ozaki_apply_mn(M, nb, K, alpha, sl->x_tn.ptr, sl->e_tn.ptr, b, ldb, beta, c, ldc, sl->cs.ptr,
                              sl->z.ptr, sl->ez.ptr, h->h.gws.work, h->h.num_sms, s, h->h.lc,
                              farqb::ozaki_fp64_slices(), sl->zmax.ptr);
        sl->last_trans = -1;   // z holds the scaled B's slices: no fqb_sliced_gemm_again after this
        return FQB_OK;
    });
}

fqb_status fqb_sliced_gemm_again(fqb_handle h, fqb_sliced sl, double alpha, double beta, double* c, int64_t ldc) {
    return guarded([&]() -> fqb_status {
        bind(h);
        if (!sl) throw farqb::Error(FQB_ERR_INVALID_ARGUMENT, "null sliced operand");
        if (sl->last_trans < 0) throw farqb::Error(FQB_ERR_INVALID_ARGUMENT, "no previous fqb_sliced_gemm");
        if (sl->last_nb > 128) throw farqb::Error(FQB_ERR_INVALID_ARGUMENT, "previous product wider than 128");
        const bool ta = sl->last_trans == 1;
        const int64_t M = ta ? sl->n : sl->m, K = ta ? sl->m : sl->n;
        if (ldc < M) throw farqb::Error(FQB_ERR_DIMENSION, "leading dimension too small");
        farqb::ensure_gemm_workspace(h->h);
        farqb::ozaki_apply_presliced(M, sl->last_nb, K, alpha, ta ? sl->x_tn.ptr : sl->x_nn.ptr,
                                     ta ? sl->e_tn.ptr : sl->e_nn.ptr, beta, c, ldc, sl->z.ptr, sl->ez.ptr,
                                     h->h.gws.work, h->h.num_sms, h->h.stream, h->h.lc);
        return FQB_OK;
    });
}

fqb_status fqb_sliced_free(fqb_handle h, fqb_sliced sl) {
    return guarded([&]() -> fqb_status {
        if (!sl) return FQB_OK;
        bind(h);
        delete sl;   // device memory returns to the pool, ordered after the handle's queued work
        return FQB_OK;
    });
}

fqb_status fqb_random_orthonormal(fqb_handle h, int64_t n, int r, uint64_t seed, uint32_t stream, double* q,
                                  int64_t ldq) {
    return guarded([&]() -> fqb_status {
        bind(h);
        if (!q) throw farqb::Error(FQB_ERR_INVALID_ARGUMENT, "null output");
        if (ldq < n) throw farqb::Error(FQB_ERR_DIMENSION, "ldq < n");
        farqb::random_orthonormal_dev(h->h, n, r, seed, stream, 0, q, ldq);
        return FQB_OK;
    });
}

fqb_status fqb_gen_synthetic(fqb_handle h, int kind, int n, int d, uint64_t seed, double* a, int64_t lda,
                             int* rank_out) {
    return guarded([&]() -> fqb_status {
        bind(h);
        if (!a) throw farqb::Error(FQB_ERR_INVALID_ARGUMENT, "null output");
        const int r = farqb::gen_synthetic_dev(h->h, kind, n, d, seed, a, lda);
        if (rank_out) *rank_out = r;
        return FQB_OK;
    });
}

fqb_status fqb_gen_lowrank(fqb_handle h, int64_t m, int64_t n, int r, const double* sigma, uint64_t seed,
                           double noise, double* a, int64_t lda) {
    return guarded([&]() -> fqb_status {
        bind(h);
        if (!a || !sigma) throw farqb::Error(FQB_ERR_INVALID_ARGUMENT, "null pointer");
        farqb::gen_lowrank_dev(h->h, m, n, r, sigma, seed, noise, a, lda);
        return FQB_OK;
    });
}

fqb_status fqb_gen_lowrank_det(fqb_handle h, int64_t m, int64_t n, int r, const double* sigma, uint64_t seed,
                               double noise_scale, int64_t row0, int64_t rows, double* a, int64_t lda) {
    return guarded([&]() -> fqb_status {
        bind(h);
        if (!a || !sigma) throw farqb::Error(FQB_ERR_INVALID_ARGUMENT, "null pointer");
        farqb::gen_lowrank_det_dev(h->h, m, n, r, sigma, seed, noise_scale, row0, rows, a, lda);
        return FQB_OK;
    });
}

fqb_status fqb_checksum(fqb_handle h, const double* a, int64_t rows, int64_t cols, int64_t lda, int64_t row0,
                        int64_t m_total, uint64_t* out) {
    return guarded([&]() -> fqb_status {
        bind(h);
        if (!out || (!a && rows > 0 && cols > 0)) throw farqb::Error(FQB_ERR_INVALID_ARGUMENT, "null pointer");
        if (rows < 0 || cols < 0 || lda < rows || row0 < 0 || row0 + rows > m_total)
            throw farqb::Error(FQB_ERR_INVALID_ARGUMENT, "fqb_checksum: bad extents");
        *out = farqb::checksum_dev(h->h, a, rows, cols, lda, row0, m_total);
        return FQB_OK;
    });
}

fqb_status fqb_raw_header(const char* path, int64_t* rows, int64_t* cols, int64_t* err_offset) {
    if (err_offset) *err_offset = -1;
    try {
        if (!path || !rows || !cols) throw farqb::Error(FQB_ERR_INVALID_ARGUMENT, "null argument");
        farqb::raw_header(path, rows, cols);
        return FQB_OK;
    } catch (const farqb::FormatFailure& e) {
        if (err_offset) *err_offset = e.offset;
        return set_error(e.status, e.what());
    } catch (const farqb::Error& e) {
        return set_error(e.status, e.what());
    } catch (const std::exception& e) {
        return set_error(FQB_ERR_INVALID_ARGUMENT, e.what());
    }
}

fqb_status fqb_load_raw_rows(fqb_handle h, const char* path, int64_t row0, int64_t rows, double* dst, int64_t ld,
                             int dst_on_device, int64_t* err_offset) {
    if (err_offset) *err_offset = -1;
    try {
        if (!path || (!dst && rows > 0)) throw farqb::Error(FQB_ERR_INVALID_ARGUMENT, "null argument");
        if (dst_on_device) bind(h);
        farqb::load_raw_rows(h ? &h->h : nullptr, path, row0, rows, dst, ld, dst_on_device != 0);
        return FQB_OK;
    } catch (const farqb::FormatFailure& e) {
        if (err_offset) *err_offset = e.offset;
        return set_error(e.status, e.what());
    } catch (const farqb::Error& e) {
        return set_error(e.status, e.what());
    } catch (const std::exception& e) {
        return set_error(FQB_ERR_INVALID_ARGUMENT, e.what());
    }
}

double fqb_default_density(int kind, int64_t n) { return farqb::default_density(kind, n); }
int fqb_default_block(int64_t m, int64_t n) { return farqb::default_block(m, n); }
int fqb_default_max_iters(int64_t n, int b) { return farqb::default_max_iters(n, b); }

}  // extern "C"
