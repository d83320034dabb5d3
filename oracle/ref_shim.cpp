// ref_shim.cpp -- extern "C" face of the UNMODIFIED reference library.
//
// TEST INFRASTRUCTURE ONLY.  oracle/Makefile compiles this file together with
// the reference's own sources where they lie (/root/reference/proj/src) into
// oracle/_ref/librsvd_ref.so.  It exposes the same ABI as the C restatement
// (farqb_oracle.h, prefix ref_ instead of fqo_) so tests can pin the
// restatement against the reference and bench.py --impl reference can time the
// reference's own run_fixed_precision on the box's host cores.
//
// Nothing here re-implements reference logic except the block loop of
// run_fixed_precision / run_fixed_rank (driver.cpp:134-160, 347-413), which
// is re-driven through the reference's public granular API (make_state,
// centering_column, power_iterate_block, accept_block, assemble_svd) solely
// to record the residual after every accepted block.
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <exception>
#include <string>
#include <vector>

#include "rsvd/driver.hpp"
#include "rsvd/errors.hpp"
#include "rsvd/experiment.hpp"
#include "rsvd/matrix_io.hpp"
#include "rsvd/matrix_core.hpp"
#include "rsvd/rng.hpp"
#include "rsvd/sketch.hpp"
#include "rsvd/synthetic.hpp"

extern "C" {
#include "farqb_oracle.h"
}

using namespace rsvd;

namespace {

void set_msg(fqo_result* out, const std::string& m) {
    std::snprintf(out->message, sizeof out->message, "%s", m.c_str());
}

template <typename T>
T* copy_out(const T* src, std::size_t count) {
    T* p = static_cast<T*>(std::calloc(count ? count : 1, sizeof(T)));
    if (count) std::memcpy(p, src, count * sizeof(T));
    return p;
}

SketchBlock to_block(const fqo_block& b) {
    SketchBlock out;
    out.is_dense = b.is_dense != 0;
    out.centered = b.centered != 0;
    out.p = b.p;
    out.std_scale = b.std_scale;
    if (out.is_dense) {
        out.dense = DenseMatrix(b.rows, b.cols);
        std::memcpy(out.dense.data.data(), b.dense, sizeof(double) * std::size_t(b.rows) * b.cols);
    } else {
        out.sparse.rows = b.rows;
        out.sparse.cols = b.cols;
        out.sparse.col_ptr.assign(b.col_ptr, b.col_ptr + b.cols + 1);
        out.sparse.row_idx.assign(b.row_idx, b.row_idx + b.nnz);
        out.sparse.values.assign(b.values, b.values + b.nnz);
    }
    return out;
}

struct CallbackSource final : BlockSource {
    fqo_source_fn fn;
    void* user;
    fqo_result* out;
    SketchSpec spec;
    SketchBlock next(int n, int b, int block_id) override {
        out->block_ids = static_cast<int*>(std::realloc(out->block_ids, sizeof(int) * (out->n_ids + 1)));
        out->block_ids[out->n_ids++] = block_id;
        if (!fn) return gen_sketch(spec, n, b, block_id);
        fqo_block blk;
        std::memset(&blk, 0, sizeof blk);
        if (fn(user, n, b, block_id, &blk) != 0) throw std::runtime_error("block source failed");
        return to_block(blk);
    }
};

FarpcaConfig to_cfg(const fqo_config& c) {
    FarpcaConfig cfg;
    cfg.eps = c.eps;
    cfg.power = c.power;
    cfg.block = c.block;
    cfg.sketch.kind = static_cast<SketchKind>(c.kind);
    cfg.sketch.p = c.p;
    cfg.sketch.seed = c.seed;
    cfg.max_iters = c.max_iters;
    cfg.shift_convention = c.shift_convention ? ShiftConvention::FirstDiagonal : ShiftConvention::LastDiagonal;
    cfg.relative = c.relative != 0;
    return cfg;
}

// Mirror of the reference's private resolve() (driver.cpp:116-132) so the block
// loop below uses the same resolved parameters.
FarpcaConfig resolve_like_ref(int m, int n, FarpcaConfig cfg, bool fixed_precision) {
    if (m < 1 || n < 1) throw ConfigError("matrix must be non-empty");
    if (cfg.block == 0) cfg.block = default_block(m, n);
    if (cfg.block < 1) throw ConfigError("block size must be at least 1");
    if (cfg.block > std::min(m, n)) throw ConfigError("block size exceeds matrix dimensions");
    if (cfg.max_iters == 0) cfg.max_iters = default_max_iters(n, cfg.block);
    if (cfg.max_iters < 1) throw ConfigError("max_iters must be at least 1");
    if (cfg.power < 0) throw ConfigError("power must be non-negative");
    if (cfg.sketch.kind != SketchKind::Gaussian && cfg.sketch.p == 0.0)
        cfg.sketch.p = default_density(cfg.sketch.kind, n);
    if (fixed_precision && !(cfg.eps > 0.0))
        throw ConfigError("fixed-precision mode needs a positive tolerance");
    return cfg;
}

void process_block_like_ref(FactorState& st, const DenseMatrix& a, const FarpcaConfig& cfg,
                            BlockSource& src, const std::vector<double>& zc, int index) {
    for (int attempt = 0;; ++attempt) {
        try {
            SketchBlock raw = src.next(a.cols, cfg.block, index + 1000 * attempt);
            if (cfg.power >= 1) {
                DenseMatrix gd = power_iterate_block(st, a, raw, cfg.power, cfg.shift_convention, zc);
                SketchBlock it;
                it.is_dense = true;
                it.dense = std::move(gd);
                accept_block(st, a, it, zc);
            } else {
                st.alpha = 0.0;
                accept_block(st, a, raw, zc);
            }
            return;
        } catch (const BlockDegenerate&) {
            if (attempt >= 3) throw;
        }
    }
}

void fill_svd(const ApproxSvd& svd, int want_vectors, fqo_result* out) {
    out->rank = svd.rank();
    out->blocks = svd.blocks;
    out->converged = svd.converged;
    out->residual_sq = svd.residual_sq;
    out->norm_a_sq = svd.norm_a_sq;
    out->sigma = copy_out(svd.sigma.data(), svd.sigma.size());
    if (want_vectors) {
        out->u = copy_out(svd.u.data.data(), svd.u.data.size());
        out->v = copy_out(svd.v.data.data(), svd.v.data.size());
    }
}

int run(const double* a_ptr, int m, int n, int rank, bool fixed_precision, const fqo_config* c,
        fqo_source_fn fn, void* user, int want_vectors, fqo_result* out, bool granular) {
    std::memset(out, 0, sizeof *out);
    out->m = m;
    out->n = n;
    std::vector<double> residuals;
    try {
        DenseMatrix a(m, n);
        std::memcpy(a.data.data(), a_ptr, sizeof(double) * std::size_t(m) * n);
        FarpcaConfig cfg0 = to_cfg(*c);
        CallbackSource src;
        src.fn = fn;
        src.user = user;
        src.out = out;
        if (!granular) {
            // The reference's own entry points, untouched.
            FarpcaConfig r = resolve_like_ref(m, n, cfg0, fixed_precision);
            src.spec = r.sketch;
            out->resolved_block = r.block;
            out->resolved_max_iters = r.max_iters;
            out->resolved_p = r.sketch.p;
            ApproxSvd svd = fixed_precision ? run_fixed_precision(a, cfg0, &src)
                                            : run_fixed_rank(a, rank, cfg0, &src);
            fill_svd(svd, want_vectors, out);
            return out->status = FQO_OK;
        }
        FarpcaConfig cfg = resolve_like_ref(m, n, cfg0, fixed_precision);
        src.spec = cfg.sketch;
        out->resolved_block = cfg.block;
        out->resolved_max_iters = cfg.max_iters;
        out->resolved_p = cfg.sketch.p;
        if (!fixed_precision) {
            if (rank < 1) throw ConfigError("rank must be at least 1");
            if (rank > std::min(m, n)) throw ConfigError("rank exceeds matrix dimensions");
        }
        FactorState st = make_state(a, cfg.block);
        std::vector<double> zc;
        if (cfg.sketch.kind == SketchKind::StdBernoulli) zc = centering_column(a, cfg.sketch.p);
        bool converged = false;
        if (fixed_precision) {
            double norm_a = std::sqrt(st.norm_a_sq);
            double eps_abs = cfg.relative ? cfg.eps * norm_a : cfg.eps;
            double eps_sq = eps_abs * eps_abs;
            if (st.residual() <= eps_sq) converged = true;
            for (int j = 0; !converged && j < cfg.max_iters; ++j) {
                process_block_like_ref(st, a, cfg, src, zc, j);
                residuals.push_back(st.residual());
                if (st.residual() < eps_sq) converged = true;
            }
        } else {
            int nblocks = (rank + cfg.block - 1) / cfg.block;
            for (int j = 0; j < nblocks; ++j) {
                process_block_like_ref(st, a, cfg, src, zc, j);
                residuals.push_back(st.residual());
            }
            converged = true;
        }
        ApproxSvd svd = assemble_svd(st);
        svd.converged = converged;
        if (!fixed_precision) {
            // The reference's private drop_smallest (driver.cpp:85-106, 406-411):
            // the rank overshoot leaves the small end, its energy returns to E.
            int extra = ((rank + cfg.block - 1) / cfg.block) * cfg.block - rank;
            for (int i = 0; i < extra; ++i) svd.residual_sq += svd.sigma[i] * svd.sigma[i];
            svd.sigma.erase(svd.sigma.begin(), svd.sigma.begin() + extra);
            auto drop_cols = [extra](DenseMatrix& mtx) {
                if (mtx.cols <= extra) return;
                DenseMatrix r(mtx.rows, mtx.cols - extra);
                std::memcpy(r.data.data(), mtx.col(extra), sizeof(double) * r.data.size());
                mtx = std::move(r);
            };
            drop_cols(svd.u);
            drop_cols(svd.v);
        }
        fill_svd(svd, want_vectors, out);
        out->block_residuals = copy_out(residuals.data(), residuals.size());
        out->status = converged ? FQO_OK : FQO_ERR_TOLERANCE_NOT_REACHED;
        if (!converged) set_msg(out, "tolerance not reached");
        return out->status;
    } catch (const ToleranceNotReached& e) {
        fill_svd(e.partial, want_vectors, out);
        set_msg(out, e.what());
        return out->status = FQO_ERR_TOLERANCE_NOT_REACHED;
    } catch (const BlockDegenerate& e) {
        out->blocks = e.blocks_accepted;
        out->residual_sq = e.residual_sq;
        out->norm_a_sq = e.norm_a_sq;
        out->block_residuals = copy_out(residuals.data(), residuals.size());
        set_msg(out, e.what());
        return out->status = FQO_ERR_BLOCK_DEGENERATE;
    } catch (const ConfigError& e) {
        set_msg(out, e.what());
        return out->status = FQO_ERR_CONFIG;
    } catch (const DimensionError& e) {
        set_msg(out, e.what());
        return out->status = FQO_ERR_DIMENSION;
    } catch (const ConvergenceFailure& e) {
        set_msg(out, e.what());
        return out->status = FQO_ERR_CONVERGENCE;
    } catch (const std::exception& e) {
        set_msg(out, e.what());
        return out->status = FQO_ERR_CALLBACK;
    }
}

}  // namespace

extern "C" {

void ref_philox_u32(uint64_t seed, uint32_t block_id, uint32_t column, int count, uint32_t* out) {
    Philox r(seed, block_id, column);
    for (int i = 0; i < count; ++i) out[i] = r.next_u32();
}

void ref_philox_units(uint64_t seed, uint32_t block_id, uint32_t column, int count, double* out) {
    Philox r(seed, block_id, column);
    for (int i = 0; i < count; ++i) out[i] = r.next_unit();
}

void ref_philox_gaussians(uint64_t seed, uint32_t block_id, uint32_t column, int count, double* out) {
    Philox r(seed, block_id, column);
    for (int i = 0; i < count; ++i) out[i] = r.next_gaussian();
}

// The reference generator has no fixed-zeta mode, so zeta must be 0.
int ref_gen_sketch(int kind, double p, uint64_t seed, int zeta, int n, int l, int block_id,
                   fqo_block* out) {
    std::memset(out, 0, sizeof *out);
    if (zeta != 0) return FQO_ERR_CONFIG;
    try {
        SketchSpec spec;
        spec.kind = static_cast<SketchKind>(kind);
        spec.p = p;
        spec.seed = seed;
        SketchBlock blk = gen_sketch(spec, n, l, block_id);
        out->is_dense = blk.is_dense;
        out->rows = n;
        out->cols = l;
        out->centered = blk.centered;
        out->p = blk.p;
        out->std_scale = blk.std_scale;
        if (blk.is_dense) {
            out->dense = copy_out(blk.dense.data.data(), blk.dense.data.size());
        } else {
            out->col_ptr = copy_out(blk.sparse.col_ptr.data(), blk.sparse.col_ptr.size());
            out->row_idx = copy_out(blk.sparse.row_idx.data(), blk.sparse.row_idx.size());
            out->values = copy_out(blk.sparse.values.data(), blk.sparse.values.size());
            out->nnz = int64_t(blk.sparse.nnz());
        }
        return FQO_OK;
    } catch (const ConfigError&) {
        return FQO_ERR_CONFIG;
    }
}

void ref_block_free(fqo_block* blk) {
    std::free(blk->dense);
    std::free(blk->col_ptr);
    std::free(blk->row_idx);
    std::free(blk->values);
    std::memset(blk, 0, sizeof *blk);
}

void ref_sparse_dense_mul(const double* a, int m, int n, const int* col_ptr, const int* row_idx,
                          const double* values, int l, double* c) {
    DenseMatrix am(m, n);
    std::memcpy(am.data.data(), a, sizeof(double) * std::size_t(m) * n);
    SparseSketch s;
    s.rows = n;
    s.cols = l;
    s.col_ptr.assign(col_ptr, col_ptr + l + 1);
    s.row_idx.assign(row_idx, row_idx + col_ptr[l]);
    s.values.assign(values, values + col_ptr[l]);
    DenseMatrix r = sparse_dense_mul(am, s);
    std::memcpy(c, r.data.data(), sizeof(double) * r.data.size());
}

void ref_centering_column(const double* a, int m, int n, double p, double* z) {
    DenseMatrix am(m, n);
    std::memcpy(am.data.data(), a, sizeof(double) * std::size_t(m) * n);
    std::vector<double> v = centering_column(am, p);
    std::memcpy(z, v.data(), sizeof(double) * v.size());
}

int ref_run_fixed_precision(const double* a, int m, int n, const fqo_config* cfg, fqo_source_fn src,
                            void* user, int want_vectors, fqo_result* out) {
    return run(a, m, n, 0, true, cfg, src, user, want_vectors, out, false);
}

int ref_run_fixed_rank(const double* a, int m, int n, int rank, const fqo_config* cfg,
                       fqo_source_fn src, void* user, int want_vectors, fqo_result* out) {
    return run(a, m, n, rank, false, cfg, src, user, want_vectors, out, false);
}

// Same loop driven through the granular public API so the per-block residual
// trace is recorded (block_residuals).  Numerically identical to the above.
int ref_run_traced(const double* a, int m, int n, int rank, int fixed_precision, const fqo_config* cfg,
                   fqo_source_fn src, void* user, int want_vectors, fqo_result* out) {
    return run(a, m, n, rank, fixed_precision != 0, cfg, src, user, want_vectors, out, true);
}

void ref_result_free(fqo_result* r) {
    std::free(r->sigma);
    std::free(r->u);
    std::free(r->v);
    std::free(r->block_residuals);
    std::free(r->block_ids);
    r->sigma = r->u = r->v = r->block_residuals = nullptr;
    r->block_ids = nullptr;
}

// gen_synthetic (synthetic.cpp:159-180): square n x n, column-major into out.
int ref_gen_synthetic(int kind, int n, uint64_t seed, double* out) {
    try {
        SyntheticSpec spec;
        spec.kind = static_cast<SyntheticKind>(kind);
        spec.n = n;
        spec.seed = seed;
        DenseMatrix a = gen_synthetic(spec, std::size_t(1) << 40);
        std::memcpy(out, a.data.data(), sizeof(double) * a.data.size());
        return FQO_OK;
    } catch (const std::exception&) {
        return FQO_ERR_CONFIG;
    }
}

int ref_random_orthonormal(int n, int r, uint64_t seed, uint32_t stream, double* out) {
    try {
        DenseMatrix q = random_orthonormal(n, r, seed, stream);
        std::memcpy(out, q.data.data(), sizeof(double) * q.data.size());
        return FQO_OK;
    } catch (const std::exception&) {
        return FQO_ERR_CONFIG;
    }
}

// ---- matrix files and the experiment driver (callers of the path) -----------
// Status: 0 ok, 1 FormatError (offset set), 2 ConfigError, 3 DimensionError,
// 4 other; message into err.

static int io_status(const std::exception& e, char* err, int errlen, long long* offset) {
    if (err && errlen > 0) std::snprintf(err, size_t(errlen), "%s", e.what());
    if (auto* f = dynamic_cast<const FormatError*>(&e)) {
        if (offset) *offset = (long long)f->byte_offset;
        return 1;
    }
    if (dynamic_cast<const ConfigError*>(&e)) return 2;
    if (dynamic_cast<const DimensionError*>(&e)) return 3;
    return 4;
}

// load_matrix (matrix_io.cpp); *data is malloc'ed (free with ref_free).
int ref_load_matrix(const char* path, const char* format, int* rows, int* cols, double** data, char* err,
                    int errlen, long long* offset) {
    try {
        DenseMatrix a = load_matrix(path, matrix_format_from_name(format));
        *rows = a.rows;
        *cols = a.cols;
        *data = static_cast<double*>(std::malloc(sizeof(double) * (a.data.size() ? a.data.size() : 1)));
        if (!a.data.empty()) std::memcpy(*data, a.data.data(), sizeof(double) * a.data.size());
        return 0;
    } catch (const std::exception& e) {
        return io_status(e, err, errlen, offset);
    }
}

int ref_save_matrix(const double* data, int rows, int cols, const char* path, const char* format, char* err,
                    int errlen) {
    try {
        DenseMatrix a(rows, cols);
        if (!a.data.empty()) std::memcpy(a.data.data(), data, sizeof(double) * a.data.size());
        save_matrix(a, path, matrix_format_from_name(format));
        return 0;
    } catch (const std::exception& e) {
        return io_status(e, err, errlen, nullptr);
    }
}

void ref_free(void* p) { std::free(p); }

// load_experiment_config + run_experiment (experiment.cpp): the reference's own
// experiment grid on this host, files under the config's out_prefix.
int ref_run_experiment(const char* config_path, char* err, int errlen) {
    try {
        run_experiment(load_experiment_config(config_path));
        return 0;
    } catch (const std::exception& e) {
        return io_status(e, err, errlen, nullptr);
    }
}

// load_experiment_config alone (validation errors)
int ref_check_experiment_config(const char* config_path, char* err, int errlen) {
    try {
        load_experiment_config(config_path);
        return 0;
    } catch (const std::exception& e) {
        return io_status(e, err, errlen, nullptr);
    }
}

// read_report_csv: record count (>= 0) or -status
int ref_read_report_csv(const char* path, char* err, int errlen, long long* offset) {
    try {
        return int(read_report_csv(path).size());
    } catch (const std::exception& e) {
        return -io_status(e, err, errlen, offset);
    }
}

}  // extern "C"
