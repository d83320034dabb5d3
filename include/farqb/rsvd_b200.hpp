// rsvd_b200.hpp -- header-only C++ drop-in for the reference's QB API, backed by
// libfarqb.so (the sm_100a engine) through the C-ABI in include/farqb.h.
//
// Mirrors /root/reference/proj/include/rsvd/{driver,sketch,dense_matrix,errors}.hpp:
//
//   rsvd::DenseMatrix              -> rsvd_b200::DenseMatrix (same fields and layout)
//   rsvd::SketchKind / SketchSpec  -> rsvd_b200::SketchKind / SketchSpec (+ zeta)
//   rsvd::FarpcaConfig             -> rsvd_b200::FarpcaConfig (same fields)
//   rsvd::BlockSource::next        -> rsvd_b200::BlockSource::next (same signature)
//   rsvd::run_fixed_precision      -> rsvd_b200::run_fixed_precision  -> QbResult
//   rsvd::run_fixed_rank           -> rsvd_b200::run_fixed_rank       -> QbResult
//   rsvd::gen_sketch               -> rsvd_b200::gen_sketch (generated on the device)
//   ConfigError, DimensionError, BlockDegenerate, ToleranceNotReached
//   (with .partial), ConvergenceFailure  -> same names, same base classes
//
// run_* accept any matrix type with `rows`, `cols` and a contiguous column-major
// `data` vector, so an existing rsvd::DenseMatrix can be passed unchanged.
// The result is the north-star QB output: Q (m x l, orthonormal), B' (n x l),
// rank l, block count and the error indicator E = ||A||_F^2 - sum ||B_j||_F^2.
#pragma once

#include <algorithm>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <stdexcept>
#include <string>
#include <type_traits>
#include <utility>
#include <vector>

#include "../farqb.h"

namespace rsvd_b200 {

struct DenseMatrix {
    int rows = 0;
    int cols = 0;
    std::vector<double> data;  // column-major
    DenseMatrix() = default;
    DenseMatrix(int r, int c) : rows(r), cols(c), data(std::size_t(r) * c, 0.0) {}
    double& operator()(int i, int j) { return data[std::size_t(j) * rows + i]; }
    double operator()(int i, int j) const { return data[std::size_t(j) * rows + i]; }
    double* col(int j) { return data.data() + std::size_t(j) * rows; }
    const double* col(int j) const { return data.data() + std::size_t(j) * rows; }
};

// FP32 input (BASELINE config 5): same layout as DenseMatrix with float storage.
// Engine::run_* on a FloatMatrix takes the FP32 input mode (A stays FP32 on the
// device, every product is formed in FP64).
struct FloatMatrix {
    int rows = 0;
    int cols = 0;
    std::vector<float> data;  // column-major
    FloatMatrix() = default;
    FloatMatrix(int r, int c) : rows(r), cols(c), data(std::size_t(r) * c, 0.0f) {}
    float& operator()(int i, int j) { return data[std::size_t(j) * rows + i]; }
    float operator()(int i, int j) const { return data[std::size_t(j) * rows + i]; }
};

enum class SketchKind { Gaussian = FQB_GAUSSIAN, Bernoulli = FQB_BERNOULLI, StdBernoulli = FQB_STD_BERNOULLI,
                        SparseSign = FQB_SPARSE_SIGN, SparseGaussian = FQB_SPARSE_GAUSSIAN };
enum class ShiftConvention { LastDiagonal = 0, FirstDiagonal = 1 };

struct SketchSpec {
    SketchKind kind = SketchKind::Gaussian;
    double p = 0.0;
    std::uint64_t seed = 0;
    int zeta = 0;  // > 0: exactly zeta nonzeros per column (sparse sign / Gaussian)
};

struct FarpcaConfig {
    double eps = 0.0;
    int power = 0;
    int block = 0;
    SketchSpec sketch;
    int max_iters = 0;
    ShiftConvention shift_convention = ShiftConvention::LastDiagonal;
    bool relative = false;
};

struct SparseSketch {
    int rows = 0, cols = 0;
    std::vector<int> col_ptr, row_idx;
    std::vector<double> values;
    std::size_t nnz() const { return row_idx.size(); }
};

struct SketchBlock {
    bool is_dense = false;
    DenseMatrix dense;
    SparseSketch sparse;
    bool centered = false;
    double p = 0.0;
    double std_scale = 0.0;
};

class BlockSource {
  public:
    virtual ~BlockSource() = default;
    virtual SketchBlock next(int n, int b, int block_id) = 0;
};

// QB factors plus the reference's ApproxSvd fields (driver.hpp:45-58).
struct QbResult {
    DenseMatrix q;   // m x rank
    DenseMatrix bt;  // n x rank  (B = bt')
    int rank = 0;    // QB rank l = blocks * b
    int blocks = 0;
    bool converged = false;
    double residual_sq = 0.0;  // ApproxSvd::residual_sq (includes a fixed-rank drop)
    double norm_a_sq = 0.0;
    DenseMatrix u;                 // m x r
    std::vector<double> sigma;     // ascending
    DenseMatrix v;                 // n x r
    std::vector<char> v_flagged;
    double qb_residual_sq = 0.0;   // E of the QB factors themselves
    std::vector<double> block_residuals;
    std::vector<int> block_ids;
    double device_ms = 0.0;
    int svd_rank() const { return int(sigma.size()); }
};

// ---- exceptions (errors.hpp:9-46, driver.hpp:60-65) -------------------------
struct DimensionError : std::invalid_argument { using std::invalid_argument::invalid_argument; };
struct ConfigError : std::invalid_argument { using std::invalid_argument::invalid_argument; };
struct ConvergenceFailure : std::runtime_error { using std::runtime_error::runtime_error; };
struct CudaError : std::runtime_error { using std::runtime_error::runtime_error; };
struct BlockDegenerate : std::runtime_error {
    BlockDegenerate(std::string msg, int blocks, double res, double na)
        : std::runtime_error(std::move(msg)), blocks_accepted(blocks), residual_sq(res), norm_a_sq(na) {}
    int blocks_accepted;
    double residual_sq;
    double norm_a_sq;
};
class ToleranceNotReached : public std::runtime_error {
  public:
    QbResult partial;
    ToleranceNotReached(std::string msg, QbResult p) : std::runtime_error(std::move(msg)), partial(std::move(p)) {}
};

namespace detail {

[[noreturn]] inline void raise(int status, const char* where) {
    std::string msg = std::string(where) + ": " + fqb_last_error();
    switch (status) {
        case FQB_ERR_CONFIG: throw ConfigError(msg);
        case FQB_ERR_DIMENSION: throw DimensionError(msg);
        case FQB_ERR_CONVERGENCE: throw ConvergenceFailure(msg);
        case FQB_ERR_CUDA: throw CudaError(msg);
        default: throw std::runtime_error(msg);
    }
}

inline fqb_config to_c(const FarpcaConfig& c) {
    fqb_config r{};
    r.eps = c.eps;
    r.power = c.power;
    r.block = c.block;
    r.sketch.kind = static_cast<int>(c.sketch.kind);
    r.sketch.p = c.sketch.p;
    r.sketch.seed = c.sketch.seed;
    r.sketch.zeta = c.sketch.zeta;
    r.max_iters = c.max_iters;
    r.shift_convention = static_cast<int>(c.shift_convention);
    r.relative = c.relative ? 1 : 0;
    return r;
}

struct SourceCtx {
    BlockSource* src;
    SketchBlock current;  // keeps the arrays alive until the next call
    std::exception_ptr error;
};

inline int source_trampoline(void* user, int n, int b, int block_id, fqb_block* out) {
    auto* ctx = static_cast<SourceCtx*>(user);
    try {
        ctx->current = ctx->src->next(n, b, block_id);
        const SketchBlock& s = ctx->current;
        *out = fqb_block{};
        out->is_dense = s.is_dense ? 1 : 0;
        out->rows = n;
        out->cols = b;
        out->centered = s.centered ? 1 : 0;
        out->p = s.p;
        out->std_scale = s.std_scale;
        if (s.is_dense) {
            out->rows = s.dense.rows;
            out->cols = s.dense.cols;
            out->dense = s.dense.data.data();
        } else {
            out->rows = s.sparse.rows;
            out->cols = s.sparse.cols;
            out->col_ptr = s.sparse.col_ptr.data();
            out->row_idx = s.sparse.row_idx.data();
            out->values = s.sparse.values.data();
            out->nnz = static_cast<int64_t>(s.sparse.nnz());
        }
        return 0;
    } catch (...) {
        ctx->error = std::current_exception();
        return 1;
    }
}

}  // namespace detail

// One libfarqb handle: one device, one stream, reusable device workspace.
class Engine {
  public:
    explicit Engine(int device = 0) {
        const fqb_status st = fqb_create(device, &h_);
        if (st != FQB_OK) detail::raise(st, "fqb_create");
    }
    ~Engine() { fqb_destroy(h_); }
    Engine(const Engine&) = delete;
    Engine& operator=(const Engine&) = delete;

    template <typename Matrix>
    QbResult run_fixed_precision(const Matrix& a, const FarpcaConfig& cfg, BlockSource* source = nullptr) {
        return run(a, cfg, source, -1);
    }
    template <typename Matrix>
    QbResult run_fixed_rank(const Matrix& a, int rank, const FarpcaConfig& cfg, BlockSource* source = nullptr) {
        return run(a, cfg, source, rank);
    }

    SketchBlock gen_sketch(const SketchSpec& spec, int n, int l, int block_id) {
        fqb_sketch_spec cs{static_cast<int>(spec.kind), spec.p, spec.seed, spec.zeta};
        fqb_sketch_host s{};
        const fqb_status st = fqb_gen_sketch(h_, &cs, n, l, block_id, &s);
        if (st != FQB_OK) detail::raise(st, "fqb_gen_sketch");
        SketchBlock out;
        out.is_dense = s.is_dense != 0;
        out.centered = s.centered != 0;
        out.p = s.p;
        out.std_scale = s.std_scale;
        if (out.is_dense) {
            out.dense = DenseMatrix(n, l);
            out.dense.data.assign(s.dense, s.dense + std::size_t(n) * l);
        } else {
            out.sparse.rows = n;
            out.sparse.cols = l;
            out.sparse.col_ptr.assign(s.col_ptr, s.col_ptr + l + 1);
            out.sparse.row_idx.assign(s.row_idx, s.row_idx + s.nnz);
            out.sparse.values.assign(s.values, s.values + s.nnz);
        }
        fqb_sketch_free(&s);
        return out;
    }

    fqb_handle handle() const { return h_; }

  private:
    template <typename Matrix>
    QbResult run(const Matrix& a, const FarpcaConfig& cfg, BlockSource* source, int rank) {
        const fqb_config c = detail::to_c(cfg);
        detail::SourceCtx ctx{source, {}, nullptr};
        fqb_qb_result r{};
        const int m = a.rows, n = a.cols;
        auto* cb = source ? detail::source_trampoline : nullptr;
        const unsigned fl = FQB_OUT_HOST | FQB_OUT_SVD;
        fqb_status st;
        if constexpr (std::is_same_v<std::decay_t<decltype(a.data[0])>, float>) {
            // FP32 input mode (fqb_qb_*_f32): A kept in FP32, products in FP64
            st = rank < 0 ? fqb_qb_fixed_precision_f32(h_, a.data.data(), m, n, m, 0, &c, cb, &ctx, fl, &r)
                          : fqb_qb_fixed_rank_f32(h_, a.data.data(), m, n, m, 0, rank, &c, cb, &ctx, fl, &r);
        } else {
            st = rank < 0 ? fqb_qb_fixed_precision(h_, a.data.data(), m, n, m, 0, &c, cb, &ctx, fl, &r)
                          : fqb_qb_fixed_rank(h_, a.data.data(), m, n, m, 0, rank, &c, cb, &ctx, fl, &r);
        }
        if (ctx.error) {
            fqb_result_free(&r);
            std::rethrow_exception(ctx.error);
        }
        if (st != FQB_OK && st != FQB_ERR_TOLERANCE_NOT_REACHED && st != FQB_ERR_BLOCK_DEGENERATE) {
            fqb_result_free(&r);
            detail::raise(st, rank < 0 ? "run_fixed_precision" : "run_fixed_rank");
        }
        QbResult out;
        out.rank = r.rank;
        out.blocks = r.blocks;
        out.converged = r.converged != 0;
        out.residual_sq = r.residual_sq;
        out.norm_a_sq = r.norm_a_sq;
        out.device_ms = r.elapsed_ms;
        if (r.rank > 0 && r.q) {
            out.q = DenseMatrix(m, r.rank);
            out.q.data.assign(r.q, r.q + std::size_t(m) * r.rank);
            out.bt = DenseMatrix(n, r.rank);
            out.bt.data.assign(r.bt, r.bt + std::size_t(n) * r.rank);
        }
        out.qb_residual_sq = r.residual_sq;
        if (r.sigma) {
            out.sigma.assign(r.sigma, r.sigma + r.svd_rank);
            out.v_flagged.assign(r.v_flagged, r.v_flagged + r.svd_rank);
            out.residual_sq = r.svd_residual_sq;
            if (r.svd_rank > 0 && r.u) {
                out.u = DenseMatrix(m, r.svd_rank);
                out.u.data.assign(r.u, r.u + std::size_t(m) * r.svd_rank);
                out.v = DenseMatrix(n, r.svd_rank);
                out.v.data.assign(r.v, r.v + std::size_t(n) * r.svd_rank);
            }
        }
        out.block_residuals.assign(r.block_residuals, r.block_residuals + r.blocks);
        out.block_ids.assign(r.block_ids, r.block_ids + r.n_ids);
        const std::string msg = fqb_last_error();
        fqb_result_free(&r);
        if (st == FQB_ERR_TOLERANCE_NOT_REACHED) throw ToleranceNotReached(msg, std::move(out));
        if (st == FQB_ERR_BLOCK_DEGENERATE) throw BlockDegenerate(msg, out.blocks, out.residual_sq, out.norm_a_sq);
        return out;
    }

    fqb_handle h_ = nullptr;
};

inline Engine& default_engine() {
    thread_local std::unique_ptr<Engine> e;
    if (!e) e = std::make_unique<Engine>(0);
    return *e;
}

template <typename Matrix>
QbResult run_fixed_precision(const Matrix& a, const FarpcaConfig& cfg, BlockSource* source = nullptr) {
    return default_engine().run_fixed_precision(a, cfg, source);
}

template <typename Matrix>
QbResult run_fixed_rank(const Matrix& a, int rank, const FarpcaConfig& cfg, BlockSource* source = nullptr) {
    return default_engine().run_fixed_rank(a, rank, cfg, source);
}

inline SketchBlock gen_sketch(const SketchSpec& spec, int n, int l, int block_id) {
    return default_engine().gen_sketch(spec, n, l, block_id);
}

// truncate_to_tolerance (driver.cpp:415-433)
inline QbResult truncate_to_tolerance(const QbResult& svd, double eps_rel, double norm_a) {
    if (eps_rel < 0.0 || norm_a < 0.0) throw ConfigError("truncate_to_tolerance: negative tolerance or norm");
    const double target = eps_rel * norm_a;
    const double budget = target * target * (1.0 + 1e-12);
    const int l = svd.svd_rank();
    double acc = svd.residual_sq;
    int drop = 0;
    while (drop < l) {
        const double next = acc + svd.sigma[drop] * svd.sigma[drop];
        if (next > budget) break;
        acc = next;
        ++drop;
    }
    if (drop == 0) return svd;
    QbResult out = svd;
    out.residual_sq = acc;
    out.sigma.assign(svd.sigma.begin() + drop, svd.sigma.end());
    out.v_flagged.assign(svd.v_flagged.begin() + drop, svd.v_flagged.end());
    const int r = l - drop;
    out.u = DenseMatrix(svd.u.rows, r);
    out.v = DenseMatrix(svd.v.rows, r);
    for (int j = 0; j < r; ++j) {
        std::copy(svd.u.col(drop + j), svd.u.col(drop + j) + svd.u.rows, out.u.col(j));
        std::copy(svd.v.col(drop + j), svd.v.col(drop + j) + svd.v.rows, out.v.col(j));
    }
    return out;
}

// relative_error (experiment.cpp:317-342): exact ||A - U diag(sigma) V'||_F / ||A||_F on the
// device (one pass over A in column strips); a QB result without the SVD uses Q and B.
inline double relative_error(const DenseMatrix& a, const QbResult& res, Engine& eng = default_engine()) {
    const bool svd = !res.sigma.empty();
    const DenseMatrix& u = svd ? res.u : res.q;
    const DenseMatrix& v = svd ? res.v : res.bt;
    const int r = svd ? res.svd_rank() : res.rank;
    if (r > 0 && (u.rows != a.rows || v.rows != a.cols)) throw DimensionError("relative_error: factor shape mismatch");
    double out = 0.0;
    const fqb_status st = fqb_relative_error(eng.handle(), a.data.data(), a.rows, a.cols, std::max(a.rows, 1), 0,
                                             u.data.data(), std::max(u.rows, 1), svd ? res.sigma.data() : nullptr,
                                             v.data.data(), std::max(v.rows, 1), r, 0, &out);
    if (st != FQB_OK) detail::raise(st, "relative_error");
    return out;
}

// RawF64 interchange format (matrix_io.cpp:141-200): "SKLR", u32 rows, u32 cols,
// u32 reserved, then column-major little-endian f64.
struct FormatError : std::runtime_error {
    std::size_t offset;
    FormatError(const std::string& m, std::size_t off) : std::runtime_error(m), offset(off) {}
};

inline DenseMatrix load_raw(const std::string& buf) {
    auto u32 = [&](std::size_t at) {
        const auto* b = reinterpret_cast<const unsigned char*>(buf.data()) + at;
        return std::uint32_t(b[0]) | (std::uint32_t(b[1]) << 8) | (std::uint32_t(b[2]) << 16) |
               (std::uint32_t(b[3]) << 24);
    };
    if (buf.size() < 16) throw FormatError("truncated header, need 16 bytes", buf.size());
    if (buf.compare(0, 4, "SKLR") != 0) throw FormatError("bad magic, expected SKLR", 0);
    const std::uint64_t rows = u32(4), cols = u32(8);
    if (rows > 0x7FFFFFFFull) throw FormatError("dimension overflow in row count", 4);
    if (cols > 0x7FFFFFFFull) throw FormatError("dimension overflow in column count", 8);
    const std::uint64_t need = rows * cols * 8;
    if (buf.size() - 16 < need) throw FormatError("truncated payload", buf.size());
    if (buf.size() - 16 > need) throw FormatError("trailing bytes after payload", std::size_t(16 + need));
    DenseMatrix a(static_cast<int>(rows), static_cast<int>(cols));
    for (std::size_t k = 0; k < a.data.size(); ++k) {   // little-endian payload, any host byte order
        std::uint64_t bits = 0;
        const auto* q = reinterpret_cast<const unsigned char*>(buf.data()) + 16 + 8 * k;
        for (int i = 7; i >= 0; --i) bits = (bits << 8) | q[i];
        std::memcpy(&a.data[k], &bits, 8);
    }
    return a;
}

inline void save_raw(const DenseMatrix& a, std::string& out) {
    auto put = [&](std::uint32_t v) {
        for (int i = 0; i < 4; ++i) out.push_back(char((v >> (8 * i)) & 0xFF));
    };
    out.reserve(out.size() + 16 + 8 * a.data.size());
    out += "SKLR";
    put(std::uint32_t(a.rows));
    put(std::uint32_t(a.cols));
    put(0);
    for (double x : a.data) {
        std::uint64_t bits;
        std::memcpy(&bits, &x, 8);
        for (int i = 0; i < 8; ++i) out.push_back(char((bits >> (8 * i)) & 0xFF));
    }
}

inline double default_density(SketchKind kind, int n) { return fqb_default_density(static_cast<int>(kind), n); }
inline int default_block(int m, int n) { return fqb_default_block(m, n); }
inline int default_max_iters(int n, int b) { return fqb_default_max_iters(n, b); }

}  // namespace rsvd_b200
