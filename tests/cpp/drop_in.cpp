// drop_in.cpp -- the reference's own usage pattern (tools/main.cpp:61-112,
// tests/test_driver.cpp) written against include/farqb/rsvd_b200.hpp.
//
//   drop_in cpu   : boundary checks that need no device (defaults, loud failure)
//   drop_in gpu   : a fixed-precision QB run of a 600 x 400 low-rank matrix for
//                   every sketch kind, with an injected BlockSource, checking Q'Q = I
//                   and E = ||A - Q B||_F^2.
#include <cmath>
#include <cstdio>
#include <cstring>
#include <random>
#include <string>

#include "farqb/rsvd_b200.hpp"

namespace rb = rsvd_b200;

static rb::DenseMatrix lowrank(int m, int n, int r, unsigned seed) {
    std::mt19937_64 g(seed);
    std::normal_distribution<double> nd;
    rb::DenseMatrix u(m, r), v(n, r), a(m, n);
    for (double& x : u.data) x = nd(g);
    for (double& x : v.data) x = nd(g);
    for (int k = 0; k < r; ++k) {
        const double s = std::pow(0.95, k) / std::sqrt(double(m) * n);
        for (int j = 0; j < n; ++j)
            for (int i = 0; i < m; ++i) a(i, j) += s * u(i, k) * v(j, k);
    }
    return a;
}

struct ZetaSource final : rb::BlockSource {
    rb::Engine* eng;
    rb::SketchBlock next(int n, int b, int block_id) override {
        rb::SketchSpec s;
        s.kind = rb::SketchKind::SparseSign;
        s.seed = 5;
        s.zeta = 8;
        return eng->gen_sketch(s, n, b, block_id);
    }
};

static int cpu_checks() {
    int fails = 0;
    fails += rb::default_block(20000, 20000) != 50;
    fails += rb::default_max_iters(401, 20) != 11;
    fails += std::fabs(rb::default_density(rb::SketchKind::SparseSign, 1000) - 0.01) > 1e-15;
    {   // RawF64 round trip and a malformed file (matrix_io.cpp:141-200)
        rb::DenseMatrix a(3, 2);
        for (int k = 0; k < 6; ++k) a.data[k] = 0.5 * k - 1.0;
        std::string buf;
        rb::save_raw(a, buf);
        const rb::DenseMatrix b = rb::load_raw(buf);
        fails += buf.size() != 16 + 48 || b.rows != 3 || b.cols != 2 || b.data != a.data;
        try {
            rb::load_raw(buf + "x");
            ++fails;
        } catch (const rb::FormatError& e) {
            fails += e.offset != 64;
        }
    }
    try {
        rb::Engine e(0);
        std::printf("unexpected: a device is present\n");
    } catch (const rb::CudaError& e) {
        std::printf("no device -> CudaError: %s\n", e.what());
    }
    std::printf(fails ? "FAIL\n" : "PASS\n");
    return fails;
}

static int gpu_checks() {
    int fails = 0;
    rb::Engine eng(0);
    const rb::DenseMatrix a = lowrank(600, 400, 120, 7);
    for (int kind = 0; kind < 5; ++kind) {
        rb::FarpcaConfig cfg;
        cfg.eps = 1e-2;  // rank ~90 of 120: far from the 1e-12 relative pivot floor
        cfg.relative = true;
        cfg.power = 1;
        cfg.block = 16;
        cfg.sketch.kind = static_cast<rb::SketchKind>(kind);
        cfg.sketch.seed = 11;
        if (kind == 3 || kind == 4) cfg.sketch.zeta = 8;
        rb::QbResult r = eng.run_fixed_precision(a, cfg);
        double orth = 0.0, err = 0.0;
        for (int j = 0; j < r.rank; ++j)
            for (int k = 0; k < r.rank; ++k) {
                double s = 0.0;
                for (int i = 0; i < a.rows; ++i) s += r.q(i, j) * r.q(i, k);
                orth = std::fmax(orth, std::fabs(s - (j == k)));
            }
        for (int j = 0; j < a.cols; ++j)
            for (int i = 0; i < a.rows; ++i) {
                double s = 0.0;
                for (int k = 0; k < r.rank; ++k) s += r.q(i, k) * r.bt(j, k);
                err += (a(i, j) - s) * (a(i, j) - s);
            }
        double recon = 0.0;  // U diag(sigma) V' == Q B
        for (int j = 0; j < a.cols; j += 37)
            for (int i = 0; i < a.rows; i += 29) {
                double s1 = 0.0, s2 = 0.0;
                for (int k = 0; k < r.rank; ++k) s1 += r.q(i, k) * r.bt(j, k);
                for (int k = 0; k < r.svd_rank(); ++k) s2 += r.u(i, k) * r.sigma[k] * r.v(j, k);
                recon = std::fmax(recon, std::fabs(s1 - s2));
            }
        const bool ok = r.converged && orth < 1e-12 && std::fabs(err - r.residual_sq) <= 1e-10 * r.norm_a_sq &&
                        r.svd_rank() == r.rank && recon < 1e-12;
        std::printf("kind %d rank %d blocks %d E %.6e true %.6e orth %.1e %s\n", kind, r.rank, r.blocks,
                    r.residual_sq, err, orth, ok ? "ok" : "FAIL");
        fails += !ok;
    }
    ZetaSource src;
    src.eng = &eng;
    rb::FarpcaConfig cfg;
    cfg.eps = 1e-2;
    cfg.relative = true;
    cfg.block = 16;
    cfg.power = 2;
    rb::QbResult r = eng.run_fixed_precision(a, cfg, &src);
    std::printf("injected source: rank %d ids %zu\n", r.rank, r.block_ids.size());
    fails += !r.converged;
    try {
        cfg.eps = 1e-14;
        cfg.max_iters = 2;
        eng.run_fixed_precision(a, cfg, &src);
        ++fails;
    } catch (const rb::ToleranceNotReached& e) {
        std::printf("ToleranceNotReached with partial rank %d\n", e.partial.rank);
        fails += e.partial.rank != 32;
    }
    try {
        cfg.block = 1000;
        eng.run_fixed_precision(a, cfg);
        ++fails;
    } catch (const rb::ConfigError&) {
    }
    {   // FP32 input mode: a FloatMatrix gives the FP64 loop on double(A)
        rb::FloatMatrix af(a.rows, a.cols);
        rb::DenseMatrix ad(a.rows, a.cols);
        for (std::size_t e = 0; e < a.data.size(); ++e) {
            af.data[e] = float(a.data[e]);
            ad.data[e] = double(af.data[e]);
        }
        rb::FarpcaConfig c2;
        c2.eps = 1e-2;
        c2.relative = true;
        c2.block = 16;
        c2.power = 1;
        c2.sketch.kind = rb::SketchKind::StdBernoulli;
        c2.sketch.seed = 3;
        const rb::QbResult r32 = eng.run_fixed_precision(af, c2);
        const rb::QbResult r64 = eng.run_fixed_precision(ad, c2);
        const bool ok = r32.rank == r64.rank && r32.blocks == r64.blocks &&
                        std::fabs(r32.qb_residual_sq - r64.qb_residual_sq) <= 1e-12 * r64.norm_a_sq;
        std::printf("fp32 input: rank %d / %d, E %.6e / %.6e %s\n", r32.rank, r64.rank, r32.qb_residual_sq,
                    r64.qb_residual_sq, ok ? "ok" : "FAIL");
        fails += !ok;
        // exact error of the SVD (experiment.cpp:317-342) vs the indicator
        const double rel = rb::relative_error(ad, r64, eng);
        const bool ok2 = std::fabs(rel * rel * r64.norm_a_sq - r64.residual_sq) <= 1e-10 * r64.norm_a_sq;
        std::printf("relative_error %.6e vs sqrt(E/|A|^2) %.6e %s\n", rel, std::sqrt(r64.residual_sq / r64.norm_a_sq),
                    ok2 ? "ok" : "FAIL");
        fails += !ok2;
    }
    std::printf(fails ? "FAIL\n" : "PASS\n");
    return fails;
}

int main(int argc, char** argv) {
    std::setvbuf(stdout, nullptr, _IONBF, 0);
    const bool gpu = argc > 1 && std::strcmp(argv[1], "gpu") == 0;
    return gpu ? gpu_checks() : cpu_checks();
}
