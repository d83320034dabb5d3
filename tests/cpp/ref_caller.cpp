// ref_caller.cpp -- a caller written against the REFERENCE's public C++ API only
// (rsvd/driver.hpp, rsvd/synthetic.hpp, rsvd/sketch.hpp), the way the reference's own
// tools and tests use it: build a DenseMatrix, fill a FarpcaConfig, call
// rsvd::run_fixed_precision / run_fixed_rank, plug in a BlockSource, catch the
// reference's exceptions.
//
// oracle/Makefile links it twice, unmodified:
//   _ref/ref_caller_ref  against the reference library alone (the CPU reference);
//   _ref/ref_caller_b200 with paper_2506_03859_b200/lib/librsvd_b200.so ahead of it,
//                        so run_fixed_precision / run_fixed_rank resolve to the B200
//                        engine and everything else (gen_synthetic, gen_sketch) to
//                        the reference.
// tests/test_cpp_dropin.py runs both on the GPU box and compares the printed results.
// Output: one line per case, "case key=value ...", doubles in %.17g.
#include <cmath>
#include <cstdio>
#include <exception>
#include <string>
#include <vector>

#include "rsvd/driver.hpp"
#include "rsvd/sketch.hpp"
#include "rsvd/synthetic.hpp"

using namespace rsvd;

namespace {

void print_svd(const char* name, const ApproxSvd& s, const std::vector<int>* ids = nullptr) {
    std::printf("%s status=ok rank=%d blocks=%d converged=%d residual_sq=%.17g norm_a_sq=%.17g", name, s.rank(),
                s.blocks, int(s.converged), s.residual_sq, s.norm_a_sq);
    std::printf(" sigma=");
    for (int i = 0; i < s.rank(); ++i) std::printf("%s%.17g", i ? "," : "", s.sigma[i]);
    // the reconstruction U diag(sigma) V' on a fixed probe: (U S V') x for x_j = 1/(1+j)
    std::vector<double> vx(s.rank(), 0.0);
    for (int k = 0; k < s.rank(); ++k) {
        double t = 0.0;
        for (int j = 0; j < s.v.rows; ++j) t += s.v(j, k) / (1.0 + j);
        vx[k] = t * s.sigma[k];
    }
    std::printf(" probe=");
    for (int i = 0; i < s.u.rows; i += std::max(1, s.u.rows / 16)) {
        double y = 0.0;
        for (int k = 0; k < s.rank(); ++k) y += s.u(i, k) * vx[k];
        std::printf("%s%.17g", i ? "," : "", y);
    }
    int flagged = 0;
    for (char f : s.v_flagged) flagged += f ? 1 : 0;
    std::printf(" flagged=%d", flagged);
    if (ids) {
        std::printf(" ids=");
        for (size_t i = 0; i < ids->size(); ++i) std::printf("%s%d", i ? "," : "", (*ids)[i]);
    }
    std::printf("\n");
}

// Serves the reference's own gen_sketch blocks, recording every id it is asked for.
struct RecordingSource final : BlockSource {
    SketchSpec spec;
    std::vector<int> seen;
    explicit RecordingSource(const SketchSpec& s) : spec(s) {}
    SketchBlock next(int n, int b, int block_id) override {
        seen.push_back(block_id);
        return gen_sketch(spec, n, b, block_id);
    }
};

// Rank-one (degenerate) blocks below `bad_below`, Gaussian gen_sketch blocks after.
struct DegenerateSource final : BlockSource {
    std::vector<int> seen;
    int bad_below = 0;
    SketchBlock next(int n, int b, int block_id) override {
        seen.push_back(block_id);
        if (block_id < bad_below) {
            SketchBlock out;
            out.is_dense = true;
            out.dense = DenseMatrix(n, b);
            for (double& x : out.dense.data) x = 1.0;
            return out;
        }
        SketchSpec g;
        g.kind = SketchKind::Gaussian;
        g.seed = 77;
        return gen_sketch(g, n, b, block_id);
    }
};

struct ThrowingSource final : BlockSource {
    SketchBlock next(int, int, int) override { throw std::runtime_error("source exhausted"); }
};

FarpcaConfig config(SketchKind kind, double p, int power, int block, double eps, std::uint64_t seed) {
    FarpcaConfig c;
    c.sketch.kind = kind;
    c.sketch.p = p;
    c.sketch.seed = seed;
    c.power = power;
    c.block = block;
    c.eps = eps;
    c.relative = true;
    return c;
}

}  // namespace

int main() {
    SyntheticSpec ss;
    ss.kind = SyntheticKind::SlowDecay;
    ss.n = 600;
    ss.seed = 42;
    const DenseMatrix a = gen_synthetic(ss);
    SyntheticSpec fs = ss;
    fs.kind = SyntheticKind::FastDecay;
    fs.n = 500;
    const DenseMatrix f = gen_synthetic(fs);

    // 1. every kind, the library's own sketch generator (no BlockSource)
    const SketchKind kinds[] = {SketchKind::Gaussian, SketchKind::Bernoulli, SketchKind::StdBernoulli,
                                SketchKind::SparseSign, SketchKind::SparseGaussian};
    const char* names[] = {"gaussian", "bernoulli", "stdbernoulli", "sparsesign", "sparsegaussian"};
    for (int k = 0; k < 5; ++k)
        for (int power : {1, 2}) {
            const double p = kinds[k] == SketchKind::StdBernoulli ? 0.5 : 0.0;
            const std::string tag = std::string("fp_") + names[k] + "_P" + std::to_string(power);
            print_svd(tag.c_str(), run_fixed_precision(f, config(kinds[k], p, power, 20, 1e-3, 7)));
        }
    // 2. a BlockSource plugin: ids requested in order
    {
        RecordingSource src(config(SketchKind::SparseSign, 0.05, 1, 16, 0, 3).sketch);
        const ApproxSvd s = run_fixed_precision(a, config(SketchKind::SparseSign, 0.05, 1, 16, 1e-2, 3), &src);
        print_svd("source_sparsesign", s, &src.seen);
    }
    // 3. fixed rank, rank not a block multiple (drop_smallest)
    print_svd("fixed_rank_37", run_fixed_rank(f, 37, config(SketchKind::Gaussian, 0.0, 2, 10, 0.0, 5)));
    // 4. ToleranceNotReached carries the partial factorization
    try {
        FarpcaConfig c = config(SketchKind::Gaussian, 0.0, 1, 10, 1e-6, 9);
        c.max_iters = 3;
        run_fixed_precision(a, c);
        std::printf("tolerance status=missing\n");
    } catch (const ToleranceNotReached& e) {
        std::printf("tolerance status=ToleranceNotReached what=\"%s\"\n", e.what());
        print_svd("tolerance_partial", e.partial);
    }
    // 5. degenerate blocks: redraw ids j + 1000 attempt, BlockDegenerate after 3 redraws
    {
        DegenerateSource src;
        src.bad_below = 2000;   // every block fails twice, then succeeds at id j + 2000
        const ApproxSvd s = run_fixed_precision(f, config(SketchKind::Gaussian, 0.0, 1, 10, 1e-1, 1), &src);
        print_svd("redraw", s, &src.seen);
    }
    try {
        DegenerateSource src;
        src.bad_below = 1 << 30;
        run_fixed_precision(f, config(SketchKind::Gaussian, 0.0, 1, 10, 1e-2, 1), &src);
        std::printf("degenerate status=missing\n");
    } catch (const BlockDegenerate& e) {
        std::printf("degenerate status=BlockDegenerate blocks=%d residual_sq=%.17g norm_a_sq=%.17g\n",
                    e.blocks_accepted, e.residual_sq, e.norm_a_sq);
    }
    // 6. configuration errors and a throwing source
    try {
        run_fixed_precision(f, config(SketchKind::Gaussian, 0.0, 1, 501, 1e-2, 1));
        std::printf("config status=missing\n");
    } catch (const ConfigError& e) {
        std::printf("config status=ConfigError what=\"%s\"\n", e.what());
    }
    try {
        run_fixed_precision(f, config(SketchKind::Gaussian, 0.0, 1, 10, 0.0, 1));
        std::printf("config_eps status=missing\n");
    } catch (const ConfigError& e) {
        std::printf("config_eps status=ConfigError what=\"%s\"\n", e.what());
    }
    try {
        ThrowingSource src;
        run_fixed_precision(f, config(SketchKind::Gaussian, 0.0, 1, 10, 1e-2, 1), &src);
        std::printf("throwing status=missing\n");
    } catch (const std::runtime_error& e) {
        std::printf("throwing status=runtime_error what=\"%s\"\n", e.what());
    }
    return 0;
}
