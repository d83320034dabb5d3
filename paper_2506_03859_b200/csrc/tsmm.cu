// tsmm.cu -- the tall-skinny Gram matrices of the CholeskyQR steps on the DMMA pipe.
//
// Replaces, for b <= 128, the general split-K GEMM (gemm.cu) on the shape every block
// runs four times (engine.cu orth_power / accept: S = W'W over n rows, S = Y'Y over m
// rows; reference: the Grams of eig_svd / accept_block, matrix_core.cpp:193-215,
// driver.cpp:230-294):
//
//   ts_gram : S = Y' Y  (Y: K x b)  -- only the 8 x 8 tiles on and above the diagonal
//             are formed (91 of 169 at b = 100), the lower triangle is mirrored, so S is
//             exactly symmetric.  Each CTA reduces a contiguous slab of rows with every
//             fragment of a k-step loaded before its MMAs; the per-CTA partials are
//             summed in a fixed order by a second kernel: deterministic.
//             C4 (ncu): 121 -> 67 us over m = 100000 rows, 31 -> 21 us over n = 20000.
//
// (A triangular-aware Y R kernel for the R^-1 products was measured no faster than the
// general GEMM -- 79-92 us vs 96 us at m = 100000, slower at n = 20000 -- and dropped.)
//
// DMMA: mma.sync.m8n8k4 f64 (SASS DMMA.8x8x4), the only FP64 tensor path on sm_100a.
#include <algorithm>
#include <cstdint>

#include "kernels.hpp"

namespace farqb {
namespace {

constexpr int kMaxB = 128;
constexpr int kGramRows = 32;      // rows of Y per stage
constexpr int kGramPitch = kGramRows + 4;   // Ys[c][k]: fragment loads hit 2 wavefronts
constexpr int kGramStages = 4;
constexpr int kGramThreads = 256;

__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                 : "+d"(d0), "+d"(d1)
                 : "d"(a), "d"(b));
}
__device__ __forceinline__ void cp16(void* smem, const void* gmem, int bytes) {
    const unsigned s = unsigned(__cvta_generic_to_shared(smem));
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(s), "l"(gmem), "r"(bytes));
}
__device__ __forceinline__ void cp8(void* smem, const void* gmem, int bytes) {
    const unsigned s = unsigned(__cvta_generic_to_shared(smem));
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(s), "l"(gmem), "r"(bytes));
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

// ---- Gram --------------------------------------------------------------------
// upper-triangular tile t (row-major over i <= j) of an nt x nt tile grid
__host__ __device__ inline void tri_tile(int t, int nt, int& i, int& j) {
    i = 0;
    int row = nt;
    while (t >= row) {
        t -= row;
        --row;
        ++i;
    }
    j = i + t;
}

struct GramArgs {
    const double* Y;
    int64_t K, ldy;
    int b, nt, tiles;
    int64_t rows_per_cta;   // multiple of kGramRows
    bool vec2;              // ldy even and Y 16-byte aligned
    double* work;           // gridDim.x x tiles x 64
};

// MAXT: tiles per warp (ceil(tiles / 8))
template <int MAXT>
__global__ void __launch_bounds__(kGramThreads, 1) k_ts_gram(const GramArgs p) {
    FQB_PDL_ENTRY();
    extern __shared__ __align__(16) double smem[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, g = lane >> 2, t4 = lane & 3;
    const int bp = p.nt * 8;
    const int stage_elems = bp * kGramPitch;
    const int64_t r0 = int64_t(blockIdx.x) * p.rows_per_cta;
    const int64_t r1 = min(p.K, r0 + p.rows_per_cta);
    const int nsteps = r1 > r0 ? int((r1 - r0 + kGramRows - 1) / kGramRows) : 0;
    // this warp's contiguous run of upper tiles
    const int per = (p.tiles + 7) / 8;
    const int t0 = warp * per;
    int ti[MAXT], tj[MAXT];
#pragma unroll
    for (int q = 0; q < MAXT; ++q) {
        const int t = t0 + q;
        if (q < per && t < p.tiles) tri_tile(t, p.nt, ti[q], tj[q]);
        else ti[q] = tj[q] = -1;
    }
    double acc[MAXT][2];
#pragma unroll
    for (int q = 0; q < MAXT; ++q) acc[q][0] = acc[q][1] = 0.0;

    auto load = [&](int step, int stage) {
        double* ys = smem + stage * stage_elems;
        const int64_t k0 = r0 + int64_t(step) * kGramRows;
        if (p.vec2) {
            constexpr int CH = kGramRows / 2;
            for (int c = threadIdx.x; c < bp * CH; c += kGramThreads) {
                const int col = c / CH, kk = (c % CH) * 2;
                const int64_t gk = k0 + kk;
                int bytes = 0;
                const double* src = p.Y;
                if (col < p.b && gk < r1) {
                    src = p.Y + int64_t(col) * p.ldy + gk;
                    bytes = (r1 - gk >= 2 ? 2 : 1) * 8;
                }
                cp16(ys + col * kGramPitch + kk, src, bytes);
            }
        } else {
            for (int c = threadIdx.x; c < bp * kGramRows; c += kGramThreads) {
                const int col = c / kGramRows, kk = c % kGramRows;
                const int64_t gk = k0 + kk;
                const bool ok = col < p.b && gk < r1;
                cp8(ys + col * kGramPitch + kk, ok ? p.Y + int64_t(col) * p.ldy + gk : p.Y, ok ? 8 : 0);
            }
        }
    };
#pragma unroll
    for (int s = 0; s < kGramStages - 1; ++s) {
        if (s < nsteps) load(s, s);
        cp_commit();
    }
    for (int step = 0; step < nsteps; ++step) {
        cp_wait<kGramStages - 2>();
        __syncthreads();
        if (step + kGramStages - 1 < nsteps) load(step + kGramStages - 1, (step + kGramStages - 1) % kGramStages);
        cp_commit();
        const double* ys = smem + (step % kGramStages) * stage_elems;
#pragma unroll
        for (int kk = 0; kk < kGramRows; kk += 4) {
            // all of the k-step's fragments first (loads in flight together), then the MMAs
            double af[MAXT], bf[MAXT];
#pragma unroll
            for (int q = 0; q < MAXT; ++q) {
                const int i = ti[q] < 0 ? 0 : ti[q], j = tj[q] < 0 ? 0 : tj[q];
                af[q] = (q > 0 && ti[q] == ti[q - 1]) ? af[q - 1] : ys[(i * 8 + g) * kGramPitch + kk + t4];
                bf[q] = ys[(j * 8 + g) * kGramPitch + kk + t4];
            }
#pragma unroll
            for (int q = 0; q < MAXT; ++q)
                if (ti[q] >= 0) dmma(acc[q][0], acc[q][1], af[q], bf[q]);   // warp-uniform
        }
    }
    cp_wait<0>();
    // partials: work[cta][tile][g * 8 + 2 t4 + h]
    double* w = p.work + int64_t(blockIdx.x) * p.tiles * 64;
#pragma unroll
    for (int q = 0; q < MAXT; ++q) {
        if (ti[q] < 0) continue;
        const int t = t0 + q;
        w[int64_t(t) * 64 + g * 8 + 2 * t4] = acc[q][0];
        w[int64_t(t) * 64 + g * 8 + 2 * t4 + 1] = acc[q][1];
    }
}

// S (b x b, lds) = alpha * sum over CTAs of the tile partials; both triangles written
// from the same sum.  A warp per upper-tile element: lane q sums CTAs q, q + 32, ... in
// order, then a fixed shuffle tree -- deterministic, and every load of the element in
// flight at once.
__global__ void __launch_bounds__(256) k_ts_gram_reduce(const double* __restrict__ work, int ctas, int tiles, int nt,
                                                        int b, double alpha, double beta, double* S, int64_t lds) {
    FQB_PDL_ENTRY();
    const int64_t e = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) / 32;
    const int q = threadIdx.x & 31;
    if (e >= int64_t(tiles) * 64) return;   // warp-uniform
    double v = 0.0;
    for (int c = q; c < ctas; c += 32) v += work[int64_t(c) * tiles * 64 + e];
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) v += __shfl_xor_sync(0xFFFFFFFFu, v, o);
    if (q != 0) return;
    const int t = int(e / 64), r = int(e % 64);
    int ti, tj;
    tri_tile(t, nt, ti, tj);
    const int row = ti * 8 + r / 8, col = tj * 8 + r % 8;
    if (row >= b || col >= b || (ti == tj && col < row)) return;
    const double s = alpha * v;
    double* up = S + int64_t(col) * lds + row;
    *up = beta != 0.0 ? fma(beta, *up, s) : s;
    if (row != col) {
        double* lo = S + int64_t(row) * lds + col;
        *lo = beta != 0.0 ? fma(beta, *lo, s) : s;
    }
}

template <int MAXT>
void launch_gram(const GramArgs& a, int grid, size_t smem, cudaStream_t s) {
    static bool configured[64] = {};
    int dev = 0;
    FQB_CUDA(cudaGetDevice(&dev));
    if (dev < 0 || dev >= 64 || !configured[dev]) {
        const int mx = kGramStages * kMaxB * kGramPitch * int(sizeof(double));
        FQB_CUDA(cudaFuncSetAttribute(k_ts_gram<MAXT>, cudaFuncAttributeMaxDynamicSharedMemorySize, mx));
        if (dev >= 0 && dev < 64) configured[dev] = true;
    }
    launch_k(k_ts_gram<MAXT>, grid, kGramThreads, smem, s, a);
}

}  // namespace

bool ts_enabled() {
    static const bool on = [] {
        const char* e = std::getenv("FQB_TSMM");
        return !(e && e[0] == '0');
    }();
    return on;
}

int64_t ts_gram_workspace_doubles(int b, int num_sms) {
    const int nt = (b + 7) / 8;
    return int64_t(num_sms) * (nt * (nt + 1) / 2) * 64;
}

void ts_gram(const double* Y, int64_t K, int b, int64_t ldy, double alpha, double beta, double* S, int64_t lds,
             double* work, int64_t work_doubles, int num_sms, cudaStream_t s, LaunchCounter& lc) {
    if (b <= 0) return;
    if (b > kMaxB) throw Error(kStatusConfig, "ts_gram: b above 128");
    GramArgs a{};
    a.Y = Y;
    a.K = K;
    a.ldy = ldy;
    a.b = b;
    a.nt = (b + 7) / 8;
    a.tiles = a.nt * (a.nt + 1) / 2;
    a.vec2 = ldy % 2 == 0 && reinterpret_cast<uintptr_t>(Y) % 16 == 0;
    const int64_t steps = std::max<int64_t>(1, (K + kGramRows - 1) / kGramRows);
    int grid = int(std::min<int64_t>(num_sms, steps));
    grid = int(std::min<int64_t>(grid, std::max<int64_t>(1, work_doubles / (int64_t(a.tiles) * 64))));
    a.rows_per_cta = ((steps + grid - 1) / grid) * kGramRows;
    grid = int((K + a.rows_per_cta - 1) / a.rows_per_cta);
    if (grid < 1) grid = 1;
    a.work = work;
    const size_t smem = size_t(kGramStages) * a.nt * 8 * kGramPitch * sizeof(double);
    const int per = (a.tiles + 7) / 8;
    if (per <= 6) launch_gram<6>(a, grid, smem, s);          // b <= 48
    else if (per <= 12) launch_gram<12>(a, grid, smem, s);   // b <= 104
    else launch_gram<17>(a, grid, smem, s);                  // b <= 128
    FQB_LAUNCHED();
    const int64_t outs = int64_t(a.tiles) * 64 * 32;
    launch_k(k_ts_gram_reduce, unsigned((outs + 255) / 256), 256, 0, s, static_cast<const double*>(work), grid,
             a.tiles, a.nt, b, alpha, beta, S, lds);
    FQB_LAUNCHED();
    lc.bump(2);
}

}  // namespace farqb
