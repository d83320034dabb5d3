// tsmm.cu -- the tall-skinny b x b products of the CholeskyQR steps on the DMMA pipe.
//
// Replace, for small b, the general split-K / stream-K GEMMs (gemm.cu, gemm_tma.cu) on the
// two shapes every block runs several times (engine.cu orth_power / accept; reference:
// the Grams of eig_svd / accept_block and the triangular solves against the Cholesky
// factors, matrix_core.cpp:117-215, driver.cpp:230-294):
//
//   ts_gram : S = Y' Y  (Y: K x b, b <= 128)  -- only the 8 x 8 tiles on and above the
//             diagonal are formed (91 of 169 at b = 100), the lower triangle is mirrored,
//             so S is exactly symmetric.  Each CTA reduces a contiguous slab of rows with
//             every fragment of a k-step loaded before its MMAs; the per-CTA partials are
//             summed in a fixed order by a second kernel: deterministic.
//             C4 (ncu): 121 -> 67 us over m = 100000 rows, 31 -> 21 us over n = 20000.
//   ts_trmm : Z = Y R  (R: b x b upper triangular, b <= 104 -- the R^-1 factors)
//             persistent, R staged once per CTA, 64-row blocks of Y double-buffered by
//             cp.async; the k-steps below R's diagonal are not emitted: every (tile,
//             k-step) pair is a compile-time constant, warps split by column-tile
//             parity (a first version chose them at run time -- the DMMAs were
//             predicated off, not skipped, and a predicated-off DMMA still occupies the
//             tensor pipe: all 2704 MMAs per block ran instead of 1456).
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
constexpr int kGramThreads = 512;   // 16 warps: more independent DMMA chains per SM partition
constexpr int kGramWarps = kGramThreads / 32;
constexpr int kTrmmRows = 64;      // rows of Y per block
constexpr int kTrmmThreads = 512;  // 8 row groups of 8 x 2 column-tile parities
constexpr int kTrmmMaxB = 104;     // R (b x b+4) + 2 x Y (b x 72) within 227 KB

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

// MAXT: tiles per warp (ceil(tiles / kGramWarps))
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
    const int per = (p.tiles + kGramWarps - 1) / kGramWarps;
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
// from the same sum.  A CTA per 32 consecutive upper-tile elements: warp w sums CTAs
// w, w + 8, ... (coalesced 256-byte rows of the partials), the 8 warp sums are added in
// warp order -- deterministic.
__global__ void __launch_bounds__(256) k_ts_gram_reduce(const double* __restrict__ work, int ctas, int tiles, int nt,
                                                        int b, double alpha, double beta, double* S, int64_t lds) {
    FQB_PDL_ENTRY();
    __shared__ double part[8][32];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t e = int64_t(blockIdx.x) * 32 + lane;
    const int64_t total = int64_t(tiles) * 64;
    double v = 0.0;
    if (e < total) {
#pragma unroll 4
        for (int c = warp; c < ctas; c += 8) v += work[int64_t(c) * total + e];
    }
    part[warp][lane] = v;
    __syncthreads();
    if (warp != 0 || e >= total) return;
    double sum = 0.0;
#pragma unroll
    for (int w = 0; w < 8; ++w) sum += part[w][lane];
    const int t = int(e / 64), r = int(e % 64);
    int ti, tj;
    tri_tile(t, nt, ti, tj);
    const int row = ti * 8 + r / 8, col = tj * 8 + r % 8;
    if (row >= b || col >= b || (ti == tj && col < row)) return;
    const double s = alpha * sum;
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

// ---- Y R with R upper triangular -----------------------------------------------
struct TrmmArgs {
    const double* Y;
    int64_t M, ldy;
    const double* R;
    int64_t ldr;
    double* Z;
    int64_t ldz;
    int b;
    bool vec2;
};

// One 64-row block of Z = Y R for warp (rows wm .. wm + 7, 8-column tiles j = WJ, WJ + 2,
// ...): every tile / k-step pair is a compile-time constant, so the k-steps below R's
// diagonal are not emitted at all (a predicated-off DMMA still occupies the pipe).
template <int NT, int WJ>
__device__ __forceinline__ void trmm_block(const double* ys, const double* Rs, int wm, int g, int t4, int64_t m0,
                                           const TrmmArgs& p) {
    constexpr int BP = NT * 8, RP = BP + 4, YP = kTrmmRows + 8;
    constexpr int JT = (NT - WJ + 1) / 2;
    double acc[JT > 0 ? JT : 1][2];
#pragma unroll
    for (int q = 0; q < JT; ++q) acc[q][0] = acc[q][1] = 0.0;
#pragma unroll
    for (int kk = 0; kk < BP; kk += 4) {
        const double a0 = ys[(kk + t4) * YP + wm + g];
        double bf[JT > 0 ? JT : 1];
#pragma unroll
        for (int q = 0; q < JT; ++q) {
            const int j = 2 * q + WJ;
            if (j * 8 + 7 >= kk) bf[q] = Rs[(j * 8 + g) * RP + kk + t4];
        }
#pragma unroll
        for (int q = 0; q < JT; ++q) {
            const int j = 2 * q + WJ;
            if (j * 8 + 7 < kk) continue;   // R(k, n) = 0 for k > n: resolved at compile time
            dmma(acc[q][0], acc[q][1], a0, bf[q]);
        }
    }
    const int64_t row = m0 + wm + g;
    if (row < p.M) {
#pragma unroll
        for (int q = 0; q < JT; ++q)
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const int col = (2 * q + WJ) * 8 + 2 * t4 + h;
                if (col < p.b) p.Z[int64_t(col) * p.ldz + row] = acc[q][h];
            }
    }
}

// NT: 8-column tiles of b (b <= 8 NT).  Persistent: R staged once per CTA as Rs[n][k]
// (pitch 8 NT + 4, zero below the diagonal), 64-row blocks of Y double-buffered by
// cp.async as Ys[k][m] (pitch 72).  16 warps: 8 row groups of 8 x the two parities of
// the column tiles (alternate tiles balance the triangle).
template <int NT>
__global__ void __launch_bounds__(kTrmmThreads, 1) k_ts_trmm(const TrmmArgs p) {
    FQB_PDL_ENTRY();
    extern __shared__ __align__(16) double smem[];
    constexpr int BP = NT * 8;
    constexpr int RP = BP + 4;
    constexpr int YP = kTrmmRows + 8;
    double* Rs = smem;
    double* Ys0 = smem + BP * RP;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, g = lane >> 2, t4 = lane & 3;
    for (int e = threadIdx.x; e < BP * BP; e += kTrmmThreads) {
        const int n = e / BP, k = e % BP;
        Rs[n * RP + k] = (n < p.b && k < p.b && k <= n) ? p.R[int64_t(n) * p.ldr + k] : 0.0;
    }
    const int64_t nblocks = (p.M + kTrmmRows - 1) / kTrmmRows;
    auto load = [&](int64_t blk, int stage) {
        double* ys = Ys0 + stage * (BP * YP);
        const int64_t m0 = blk * kTrmmRows;
        if (p.vec2) {
            constexpr int CH = kTrmmRows / 2;
            for (int c = threadIdx.x; c < BP * CH; c += kTrmmThreads) {
                const int k = c / CH, mm = (c % CH) * 2;
                const int64_t gm = m0 + mm;
                int bytes = 0;
                const double* src = p.Y;
                if (k < p.b && gm < p.M) {
                    src = p.Y + int64_t(k) * p.ldy + gm;
                    bytes = (p.M - gm >= 2 ? 2 : 1) * 8;
                }
                cp16(ys + k * YP + mm, src, bytes);
            }
        } else {
            for (int c = threadIdx.x; c < BP * kTrmmRows; c += kTrmmThreads) {
                const int k = c / kTrmmRows, mm = c % kTrmmRows;
                const int64_t gm = m0 + mm;
                const bool ok = k < p.b && gm < p.M;
                cp8(ys + k * YP + mm, ok ? p.Y + int64_t(k) * p.ldy + gm : p.Y, ok ? 8 : 0);
            }
        }
    };
    int64_t blk = blockIdx.x;
    if (blk < nblocks) load(blk, 0);
    cp_commit();
    const int wm = (warp & 7) * 8;
    for (int it = 0; blk < nblocks; ++it, blk += gridDim.x) {
        const int64_t nxt = blk + gridDim.x;
        if (nxt < nblocks) load(nxt, (it + 1) & 1);
        cp_commit();
        cp_wait<1>();
        __syncthreads();
        const double* ys = Ys0 + (it & 1) * (BP * YP);
        if (warp < 8) trmm_block<NT, 0>(ys, Rs, wm, g, t4, blk * kTrmmRows, p);
        else trmm_block<NT, 1>(ys, Rs, wm, g, t4, blk * kTrmmRows, p);
        __syncthreads();   // the stage is refilled next iteration
    }
    cp_wait<0>();
}

template <int NT>
void launch_trmm(const TrmmArgs& a, int grid, cudaStream_t s) {
    constexpr int BP = NT * 8;
    const size_t smem = size_t(BP) * (BP + 4) * sizeof(double) + 2 * size_t(BP) * (kTrmmRows + 8) * sizeof(double);
    static bool configured[64] = {};
    int dev = 0;
    FQB_CUDA(cudaGetDevice(&dev));
    if (dev < 0 || dev >= 64 || !configured[dev]) {
        FQB_CUDA(cudaFuncSetAttribute(k_ts_trmm<NT>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
        if (dev >= 0 && dev < 64) configured[dev] = true;
    }
    launch_k(k_ts_trmm<NT>, grid, kTrmmThreads, smem, s, a);
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
    const int per = (a.tiles + kGramWarps - 1) / kGramWarps;
    if (per <= 3) launch_gram<3>(a, grid, smem, s);          // b <= 48
    else if (per <= 6) launch_gram<6>(a, grid, smem, s);     // b <= 104
    else launch_gram<9>(a, grid, smem, s);                   // b <= 128
    FQB_LAUNCHED();
    const int64_t outs = int64_t(a.tiles) * 64;
    launch_k(k_ts_gram_reduce, unsigned((outs + 31) / 32), 256, 0, s, static_cast<const double*>(work), grid,
             a.tiles, a.nt, b, alpha, beta, S, lds);
    FQB_LAUNCHED();
    lc.bump(2);
}

bool ts_trmm(const double* Y, int64_t M, int b, int64_t ldy, const double* R, int64_t ldr, double* Z, int64_t ldz,
             int num_sms, cudaStream_t s, LaunchCounter& lc) {
    if (b > kTrmmMaxB || b <= 0) return false;   // R and two Y stages no longer fit in shared memory
    if (M <= 0) return true;
    TrmmArgs a{};
    a.Y = Y;
    a.M = M;
    a.ldy = ldy;
    a.R = R;
    a.ldr = ldr;
    a.Z = Z;
    a.ldz = ldz;
    a.b = b;
    a.vec2 = ldy % 2 == 0 && reinterpret_cast<uintptr_t>(Y) % 16 == 0;
    const int64_t nblocks = (M + kTrmmRows - 1) / kTrmmRows;
    const int grid = int(std::min<int64_t>(num_sms, nblocks));
    switch ((b + 7) / 8) {
        case 1: launch_trmm<1>(a, grid, s); break;
        case 2: launch_trmm<2>(a, grid, s); break;
        case 3: launch_trmm<3>(a, grid, s); break;
        case 4: launch_trmm<4>(a, grid, s); break;
        case 5: launch_trmm<5>(a, grid, s); break;
        case 6: launch_trmm<6>(a, grid, s); break;
        case 7: launch_trmm<7>(a, grid, s); break;
        case 8: launch_trmm<8>(a, grid, s); break;
        case 9: launch_trmm<9>(a, grid, s); break;
        case 10: launch_trmm<10>(a, grid, s); break;
        case 11: launch_trmm<11>(a, grid, s); break;
        case 12: launch_trmm<12>(a, grid, s); break;
        default: launch_trmm<13>(a, grid, s); break;
    }
    FQB_LAUNCHED();
    lc.bump();
    return true;
}

}  // namespace farqb
