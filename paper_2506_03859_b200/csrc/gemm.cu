// gemm.cu -- FP64 tall-skinny GEMM on the sm_100a DMMA tensor pipe.
//
// Replaces the reference's CPU micro-kernels kern::Ops::gemm_nn / gemm_tn
// (/root/reference/proj/include/rsvd/kernels.hpp:9-19, src/kernels_avx2.cpp:
// 18-218) for every product of the QB loop: Y = A*G, W = A'*Y, the Gram
// matrices, the block Gram-Schmidt projections and the B updates.
//
// FP64 tensor cores on sm_100a are reachable only through warp-level
// mma.sync ... f64 (SASS DMMA.8x8x4); tcgen05 has no kind::f64 (SURVEY.md
// section 0.6).  Measured peak on this pool: 37.1 TFLOP/s (profiles/).
//
// Shape: the outputs are skinny (N = block size b <= 128), so one CTA owns a
// BM x BN tile with BN = 8*NT covering all of b -- A is streamed exactly once
// per product -- and eight warps split BM.  K is streamed through a
// STAGES-deep cp.async ring.  Shared-memory layouts are padded so every DMMA
// fragment load (8 rows x 4 k) costs the minimum two wavefronts:
//   A (NN, m contiguous)  As[k][BM+8]     row pitch = 64 (mod 128) bytes
//   A (TN, k contiguous)  As[m][BK+4]     row pitch 160 B
//   B (k contiguous)      Bs[n][BK+4]
// Split-K partials go to a workspace and are reduced in a fixed order, so
// results are bitwise reproducible run to run.
#include <algorithm>
#include <cstdint>

#include "kernels.hpp"

namespace farqb {
namespace {

constexpr int BK = 16;
constexpr int STAGES = 4;
constexpr int THREADS = 256;
constexpr int WARPS = THREADS / 32;

struct GemmArgs {
    int64_t M, N, K;
    double alpha, beta;
    const double* A;
    int64_t lda;
    const double* B;
    int64_t ldb;
    double* C;
    int64_t ldc;
    double* work;     // split-K partials: splits x (M x N), ld = M
    int64_t kchunk;   // K per split, multiple of BK
    int splits;
    unsigned* counters;  // per-tile arrival counters (zero between launches)
};

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem, int src_bytes) {
    const unsigned s = unsigned(__cvta_generic_to_shared(smem));
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(s), "l"(gmem), "r"(src_bytes));
}
__device__ __forceinline__ void cp_async8(void* smem, const void* gmem, int src_bytes) {
    const unsigned s = unsigned(__cvta_generic_to_shared(smem));
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(s), "l"(gmem), "r"(src_bytes));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                 : "+d"(d0), "+d"(d1)
                 : "d"(a), "d"(b));
}

template <bool TRANS_A, int NT, int WM, int VEC>
struct Cfg {
    static constexpr int BM = WM * WARPS;
    static constexpr int BN = 8 * NT;
    static constexpr int MT = WM / 8;  // m8 tiles per warp
    // NN: As[k][BM+8]; TN: As[m][BK+4]
    static constexpr int A_PITCH = TRANS_A ? (BK + 4) : (BM + 8);
    static constexpr int A_ELEMS = TRANS_A ? BM * (BK + 4) : BK * (BM + 8);
    static constexpr int B_PITCH = BK + 4;
    static constexpr int B_ELEMS = BN * (BK + 4);
    static constexpr int STAGE_ELEMS = A_ELEMS + B_ELEMS;
    static constexpr size_t SMEM = size_t(STAGES) * STAGE_ELEMS * sizeof(double);
};

template <bool TRANS_A, int NT, int WM, int VEC>
__device__ __forceinline__ void load_stage(const GemmArgs& p, double* As, double* Bs, int64_t m0,
                                           int64_t n0, int64_t k0, int64_t kend) {
    using C = Cfg<TRANS_A, NT, WM, VEC>;
    const int tid = threadIdx.x;
    // ---- A ----
    if (!TRANS_A) {
        constexpr int CH_M = C::BM / VEC;  // chunks per k row
        constexpr int CHUNKS = BK * CH_M;
        for (int c = tid; c < CHUNKS; c += THREADS) {
            const int kk = c / CH_M, mm = (c % CH_M) * VEC;
            const int64_t gk = k0 + kk, gm = m0 + mm;
            int bytes = 0;
            const double* src = p.A;
            if (gk < kend && gm < p.M) {
                src = p.A + gk * p.lda + gm;
                const int64_t rem = p.M - gm;
                bytes = int(rem >= VEC ? VEC : rem) * 8;
            }
            double* dst = As + kk * C::A_PITCH + mm;
            if (VEC == 2) cp_async16(dst, src, bytes); else cp_async8(dst, src, bytes);
        }
    } else {
        constexpr int CH_K = BK / VEC;
        constexpr int CHUNKS = C::BM * CH_K;
        for (int c = tid; c < CHUNKS; c += THREADS) {
            const int mm = c / CH_K, kk = (c % CH_K) * VEC;
            const int64_t gk = k0 + kk, gm = m0 + mm;
            int bytes = 0;
            const double* src = p.A;
            if (gk < kend && gm < p.M) {
                src = p.A + gm * p.lda + gk;
                const int64_t rem = kend - gk;
                bytes = int(rem >= VEC ? VEC : rem) * 8;
            }
            double* dst = As + mm * C::A_PITCH + kk;
            if (VEC == 2) cp_async16(dst, src, bytes); else cp_async8(dst, src, bytes);
        }
    }
    // ---- B (k contiguous) ----
    {
        constexpr int CH_K = BK / VEC;
        constexpr int CHUNKS = C::BN * CH_K;
        for (int c = tid; c < CHUNKS; c += THREADS) {
            const int nn = c / CH_K, kk = (c % CH_K) * VEC;
            const int64_t gk = k0 + kk, gn = n0 + nn;
            int bytes = 0;
            const double* src = p.B;
            if (gk < kend && gn < p.N) {
                src = p.B + gn * p.ldb + gk;
                const int64_t rem = kend - gk;
                bytes = int(rem >= VEC ? VEC : rem) * 8;
            }
            double* dst = Bs + nn * C::B_PITCH + kk;
            if (VEC == 2) cp_async16(dst, src, bytes); else cp_async8(dst, src, bytes);
        }
    }
}

template <bool TRANS_A, int NT, int WM, int VEC>
__global__ void __launch_bounds__(THREADS, 1) k_gemm(const GemmArgs p) {
    FQB_PDL_ENTRY();
    using C = Cfg<TRANS_A, NT, WM, VEC>;
    extern __shared__ __align__(16) double smem[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int g = lane >> 2, t = lane & 3;
    const int64_t m0 = int64_t(blockIdx.x) * C::BM;
    const int64_t n0 = int64_t(blockIdx.y) * C::BN;
    const int64_t kbeg = int64_t(blockIdx.z) * p.kchunk;
    const int64_t kend = kbeg + p.kchunk < p.K ? kbeg + p.kchunk : p.K;
    const int ktiles = int((kend - kbeg + BK - 1) / BK);

    double acc[C::MT][NT][2];
#pragma unroll
    for (int i = 0; i < C::MT; ++i)
#pragma unroll
        for (int j = 0; j < NT; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

    auto stage_a = [&](int s) { return smem + s * C::STAGE_ELEMS; };
    auto stage_b = [&](int s) { return smem + s * C::STAGE_ELEMS + C::A_ELEMS; };

#pragma unroll
    for (int s = 0; s < STAGES - 1; ++s) {
        if (s < ktiles) load_stage<TRANS_A, NT, WM, VEC>(p, stage_a(s), stage_b(s), m0, n0, kbeg + s * BK, kend);
        cp_async_commit();
    }
    const int wm0 = warp * WM;
    for (int kt = 0; kt < ktiles; ++kt) {
        cp_async_wait<STAGES - 2>();
        __syncthreads();
        {
            const int nk = kt + STAGES - 1;
            if (nk < ktiles) {
                const int s = nk % STAGES;
                load_stage<TRANS_A, NT, WM, VEC>(p, stage_a(s), stage_b(s), m0, n0, kbeg + int64_t(nk) * BK, kend);
            }
            cp_async_commit();
        }
        const double* As = stage_a(kt % STAGES);
        const double* Bs = stage_b(kt % STAGES);
#pragma unroll
        for (int kk = 0; kk < BK; kk += 4) {
            double af[C::MT], bf[NT];
#pragma unroll
            for (int i = 0; i < C::MT; ++i) {
                const int row = wm0 + i * 8 + g;
                af[i] = TRANS_A ? As[row * C::A_PITCH + kk + t] : As[(kk + t) * C::A_PITCH + row];
            }
#pragma unroll
            for (int j = 0; j < NT; ++j) bf[j] = Bs[(j * 8 + g) * C::B_PITCH + kk + t];
#pragma unroll
            for (int i = 0; i < C::MT; ++i)
#pragma unroll
                for (int j = 0; j < NT; ++j) dmma(acc[i][j][0], acc[i][j][1], af[i], bf[j]);
        }
    }
    cp_async_wait<0>();

    // ---- epilogue: c0, c1 = C[g][2t], C[g][2t+1] of each 8x8 tile ----
    if (p.splits == 1) {
#pragma unroll
        for (int i = 0; i < C::MT; ++i) {
            const int64_t row = m0 + wm0 + i * 8 + g;
            if (row >= p.M) continue;
#pragma unroll
            for (int j = 0; j < NT; ++j) {
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    const int64_t col = n0 + j * 8 + 2 * t + h;
                    if (col >= p.N) continue;
                    double* cp = p.C + col * p.ldc + row;
                    const double v = p.alpha * acc[i][j][h];
                    *cp = p.beta != 0.0 ? fma(p.beta, *cp, v) : v;
                }
            }
        }
    } else {
        double* w = p.work + int64_t(blockIdx.z) * p.M * p.N;
#pragma unroll
        for (int i = 0; i < C::MT; ++i) {
            const int64_t row = m0 + wm0 + i * 8 + g;
            if (row >= p.M) continue;
#pragma unroll
            for (int j = 0; j < NT; ++j) {
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    const int64_t col = n0 + j * 8 + 2 * t + h;
                    if (col < p.N) w[col * p.M + row] = acc[i][j][h];
                }
            }
        }
    }
}

// C = alpha * sum_z work[z] + beta * C.  A CTA covers 32 outputs x 8 split
// lanes: lane q sums splits q, q+8, q+16, ... in order, then the 8 lane sums are
// combined by a fixed shuffle tree -- deterministic, and only splits/8 dependent
// loads per thread instead of `splits`.
__global__ void __launch_bounds__(256) k_splitk_reduce(const double* __restrict__ work, int splits, int64_t M,
                                                       int64_t N, double alpha, double beta, double* C,
                                                       int64_t ldc) {
    FQB_PDL_ENTRY();
    const int q = threadIdx.x & 7;
    const int64_t idx = int64_t(blockIdx.x) * 32 + (threadIdx.x >> 3);
    const int64_t total = M * N;
    double s = 0.0;
    if (idx < total)
        for (int z = q; z < splits; z += 8) s += __ldcg(work + int64_t(z) * total + idx);
    s += __shfl_xor_sync(0xffffffffu, s, 1);
    s += __shfl_xor_sync(0xffffffffu, s, 2);
    s += __shfl_xor_sync(0xffffffffu, s, 4);
    if (q != 0 || idx >= total) return;
    const int64_t col = idx / M, row = idx - col * M;
    double* cp = C + col * ldc + row;
    const double v = alpha * s;
    *cp = beta != 0.0 ? fma(beta, *cp, v) : v;
}

__global__ void k_scale(double* C, int64_t M, int64_t N, int64_t ldc, double beta) {
    FQB_PDL_ENTRY();
    const int64_t idx = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (idx >= M * N) return;
    const int64_t col = idx / M, row = idx - col * M;
    double* cp = C + col * ldc + row;
    *cp = beta != 0.0 ? beta * *cp : 0.0;
}

using KernelFn = void (*)(const GemmArgs);

template <bool TRANS_A, int NT, int WM, int VEC>
KernelFn kernel_for(size_t& smem, int& bm, int& bn) {
    using C = Cfg<TRANS_A, NT, WM, VEC>;
    smem = C::SMEM;
    bm = C::BM;
    bn = C::BN;
    static bool configured[64] = {};  // per device ordinal
    int dev = 0;
    FQB_CUDA(cudaGetDevice(&dev));
    if (dev < 0 || dev >= 64 || !configured[dev]) {
        FQB_CUDA(cudaFuncSetAttribute(k_gemm<TRANS_A, NT, WM, VEC>,
                                      cudaFuncAttributeMaxDynamicSharedMemorySize, int(C::SMEM)));
        if (dev >= 0 && dev < 64) configured[dev] = true;
    }
    return k_gemm<TRANS_A, NT, WM, VEC>;
}

// WM = rows per warp (8, 16 or 32; 32 only while the accumulators fit, NT <= 8)
template <bool TRANS_A, int NT>
KernelFn pick_wm(int wm, size_t& smem, int& bm, int& bn) {
    if constexpr (NT <= 8) {
        if (wm >= 32) return kernel_for<TRANS_A, NT, 32, 2>(smem, bm, bn);
    }
    if (wm >= 16) return kernel_for<TRANS_A, NT, 16, 2>(smem, bm, bn);
    return kernel_for<TRANS_A, NT, 8, 2>(smem, bm, bn);
}

template <bool TRANS_A>
KernelFn pick_vec2(int nt, int wm, size_t& smem, int& bm, int& bn) {
    switch (nt) {
        case 1: return pick_wm<TRANS_A, 1>(wm, smem, bm, bn);
        case 2: return pick_wm<TRANS_A, 2>(wm, smem, bm, bn);
        case 3: return pick_wm<TRANS_A, 3>(wm, smem, bm, bn);
        case 4: return pick_wm<TRANS_A, 4>(wm, smem, bm, bn);
        case 5: return pick_wm<TRANS_A, 5>(wm, smem, bm, bn);
        case 6: return pick_wm<TRANS_A, 6>(wm, smem, bm, bn);
        case 7: return pick_wm<TRANS_A, 7>(wm, smem, bm, bn);
        case 8: return pick_wm<TRANS_A, 8>(wm, smem, bm, bn);
        case 9: return pick_wm<TRANS_A, 9>(wm, smem, bm, bn);
        case 10: return pick_wm<TRANS_A, 10>(wm, smem, bm, bn);
        case 11: return pick_wm<TRANS_A, 11>(wm, smem, bm, bn);
        case 12: return pick_wm<TRANS_A, 12>(wm, smem, bm, bn);
        case 13: return pick_wm<TRANS_A, 13>(wm, smem, bm, bn);
        case 14: return pick_wm<TRANS_A, 14>(wm, smem, bm, bn);
        case 15: return pick_wm<TRANS_A, 15>(wm, smem, bm, bn);
        default: return pick_wm<TRANS_A, 16>(wm, smem, bm, bn);
    }
}

struct Plan {
    KernelFn fn;
    size_t smem;
    int bm, bn;
    int64_t mt, nt_tiles;
    int splits;
    int64_t kchunk;
};

Plan make_plan(bool trans_a, bool vec2, int64_t M, int64_t N, int64_t K, int num_sms) {
    Plan pl{};
    const int nt = int(std::min<int64_t>(16, ceil_div(std::max<int64_t>(N, 1), 8)));
    // the largest warp tile that still yields half a wave of CTAs without split-K
    int wm = nt <= 8 ? 32 : 16;
    while (wm > 8 && ceil_div(M, int64_t(wm) * WARPS) * ceil_div(N, 8 * nt) < num_sms / 2) wm /= 2;
    if (vec2) {
        pl.fn = trans_a ? pick_vec2<true>(nt, wm, pl.smem, pl.bm, pl.bn)
                        : pick_vec2<false>(nt, wm, pl.smem, pl.bm, pl.bn);
    } else {
        pl.fn = trans_a ? kernel_for<true, 16, 16, 1>(pl.smem, pl.bm, pl.bn)
                        : kernel_for<false, 16, 16, 1>(pl.smem, pl.bm, pl.bn);
    }
    pl.mt = ceil_div(M, pl.bm);
    pl.nt_tiles = ceil_div(N, pl.bn);
    const int64_t tiles = pl.mt * pl.nt_tiles;
    const int64_t ktiles = ceil_div(std::max<int64_t>(K, 1), BK);
    int64_t splits = 1;
    if (tiles < num_sms) {
        splits = std::max<int64_t>(1, num_sms / tiles);
        splits = std::min<int64_t>(splits, std::max<int64_t>(1, ktiles / 4));
    }
    pl.splits = int(splits);
    pl.kchunk = ceil_div(ktiles, splits) * BK;
    pl.splits = int(ceil_div(std::max<int64_t>(K, 1), pl.kchunk));
    return pl;
}

}  // namespace

int64_t gemm_workspace_doubles(int64_t m, int64_t n, int64_t k, int num_sms) {
    const Plan pl = make_plan(true, true, m, n, k, num_sms);
    const Plan pn = make_plan(false, true, m, n, k, num_sms);
    const int s = std::max(pl.splits, pn.splits);
    return s > 1 ? int64_t(s) * m * n : 0;
}

void gemm(bool trans_a, int64_t M, int64_t N, int64_t K, double alpha, const double* A, int64_t lda,
          const double* B, int64_t ldb, double beta, double* C, int64_t ldc, GemmWorkspace& ws,
          int num_sms, cudaStream_t s, LaunchCounter& lc) {
    if (M <= 0 || N <= 0) return;
    if (K <= 0 || alpha == 0.0) {
        launch_k(k_scale, unsigned(ceil_div(M * N, 256)), 256, 0, s, C, M, N, ldc, beta);
        FQB_LAUNCHED();
        lc.bump();
        return;
    }
    if (ws.use_tma && ws.flags && gemm_tma_supported(trans_a, M, N, K, lda, ldb, A, B, num_sms) &&
        ws.work_doubles >= gemm_tma_workspace_doubles(num_sms)) {
        if (++ws.epoch == 0) ws.epoch = 1;
        gemm_tma(trans_a, M, N, K, alpha, A, lda, B, ldb, beta, C, ldc, ws.work, ws.flags, ws.epoch, num_sms, s,
                 false);
        lc.bump();
        return;
    }
    double* work = ws.work;
    const int64_t work_doubles = ws.work_doubles;
    const bool vec2 = (lda % 2 == 0) && (ldb % 2 == 0) && (reinterpret_cast<uintptr_t>(A) % 16 == 0) &&
                      (reinterpret_cast<uintptr_t>(B) % 16 == 0);
    Plan pl = make_plan(trans_a, vec2, M, N, K, num_sms);
    if (pl.splits > 1 && int64_t(pl.splits) * M * N > work_doubles) {
        // not enough workspace: fall back to fewer splits on the same kernel
        int64_t fit = work_doubles / (M * N);
        const int64_t ktiles = ceil_div(K, BK);
        if (fit < 2) {
            pl.splits = 1;
            pl.kchunk = ktiles * BK;
        } else {
            pl.kchunk = ceil_div(ktiles, fit) * BK;
            pl.splits = int(ceil_div(K, pl.kchunk));
        }
    }
    GemmArgs a{M, N, K, alpha, beta, A, lda, B, ldb, C, ldc, work, pl.kchunk, pl.splits, nullptr};
    dim3 grid(unsigned(pl.mt), unsigned(pl.nt_tiles), unsigned(pl.splits));
    launch_k(pl.fn, grid, THREADS, pl.smem, s, a);
    FQB_LAUNCHED();
    lc.bump();
    if (pl.splits > 1) {
        launch_k(k_splitk_reduce, unsigned(ceil_div(M * N, 32)), 256, 0, s, work, pl.splits, M, N, alpha, beta, C, ldc);
        FQB_LAUNCHED();
        lc.bump();
    }
}

}  // namespace farqb
