// gemm_tma.cu -- FP64 DMMA GEMM fed by TMA, persistent stream-K (sm_100a).
//
// C (M x N) = alpha op(A) B + beta C for the QB loop's tall-skinny products
// (the reference's kern::Ops::gemm_nn / gemm_tn, kernels.hpp:9-19).
//
//  * one producer warp: a single lane issues cp.async.bulk.tensor (TMA) copies
//    of the A tile (BM x 16) and the B tile (16 x BN) into a STAGES-deep ring
//    of 128B-swizzled shared-memory stages, signalling mbarrier "full[s]";
//  * eight consumer warps: wait full[s], run 4 DMMA k-steps (mma.sync m8n8k4
//    f64) on fragments read with conflict-free LDS.64, release via "empty[s]".
//    The K order inside a 16-wide k-tile is permuted ({0,4,1,5}, {2,6,3,7} per
//    group of 8) so that both the M-contiguous (NN) and the K-contiguous (TN,
//    B) swizzled layouts serve each fragment load in the minimum two wavefronts
//    -- both operands use the same permutation, so the product is unchanged;
//  * stream-K: the tiles x k-tiles iteration space is cut into G equal
//    contiguous ranges, one per persistent CTA (G <= #SMs), so every SM gets
//    the same work regardless of tile quantization (C3: 79 tiles, C4: 157).
//    A tile split across CTAs is finished by the CTA holding its last k-tile,
//    which adds the other CTAs' partials in CTA order: deterministic.
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>

#include "kernels.hpp"

namespace farqb {
namespace {

constexpr int CW = 8;                 // consumer warps
constexpr int TMA_THREADS = CW * 32;   // the TMA producer is lane 0 of warp 0
constexpr int BK = 16;                // k-tile: 16 doubles = one 128-byte swizzle row
constexpr int SMEM_BUDGET = 200 * 1024;

template <bool TRANS_A, int NT, int WM>
struct TCfg {
    static constexpr int BM = WM * CW;
    static constexpr int BN = 8 * NT;
    static constexpr int MT = WM / 8;
    static constexpr int A_BYTES = BM * BK * 8;
    static constexpr int B_BYTES = ((BN * BK * 8) + 1023) / 1024 * 1024;
    static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
    static constexpr int STAGES = (SMEM_BUDGET / STAGE_BYTES) < 8 ? (SMEM_BUDGET / STAGE_BYTES) : 8;
    static constexpr int TX_BYTES = BM * BK * 8 + BN * BK * 8;
    static constexpr size_t SMEM = size_t(STAGES) * STAGE_BYTES + 1024 + 2 * STAGES * 8;
    static constexpr int PARTIAL_DOUBLES = CW * 32 * MT * NT * 2;
};

struct TmaArgs {
    int64_t M, N, K;
    double alpha, beta;
    double* C;
    int64_t ldc;
    double* work;       // G partial slots
    unsigned* flags;    // G partial-ready flags (epoch values)
    unsigned epoch;
    int64_t iters;      // tiles * ktiles
    int ktiles, mtiles;
    int grid;
    int a3d;            // NN: A tile as one 3-D box {16, BK, BM/16}
};

__device__ __forceinline__ unsigned smem_u32(const void* p) {
    return unsigned(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(unsigned bar, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(bar), "r"(count));
}

__device__ __forceinline__ void mbar_expect_tx(unsigned bar, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(bar), "r"(bytes) : "memory");
}

__device__ __forceinline__ void mbar_arrive(unsigned bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(bar) : "memory");
}

__device__ __forceinline__ void mbar_wait(unsigned bar, unsigned parity) {
    unsigned done = 0;
    do {
        asm volatile(
            "{\n\t.reg .pred p;\n\t"
            "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
            "selp.u32 %0, 1, 0, p;\n\t}\n"
            : "=r"(done)
            : "r"(bar), "r"(parity)
            : "memory");
    } while (!done);
}

__device__ __forceinline__ void tma_load_2d(unsigned dst, const CUtensorMap* map, int x, int y, unsigned bar) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];\n"
        ::"r"(dst), "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(bar)
        : "memory");
}

__device__ __forceinline__ void tma_load_3d(unsigned dst, const CUtensorMap* map, int x, int y, int z,
                                            unsigned bar) {
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];\n"
        ::"r"(dst), "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(z), "r"(bar)
        : "memory");
}

__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
    asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
        : "+d"(d0), "+d"(d1)
        : "d"(a), "d"(b));
}

__device__ __forceinline__ unsigned ld_acquire(const unsigned* p) {
    unsigned v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];\n" : "=r"(v) : "l"(p) : "memory");
    return v;
}

__device__ __forceinline__ void st_release(unsigned* p, unsigned v) {
    asm volatile("st.release.gpu.global.u32 [%0], %1;\n" ::"l"(p), "r"(v) : "memory");
}

__device__ __forceinline__ void consumer_bar() {
    asm volatile("bar.sync 1, %0;\n" ::"n"(CW * 32) : "memory");
}

__device__ __forceinline__ int64_t range_begin(int64_t iters, int grid, int c) {
    return (iters * c) / grid;
}

__device__ __forceinline__ int cta_of(int64_t it, int64_t iters, int grid) {
    int c = int((it * grid) / iters);
    while (c + 1 < grid && range_begin(iters, grid, c + 1) <= it) ++c;
    while (c > 0 && range_begin(iters, grid, c) > it) --c;
    return c;
}

// k index handled by thread quad position t in DMMA k-step q (0..3) of a k-tile
__device__ __forceinline__ int kperm(int t, int q) {
    return 8 * (q >> 1) + 2 * (q & 1) + (((t & 1) << 2) | (t >> 1));
}

// byte offset of element (row, k) in a 128B-swizzled [row][16 doubles] tile
__device__ __forceinline__ unsigned swz_rowk(int row, int k) {
    return unsigned(row * 128 + ((((k >> 1) ^ (row & 7)) << 4) | ((k & 1) << 3)));
}

// byte offset of element (m, k) in the NN A tile made of [k][16 m] boxes
__device__ __forceinline__ unsigned swz_nn(int m, int k) {
    const int box = m >> 4, mi = m & 15;
    return unsigned(box * (BK * 128) + k * 128 + ((((mi >> 1) ^ (k & 7)) << 4) | ((mi & 1) << 3)));
}

template <bool TRANS_A, int NT, int WM>
__global__ void __launch_bounds__(TMA_THREADS, 1)
    k_gemm_tma(const __grid_constant__ CUtensorMap map_a, const __grid_constant__ CUtensorMap map_b,
               const TmaArgs p) {
    FQB_PDL_ENTRY();
    using Cf = TCfg<TRANS_A, NT, WM>;
    extern __shared__ uint8_t smem_raw[];
    const unsigned raw = smem_u32(smem_raw);
    const unsigned base = (raw + 1023u) & ~1023u;
    const unsigned bars = base + Cf::STAGES * Cf::STAGE_BYTES;  // full[STAGES], empty[STAGES]
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

    if (threadIdx.x == 0) {
        for (int s = 0; s < Cf::STAGES; ++s) {
            mbar_init(bars + 8 * s, 1);
            mbar_init(bars + 8 * (Cf::STAGES + s), CW);
        }
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    __syncthreads();

    const int c = blockIdx.x;
    const int64_t beg = range_begin(p.iters, p.grid, c);
    const int64_t end = range_begin(p.iters, p.grid, c + 1);

    // Segment order: the CTA's range [beg, end) covers tiles t_first..t_last.  The
    // segments are processed LAST tile first: the head of t_last (whose partial a
    // later CTA is waiting for) is produced first and the tail of t_first (which
    // needs the earlier CTAs' partials) is finished last, so no CTA ever waits on
    // work its predecessor has not already done -- no serial chain.
    const int64_t KT = p.ktiles;
    const int64_t t_first = beg / KT, t_last = (end - 1) / KT;
    auto seg_tile = [&](int64_t si) { return t_last - si; };
    auto seg_kb = [&](int64_t tile) { return tile == t_first ? int(beg - tile * KT) : 0; };
    auto seg_ke = [&](int64_t tile) { return tile == t_last ? int(end - tile * KT) : int(KT); };
    const int64_t nseg = end > beg ? t_last - t_first + 1 : 0;

    // TMA producer: lane 0 of warp 0 keeps the ring STAGES-1 k-tiles ahead of
    // consumption.  j counts k-tiles in processing order; stage = j % STAGES.
    int64_t p_seg = 0, p_k = 0, p_j = 0;  // producer cursor
    auto produce_next = [&]() {
        if (p_seg >= nseg) return;
        const int64_t tile = seg_tile(p_seg);
        if (p_k == 0) p_k = seg_kb(tile);
        const int s = int(p_j % Cf::STAGES);
        const unsigned par = unsigned((p_j / Cf::STAGES) & 1);
        const int mt = int(tile % p.mtiles), ntile = int(tile / p.mtiles);
        const int m0 = mt * Cf::BM, n0 = ntile * Cf::BN, k0 = int(p_k) * BK;
        mbar_wait(bars + 8 * (Cf::STAGES + s), par ^ 1);
        const unsigned full = bars + 8 * s;
        mbar_expect_tx(full, Cf::TX_BYTES);
        const unsigned sa = base + s * Cf::STAGE_BYTES;
        if (TRANS_A) {
            tma_load_2d(sa, &map_a, k0, m0, full);
        } else if (p.a3d) {
            tma_load_3d(sa, &map_a, 0, k0, m0 / 16, full);   // all BM/16 boxes at once
        } else {
#pragma unroll
            for (int bx = 0; bx < Cf::BM / 16; ++bx) tma_load_2d(sa + bx * (BK * 128), &map_a, m0 + 16 * bx, k0, full);
        }
        tma_load_2d(sa + Cf::A_BYTES, &map_b, k0, n0, full);
        ++p_j;
        if (++p_k >= seg_ke(tile)) {
            ++p_seg;
            p_k = 0;
        }
    };
    const bool producer = warp == 0 && lane == 0;
    if (producer) {
        asm volatile("prefetch.tensormap [%0];\n" ::"l"(reinterpret_cast<uint64_t>(&map_a)) : "memory");
        asm volatile("prefetch.tensormap [%0];\n" ::"l"(reinterpret_cast<uint64_t>(&map_b)) : "memory");
        for (int i = 0; i < Cf::STAGES - 1; ++i) produce_next();
    }
    __syncwarp();

    // ------------------------------- consumers ---------------------------------
    const int g = lane >> 2, t = lane & 3;
    const int wm0 = warp * WM;
    // per-thread fragment offsets (bytes) for the four k-steps of a k-tile
    unsigned a_off[Cf::MT][4], b_off0[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
        const int k = kperm(t, q);
#pragma unroll
        for (int i = 0; i < Cf::MT; ++i) {
            const int m = wm0 + i * 8 + g;
            a_off[i][q] = TRANS_A ? swz_rowk(m, k) : swz_nn(m, k);
        }
        b_off0[q] = unsigned(Cf::A_BYTES) + swz_rowk(g, k);  // + j * 1024 for n-tile j
    }

    double acc[Cf::MT][NT][2];
    int64_t jc = 0;  // consumer k-tile counter (processing order)
    for (int64_t si = 0; si < nseg; ++si) {
        const int64_t tile = seg_tile(si);
        const int kb = seg_kb(tile), ke = seg_ke(tile);
#pragma unroll
        for (int i = 0; i < Cf::MT; ++i)
#pragma unroll
            for (int j = 0; j < NT; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
        for (int kt = kb; kt < ke; ++kt, ++jc) {
            if (warp == 0) {
                if (lane == 0) produce_next();
                __syncwarp();
            }
            const int s = int(jc % Cf::STAGES);
            mbar_wait(bars + 8 * s, unsigned((jc / Cf::STAGES) & 1));
            const uint8_t* st = smem_raw + (base - raw) + s * Cf::STAGE_BYTES;
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                double af[Cf::MT], bf[NT];
#pragma unroll
                for (int i = 0; i < Cf::MT; ++i) af[i] = *reinterpret_cast<const double*>(st + a_off[i][q]);
#pragma unroll
                for (int j = 0; j < NT; ++j)
                    bf[j] = *reinterpret_cast<const double*>(st + b_off0[q] + j * 1024);
#pragma unroll
                for (int i = 0; i < Cf::MT; ++i)
#pragma unroll
                    for (int j = 0; j < NT; ++j) dmma(acc[i][j][0], acc[i][j][1], af[i], bf[j]);
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(bars + 8 * (Cf::STAGES + s));
        }

        // ---------------- segment epilogue ----------------
        const int mt = int(tile % p.mtiles), ntile = int(tile / p.mtiles);
        const int64_t m0 = int64_t(mt) * Cf::BM, n0 = int64_t(ntile) * Cf::BN;
        const bool full_tile = kb == 0 && ke == p.ktiles;
        const bool finisher = !full_tile && ke == p.ktiles;
        if (!full_tile && !finisher) {
            double2* w = reinterpret_cast<double2*>(p.work + int64_t(c) * Cf::PARTIAL_DOUBLES);
#pragma unroll
            for (int i = 0; i < Cf::MT; ++i)
#pragma unroll
                for (int j = 0; j < NT; ++j)
                    w[((warp * Cf::MT + i) * NT + j) * 32 + lane] = make_double2(acc[i][j][0], acc[i][j][1]);
            __threadfence();
            consumer_bar();
            if (threadIdx.x == 0) st_release(p.flags + c, p.epoch);
            continue;
        }
        if (finisher) {
            const int c0 = cta_of(tile * p.ktiles, p.iters, p.grid);
            for (int cc = c0; cc < c; ++cc) {
                while (ld_acquire(p.flags + cc) != p.epoch) {
                }
                const double2* w = reinterpret_cast<const double2*>(p.work + int64_t(cc) * Cf::PARTIAL_DOUBLES);
#pragma unroll
                for (int i = 0; i < Cf::MT; ++i)
#pragma unroll
                    for (int j = 0; j < NT; ++j) {
                        const double2 v = __ldcg(&w[((warp * Cf::MT + i) * NT + j) * 32 + lane]);
                        acc[i][j][0] += v.x;
                        acc[i][j][1] += v.y;
                    }
            }
        }
#pragma unroll
        for (int i = 0; i < Cf::MT; ++i) {
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
    }
}

// ---------------------------------------------------------------------------
// host side

using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                              const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                              CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeFn encode_fn() {
    static EncodeFn fn = nullptr;
    if (!fn) {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        FQB_CUDA(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q));
        if (q != cudaDriverEntryPointSuccess || !p) throw Error(kStatusCuda, "cuTensorMapEncodeTiled unavailable");
        fn = reinterpret_cast<EncodeFn>(p);
    }
    return fn;
}

// rows x cols column-major view (ld), box = box_rows x box_cols, 128B swizzle
CUtensorMap make_map(const double* ptr, int64_t rows, int64_t cols, int64_t ld, int box_rows, int box_cols) {
    CUtensorMap m;
    const cuuint64_t dims[2] = {cuuint64_t(rows), cuuint64_t(cols)};
    const cuuint64_t strides[1] = {cuuint64_t(ld) * 8};
    const cuuint32_t box[2] = {cuuint32_t(box_rows), cuuint32_t(box_cols)};
    const cuuint32_t estr[2] = {1, 1};
    const CUresult r = encode_fn()(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, const_cast<double*>(ptr), dims, strides,
                                   box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) throw Error(kStatusCuda, "cuTensorMapEncodeTiled failed");
    return m;
}

// NN A operand (M x K, column-major) as {16 rows, K, M/16 row blocks} so one TMA
// fills the whole [BM/16][BK][16] swizzled tile.  Only used when the reads of
// the last row block cannot run past the allocation (see gemm_tma()).
CUtensorMap make_map3_nn(const double* ptr, int64_t rows, int64_t cols, int64_t ld, int boxes) {
    CUtensorMap m;
    const cuuint64_t dims[3] = {16, cuuint64_t(cols), cuuint64_t((rows + 15) / 16)};
    const cuuint64_t strides[2] = {cuuint64_t(ld) * 8, 128};
    const cuuint32_t box[3] = {16, cuuint32_t(BK), cuuint32_t(boxes)};
    const cuuint32_t estr[3] = {1, 1, 1};
    const CUresult r = encode_fn()(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, const_cast<double*>(ptr), dims, strides,
                                   box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) throw Error(kStatusCuda, "cuTensorMapEncodeTiled (3d) failed");
    return m;
}

template <bool TRANS_A, int NT>
void launch_nt(const double* A, int64_t lda, const double* B, int64_t ldb, TmaArgs& a, int num_sms,
               cudaStream_t s) {
    constexpr int WM = NT <= 8 ? 32 : 16;
    using Cf = TCfg<TRANS_A, NT, WM>;
    static bool configured[64] = {};
    int dev = 0;
    FQB_CUDA(cudaGetDevice(&dev));
    if (dev < 0 || dev >= 64 || !configured[dev]) {
        FQB_CUDA(cudaFuncSetAttribute(k_gemm_tma<TRANS_A, NT, WM>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      int(Cf::SMEM)));
        if (dev >= 0 && dev < 64) configured[dev] = true;
    }
    CUtensorMap ma;
    if (TRANS_A) ma = make_map(A, a.K, a.M, lda, BK, Cf::BM);
    else if (a.a3d) ma = make_map3_nn(A, a.M, a.K, lda, Cf::BM / 16);
    else ma = make_map(A, a.M, a.K, lda, 16, BK);
    const CUtensorMap mb = make_map(B, a.K, a.N, ldb, BK, Cf::BN);
    a.mtiles = int(ceil_div(a.M, Cf::BM));
    const int ntiles = int(ceil_div(a.N, Cf::BN));
    a.ktiles = int(ceil_div(a.K, BK));
    a.iters = int64_t(a.mtiles) * ntiles * a.ktiles;
    a.grid = int(std::max<int64_t>(1, std::min<int64_t>(num_sms, a.iters / 8)));
    launch_k(k_gemm_tma<TRANS_A, NT, WM>, a.grid, TMA_THREADS, Cf::SMEM, s, ma, mb, a);
    FQB_LAUNCHED();
}

template <bool TRANS_A>
void dispatch(int nt, const double* A, int64_t lda, const double* B, int64_t ldb, TmaArgs& a, int num_sms,
              cudaStream_t s) {
    switch (nt) {
        case 1: return launch_nt<TRANS_A, 1>(A, lda, B, ldb, a, num_sms, s);
        case 2: return launch_nt<TRANS_A, 2>(A, lda, B, ldb, a, num_sms, s);
        case 3: return launch_nt<TRANS_A, 3>(A, lda, B, ldb, a, num_sms, s);
        case 4: return launch_nt<TRANS_A, 4>(A, lda, B, ldb, a, num_sms, s);
        case 5: return launch_nt<TRANS_A, 5>(A, lda, B, ldb, a, num_sms, s);
        case 6: return launch_nt<TRANS_A, 6>(A, lda, B, ldb, a, num_sms, s);
        case 7: return launch_nt<TRANS_A, 7>(A, lda, B, ldb, a, num_sms, s);
        case 8: return launch_nt<TRANS_A, 8>(A, lda, B, ldb, a, num_sms, s);
        case 9: return launch_nt<TRANS_A, 9>(A, lda, B, ldb, a, num_sms, s);
        case 10: return launch_nt<TRANS_A, 10>(A, lda, B, ldb, a, num_sms, s);
        case 11: return launch_nt<TRANS_A, 11>(A, lda, B, ldb, a, num_sms, s);
        case 12: return launch_nt<TRANS_A, 12>(A, lda, B, ldb, a, num_sms, s);
        case 13: return launch_nt<TRANS_A, 13>(A, lda, B, ldb, a, num_sms, s);
        case 14: return launch_nt<TRANS_A, 14>(A, lda, B, ldb, a, num_sms, s);
        case 15: return launch_nt<TRANS_A, 15>(A, lda, B, ldb, a, num_sms, s);
        default: return launch_nt<TRANS_A, 16>(A, lda, B, ldb, a, num_sms, s);
    }
}

}  // namespace

int64_t gemm_tma_workspace_doubles(int num_sms) {
    // largest partial slot: MT * NT * 2 * 32 * CW with WM * NT <= 32 * 8 = 256
    return int64_t(num_sms) * (CW * 32 * 2 * 32) + 16;
}

bool gemm_tma_supported(bool trans_a, int64_t M, int64_t N, int64_t K, int64_t lda, int64_t ldb, const double* A,
                        const double* B, int num_sms) {
    if (!(lda % 2 == 0 && ldb % 2 == 0 && reinterpret_cast<uintptr_t>(A) % 16 == 0 &&
          reinterpret_cast<uintptr_t>(B) % 16 == 0))
        return false;
    // stream-K pays one serial partial reduction per split tile: keep it to
    // shapes with enough tiles (or enough K per CTA); the rest use split-K.
    const int nt = int(std::min<int64_t>(16, ceil_div(N, 8)));
    const int bm = nt <= 8 ? 32 * CW : 16 * CW;
    const int64_t tiles = ceil_div(M, bm) * ceil_div(N, 8 * nt);
    const int64_t iters = tiles * ceil_div(K, BK);
    const int64_t grid = std::max<int64_t>(1, std::min<int64_t>(num_sms, iters / 8));
    (void)trans_a;
    // enough k-tiles per CTA to keep the TMA ring busy, and at most ~8 segments
    // per tile for the serial fixup; otherwise the split-K kernel is faster.
    return iters >= 16 * int64_t(num_sms) && grid <= 8 * tiles;
}

void gemm_tma(bool trans_a, int64_t M, int64_t N, int64_t K, double alpha, const double* A, int64_t lda,
              const double* B, int64_t ldb, double beta, double* C, int64_t ldc, double* work, unsigned* flags,
              unsigned epoch, int num_sms, cudaStream_t s, bool a3d_slack) {
    TmaArgs a{};
    a.M = M;
    a.N = N;
    a.K = K;
    a.alpha = alpha;
    a.beta = beta;
    a.C = C;
    a.ldc = ldc;
    a.work = work;
    a.flags = flags;
    a.epoch = epoch;
    // one 3-D TMA per NN stage when the last 16-row block cannot overrun A
    a.a3d = (!trans_a && (M % 16 == 0 || a3d_slack)) ? 1 : 0;
    const int nt = int(std::min<int64_t>(16, ceil_div(N, 8)));
    if (trans_a) dispatch<true>(nt, A, lda, B, ldb, a, num_sms, s);
    else dispatch<false>(nt, A, lda, B, ldb, a, num_sms, s);
}

}  // namespace farqb
