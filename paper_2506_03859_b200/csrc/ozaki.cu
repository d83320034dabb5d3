// ozaki.cu -- FP64 GEMM emulated on the INT8 tcgen05 tensor cores (Ozaki scheme I).
//
// For the passes over A the FP64 DMMA pipe (37 TFLOP/s) is the bound; B200's INT8
// tensor cores (tcgen05 kind::i8, 4.5 POPS dense) are not.  Each operand is cut
// into signed integer slices with a power-of-two scale per output row / column.
// Default (NSL = 7): for a row x of A with 2^(e-1) <= max|x| < 2^e,
//     x = 2^e ( 2^-6 x_0 + 2^-14 x_1 + ... + 2^-54 x_6 ) + r,
//     |x_0| <= 64, |x_p| <= 128, |r| <= 2^(e-55)
// (8-bit digits of R = rint(x 2^(54-e)), see digits7).  Then
//     (A Z)_ij = 2^(e_i + f_j) sum_{p+q <= 7} 2^(-12 - 8(p+q)) (A_p Z_q)_ij
// where every A_p Z_q is an exact int32 product on the tensor cores and the 34
// products collapse into 8 diagonals d = p+q (same power of two), accumulated
// in TMEM (8 x 64 int32 columns = all 512).  The epilogue adds the diagonals
// from the least significant up in FP64 and applies the exponents.  The
// dropped terms (d >= 8: 5 products, ~2^-59) and r are below 2^-54 relative to
// max|row| * max|col|.  The bound is NORMWISE per line, not elementwise: an entry
// much smaller than its line's maximum keeps only ~54 - log2(max/|x|) bits, so a
// product is FP64-class relative to max|row_i(A)| * max|col_j(Z)|, which is the
// class of the normwise FP64 GEMM bound K u |A_i| |Z_j| the QB loop's parity bars
// rest on (tests/test_gpu_ozaki.py: graded-line products and QB runs on matrices
// whose lines span 1e-8..1, against the oracle).  NSL = 8 is the
// same with 7-bit digits (R = rint(x 2^(55-e)), 36 products, 8 bytes per element);
// NSL = 4 the FP32-class variant for FP32 input.
//
// The slices of A are made once per run (A is fixed for all 2P+2 passes), in
// two layouts: scaled per column for A'Y (K = m contiguous, A's own layout)
// and per row, transposed, for A G (K = n contiguous).  A pass then streams
// 7 bytes of slices per element of A -- less than FP64's 8 -- so it becomes
// HBM bound instead of FP64 bound.
//
// Slices are stored pre-tiled and pre-swizzled: tile (row tile, k-block, slice)
// is one contiguous TR x 64 B block already in the 64B-swizzle arrangement
// tcgen05 expects, so every pipeline stage is a single 1-D bulk copy
// (cp.async.bulk) -- no per-row TMA requests.  Kernel: one producer warp (8 KB
// A-slice tiles, all Z slices of a k-block in one copy, ~165 KB of A in
// flight), one MMA warp (tcgen05.mma.cta_group::1.kind::i8, M=128, K=32, N = 64
// per Z slice: the products of one A slice with up to 4 consecutive Z slices
// land on consecutive TMEM diagonals, so one N<=256 MMA covers them and A is
// read from shared memory once per 4 products; chunks of <= 56 columns use 56-row Z
// slices and the wide schedule of issue_s56: 12 MMAs of N <= 256 per k-step for all 34
// products), four epilogue warps (tcgen05.ld 32x32b -> FP64).  Tiles are split over the persistent grid
// stream-K style; a CTA writes pieces of split tiles, already scaled, to its
// partial slots and k_ozaki_fixup sums them in CTA order (deterministic).
//
// Measured (C2, A'Y 8000x50x8000, B200, NSL = 7): 104-106 us + 3 us fixup, vs 235 us
// for the FP64 DMMA GEMM; HBM floor for the 448 MB of A slices ~70 us.
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdint>
#include <cstdlib>

#include "kernels.hpp"

namespace farqb {
namespace {

constexpr int OZ_BM = 128;               // rows per tile (UMMA M)
// K bytes per k-block: one 64-byte swizzle row.  64 rather than 128 halves the Z
// stage (all 8 slices of a k-block) and so doubles the A-slice bytes in flight.
constexpr int OZ_BK = 64;
constexpr int SWZ_ROWS = 1024 / 128;     // the swizzle pattern repeats every 8 rows (SBO = 8 rows)
constexpr int OZ_BN = 64;                // max N (8 diagonals x 64 = 512 TMEM columns)
constexpr int A_TILE = OZ_BM * OZ_BK;             // 8 KB, one slice
constexpr int B_TILE = OZ_BN * OZ_BK;             // 4 KB per slice (bn = 64)
// Per slice count NSL: 7 (FP64-class, the default: 8-bit digits, diagonals d = p+q <= 7,
// 34 products), 8 (FP64-class, 7-bit digits, d <= 7, 36 products), 4 (FP32-class for FP32
// input, 7-bit digits, d <= 3, 10 products), 3 (FP32-class, 8-bit digits, d <= 3, 8 products).  The Z stage holds all NSL slices of a k-block, the rest
// of 225 KB is the A ring, TMEM holds ND diagonals of 64 columns.
// Z rows per k-block of the slices of one column chunk: NSL slices of S rows each (S = 64,
// or S = 56 for chunks of <= 56 columns, then with 8 zero rows after the last slice that
// the N = 64 lone products of the S = 56 schedule read past it)
// Zero rows after the last slice that the schedules read past it: 8 for S = 56 (the N = 64
// lone products), 2 for S = 50 (the N = 96 MMAs of slices 0 / 1 cover rows 256..351).
__host__ __device__ constexpr int z_pad_rows(int S) { return S == 56 ? 8 : S == 50 ? 2 : 0; }
__host__ __device__ constexpr int z_block_rows(int nsl, int S) { return nsl * S + z_pad_rows(S); }

template <int NSL, int BS = 2, int S = 64, int NDK = 0>
struct Sl {
    static constexpr int B_STAGES = BS;                                            // Z stages (2 or 3)
    static constexpr int W = (NSL == 7 || NSL == 3) ? 8 : 7;                        // bits per digit
    // diagonals kept (NDK = 7 with NSL = 7: the trimmed variant, FQB_OZ_DIAGS=7)
    static constexpr int ND = NDK ? NDK : NSL == 7 ? 8 : NSL == 3 ? 4 : NSL;
    static constexpr int B_STAGE = z_block_rows(NSL, S) * OZ_BK;                   // 28 / 32 / 16 KB (25 KB at S = 56)
    static constexpr int A_STAGES = (225 * 1024 - B_STAGES * B_STAGE) / A_TILE;     // 21 / 20 / 24
    static constexpr size_t SMEM = size_t(A_STAGES) * A_TILE + size_t(B_STAGES) * B_STAGE + 1024;
    static constexpr unsigned TMEM_COLS = ND > 4 ? 512u : unsigned(ND * OZ_BN);    // a power of two: 512 / 256
    // k-blocks per TMEM accumulation (int32 headroom).  7-bit digits: at most 8 products
    // of |d| <= 64 per diagonal, 8 * 64^2 * 32768 = 2^30.  8-bit digits (|d| <= 128, the top
    // digit |d_0| <= 64): diagonal d sums the products p + q = d, at most 6 of size 2^14
    // (d = 6: two with the top digit, 2^13 each, plus five; d = 7: six) -> 6 * 2^14 per
    // element of K, so K <= 21845; 336 k-blocks (21504) keep every diagonal < 2^31.  (What
    // the schedules spill onto diagonal 8 is never read.)  The 4-diagonal FP32 scheme keeps
    // the old 256.  336 puts a whole K = 20000 A G pass into one accumulation (two with 256).
    static constexpr int CHUNK_KB = W == 7 ? 32768 / OZ_BK : (ND >= 7 ? 336 : 16384 / OZ_BK);
};
constexpr int OZ_THREADS = 192;                   // producer, MMA, 4 epilogue warps
// the MN-major (AMN) products have short K, so each row tile's TMEM drain is on the MMA's
// critical path: they split it over 8 epilogue warps (two per TMEM lane quarter, each
// draining half of the column groups)
constexpr int oz_threads(bool amn) { return amn ? OZ_THREADS + 128 : OZ_THREADS; }
constexpr int OZ_PARTIAL = OZ_BM * OZ_BN;         // doubles per CTA partial slot

// 64-bit quotient through a double reciprocal and one correction step (operands are
// far below 2^48).  The kernel must not contain a division subroutine call: a call
// anywhere in it pushes the MMA issue path out of the uniform datapath (~1.3x slower).
// inv_b is 1/b rounded on the host.
__device__ __forceinline__ int64_t qdiv(int64_t a, int64_t b, double inv_b) {
    int64_t q = int64_t(double(a) * inv_b);
    if (q * b > a) --q;
    else if ((q + 1) * b <= a) ++q;
    return q;
}

// x * 2^k without ldexp() (a long library routine: 64 of them per thread made the
// finishing epilogue take ~14 us).  Exact whenever the result is a normal number;
// |k| up to 2046 through two factors.
__device__ __forceinline__ int64_t round_up_dev(int64_t x, int64_t r) { return (x + r - 1) / r * r; }
__device__ __forceinline__ double pow2i(int k) {   // k in [-1022, 1023]
    return __longlong_as_double(static_cast<long long>(k + 1023) << 52);
}
constexpr int kNonFiniteE = 1 << 20;   // line exponent of a line holding Inf/NaN
__device__ __forceinline__ double mul_pow2(double x, int k) {
    if (k >= -1022 && k <= 1023) return x * pow2i(k);
    // an output touching a non-finite input line is NaN (the digits are meaningless)
    if (k > kNonFiniteE / 2) return __longlong_as_double(0x7FF8000000000000LL);
    const int k1 = max(-1022, min(1023, k / 2));
    const int k2 = max(-1022, min(1023, k - k1));
    return x * pow2i(k1) * pow2i(k2);
}

struct OzArgs {
    const int8_t* xs;     // tiled slices of the K x M operand
    const int8_t* zs;     // tiled slices of the K x N operand (one row tile of bn)
    int64_t M, N, K;
    double alpha, beta;
    double* C;
    int64_t ldc;
    const int* ex;        // per output row exponent
    const int* ez;        // per output column exponent
    double* work;         // 2 * grid slots: partials, then carries
    int64_t iters;        // tiles * kblocks
    int kblocks, mtiles, grid, bn;
    double inv_grid, inv_kblocks, inv_iters;
    // paired launch (pair = 1): clusters of two CTAs stream the same A tiles, each
    // loading half of every k-block's slices multicast into both; CTA rank r
    // computes column chunk r: zs + r zs_stride, ez + 64 r, C + r cw ldc, N_r =
    // min(cw, N - r cw), work + r work_stride.  grid counts clusters.
    int pair;
    int64_t zs_stride, cw, work_stride;
    // L2 policy of the bulk copies: A slices evict-first (streamed once per pass), Z
    // slices evict-last (re-read by every row tile; the pairs walk different k ranges)
    int l2hint;
    // AMN launches: xs are the A'Y-layout (column-scaled, K-major) slices of an operand X
    // (rows = K of this product, x_kb k-blocks of 64 of them), read MN-major as A = X
    int64_t x_kb;
    // k-blocks per TMEM accumulation, <= Sl::CHUNK_KB (int32 headroom); FQB_OZ_CHUNK lowers it
    int chunk_kb;
};

// this CTA's (or fixup block's) column chunk of a paired launch
__device__ __forceinline__ OzArgs chunk_args(const OzArgs& p, int r) {
    OzArgs q = p;
    if (p.pair) {
        q.zs = p.zs + r * p.zs_stride;
        q.ez = p.ez + r * OZ_BN;
        q.C = p.C + r * p.cw * p.ldc;
        q.N = min(p.cw, p.N - r * p.cw);
        q.work = p.work + r * p.work_stride;
    }
    return q;
}

__device__ __forceinline__ int64_t range_begin(const OzArgs& p, int c) { return qdiv(p.iters * c, p.grid, p.inv_grid); }
// the CTA whose range holds iteration it: largest c with range_begin(c) <= it
__device__ __forceinline__ int cta_of(const OzArgs& p, int64_t it) {
    return int(qdiv((it + 1) * p.grid - 1, p.iters, p.inv_iters));
}

__device__ __forceinline__ unsigned smem_u32(const void* p) { return unsigned(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ void mbar_init(unsigned bar, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(bar), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(unsigned bar, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(bar), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(unsigned bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(bar) : "memory");
}
// the spin loop lives inside the asm (no outputs), so the compiler does not treat the
// code after a wait as divergent and keeps the MMA descriptors in uniform registers
__device__ __forceinline__ void mbar_wait(unsigned bar, unsigned parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra WAIT_%=;\n\t}\n" ::"r"(bar), "r"(parity) : "memory");
}
// one 1-D bulk copy landing at the same offset in both CTAs of the pair, completing
// transaction bytes on the mbarrier at the same offset in each
__device__ __forceinline__ void bulk_load_mc2(unsigned dst, const void* src, unsigned bytes, unsigned bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.multicast::cluster [%0], [%1], %2, [%3], "
        "%4;\n" ::"r"(dst),
        "l"(reinterpret_cast<uint64_t>(src)), "r"(bytes), "r"(bar), "h"((unsigned short)3)
        : "memory");
}
__device__ __forceinline__ void bulk_load_mc2_hint(unsigned dst, const void* src, unsigned bytes, unsigned bar,
                                                   uint64_t pol) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.multicast::cluster.L2::cache_hint [%0], "
        "[%1], %2, [%3], %4, %5;\n" ::"r"(dst),
        "l"(reinterpret_cast<uint64_t>(src)), "r"(bytes), "r"(bar), "h"((unsigned short)3), "l"(pol)
        : "memory");
}
__device__ __forceinline__ void bulk_load_hint(unsigned dst, const void* src, unsigned bytes, unsigned bar,
                                               uint64_t pol) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;\n"
        ::"r"(dst), "l"(reinterpret_cast<uint64_t>(src)), "r"(bytes), "r"(bar), "l"(pol) : "memory");
}
__device__ __forceinline__ uint64_t policy_evict_first() {
    uint64_t pol;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;\n" : "=l"(pol));
    return pol;
}
__device__ __forceinline__ uint64_t policy_evict_last() {
    uint64_t pol;
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;\n" : "=l"(pol));
    return pol;
}
__device__ __forceinline__ void cluster_sync() {
    asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;\n" ::: "memory");
}
__device__ __forceinline__ void bulk_load(unsigned dst, const void* src, unsigned bytes, unsigned bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n"
                 ::"r"(dst), "l"(reinterpret_cast<uint64_t>(src)), "r"(bytes), "r"(bar) : "memory");
}
// K-major, 64B swizzle canonical layout (8-row atoms of 512 B), descriptor version 1,
// layout type 4 = SWIZZLE_64B
static_assert(OZ_BK == 64, "descriptor and swz() below are written for 64-byte rows");
__device__ __forceinline__ uint64_t smem_desc(unsigned addr) {
    return uint64_t((addr >> 4) & 0x3FFF) | (uint64_t(1) << 16) | (uint64_t((8 * OZ_BK) >> 4) << 32) |
           (uint64_t(1) << 46) | (uint64_t(4) << 61);
}
// descriptors passed as (low, high) 32-bit halves: only the low half (start address) varies
__device__ __forceinline__ void umma_i8(unsigned tmem_d, unsigned da_lo, unsigned db_lo, unsigned d_hi, unsigned idesc,
                                        unsigned acc) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t.reg .b64 da, db;\n\t"
        "mov.b64 da, {%1, %3};\n\tmov.b64 db, {%2, %3};\n\t"
        "setp.ne.b32 p, %5, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::i8 [%0], da, db, %4, p;\n\t}\n"
        ::"r"(tmem_d), "r"(da_lo), "r"(db_lo), "r"(d_hi), "r"(idesc), "r"(acc));
}
__device__ __forceinline__ void umma_commit(unsigned bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(bar)
                 : "memory");
}
// arrive on the mbarrier at this offset in both CTAs of the pair
__device__ __forceinline__ void umma_commit_mc2(unsigned bar) {
    asm volatile(
        "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;\n" ::"r"(
            bar),
        "h"((unsigned short)3)
        : "memory");
}
__device__ __forceinline__ void tmem_ld16(unsigned taddr, unsigned (&v)[16]) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];\n"
        : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
          "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
        : "r"(taddr));
}

__device__ __forceinline__ void tmem_ld8(unsigned taddr, unsigned (&v)[8]) {
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];\n"
                 : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7])
                 : "r"(taddr));
}
template <int GW>
__device__ __forceinline__ void tmem_ld_g(unsigned taddr, unsigned (&v)[GW]) {
    if constexpr (GW == 16) tmem_ld16(taddr, v);
    else tmem_ld8(taddr, v);
}

// zero 16 columns of this warp's 32 TMEM lanes
__device__ __forceinline__ void tmem_st16_zero(unsigned taddr) {
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1};\n" ::"r"(taddr),
        "r"(0u)
        : "memory");
}

// Work item sequence shared by the three roles: the CTA's iteration range is cut
// into segments (one per tile, processed last tile first, as in gemm_tma.cu) and
// each segment into chunks of at most CHUNK_KB k-blocks (int32 headroom).
struct Walk {
    int64_t beg, end, KT, t_first, t_last, nseg;
    __device__ Walk(int64_t b, int64_t e, int64_t kt, double inv_kt) : beg(b), end(e), KT(kt) {
        t_first = qdiv(b, kt, inv_kt);
        t_last = qdiv(e - 1, kt, inv_kt);
        nseg = e > b ? t_last - t_first + 1 : 0;
    }
    __device__ int64_t tile(int64_t si) const { return t_last - si; }
    __device__ int kb(int64_t t) const { return t == t_first ? int(beg - t * KT) : 0; }
    __device__ int ke(int64_t t) const { return t == t_last ? int(end - t * KT) : int(KT); }
};

// PAIR: the clustered two-chunk variant (a separate instantiation, so the single
// chunk kernel carries none of its branches -- they cost ~4 us per pass when shared)
// One k-step (32 bytes of K) of the S = 56 schedule for A slice SP (NSL = 7): 34 products
// in 14 MMAs.  Z slice q sits at B rows 56 q, its products with A slice SP accumulate on
// TMEM diagonal SP + q at column 56 (SP + q).  Runs of 4 / 2 slices are N = 224 / 112
// MMAs; a lone product is an N = 64 MMA whose last 8 columns read the next slice (or the
// 8 zero rows after slice 6) into the next diagonal -- placed so that spill is either
// zero or lands on diagonal 8 (columns 448..511, never read).  `init` (first k-step of an
// accumulation) starts a diagonal at its first writer: (0, 0..6) for diagonals 0..6,
// (1, 6) for diagonal 7 (issued after (0, 6), whose spill into diagonal 7 is zero).
//
// WIDE (the default; FQB_OZ_WIDE=0 for the schedule above): the same products in fewer, wider MMAs -- a slice's Z rows are
// covered by N = 256 MMAs split at row 256 (a swizzle-atom boundary inside slice 4), so
// A is read from shared memory 12 (ND = 8) / 10 (ND = 7) times per k-step instead of
// 14 / 11.  Spilled rows (past the slices a product needs) land on diagonal 8 (ND = 8) or
// 7 (ND = 7), never read; diagonal 7 of ND = 8 starts with its own lone MMA in SP = 1.
// AK: advance of the A descriptor per 32-element k-step (16-byte units): 2 (K-major), 128
// (MN-major: 32 K rows of 64 bytes)
template <int SP, int ND, bool WIDE, unsigned AK = (32 >> 4)>
__device__ __forceinline__ void issue_s56(unsigned tmem, unsigned da_lo, unsigned db_lo, unsigned d_hi,
                                          unsigned idesc, bool init) {
    constexpr unsigned kstep = 32 >> 4;
    if constexpr (WIDE) {
        // rows [r0, r0 + n) of the Z stage -> TMEM columns 56 SP + r0 ..
        auto mmr = [&](int r0, int n, bool first_writer) {
            const unsigned id = idesc | (unsigned(n >> 3) << 17);
            const unsigned dt = tmem + unsigned(SP * 56 + r0);
            const unsigned bl = db_lo + unsigned((r0 * OZ_BK) >> 4);
            umma_i8(dt, da_lo, bl, d_hi, id, (first_writer && init) ? 0u : 1u);
            umma_i8(dt, da_lo + AK, bl + kstep, d_hi, id, 1u);
        };
        if constexpr (SP == 0) { mmr(0, 256, true); mmr(256, 144, true); }
        else if constexpr (SP == 1) {
            mmr(0, 256, false);
            mmr(256, 80, false);
            if constexpr (ND == 8) mmr(336, 64, true);
        } else if constexpr (SP == 2) { mmr(0, 256, false); mmr(256, ND == 8 ? 80 : 32, false); }
        else if constexpr (SP == 3) {
            if constexpr (ND == 8) { mmr(0, 256, false); mmr(256, 32, false); }
            else mmr(0, 224, false);
        } else if constexpr (SP == 4) mmr(0, ND == 8 ? 224 : 176, false);
        else if constexpr (SP == 5) mmr(0, ND == 8 ? 176 : 112, false);
        else mmr(0, ND == 8 ? 112 : 64, false);
        return;
    }
    auto mma = [&](int q0, int n, bool first_writer) {
        const unsigned id = idesc | (unsigned(n >> 3) << 17);
        const unsigned dt = tmem + unsigned((SP + q0) * 56);
        const unsigned bl = db_lo + unsigned((q0 * 56 * OZ_BK) >> 4);
        umma_i8(dt, da_lo, bl, d_hi, id, (first_writer && init) ? 0u : 1u);
        umma_i8(dt, da_lo + AK, bl + kstep, d_hi, id, 1u);
    };
    if constexpr (ND == 7) {
        // diagonals 0..6 only (p + q <= 6: 28 products in 11 MMAs); every diagonal starts
        // with SP = 0, and the N = 64 spills land on diagonal 7, which is never read
        if constexpr (SP == 0) { mma(0, 224, true); mma(4, 112, true); mma(6, 64, true); }
        else if constexpr (SP == 1) { mma(0, 224, false); mma(4, 112, false); }
        else if constexpr (SP == 2) { mma(0, 224, false); mma(4, 64, false); }
        else if constexpr (SP == 3) { mma(0, 224, false); }
        else if constexpr (SP == 4) { mma(0, 112, false); mma(2, 64, false); }
        else if constexpr (SP == 5) { mma(0, 112, false); }
        else { mma(0, 64, false); }
        return;
    }
    if constexpr (SP == 0) { mma(0, 224, true); mma(4, 112, true); mma(6, 64, true); }
    else if constexpr (SP == 1) { mma(0, 224, false); mma(4, 112, false); mma(6, 64, true); }
    else if constexpr (SP == 2) { mma(0, 224, false); mma(4, 112, false); }
    else if constexpr (SP == 3) { mma(0, 224, false); mma(4, 64, false); }
    else if constexpr (SP == 4) { mma(0, 224, false); }
    else if constexpr (SP == 5) { mma(0, 112, false); mma(2, 64, false); }
    else { mma(0, 112, false); }
}

// One k-step of the S = 50 schedule (chunks of <= 50 columns, NSL = 7, all 8 diagonals):
// Z slice q sits at B rows 50 q (2 zero rows after slice 6), diagonal d at TMEM columns
// 50 d .. 50 d + 49.  Every MMA starts at B row 0 or 256 (swizzle-atom aligned) and covers
// the rows a slice's products need, N rounded up to a multiple of 16:
//     SP 0, 1: rows 0..255, 256..351    SP 2: 0..255, 256..303    SP 3: 0..255
//     SP 4: 0..207    SP 5: 0..159    SP 6: 0..111
// 10 MMAs, 1744 B rows per k-step (S = 56 wide: 12 MMAs, 1936 rows).  Rows past the needed
// slices read the zero pad rows (SP 0, 1) or land on diagonal 8 (columns 400..411, never
// read).  SP 0 writes columns 0..351 first (accumulate = 0 at `init`); the rest of
// diagonal 7 (columns 352..399) is zeroed by the epilogue (tcgen05.st) before each
// accumulation, so every other MMA accumulates.
template <int SP, unsigned AK = (32 >> 4)>
__device__ __forceinline__ void issue_s50(unsigned tmem, unsigned da_lo, unsigned db_lo, unsigned d_hi,
                                          unsigned idesc, bool init) {
    constexpr unsigned kstep = 32 >> 4;
    auto mmr = [&](int r0, int n) {
        const unsigned id = idesc | (unsigned(n >> 3) << 17);
        const unsigned dt = tmem + unsigned(SP * 50 + r0);
        const unsigned bl = db_lo + unsigned((r0 * OZ_BK) >> 4);
        umma_i8(dt, da_lo, bl, d_hi, id, (SP == 0 && init) ? 0u : 1u);
        umma_i8(dt, da_lo + AK, bl + kstep, d_hi, id, 1u);
    };
    if constexpr (SP <= 1) { mmr(0, 256); mmr(256, 96); }
    else if constexpr (SP == 2) { mmr(0, 256); mmr(256, 48); }
    else if constexpr (SP == 3) mmr(0, 256);
    else if constexpr (SP == 4) mmr(0, 208);
    else if constexpr (SP == 5) mmr(0, 160);
    else mmr(0, 112);
}
// diagonal 7's columns the S = 50 schedule does not initialise (352..399, in 16s)
constexpr int kS50ZeroCol = 352, kS50ZeroGroups = 3;

// AMN: A is read MN-major from the A'Y-layout slices of an operand X (p.x_kb): the
// products Y (rows of X) = X C with K = columns of X, e.g. Y -= Q C in the block
// Gram-Schmidt, on the slices of Q the Q'Y products already made.  A k-block (64 columns
// of X, 128 rows) per slice is two 4 KB halves of A'Y tiles: the rows 0..63 and 64..127
// halves sit 4 KB apart (LBO), 8 columns per 512-byte swizzle atom (SBO); the row
// exponents are 0 (each column's scale is folded into C by the caller).
template <bool PAIR, int NSL, int BS, int S, int NDK = 0, bool WIDE = false, bool AMN = false>
__global__ void __launch_bounds__(oz_threads(AMN), 1) k_ozaki(const OzArgs p) {
    using SL = Sl<NSL, BS, S, NDK>;
    constexpr unsigned AK = AMN ? (32u * 64u) >> 4 : 32u >> 4;
    static_assert(S == 64 || ((S == 56 || S == 50) && NSL == 7), "the 56 / 50-row spacings are scheduled for 7 slices");
    static_assert(S != 50 || (NDK == 0 && WIDE), "the 50-row spacing has one (wide, 8-diagonal) schedule");
    static_assert(NDK == 0 || (NDK == 7 && NSL == 7 && S == 56), "the trimmed variant is scheduled for S = 56");
    constexpr int A_STAGES = SL::A_STAGES;
    constexpr int B_STAGES = SL::B_STAGES;
    constexpr int B_STAGE = SL::B_STAGE;
    constexpr int ND = SL::ND;
    const int CHUNK_KB = p.chunk_kb;
    FQB_PDL_ENTRY();
    extern __shared__ uint8_t smem_raw[];
    __shared__ uint64_t bars[2 * A_STAGES + 2 * B_STAGES + 2];
    __shared__ unsigned tmem_base_s;
    __shared__ int ez_s[OZ_BN];   // column exponents (0 past N)
    const unsigned raw = smem_u32(smem_raw);
    const unsigned base = (raw + 1023u) & ~1023u;
    const unsigned a_base = base, b_base = base + A_STAGES * A_TILE;
    const unsigned a_full = smem_u32(&bars[0]), a_empty = a_full + 8 * A_STAGES;
    const unsigned b_full = a_empty + 8 * A_STAGES, b_empty = b_full + 8 * B_STAGES;
    const unsigned t_full = b_empty + 8 * B_STAGES, t_empty = t_full + 8;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int rank = PAIR ? int(blockIdx.x & 1) : 0;
    // this CTA's column chunk (PAIR), else the launch's own operands -- scalars, not a
    // copy of the parameter block (which would pin it in registers)
    const int8_t* const q_zs = PAIR ? p.zs + rank * p.zs_stride : p.zs;
    const int* const q_ez = PAIR ? p.ez + rank * OZ_BN : p.ez;
    double* const q_C = PAIR ? p.C + rank * p.cw * p.ldc : p.C;
    const int64_t q_N = PAIR ? min(p.cw, p.N - rank * p.cw) : p.N;
    double* const q_work = PAIR ? p.work + rank * p.work_stride : p.work;
    if (threadIdx.x == 0) {
        for (int s = 0; s < A_STAGES; ++s) {
            mbar_init(a_full + 8 * s, 1);
            mbar_init(a_empty + 8 * s, PAIR ? 2 : 1);   // both consumers release a shared stage
        }
        for (int s = 0; s < B_STAGES; ++s) {
            mbar_init(b_full + 8 * s, 1);
            mbar_init(b_empty + 8 * s, 1);
        }
        mbar_init(t_full, 1);
        mbar_init(t_empty, unsigned(oz_threads(AMN) - 64));   // every epilogue thread
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    if (threadIdx.x < OZ_BN) ez_s[threadIdx.x] = int(threadIdx.x) < q_N ? q_ez[threadIdx.x] : 0;
    if (warp == 1) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(
            smem_u32(&tmem_base_s)), "n"(SL::TMEM_COLS));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
    }
    asm volatile("tcgen05.fence::before_thread_sync;\n");
    __syncthreads();
    if constexpr (PAIR) cluster_sync();   // the peer's barriers exist before any multicast / remote arrive
    asm volatile("tcgen05.fence::after_thread_sync;\n");
    const unsigned tmem = tmem_base_s;

    const int c = PAIR ? int(blockIdx.x >> 1) : int(blockIdx.x);
    const Walk wk(range_begin(p, c), range_begin(p, c + 1), p.kblocks, p.inv_kblocks);

    if (warp == 0) {
        if (lane == 0) {
            const unsigned zbytes = unsigned(z_block_rows(NSL, S) * OZ_BK);
            const bool hint = p.l2hint != 0;
            const uint64_t pol_a = policy_evict_first(), pol_z = policy_evict_last();
            int64_t ja = 0, jb = 0;
            for (int64_t si = 0; si < wk.nseg; ++si) {
                const int64_t t = wk.tile(si);
                const int64_t mt = t;   // N <= 64: one column tile, tile index = row tile
                for (int kb = wk.kb(t); kb < wk.ke(t); ++kb, ++jb) {
                    const int sb = int(jb % B_STAGES);
                    mbar_wait(b_empty + 8 * sb, unsigned((jb / B_STAGES) & 1) ^ 1u);
                    mbar_expect_tx(b_full + 8 * sb, zbytes);
                    if (hint)
                        bulk_load_hint(b_base + sb * B_STAGE, q_zs + int64_t(kb) * zbytes, zbytes, b_full + 8 * sb,
                                       pol_z);
                    else
                        bulk_load(b_base + sb * B_STAGE, q_zs + int64_t(kb) * zbytes, zbytes, b_full + 8 * sb);
                    if constexpr (AMN) {
                        // columns 64 kb.. of X = half (kb & 1) of row tile kb / 2 of its A'Y
                        // slices, at X-row k-blocks 2 mt (rows 0..63) and 2 mt + 1 (64..127)
                        const int64_t kb0 = 2 * mt;
                        const bool two = kb0 + 1 < p.x_kb;
                        const int8_t* xt = p.xs + ((int64_t(kb >> 1) * p.x_kb + kb0) * NSL) * int64_t(A_TILE) +
                                           (kb & 1) * (A_TILE / 2);
                        for (int sp = 0; sp < NSL; ++sp, ++ja) {
                            const int sa = int(ja % A_STAGES);
                            mbar_wait(a_empty + 8 * sa, unsigned((ja / A_STAGES) & 1) ^ 1u);
                            mbar_expect_tx(a_full + 8 * sa, unsigned(two ? A_TILE : A_TILE / 2));
                            if (PAIR && (sp & 1) != rank) continue;
                            for (int hf = 0; hf < (two ? 2 : 1); ++hf) {
                                const int8_t* src = xt + (int64_t(hf) * NSL + sp) * A_TILE;
                                const unsigned dst = a_base + sa * A_TILE + hf * (A_TILE / 2);
                                if constexpr (PAIR) bulk_load_mc2_hint(dst, src, unsigned(A_TILE / 2), a_full + 8 * sa, pol_a);
                                else bulk_load_hint(dst, src, unsigned(A_TILE / 2), a_full + 8 * sa, pol_a);
                            }
                        }
                        continue;
                    }
                    const int8_t* xt = p.xs + (mt * p.kblocks + kb) * int64_t(NSL * A_TILE);
                    for (int sp = 0; sp < NSL; ++sp, ++ja) {
                        const int sa = int(ja % A_STAGES);
                        mbar_wait(a_empty + 8 * sa, unsigned((ja / A_STAGES) & 1) ^ 1u);
                        mbar_expect_tx(a_full + 8 * sa, unsigned(A_TILE));
                        if constexpr (!PAIR) {
                            if (hint)
                                bulk_load_hint(a_base + sa * A_TILE, xt + sp * A_TILE, unsigned(A_TILE),
                                               a_full + 8 * sa, pol_a);
                            else
                                bulk_load(a_base + sa * A_TILE, xt + sp * A_TILE, unsigned(A_TILE), a_full + 8 * sa);
                        } else if ((sp & 1) == rank) {   // the pair splits the slices, each lands in both
                            if (hint)
                                bulk_load_mc2_hint(a_base + sa * A_TILE, xt + sp * A_TILE, unsigned(A_TILE),
                                                   a_full + 8 * sa, pol_a);
                            else
                                bulk_load_mc2(a_base + sa * A_TILE, xt + sp * A_TILE, unsigned(A_TILE),
                                              a_full + 8 * sa);
                        }
                    }
                }
            }
        }
    } else if (warp == 1) {
        if (lane == 0) {
            // M = 128, S32 accumulate, signed int8 A and B, both K-major; N is set per MMA.
            // Everything below stays 32-bit and the slice loops are unrolled, so the
            // descriptors live in uniform registers (a per-MMA register->uniform
            // broadcast made the issue loop, not the tensor core, the bottleneck).
            constexpr unsigned idesc =
                (2u << 4) | (1u << 7) | (1u << 10) | (AMN ? 1u << 15 : 0u) | (unsigned(OZ_BM >> 4) << 24);
            // MN-major A: LBO = 4 KB between the two 64-row halves (SBO = 512 B as for K-major)
            const uint64_t da0 = AMN ? (smem_desc(a_base) & ~(uint64_t(0x3FFF) << 16)) | (uint64_t(4096 >> 4) << 16)
                                     : smem_desc(a_base);
            const uint64_t db0 = smem_desc(b_base);
            const unsigned da_lo0 = unsigned(da0), db_lo0 = unsigned(db0);
            const unsigned d_hi = unsigned(da0 >> 32);   // identical for both operands
            // S = 50: the epilogue zeroes part of diagonal 7 before the first accumulation
            // too (one extra phase of t_empty), so the first wait is on phase 0
            unsigned sa = 0, pa = 0, sb = 0, pb = 0, pt = S == 50 ? 1u : 0u;
            for (int64_t si = 0; si < wk.nseg; ++si) {
                const int64_t t = wk.tile(si);
                const int kb0 = wk.kb(t), kb1 = wk.ke(t);
                for (int cb = kb0; cb < kb1; cb += CHUNK_KB) {
                    const int ce = min(kb1, cb + CHUNK_KB);
                    mbar_wait(t_empty, pt ^ 1u);   // epilogue drained the accumulators
                    pt ^= 1u;
                    asm volatile("tcgen05.fence::after_thread_sync;\n");
                    for (int kb = cb; kb < ce; ++kb) {
                        mbar_wait(b_full + 8 * sb, pb);
                        const unsigned db_lo = db_lo0 + sb * unsigned(B_STAGE >> 4);
#pragma unroll
                        for (int sp = 0; sp < NSL; ++sp) {
                            mbar_wait(a_full + 8 * sa, pa);
                            asm volatile("tcgen05.fence::after_thread_sync;\n");
                            const unsigned da_lo = da_lo0 + sa * unsigned(A_TILE >> 4);
                            // products (sp, sq), sq = sq0 .. sq0+3, land on the consecutive
                            // diagonals sp+sq: one N = 64 * slices MMA covers them (A read once).
                            // Diagonals d < NSL start (accumulate = 0) with sp = 0; with ND > NSL
                            // the top diagonal ND-1 starts with (ND-NSL, NSL-1), issued alone.
                            if constexpr (S == 50) {
                                const bool init = kb == cb;
                                if (sp == 0) issue_s50<0, AK>(tmem, da_lo, db_lo, d_hi, idesc, init);
                                else if (sp == 1) issue_s50<1, AK>(tmem, da_lo, db_lo, d_hi, idesc, init);
                                else if (sp == 2) issue_s50<2, AK>(tmem, da_lo, db_lo, d_hi, idesc, init);
                                else if (sp == 3) issue_s50<3, AK>(tmem, da_lo, db_lo, d_hi, idesc, init);
                                else if (sp == 4) issue_s50<4, AK>(tmem, da_lo, db_lo, d_hi, idesc, init);
                                else if (sp == 5) issue_s50<5, AK>(tmem, da_lo, db_lo, d_hi, idesc, init);
                                else issue_s50<6, AK>(tmem, da_lo, db_lo, d_hi, idesc, init);
                                if constexpr (PAIR) umma_commit_mc2(a_empty + 8 * sa);
                                else umma_commit(a_empty + 8 * sa);
                                if (++sa == A_STAGES) sa = 0, pa ^= 1u;
                                continue;
                            }
                            if constexpr (S == 56) {
                                const bool init = kb == cb;
                                if (sp == 0) issue_s56<0, ND, WIDE, AK>(tmem, da_lo, db_lo, d_hi, idesc, init);
                                else if (sp == 1) issue_s56<1, ND, WIDE, AK>(tmem, da_lo, db_lo, d_hi, idesc, init);
                                else if (sp == 2) issue_s56<2, ND, WIDE, AK>(tmem, da_lo, db_lo, d_hi, idesc, init);
                                else if (sp == 3) issue_s56<3, ND, WIDE, AK>(tmem, da_lo, db_lo, d_hi, idesc, init);
                                else if (sp == 4) issue_s56<4, ND, WIDE, AK>(tmem, da_lo, db_lo, d_hi, idesc, init);
                                else if (sp == 5) issue_s56<5, ND, WIDE, AK>(tmem, da_lo, db_lo, d_hi, idesc, init);
                                else issue_s56<6, ND, WIDE, AK>(tmem, da_lo, db_lo, d_hi, idesc, init);
                                if constexpr (PAIR) umma_commit_mc2(a_empty + 8 * sa);
                                else umma_commit(a_empty + 8 * sa);
                                if (++sa == A_STAGES) sa = 0, pa ^= 1u;
                                continue;
                            }
                            constexpr unsigned kstep = 32 >> 4;   // 32 bytes of K per MMA
                            const int nq_all = min(NSL, ND - sp);
                            const bool split_top = ND > NSL && sp == ND - NSL;
                            const int nq_main = split_top ? nq_all - 1 : nq_all;
#pragma unroll
                            for (int sq0 = 0; sq0 < nq_main; sq0 += 4) {
                                const int nq = nq_main - sq0;
                                const unsigned id = idesc | (unsigned((nq < 4 ? nq : 4) * (OZ_BN >> 3)) << 17);
                                const unsigned dt = tmem + unsigned((sp + sq0) * OZ_BN);
                                const unsigned bl = db_lo + unsigned((sq0 * OZ_BN * OZ_BK) >> 4);
                                umma_i8(dt, da_lo, bl, d_hi, id, sp == 0 ? unsigned(kb != cb) : 1u);
#pragma unroll
                                for (int k = 1; k < OZ_BK / 32; ++k)
                                    umma_i8(dt, da_lo + k * AK, bl + k * kstep, d_hi, id, 1u);
                            }
                            if (split_top) {
                                const unsigned id = idesc | (unsigned(OZ_BN >> 3) << 17);
                                const unsigned dt = tmem + unsigned((ND - 1) * OZ_BN);
                                const unsigned bl = db_lo + unsigned(((NSL - 1) * OZ_BN * OZ_BK) >> 4);
                                umma_i8(dt, da_lo, bl, d_hi, id, unsigned(kb != cb));
#pragma unroll
                                for (int k = 1; k < OZ_BK / 32; ++k)
                                    umma_i8(dt, da_lo + k * AK, bl + k * kstep, d_hi, id, 1u);
                            }
                            if constexpr (PAIR) umma_commit_mc2(a_empty + 8 * sa);
                            else umma_commit(a_empty + 8 * sa);
                            if (++sa == A_STAGES) sa = 0, pa ^= 1u;
                        }
                        umma_commit(b_empty + 8 * sb);
                        if (++sb == B_STAGES) sb = 0, pb ^= 1u;
                    }
                    umma_commit(t_full);
                }
            }
        }
    } else {
        // ------------------------------ epilogue --------------------------------
        // 16 output columns at a time (low register pressure keeps the MMA issue
        // path in uniform registers).  A tile this CTA owns entirely goes straight to
        // C; a piece of a split tile is written, already scaled, to one of the CTA's
        // partial slots (0: its last tile, 1: its first) and k_ozaki_fixup sums the
        // pieces in CTA order afterwards -- no inter-CTA waiting inside this kernel.
        // A segment longer than CHUNK_KB k-blocks carries its running sum in slot 2.
        const int quarter = warp & 3;           // TMEM lanes 32*quarter .. +31
        constexpr int EPI = (oz_threads(AMN) - 64) / 32;   // epilogue warps: 4, or 8 (AMN)
        constexpr int GPH = EPI == 8 ? 32 : 64;             // columns drained per epilogue half
        const int g_lo = EPI == 8 ? ((warp - 2) >> 2) * GPH : 0;   // this warp's column groups
        const int g_hi = min(S, g_lo + GPH);
        constexpr int GW = EPI == 8 ? 8 : 16;               // columns per drain step (registers)
        const int r_loc = quarter * 32 + lane;  // tile row of this thread
        const unsigned lane_addr = tmem + (unsigned(quarter * 32) << 16);
        double* carry = q_work + (3 * int64_t(c) + 2) * OZ_PARTIAL;
        unsigned ph = 0;
        // S = 50: diagonal 7's columns no MMA initialises are zeroed before every
        // accumulation (here for the first, after each drain for the next)
        auto zero_d7 = [&]() {
            if constexpr (EPI == 8) {
                // both halves have read diagonal 7 before the first half zeroes it
                asm volatile("bar.sync 1, %0;\n" ::"n"(EPI * 32) : "memory");
                if (g_lo == 0) {
#pragma unroll
                    for (int z = 0; z < kS50ZeroGroups; ++z)
                        tmem_st16_zero(lane_addr + unsigned(kS50ZeroCol + 16 * z));
                    asm volatile("tcgen05.wait::st.sync.aligned;\n" ::: "memory");
                }
            } else {
#pragma unroll
                for (int z = 0; z < kS50ZeroGroups; ++z) tmem_st16_zero(lane_addr + unsigned(kS50ZeroCol + 16 * z));
                asm volatile("tcgen05.wait::st.sync.aligned;\n" ::: "memory");
            }
            asm volatile("tcgen05.fence::before_thread_sync;\n");
            mbar_arrive(t_empty);
        };
        if constexpr (S == 50) zero_d7();
        for (int64_t si = 0; si < wk.nseg; ++si) {
            const int64_t t = wk.tile(si);
            const int kb0 = wk.kb(t), kb1 = wk.ke(t);
            const int64_t row = t * OZ_BM + r_loc;
            const bool full_tile = kb0 == 0 && kb1 == p.kblocks;
            double* piece = q_work + (3 * int64_t(c) + (t == wk.t_last ? 0 : 1)) * OZ_PARTIAL;
            const int er = (!AMN && row < p.M) ? p.ex[row] : 0;   // loaded while the MMAs run
            // AMN (short K, beta != 0: Y -= Q C): each group's old C is loaded one group
            // ahead -- the first before the accumulators are ready -- so the drain, which
            // the single-buffered TMEM puts on the MMA's critical path, does not wait on it
            double pre[GW];
            const bool pre_on = AMN && p.beta != 0.0 && full_tile && row < p.M;
            auto load_old = [&](int g0) {
#pragma unroll
                for (int j = 0; j < GW; ++j) pre[j] = g0 + j < q_N ? q_C[int64_t(g0 + j) * p.ldc + row] : 0.0;
            };
            for (int cb = kb0; cb < kb1; cb += CHUNK_KB) {
                const bool first_chunk = cb == kb0, last_chunk = cb + CHUNK_KB >= kb1;
                if constexpr (AMN) {
                    if (pre_on && last_chunk) load_old(g_lo);
                }
                mbar_wait(t_full, ph);
                ph ^= 1u;
                asm volatile("tcgen05.fence::after_thread_sync;\n");
#pragma unroll 1
                for (int g = g_lo; g < g_hi; g += GW) {   // S = 56: the last group reads 8 spare columns
                    // all diagonals in flight, one wait
                    unsigned v[ND][GW];
#pragma unroll
                    for (int d = 0; d < ND; ++d) tmem_ld_g<GW>(lane_addr + unsigned(d * S + g), v[d]);
                    asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
                    double acc[GW];
#pragma unroll
                    for (int j = 0; j < GW; ++j) acc[j] = 0.0;
                    // least significant diagonal first: d = ND-1 .. 0 (scale 2^(-12-W d))
#pragma unroll
                    for (int d = ND - 1; d >= 0; --d) {
                        const double sc = pow2i(-12 - SL::W * d);
#pragma unroll
                        for (int j = 0; j < GW; ++j) acc[j] = fma(double(int(v[d][j])), sc, acc[j]);
                    }
                    if (!first_chunk) {
#pragma unroll
                        for (int j = 0; j < GW; ++j) acc[j] += carry[(g + j) * OZ_BM + r_loc];
                    }
                    if (!last_chunk) {
#pragma unroll
                        for (int j = 0; j < GW; ++j) carry[(g + j) * OZ_BM + r_loc] = acc[j];
                        continue;
                    }
                    if (!full_tile) {
#pragma unroll
                        for (int j = 0; j < GW; ++j)
                            piece[(g + j) * OZ_BM + r_loc] = mul_pow2(acc[j], er + ez_s[g + j]);
                        continue;
                    }
                    if (row < p.M) {
                        double old_c[GW];
                        if (AMN && pre_on) {
#pragma unroll
                            for (int j = 0; j < GW; ++j) old_c[j] = pre[j];
                            if (g + GW < g_hi) load_old(g + GW);
                        } else if (p.beta != 0.0) {
#pragma unroll
                            for (int j = 0; j < GW; ++j)
                                old_c[j] = g + j < q_N ? q_C[int64_t(g + j) * p.ldc + row] : 0.0;
                        }
#pragma unroll
                        for (int j = 0; j < GW; ++j) {
                            if (g + j < q_N) {
                                const double val = p.alpha * mul_pow2(acc[j], er + ez_s[g + j]);
                                q_C[int64_t(g + j) * p.ldc + row] = p.beta != 0.0 ? fma(p.beta, old_c[j], val) : val;
                            }
                        }
                    }
                }
                if constexpr (S == 50) {
                    zero_d7();
                } else {
                    asm volatile("tcgen05.fence::before_thread_sync;\n");
                    mbar_arrive(t_empty);
                }
            }
        }
    }
    asm volatile("tcgen05.fence::before_thread_sync;\n");
    __syncthreads();
    if constexpr (PAIR) cluster_sync();   // no CTA leaves while its peer may still arrive on its barriers
    if (warp == 1)
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem),
                     "n"(SL::TMEM_COLS));
}

// ---------------------------------------------------------------------------
// slicing
//
// A line (row or column) x with max|x| in [2^(e-1), 2^e) becomes the 55-bit
// integer R = rint(x 2^(55-e)) (|R| < 2^55, one FP64 multiply and one
// conversion), and R is written in balanced base 128 with a base-64 top digit:
//     R = sum_p d_p 2^(49-7p),  d_0 in [-64, 64],  d_1..d_7 in [-64, 63]
// read off as the 7-bit fields of R + sum_p 64 2^(49-7p) minus 64 (integer ops
// only).  So x = 2^e sum_p d_p 2^(-6-7p) up to the rounding of R, the weights
// the kernel's epilogue applies.  Line maxima only need the exponent, which
// lives in the high word of |x|: they are reduced as 32-bit integers.

constexpr long long kDigitBias = (64LL << 49) + (64LL << 42) + (64LL << 35) + (64LL << 28) + (64LL << 21) +
                                 (64LL << 14) + (64LL << 7) + 64LL;

// high word of |x|: monotone in |x|, exponent in bits 20..30
__device__ __forceinline__ unsigned abs_hi(double x) {
    return unsigned(static_cast<unsigned long long>(__double_as_longlong(x)) >> 32) & 0x7FFFFFFFu;
}
// e with 2^(e-1) <= max|x| < 2^e from the max high word.  All-zero lines and
// subnormal maxima get e = -1021 (their digits are 0 or just coarser); a line
// holding Inf or NaN gets kNonFiniteE, which turns its outputs into NaN.
__device__ __forceinline__ int exp_of_hi(unsigned hi) {
    return hi >= 0x7FF00000u ? kNonFiniteE : hi >= 0x00100000u ? int(hi >> 20) - 1022 : -1021;
}

// Line maxima are atomicMax'ed as (generation << 32 | high word): a word left by an
// earlier call carries a smaller generation and reads as 0, so the buffers need no
// memset between calls (a memset node would also break the programmatic-launch chain).
typedef unsigned long long u64;
__device__ __forceinline__ void max_tagged(u64* w, unsigned gen, unsigned v) {
    if (v) atomicMax(w, (u64(gen) << 32) | v);
}
__device__ __forceinline__ unsigned untag(u64 w, unsigned gen) { return unsigned(w >> 32) == gen ? unsigned(w) : 0u; }

// the 8 digits of x in line scale e, as raw fields d_p + 64 in [0, 128]: the 7-bit
// fields of U = R + sum_p 64 2^(49-7p), read from its two 32-bit halves
__device__ __forceinline__ void digits8(double x, int e, unsigned (&d)[8]) {
    const unsigned long long U = static_cast<unsigned long long>(__double2ll_rn(mul_pow2(x, 55 - e)) + kDigitBias);
    const unsigned hi = unsigned(U >> 32), lo = unsigned(U);
    d[0] = hi >> 17;
    d[1] = (hi >> 10) & 127u;
    d[2] = (hi >> 3) & 127u;
    d[3] = __funnelshift_r(lo, hi, 28) & 127u;
    d[4] = (lo >> 21) & 127u;
    d[5] = (lo >> 14) & 127u;
    d[6] = (lo >> 7) & 127u;
    d[7] = lo & 127u;
}

// NSL = 4 (FP32-class): R = rint(x 2^(27-e)), |R| <= 2^27, four digits of the same
// weights 2^(e-6-7p), p = 0..3, from the 32-bit U = R + 64 (2^21 + 2^14 + 2^7 + 1)
constexpr int kDigitBias4 = (64 << 21) + (64 << 14) + (64 << 7) + 64;
__device__ __forceinline__ void digits4(double x, int e, unsigned (&d)[4]) {
    const unsigned U = unsigned(__double2int_rn(mul_pow2(x, 27 - e)) + kDigitBias4);
    d[0] = (U >> 21) & 255u;
    d[1] = (U >> 14) & 127u;
    d[2] = (U >> 7) & 127u;
    d[3] = U & 127u;
}
// NSL = 7 (8-bit digits): R = rint(x 2^(54-e)), |R| <= 2^54, in balanced base 256,
//     R = sum_p d_p 2^(48-8p),  d_0 in [-64, 64],  d_1..d_6 in [-128, 127],
// the bytes of U = R + 0x80 80 80 80 80 80 80 (byte 6-p is d_p + 128): so
// x = 2^e sum_p d_p 2^(-6-8p) up to the rounding of R (2^(e-55)), one bit coarser
// than NSL = 8 but the products of 7 slices of 8 bits reach 2^-56 below 2^e with 34
// products instead of 36 and the A slices are 7 bytes per element instead of 8.
constexpr long long kDigitBias7 = 0x80808080808080LL;
__device__ __forceinline__ void digits7(double x, int e, unsigned (&d)[7]) {
    const unsigned long long U = static_cast<unsigned long long>(__double2ll_rn(mul_pow2(x, 54 - e)) + kDigitBias7);
    const unsigned hi = unsigned(U >> 32), lo = unsigned(U);
    d[0] = hi >> 16;
    d[1] = (hi >> 8) & 255u;
    d[2] = hi & 255u;
    d[3] = lo >> 24;
    d[4] = (lo >> 16) & 255u;
    d[5] = (lo >> 8) & 255u;
    d[6] = lo & 255u;
}
// NSL = 3 (FP32-class, 8-bit digits): R = rint(x 2^(22-e)), |R| <= 2^22, the bytes of
// U = R + 0x808080: x = 2^e sum_p d_p 2^(-6-8p), p = 0..2, up to 2^(e-23)
__device__ __forceinline__ void digits3(double x, int e, unsigned (&d)[3]) {
    const unsigned U = unsigned(__double2int_rn(mul_pow2(x, 22 - e)) + 0x808080);
    d[0] = U >> 16;
    d[1] = (U >> 8) & 255u;
    d[2] = U & 255u;
}
template <int NSL>
__device__ __forceinline__ void digits(double x, int e, unsigned (&d)[NSL]) {
    if constexpr (NSL == 8) digits8(x, e, d);
    else if constexpr (NSL == 7) digits7(x, e, d);
    else if constexpr (NSL == 3) digits3(x, e, d);
    else digits4(x, e, d);
}

// byte offset of (row r, byte c) inside a swizzled TR x OZ_BK byte tile
// (64B swizzle: the 16-byte chunk index c>>4 is XORed with address bits 7-8 = (r >> 1) & 3)
__device__ __forceinline__ int swz(int r, int c) { return r * OZ_BK + ((((c >> 4) ^ ((r >> 1) & 3)) << 4) | (c & 15)); }

// 16 consecutive K-values of one operand row -> one 16-byte chunk per slice
template <int NSL>
__device__ __forceinline__ void put_chunk16(const double (&v)[16], int e, int8_t* tile0, int64_t slice_stride, int r,
                                            int c) {
    uint32_t w[NSL][4];
#pragma unroll
    for (int sl = 0; sl < NSL; ++sl) w[sl][0] = w[sl][1] = w[sl][2] = w[sl][3] = 0;
#pragma unroll
    for (int u = 0; u < 16; ++u) {
        unsigned d[NSL];
        digits<NSL>(v[u], e, d);
#pragma unroll
        for (int sl = 0; sl < NSL; ++sl) w[sl][u >> 2] |= d[sl] << (8 * (u & 3));
    }
    // raw fields -> signed digits: (d - 2^(W-1)) mod 256 per byte, four at a time
    constexpr unsigned kOff = Sl<NSL>::W == 8 ? 0x80808080u : 0xC0C0C0C0u;
#pragma unroll
    for (int sl = 0; sl < NSL; ++sl)
#pragma unroll
        for (int q = 0; q < 4; ++q) w[sl][q] = __vadd4(w[sl][q], kOff);
    int8_t* dst = tile0 + swz(r, c);
#pragma unroll
    for (int sl = 0; sl < NSL; ++sl)
        *reinterpret_cast<uint4*>(dst + sl * slice_stride) = make_uint4(w[sl][0], w[sl][1], w[sl][2], w[sl][3]);
}

// the same for a Z stage of NSL slices spaced S rows apart: slice sl's row r is stage row
// S sl + r, swizzled by its stage row (S = 50 is not a multiple of the 8-row atom)
template <int NSL, int S>
__device__ __forceinline__ void put_chunk16_z(const double (&v)[16], int e, int8_t* tile0, int r, int c) {
    if constexpr (S % 8 == 0) {
        put_chunk16<NSL>(v, e, tile0, int64_t(S) * OZ_BK, r, c);
    } else {
        uint32_t w[NSL][4];
#pragma unroll
        for (int sl = 0; sl < NSL; ++sl) w[sl][0] = w[sl][1] = w[sl][2] = w[sl][3] = 0;
#pragma unroll
        for (int u = 0; u < 16; ++u) {
            unsigned d[NSL];
            digits<NSL>(v[u], e, d);
#pragma unroll
            for (int sl = 0; sl < NSL; ++sl) w[sl][u >> 2] |= d[sl] << (8 * (u & 3));
        }
        constexpr unsigned kOff = Sl<NSL>::W == 8 ? 0x80808080u : 0xC0C0C0C0u;
#pragma unroll
        for (int sl = 0; sl < NSL; ++sl)
#pragma unroll
            for (int q = 0; q < 4; ++q) w[sl][q] = __vadd4(w[sl][q], kOff);
#pragma unroll
        for (int sl = 0; sl < NSL; ++sl)
            *reinterpret_cast<uint4*>(tile0 + swz(S * sl + r, c)) = make_uint4(w[sl][0], w[sl][1], w[sl][2], w[sl][3]);
    }
}

// Row and column maxima (high words) of A (m x n, ld) in one pass, tagged with this
// call's generation (max_tagged).  CTA: 256 rows x 128 columns, a thread walks one row.  With
// norm_partial it also writes the CTA's sum of squares (||A||_F^2, reduced by
// ozaki_slice_a in CTA order), so the engine does not read A a third time.
template <typename T>   // double, or float A (FP32 input mode: widened exactly)
__global__ void __launch_bounds__(256) k_line_max(const T* __restrict__ a, int64_t m, int64_t n, int64_t ld,
                                                  u64* rmax, u64* cmax, unsigned gen, double* norm_partial) {
    FQB_PDL_ENTRY();
    __shared__ unsigned cm[8][128];
    __shared__ double red[8];
    const int64_t i = int64_t(blockIdx.x) * 256 + threadIdx.x;
    const int64_t j0 = int64_t(blockIdx.y) * 128;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    unsigned rm = 0;
    double sq[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll 4
    for (int c = 0; c < 128; ++c) {
        const int64_t j = j0 + c;
        const double x = (i < m && j < n) ? double(a[j * ld + i]) : 0.0;
        const unsigned h = abs_hi(x);
        sq[c & 3] = fma(x, x, sq[c & 3]);
        rm = max(rm, h);
        const unsigned wm = __reduce_max_sync(0xFFFFFFFFu, h);
        if (lane == 0) cm[warp][c] = wm;
    }
    if (i < m) max_tagged(rmax + i, gen, rm);
    if (norm_partial) {
        double t = (sq[0] + sq[1]) + (sq[2] + sq[3]);
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) t += __shfl_down_sync(0xFFFFFFFFu, t, off);
        if (lane == 0) red[warp] = t;
    }
    __syncthreads();
    if (norm_partial && threadIdx.x == 0) {
        double t = 0.0;
#pragma unroll
        for (int w = 0; w < 8; ++w) t += red[w];
        norm_partial[int64_t(blockIdx.y) * gridDim.x + blockIdx.x] = t;
    }
    if (threadIdx.x < 128 && j0 + threadIdx.x < n) {
        unsigned v = 0;
#pragma unroll
        for (int w = 0; w < 8; ++w) v = max(v, cm[w][threadIdx.x]);
        max_tagged(cmax + j0 + threadIdx.x, gen, v);
    }
}

// Sum of the per-CTA partials in index order (one CTA; deterministic)
__global__ void __launch_bounds__(1024) k_sum_ordered(const double* __restrict__ partial, int64_t count,
                                                      double* out) {
    FQB_PDL_ENTRY();
    __shared__ double red[32];
    double t = 0.0;
    for (int64_t k = threadIdx.x; k < count; k += blockDim.x) t += partial[k];
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) t += __shfl_down_sync(0xFFFFFFFFu, t, off);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = t;
    __syncthreads();
    if (threadIdx.x == 0) {
        double u = 0.0;
        for (int w = 0; w < int(blockDim.x >> 5); ++w) u += red[w];
        *out = u;
    }
}

// Both layouts of A's slices from one read of a 64 x 64 block (staged in shared
// memory); also turns the line maxima into the exponents the GEMM epilogue uses.
//   x_tn: operand rows = columns of A, K = m (A' Y),  e_tn per column
//   x_nn: operand rows = rows of A,    K = n (A G),   e_nn per row
// Either may be null.  The grid covers the padded operand rows, so every byte of
// both slice buffers is written (zeros outside A) and no memset is needed.
template <typename T, int NSL>
__global__ void __launch_bounds__(256) k_slice_a(const T* __restrict__ a, int64_t m, int64_t n, int64_t ld,
                                                 const u64* __restrict__ rmax, const u64* __restrict__ cmax, unsigned gen,
                                                 int8_t* x_tn, int* e_tn, int8_t* x_nn, int* e_nn) {
    FQB_PDL_ENTRY();
    __shared__ double t[64][65];   // t[j][i]
    const int64_t i0 = int64_t(blockIdx.x) * 64, j0 = int64_t(blockIdx.y) * 64;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    // all 16 loads of a thread in flight before the first shared store (a rolled
    // loop here left the kernel latency-bound at ~50% of HBM)
    double x[8][2];
#pragma unroll
    for (int k = 0; k < 8; ++k) {
        const int64_t j = j0 + warp + 8 * k;
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const int64_t i = i0 + lane + 32 * h;
            x[k][h] = (i < m && j < n) ? double(__ldcs(a + j * ld + i)) : 0.0;
        }
    }
#pragma unroll
    for (int k = 0; k < 8; ++k) {
#pragma unroll
        for (int h = 0; h < 2; ++h) t[warp + 8 * k][lane + 32 * h] = x[k][h];
    }
    __syncthreads();
    const int line = threadIdx.x >> 2, q = threadIdx.x & 3;   // 64 lines x 4 chunks of 16
    if (x_tn && i0 < round_up_dev(m, OZ_BK)) {                  // columns of A: rows j, K = i
        const int64_t j = j0 + line;
        const int e = j < n ? exp_of_hi(untag(cmax[j], gen)) : -1021;
        if (e_tn && blockIdx.x == 0 && j < n && q == 0) e_tn[j] = e;
        double v[16];
#pragma unroll
        for (int u = 0; u < 16; ++u) v[u] = t[line][q * 16 + u];
        const int64_t kb_count = (m + OZ_BK - 1) / OZ_BK;
        int8_t* tile0 = x_tn + ((j / OZ_BM) * kb_count + i0 / OZ_BK) * NSL * int64_t(A_TILE);
        put_chunk16<NSL>(v, e, tile0, A_TILE, int(j % OZ_BM), q * 16);
    }
    if (x_nn && j0 < round_up_dev(n, OZ_BK)) {                  // rows of A: rows i, K = j
        const int64_t i = i0 + line;
        const int e = i < m ? exp_of_hi(untag(rmax[i], gen)) : -1021;
        if (e_nn && blockIdx.y == 0 && i < m && q == 0) e_nn[i] = e;
        double v[16];
#pragma unroll
        for (int u = 0; u < 16; ++u) v[u] = t[q * 16 + u][line];
        const int64_t kb_count = (n + OZ_BK - 1) / OZ_BK;
        int8_t* tile0 = x_nn + ((i / OZ_BM) * kb_count + j0 / OZ_BK) * NSL * int64_t(A_TILE);
        put_chunk16<NSL>(v, e, tile0, A_TILE, int(i % OZ_BM), q * 16);
    }
}

// Z (k x n, ld, n <= 64): CTA (j, y) slices 16-row chunks y*ZT .. y*ZT+ZT-1 of
// column j (padded to 64 columns: zeros).  Every CTA of a column first takes the
// column max itself (the column is small and L2-resident), so one launch does it;
// (ZT = 256 measured faster than 512 at C2: 7.7 vs 9.6 us)
constexpr int ZT = 256;
template <int NSL, int S>
__global__ void __launch_bounds__(ZT) k_slice_z(const double* __restrict__ b, int64_t k, int64_t n, int64_t ld,
                                                int* ez, int8_t* out) {
    FQB_PDL_ENTRY();
    __shared__ unsigned wmax[ZT / 32];
    const int j = blockIdx.x;
    constexpr int ZR = z_block_rows(NSL, S);
    if (j >= S) {   // S = 56 / 50: the 8 / 2 zero rows after the last slice, row NSL S + (j - S)
        const int64_t kb_count = (k + OZ_BK - 1) / OZ_BK;
        const int64_t c16 = int64_t(blockIdx.y) * ZT + threadIdx.x;
        if (c16 >= kb_count * (OZ_BK / 16)) return;
        const int64_t k0 = c16 * 16;
        *reinterpret_cast<uint4*>(out + (k0 / OZ_BK) * int64_t(ZR) * OZ_BK + swz(NSL * S + (j - S), int(k0 % OZ_BK))) =
            make_uint4(0u, 0u, 0u, 0u);
        return;
    }
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const double* col = b + int64_t(j) * ld;
    const bool live = j < n;
    unsigned h = 0;
    if (live) {
        // eight loads in flight per thread (k = 8000: four round trips instead of eight)
        int64_t r = threadIdx.x;
        for (; r + 7 * ZT < k; r += 8 * ZT) {
            unsigned x[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) x[u] = abs_hi(col[r + u * ZT]);
#pragma unroll
            for (int u = 0; u < 8; ++u) h = max(h, x[u]);
        }
        unsigned x[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) x[u] = r + u * ZT < k ? abs_hi(col[r + u * ZT]) : 0u;   // the tail, also in flight
#pragma unroll
        for (int u = 0; u < 8; ++u) h = max(h, x[u]);
    }
    h = __reduce_max_sync(0xFFFFFFFFu, h);
    if (lane == 0) wmax[warp] = h;
    __syncthreads();
    unsigned mx = 0;
#pragma unroll
    for (int w = 0; w < ZT / 32; ++w) mx = max(mx, wmax[w]);
    const int e = exp_of_hi(mx);
    if (live && blockIdx.y == 0 && threadIdx.x == 0) ez[j] = e;
    const int64_t kb_count = (k + OZ_BK - 1) / OZ_BK;
    const int64_t c16 = int64_t(blockIdx.y) * ZT + threadIdx.x;
    if (c16 >= kb_count * (OZ_BK / 16)) return;
    const int64_t k0 = c16 * 16;
    double v[16];
#pragma unroll
    for (int u = 0; u < 16; ++u) v[u] = (live && k0 + u < k) ? col[k0 + u] : 0.0;
    put_chunk16_z<NSL, S>(v, e, out + (k0 / OZ_BK) * int64_t(ZR) * OZ_BK, j, int(k0 % OZ_BK));
}

// Long Z operands (k > kZFused rows: the Y of config 4's A'Y, k = m = 100000): every CTA
// of k_slice_z re-reads its whole column for the max (25x at k = 100000), so the maxima
// come from one pass first (k_zcol_max: atomicMax of the high words) and the slicer is a
// k-block per CTA with a warp per 8 rows -- each warp's stores are a contiguous 512 B.
constexpr int64_t kZFused = 16384;
constexpr int ZMAX_PER_CTA = 8192;
__global__ void __launch_bounds__(256) k_zcol_max(const double* __restrict__ b, int64_t k, int64_t n, int64_t ld,
                                                  u64* cmax, unsigned gen) {
    FQB_PDL_ENTRY();
    __shared__ unsigned wmax[8];
    const int j = blockIdx.x;
    if (j >= n) return;
    const double* col = b + int64_t(j) * ld;
    const int64_t r0 = int64_t(blockIdx.y) * ZMAX_PER_CTA;
    unsigned h = 0;
    unsigned x[8];
#pragma unroll
    for (int g = 0; g < ZMAX_PER_CTA / (256 * 8); ++g) {
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            const int64_t r = r0 + (int64_t(g) * 8 + u) * 256 + threadIdx.x;
            x[u] = r < k ? abs_hi(col[r]) : 0u;
        }
#pragma unroll
        for (int u = 0; u < 8; ++u) h = max(h, x[u]);
    }
    h = __reduce_max_sync(0xFFFFFFFFu, h);
    if ((threadIdx.x & 31) == 0) wmax[threadIdx.x >> 5] = h;
    __syncthreads();
    if (threadIdx.x == 0) {
        unsigned mx = 0;
#pragma unroll
        for (int w = 0; w < 8; ++w) mx = max(mx, wmax[w]);
        max_tagged(cmax + j, gen, mx);
    }
}

template <int NSL, int S>
__global__ void __launch_bounds__(256) k_slice_z_kb(const double* __restrict__ b, int64_t k, int64_t n, int64_t ld,
                                                    const u64* __restrict__ cmax, unsigned gen, int* ez, int8_t* out) {
    FQB_PDL_ENTRY();
    constexpr int ZR = z_block_rows(NSL, S);
    const int kb = blockIdx.x;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int j = warp * 8 + (lane >> 2), q = lane & 3;   // row j of the tile, 16-byte chunk q
    const int64_t k0 = int64_t(kb) * OZ_BK + q * 16;
    int8_t* tile0 = out + int64_t(kb) * ZR * OZ_BK;
    if (j >= S) {   // S = 56 / 50: the 8 / 2 zero rows after the last slice
        if (j - S < z_pad_rows(S))
            *reinterpret_cast<uint4*>(tile0 + swz(NSL * S + (j - S), q * 16)) = make_uint4(0u, 0u, 0u, 0u);
        return;
    }
    const bool live = j < n;
    const int e = live ? exp_of_hi(untag(cmax[j], gen)) : exp_of_hi(0u);
    if (live && kb == 0 && q == 0) ez[j] = e;
    const double* col = b + int64_t(j) * ld;
    double v[16];
#pragma unroll
    for (int u = 0; u < 16; ++u) v[u] = (live && k0 + u < k) ? col[k0 + u] : 0.0;
    put_chunk16_z<NSL, S>(v, e, tile0, j, q * 16);
}

// Sum the pieces of every split tile in CTA order (deterministic) into C.
// Pieces were written already scaled by 2^(ex + ez).  Block (tile, 8 columns),
// one thread per tile row; up to 4 pieces x 8 columns of loads in flight.
constexpr int FIX_COLS = 8;
__global__ void __launch_bounds__(OZ_BM) k_ozaki_fixup(const OzArgs p0) {
    FQB_PDL_ENTRY();
    const OzArgs p = chunk_args(p0, int(blockIdx.z));   // blockIdx.z = column chunk of a paired launch
    const int64_t t = blockIdx.x;
    const int j0 = blockIdx.y * FIX_COLS, r = threadIdx.x;
    const int c0 = cta_of(p, t * p.kblocks), c1 = cta_of(p, t * p.kblocks + p.kblocks - 1);
    const int64_t row = t * OZ_BM + r;
    if (c0 == c1 || row >= p.M) return;   // a tile owned by one CTA was written directly
    double sum[FIX_COLS];
#pragma unroll
    for (int q = 0; q < FIX_COLS; ++q) sum[q] = 0.0;
    for (int cb = c0; cb <= c1; cb += 4) {
        double v[4][FIX_COLS];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const int cc = cb + u;
            if (cc <= c1) {
                const int64_t t_last = qdiv(range_begin(p, cc + 1) - 1, p.kblocks, p.inv_kblocks);
                const double* w = p.work + (3 * int64_t(cc) + (t == t_last ? 0 : 1)) * OZ_PARTIAL + r;
#pragma unroll
                for (int q = 0; q < FIX_COLS; ++q) v[u][q] = j0 + q < p.N ? __ldcg(w + (j0 + q) * OZ_BM) : 0.0;
            }
        }
#pragma unroll
        for (int u = 0; u < 4; ++u)
            if (cb + u <= c1) {
#pragma unroll
                for (int q = 0; q < FIX_COLS; ++q) sum[q] += v[u][q];
            }
    }
#pragma unroll
    for (int q = 0; q < FIX_COLS; ++q) {
        if (j0 + q < p.N) {
            double* cp = p.C + int64_t(j0 + q) * p.ldc + row;
            const double val = p.alpha * sum[q];
            *cp = p.beta != 0.0 ? fma(p.beta, *cp, val) : val;
        }
    }
}

}  // namespace

int ozaki_slices() { return ozaki_fp64_slices(); }
int ozaki_fp64_slices() {
    static const int v = [] {
        const char* e = std::getenv("FQB_OZ_SLICES");   // 8: the 7-bit-digit FP64 scheme
        return e && std::atoi(e) == 8 ? 8 : 7;
    }();
    return v;
}
int ozaki_max_n() { return OZ_BN; }
int ozaki_bn(int64_t) { return OZ_BN; }   // Z slices padded to 64 rows: slice sq sits at TMEM diagonal spacing
int64_t ozaki_x_bytes(int64_t rows, int64_t k, int nsl) {
    return ceil_div(rows, OZ_BM) * ceil_div(k, OZ_BK) * nsl * OZ_BM * OZ_BK;
}
int64_t ozaki_z_bytes(int64_t n, int64_t k, int nsl) { return ceil_div(k, OZ_BK) * nsl * int64_t(ozaki_bn(n)) * OZ_BK; }
static void check_nsl(int nsl) {
    if (nsl != 8 && nsl != 7 && nsl != 4 && nsl != 3)
        throw Error(kStatusInvalid, "ozaki: slices per operand must be 8, 7, 4 or 3");
}

int64_t ozaki_line_max_words(int64_t m, int64_t n) { return 2 * (m + n); }   // generation-tagged 64-bit maxima
// one generation per maxima pass (host-side, process-wide, never reused before 2^32 calls)
static unsigned next_generation() {
    static std::atomic<unsigned> g{0};
    unsigned v = ++g;
    if (v == 0) v = ++g;
    return v;
}
int64_t ozaki_norm_partials(int64_t m, int64_t n) { return ceil_div(m, 256) * ceil_div(n, 128); }

template <typename T>
static void slice_a_impl(const T* a, int64_t m, int64_t n, int64_t ld, unsigned* line_max, int8_t* x_tn, int* e_tn,
                         int8_t* x_nn, int* e_nn, double* norm_partial, double* norm_out, int nsl, cudaStream_t s,
                         LaunchCounter& lc) {
    check_nsl(nsl);
    if (m <= 0 || n <= 0) {
        if (norm_out) FQB_CUDA(cudaMemsetAsync(norm_out, 0, sizeof(double), s));
        return;
    }
    u64* rmax = reinterpret_cast<u64*>(line_max);
    u64* cmax = rmax + m;
    const unsigned gen = next_generation();
    launch_k(k_line_max<T>, dim3(unsigned(ceil_div(m, 256)), unsigned(ceil_div(n, 128))), 256, 0, s, a, m, n, ld, rmax,
             cmax, gen, norm_out ? norm_partial : nullptr);
    FQB_LAUNCHED();
    if (norm_out) {
        launch_k(k_sum_ordered, 1, 1024, 0, s, norm_partial, ozaki_norm_partials(m, n), norm_out);
        FQB_LAUNCHED();
        lc.bump();
    }
    // cover the padded operand rows of both layouts (multiples of OZ_BM)
    const dim3 g(unsigned(ceil_div(m, OZ_BM) * (OZ_BM / 64)), unsigned(ceil_div(n, OZ_BM) * (OZ_BM / 64)));
    if (nsl == 8) launch_k(k_slice_a<T, 8>, g, 256, 0, s, a, m, n, ld, rmax, cmax, gen, x_tn, e_tn, x_nn, e_nn);
    else if (nsl == 7) launch_k(k_slice_a<T, 7>, g, 256, 0, s, a, m, n, ld, rmax, cmax, gen, x_tn, e_tn, x_nn, e_nn);
    else if (nsl == 3) launch_k(k_slice_a<T, 3>, g, 256, 0, s, a, m, n, ld, rmax, cmax, gen, x_tn, e_tn, x_nn, e_nn);
    else launch_k(k_slice_a<T, 4>, g, 256, 0, s, a, m, n, ld, rmax, cmax, gen, x_tn, e_tn, x_nn, e_nn);
    FQB_LAUNCHED();
    lc.bump(2);
}

void ozaki_slice_a(const double* a, int64_t m, int64_t n, int64_t ld, unsigned* line_max, int8_t* x_tn, int* e_tn,
                   int8_t* x_nn, int* e_nn, cudaStream_t s, LaunchCounter& lc, double* norm_partial,
                   double* norm_out, int nsl) {
    slice_a_impl(a, m, n, ld, line_max, x_tn, e_tn, x_nn, e_nn, norm_partial, norm_out, nsl, s, lc);
}
void ozaki_slice_a(const float* a, int64_t m, int64_t n, int64_t ld, unsigned* line_max, int8_t* x_tn, int* e_tn,
                   int8_t* x_nn, int* e_nn, cudaStream_t s, LaunchCounter& lc, double* norm_partial,
                   double* norm_out, int nsl) {
    slice_a_impl(a, m, n, ld, line_max, x_tn, e_tn, x_nn, e_nn, norm_partial, norm_out, nsl, s, lc);
}

// Z slices with row spacing S (64, or 56 for chunks of <= 56 columns of the 7-slice scheme)
template <int NSL, int S>
static void slice_z_long(const double* b, int64_t k, int64_t n, int64_t ld, int* e, int8_t* out, unsigned* cmax,
                         cudaStream_t s, LaunchCounter& lc) {
    u64* cm = reinterpret_cast<u64*>(cmax);   // OZ_BN tagged words (2 OZ_BN unsigned)
    const unsigned gen = next_generation();
    launch_k(k_zcol_max, dim3(unsigned(n), unsigned(ceil_div(k, ZMAX_PER_CTA))), 256, 0, s, b, k, n, ld, cm, gen);
    FQB_LAUNCHED();
    launch_k(k_slice_z_kb<NSL, S>, dim3(unsigned(ceil_div(k, OZ_BK))), 256, 0, s, b, k, n, ld,
             static_cast<const u64*>(cm), gen, e, out);
    FQB_LAUNCHED();
    lc.bump(2);
}

static void slice_z_s(const double* b, int64_t k, int64_t n, int64_t ld, int* e, int8_t* out, cudaStream_t s,
                      LaunchCounter& lc, int nsl, int S, unsigned* cmax = nullptr) {
    if (n <= 0 || k <= 0) return;
    check_nsl(nsl);
    if (cmax && k > kZFused) {
        if (nsl == 7 && S == 50) slice_z_long<7, 50>(b, k, n, ld, e, out, cmax, s, lc);
        else if (nsl == 7 && S == 56) slice_z_long<7, 56>(b, k, n, ld, e, out, cmax, s, lc);
        else if (nsl == 7) slice_z_long<7, 64>(b, k, n, ld, e, out, cmax, s, lc);
        else if (nsl == 8) slice_z_long<8, 64>(b, k, n, ld, e, out, cmax, s, lc);
        else if (nsl == 3) slice_z_long<3, 64>(b, k, n, ld, e, out, cmax, s, lc);
        else slice_z_long<4, 64>(b, k, n, ld, e, out, cmax, s, lc);
        return;
    }
    const int64_t chunks = ceil_div(k, OZ_BK) * (OZ_BK / 16);
    const dim3 g(unsigned(S + z_pad_rows(S)), unsigned(ceil_div(chunks, ZT)));
    if (nsl == 7 && S == 50) launch_k(k_slice_z<7, 50>, g, ZT, 0, s, b, k, n, ld, e, out);
    else if (nsl == 7 && S == 56) launch_k(k_slice_z<7, 56>, g, ZT, 0, s, b, k, n, ld, e, out);
    else if (nsl == 8) launch_k(k_slice_z<8, 64>, g, ZT, 0, s, b, k, n, ld, e, out);
    else if (nsl == 7) launch_k(k_slice_z<7, 64>, g, ZT, 0, s, b, k, n, ld, e, out);
    else if (nsl == 3) launch_k(k_slice_z<3, 64>, g, ZT, 0, s, b, k, n, ld, e, out);
    else launch_k(k_slice_z<4, 64>, g, ZT, 0, s, b, k, n, ld, e, out);
    FQB_LAUNCHED();
    lc.bump();
}

void ozaki_slice_z(const double* b, int64_t k, int64_t n, int64_t ld, int* e, int8_t* out, cudaStream_t s,
                   LaunchCounter& lc, int nsl) {
    slice_z_s(b, k, n, ld, e, out, s, lc, nsl, OZ_BN);
}

// paired (pair_cw > 0): N = 2 chunks of pair_cw columns at most, zs / ez hold both
// FQB_OZ_CHUNK=<k-blocks>: a shorter TMEM accumulation than the int32 headroom allows
// (A/B measurements; the default is the headroom, Sl::CHUNK_KB)
static int chunk_kb_limit() {
    static const int v = [] {
        const char* e = std::getenv("FQB_OZ_CHUNK");
        const int x = e ? std::atoi(e) : 0;
        return x > 0 ? x : 1 << 30;
    }();
    return v;
}

template <bool PAIR, int NSL, int BS, int S = 64, int NDK = 0, bool WIDE = false, bool AMN = false>
static void launch_variant(const OzArgs& a, cudaStream_t s) {
    static bool configured[64] = {};
    int dev = 0;
    FQB_CUDA(cudaGetDevice(&dev));
    if (dev < 0 || dev >= 64 || !configured[dev]) {
        FQB_CUDA(cudaFuncSetAttribute(k_ozaki<PAIR, NSL, BS, S, NDK, WIDE, AMN>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      int(Sl<NSL, BS, S, NDK>::SMEM)));
        if (dev >= 0 && dev < 64) configured[dev] = true;
    }
    OzArgs args = a;
    args.chunk_kb = std::min(Sl<NSL, BS, S, NDK>::CHUNK_KB, chunk_kb_limit());
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(unsigned(PAIR ? 2 * a.grid : a.grid));
    cfg.blockDim = dim3(oz_threads(AMN));
    cfg.dynamicSmemBytes = Sl<NSL, BS, S, NDK>::SMEM;
    cfg.stream = s;
    cudaLaunchAttribute attr[2];
    int na = 0;
    if (PAIR) {
        attr[na].id = cudaLaunchAttributeClusterDimension;
        attr[na].val.clusterDim.x = 2;
        attr[na].val.clusterDim.y = 1;
        attr[na].val.clusterDim.z = 1;
        ++na;
    }
    if (pdl_enabled()) {
        attr[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        attr[na].val.programmaticStreamSerializationAllowed = 1;
        ++na;
    }
    cfg.attrs = attr;
    cfg.numAttrs = na;
    FQB_CUDA(cudaLaunchKernelEx(&cfg, k_ozaki<PAIR, NSL, BS, S, NDK, WIDE, AMN>, args));
}

// A/B switches of the A-pass kernel (read once): FQB_OZ_L2HINT=0 plain bulk copies,
// FQB_OZ_BSTAGES=2|3 Z-slice stages of the 7-slice scheme
static int env_int(const char* name, int dflt) {
    const char* e = std::getenv(name);
    return e && *e ? std::atoi(e) : dflt;
}
static int l2hint_default() {
    static const int v = env_int("FQB_OZ_L2HINT", 1) != 0 ? 1 : 0;
    return v;
}
static int zstages_default() {
    static const int v = env_int("FQB_OZ_BSTAGES", 2) == 3 ? 3 : 2;
    return v;
}
static int64_t z_chunk_bytes(int64_t K, int nsl, int S) { return ceil_div(K, OZ_BK) * z_block_rows(nsl, S) * OZ_BK; }

// FQB_OZ_DIAGS=7: the 7-slice scheme keeps diagonals p + q <= 6 only (28 of 34 products,
// S = 56 chunks); see the DESIGN note on its error.  Default 8 (all d <= 7).
static int diags_default() {
    static const int v = env_int("FQB_OZ_DIAGS", 8) == 7 ? 7 : 8;
    return v;
}

// the S = 56 schedule in wide MMAs (default; FQB_OZ_WIDE=0: the 14-MMA schedule).  The
// int32 sums are exact either way, so both give identical bits.
static bool wide_default() {
    static const bool v = env_int("FQB_OZ_WIDE", 1) != 0;
    return v;
}

// Z slice spacing of a chunk of cw columns on the 7-slice scheme: 50 rows for cw <= 50 (the
// wide 8-diagonal schedule: 10 MMAs, 1744 B rows per k-step), 56 for cw <= 56 (12 MMAs,
// 1936 rows), else 64.  FQB_OZ_S50=0 / FQB_OZ_S56=0 turn the narrower spacings off.
static int z_spacing(int64_t cw, int nsl) {
    static const bool on56 = env_int("FQB_OZ_S56", 1) != 0;
    static const bool on50 = on56 && env_int("FQB_OZ_S50", 1) != 0 && wide_default() && diags_default() == 8;
    if (nsl != 7) return 64;
    if (on50 && cw <= 50) return 50;
    return (on56 && cw <= 56) ? 56 : 64;
}

template <bool PAIR>
static void launch_pair_or_not(const OzArgs& a, int nsl, int S, cudaStream_t s, bool amn) {
    const bool s56 = nsl == 7 && S == 56;
    if (nsl == 7 && S == 50) {
        if (amn) launch_variant<PAIR, 7, 2, 50, 0, true, true>(a, s);
        else launch_variant<PAIR, 7, 2, 50, 0, true>(a, s);
        return;
    }
    if (amn) {   // the MN-major reads of A'Y-layout slices: FP64-class, default schedules only
        if (s56 && wide_default()) launch_variant<PAIR, 7, 2, 56, 0, true, true>(a, s);
        else if (nsl == 7 && S == 64) launch_variant<PAIR, 7, 2, 64, 0, false, true>(a, s);
        else throw Error(kStatusInvalid, "ozaki_apply_mn: unsupported slice scheme");
        return;
    }
    if (s56 && diags_default() == 7 && wide_default()) launch_variant<PAIR, 7, 2, 56, 7, true>(a, s);
    else if (s56 && diags_default() == 7) launch_variant<PAIR, 7, 2, 56, 7>(a, s);
    else if (s56 && wide_default()) launch_variant<PAIR, 7, 2, 56, 0, true>(a, s);
    else if (s56) launch_variant<PAIR, 7, 2, 56>(a, s);
    else if (nsl == 8) launch_variant<PAIR, 8, 2>(a, s);
    else if (nsl == 7 && zstages_default() == 3) launch_variant<PAIR, 7, 3>(a, s);
    else if (nsl == 7) launch_variant<PAIR, 7, 2>(a, s);
    else if (nsl == 3) launch_variant<PAIR, 3, 2>(a, s);
    else launch_variant<PAIR, 4, 2>(a, s);
}

static thread_local LaunchTimer* t_timer = nullptr;
void ozaki_set_timer(LaunchTimer* t) { t_timer = t; }
static cudaEvent_t timer_event(LaunchTimer* t) {
    if (t->used == t->ev.size()) {
        cudaEvent_t e;
        FQB_CUDA(cudaEventCreate(&e));
        t->ev.push_back(e);
    }
    return t->ev[t->used++];
}

static void launch_ozaki(int64_t M, int64_t N, int64_t K, double alpha, const int8_t* xs, const int* ex,
                         const int8_t* zs, const int* ez, double beta, double* C, int64_t ldc, double* work,
                         int num_sms, int64_t pair_cw, int nsl, int S, cudaStream_t s, LaunchCounter& lc,
                         int64_t x_kb = 0) {
    check_nsl(nsl);
    const bool pair = pair_cw > 0;
    OzArgs a{};
    a.xs = xs;
    a.zs = zs;
    a.M = M;
    a.N = N;
    a.K = K;
    a.alpha = alpha;
    a.beta = beta;
    a.C = C;
    a.ldc = ldc;
    a.ex = ex;
    a.ez = ez;
    a.work = work;
    a.bn = S;
    a.mtiles = int(ceil_div(M, OZ_BM));
    a.kblocks = int(ceil_div(K, OZ_BK));
    a.iters = int64_t(a.mtiles) * a.kblocks;
    const int slots = pair ? num_sms / 2 : num_sms;   // CTAs (pairs) streaming distinct A ranges
    a.grid = int(std::max<int64_t>(1, std::min<int64_t>(slots, a.iters / 4)));
    a.inv_grid = 1.0 / double(a.grid);
    a.inv_kblocks = 1.0 / double(a.kblocks);
    a.inv_iters = 1.0 / double(a.iters);
    a.pair = pair ? 1 : 0;
    a.cw = pair_cw;
    a.zs_stride = z_chunk_bytes(K, nsl, S);
    a.work_stride = 3 * int64_t(a.grid) * OZ_PARTIAL;
    a.l2hint = l2hint_default();
    LaunchTimer* const tm = (t_timer && t_timer->on) ? t_timer : nullptr;
    if (tm) FQB_CUDA(cudaEventRecord(timer_event(tm), s));
    a.x_kb = x_kb;
    if (pair) launch_pair_or_not<true>(a, nsl, S, s, x_kb > 0);
    else launch_pair_or_not<false>(a, nsl, S, s, x_kb > 0);
    FQB_LAUNCHED();
    lc.bump();
    bool split = false;   // does any CTA (pair) boundary fall inside a tile?
    for (int c = 1; c < a.grid && !split; ++c) split = (a.iters * c / a.grid) % a.kblocks != 0;
    if (split) {
        const int64_t ncols = pair ? pair_cw : N;
        launch_k(k_ozaki_fixup, dim3(unsigned(a.mtiles), unsigned(ceil_div(ncols, FIX_COLS)), pair ? 2u : 1u), OZ_BM,
                 0, s, a);
        FQB_LAUNCHED();
        lc.bump();
    }
    if (tm) {
        FQB_CUDA(cudaEventRecord(timer_event(tm), s));
        tm->bytes += 8.0 * (double(M) * double(K) + double(K) * double(N) + double(M) * double(N));
    }
}

void ozaki_gemm(int64_t M, int64_t N, int64_t K, double alpha, const int8_t* xs, const int* ex, const int8_t* zs,
                const int* ez, double beta, double* C, int64_t ldc, double* work, int num_sms, cudaStream_t s,
                LaunchCounter& lc, int nsl) {
    if (N > OZ_BN) throw Error(kStatusInvalid, "ozaki_gemm: N > 64");
    launch_ozaki(M, N, K, alpha, xs, ex, zs, ez, beta, C, ldc, work, num_sms, 0, nsl, OZ_BN, s, lc);
}

static bool pairs_enabled() {
    static const bool on = [] {
        const char* e = std::getenv("FQB_OZ_PAIR");
        return !(e && e[0] == '0');
    }();
    return on;
}

static void apply_chunks(int64_t M, int64_t N, int64_t K, double alpha, const int8_t* xs, const int* ex,
                         const double* b, int64_t ldb, double beta, double* C, int64_t ldc, int8_t* z, int* ez,
                         double* work, int num_sms, cudaStream_t s, LaunchCounter& lc, int nsl, unsigned* zmax,
                         int64_t x_kb);

void ozaki_apply(int64_t M, int64_t N, int64_t K, double alpha, const int8_t* xs, const int* ex, const double* b,
                 int64_t ldb, double beta, double* C, int64_t ldc, int8_t* z, int* ez, double* work, int num_sms,
                 cudaStream_t s, LaunchCounter& lc, int nsl, unsigned* zmax) {
    apply_chunks(M, N, K, alpha, xs, ex, b, ldb, beta, C, ldc, z, ez, work, num_sms, s, lc, nsl, zmax, 0);
}

// cs (K x N, ld K) = diag(2^e) c: row k of C times 2^e_k (exact; NaN for a non-finite line)
__global__ void k_scale_rows_pow2(const double* __restrict__ c, int64_t K, int64_t N, int64_t ldc,
                                  const int* __restrict__ e, double* __restrict__ cs) {
    FQB_PDL_ENTRY();
    const int64_t k = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (k >= K) return;
    const int ek = e[k];
    for (int64_t j = blockIdx.y; j < N; j += gridDim.y) cs[j * K + k] = mul_pow2(c[j * ldc + k], ek);
}

void ozaki_apply_mn(int64_t M, int64_t N, int64_t K, double alpha, const int8_t* xs_tn, const int* xe,
                    const double* c, int64_t ldc_in, double beta, double* Y, int64_t ldy, double* cs, int8_t* z,
                    int* ez, double* work, int num_sms, cudaStream_t s, LaunchCounter& lc, int nsl,
                    unsigned* zmax) {
    if (N <= 0 || M <= 0) return;
    if (K <= 0) {   // empty sum: Y = beta Y
        throw Error(kStatusInvalid, "ozaki_apply_mn: K = 0");
    }
    launch_k(k_scale_rows_pow2, dim3(unsigned(ceil_div(K, 128)), unsigned(std::min<int64_t>(N, 64))), 128, 0, s, c,
             K, N, ldc_in, xe, cs);
    FQB_LAUNCHED();
    lc.bump();
    apply_chunks(M, N, K, alpha, xs_tn, nullptr, cs, K, beta, Y, ldy, z, ez, work, num_sms, s, lc, nsl, zmax,
                 ceil_div(M, OZ_BK));
}

static void apply_chunks(int64_t M, int64_t N, int64_t K, double alpha, const int8_t* xs, const int* ex,
                         const double* b, int64_t ldb, double beta, double* C, int64_t ldc, int8_t* z, int* ez,
                         double* work, int num_sms, cudaStream_t s, LaunchCounter& lc, int nsl, unsigned* zmax,
                         int64_t x_kb) {
    if (N <= 0) return;
    const int64_t chunks = ceil_div(N, OZ_BN);
    const int64_t cw = ceil_div(N, chunks);
    const int S = z_spacing(cw, nsl);
    const int64_t zstride = z_chunk_bytes(K, nsl, S);
    int64_t c0 = 0;
    // two chunks at a time on CTA pairs that share every A tile (multicast): A is
    // streamed once per pair of chunks instead of once per chunk
    while (pairs_enabled() && num_sms >= 2 && N - c0 > cw) {
        const int64_t nb = std::min(2 * cw, N - c0);
        slice_z_s(b + c0 * ldb, K, cw, ldb, ez, z, s, lc, nsl, S, zmax);
        slice_z_s(b + (c0 + cw) * ldb, K, nb - cw, ldb, ez + OZ_BN, z + zstride, s, lc, nsl, S,
                  zmax ? zmax + 2 * OZ_BN : nullptr);
        launch_ozaki(M, nb, K, alpha, xs, ex, z, ez, beta, C + c0 * ldc, ldc, work, num_sms, cw, nsl, S, s, lc, x_kb);
        c0 += nb;
    }
    for (; c0 < N; c0 += cw) {
        const int64_t nb = std::min(cw, N - c0);
        slice_z_s(b + c0 * ldb, K, nb, ldb, ez, z, s, lc, nsl, S, zmax);
        launch_ozaki(M, nb, K, alpha, xs, ex, z, ez, beta, C + c0 * ldc, ldc, work, num_sms, 0, nsl, S, s, lc, x_kb);
    }
}
// the products of ozaki_apply again, on the B slices its last call left in z / ez
// (N <= 128: the chunks of one launch)
void ozaki_apply_presliced(int64_t M, int64_t N, int64_t K, double alpha, const int8_t* xs, const int* ex, double beta,
                           double* C, int64_t ldc, const int8_t* z, const int* ez, double* work, int num_sms,
                           cudaStream_t s, LaunchCounter& lc, int nsl) {
    if (N <= 0) return;
    if (N > 2 * OZ_BN) throw Error(kStatusInvalid, "ozaki_apply_presliced: N > 128");
    const int64_t chunks = ceil_div(N, OZ_BN);
    const int64_t cw = ceil_div(N, chunks);
    if (chunks == 2 && !(pairs_enabled() && num_sms >= 2))
        throw Error(kStatusInvalid, "ozaki_apply_presliced: two chunks need the paired launch");
    launch_ozaki(M, N, K, alpha, xs, ex, z, ez, beta, C, ldc, work, num_sms, chunks == 2 ? cw : 0, nsl,
                 z_spacing(cw, nsl), s, lc);
}
int64_t ozaki_apply_z_bytes(int64_t K, int nsl) { return 2 * ozaki_z_bytes(OZ_BN, K, nsl); }
int ozaki_apply_ez_count() { return 4 * OZ_BN; }   // also the tagged 64-bit column maxima of two chunks
int64_t ozaki_workspace_doubles(int num_sms) { return 3 * int64_t(num_sms) * OZ_PARTIAL; }  // 2 pieces + carry

}  // namespace farqb
