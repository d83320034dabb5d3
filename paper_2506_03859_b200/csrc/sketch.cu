// sketch.cu -- on-device test-matrix generation (Omega blocks).
//
// Reproduces rsvd::gen_sketch (/root/reference/proj/src/sketch.cpp:51-102)
// from the same Philox streams, without a host-side Omega:
//
//  * Gaussian: gaussian number i of column j comes from Philox output i/2 of
//    stream (seed, block_id, j) -- one Box-Muller pair per 128-bit output --
//    so the whole n x b block is generated in parallel, one thread per pair.
//  * i.i.d. density-p kinds: the reference walks each column by geometric
//    gaps row += 1 + (long long)(log u / log1p(-p)) (sketch.cpp:35-47).  Every
//    gap and value consumes a fixed number of stream words, so the unit used
//    by nonzero t is known in closed form; a warp evaluates 32 candidate gaps
//    at once and turns them into row indices with a warp prefix sum.
//  * fixed zeta (new): one thread per column, same rule as the oracle
//    (oracle/farqb_oracle.c fqo_gen_sketch): rows r = (u32 * n) >> 32 with
//    duplicates skipped, then one sign bit / Gaussian per row, sorted by row.
#include <cmath>
#include <cstdint>

#include "kernels.hpp"
#include "philox.cuh"

namespace farqb {
namespace {

// ---- unit-index bookkeeping of the i.i.d. walks -----------------------------

// unit (pair of u32 words) used by the gap draw of candidate nonzero t
__device__ __forceinline__ uint64_t gap_unit(int kind, uint64_t t) {
    if (kind == kSparseSign) return 2 * t;                   // gap, sign, gap, sign ...
    if (kind == kSparseGaussian) return t + 2 * ((t + 1) >> 1);  // gap, pair, gap, (spare) ...
    return t;                                                // Bernoulli / StdBernoulli
}

__device__ __forceinline__ double stream_unit(PhiloxKey key, uint32_t blk, uint32_t col, uint64_t ui) {
    const uint4 o = philox_block(key, blk, col, ui >> 1);
    return (ui & 1) ? unit_from_words(o.z, o.w) : unit_from_words(o.x, o.y);
}

// value of nonzero t; returns false on an exact-zero Gaussian (reference redraw)
__device__ __forceinline__ bool nonzero_value(int kind, PhiloxKey key, uint32_t blk, uint32_t col,
                                              uint64_t t, double scale, double& v) {
    if (kind == kSparseSign) {
        const double u = stream_unit(key, blk, col, 2 * t + 1);
        v = u < 0.5 ? -scale : scale;
        return true;
    }
    if (kind == kSparseGaussian) {
        const uint64_t te = t & ~uint64_t(1);           // the even t that drew the pair
        const uint64_t g = gap_unit(kind, te);
        const double u1 = stream_unit(key, blk, col, g + 1);
        const double u2 = stream_unit(key, blk, col, g + 2);
        double z0, z1;
        box_muller(u1, u2, z0, z1);
        const double z = (t & 1) ? z1 : z0;
        v = z * scale;
        return z != 0.0;
    }
    v = 1.0;
    return true;
}

__device__ __forceinline__ long long warp_incl_scan(long long x, int lane) {
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
        const long long y = __shfl_up_sync(0xffffffffu, x, off);
        if (lane >= off) x += y;
    }
    return x;
}

enum WalkMode { kCount = 0, kFillCsc = 1, kFillDense = 2 };

// One warp per column.
template <int MODE>
__global__ void __launch_bounds__(256) k_iid_walk(int kind, PhiloxKey key, uint32_t blk, int64_t n,
                                                  int l, double denom, double scale, double shift,
                                                  int* counts, const int* col_ptr, int* row_idx,
                                                  double* values, double* dense, int64_t ld,
                                                  unsigned* status) {
    FQB_PDL_ENTRY();
    const int lane = threadIdx.x & 31;
    const int col = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    if (col >= l) return;
    long long row = -1;
    uint64_t t_base = 0;
    int base_out = MODE == kFillCsc ? col_ptr[col] : 0;
    const double nd = double(n);
    for (;;) {
        const uint64_t t = t_base + lane;
        const double u = stream_unit(key, blk, uint32_t(col), gap_unit(kind, t));
        const double ratio = log(u) / denom;
        const bool stop = ratio >= nd;
        const long long gap = stop ? (long long)n : 1 + (long long)ratio;
        const long long r = row + warp_incl_scan(gap, lane);
        const bool bad = stop || r >= n;
        const unsigned badmask = __ballot_sync(0xffffffffu, bad);
        const int first_bad = badmask ? __ffs(badmask) - 1 : 32;
        if (lane < first_bad) {
            if (MODE != kCount) {
                double v;
                if (!nonzero_value(kind, key, blk, uint32_t(col), t, scale, v))
                    atomicOr(status, kGenZeroGaussian);
                if (MODE == kFillCsc) {
                    row_idx[base_out + t] = int(r);
                    values[base_out + t] = v;
                } else {
                    dense[int64_t(col) * ld + r] = v - shift;
                }
            }
        }
        if (first_bad < 32) {
            if (MODE == kCount && lane == 0) counts[col] = int(t_base + first_bad);
            return;
        }
        row = __shfl_sync(0xffffffffu, r, 31);
        t_base += 32;
    }
}

// One CTA (1024 threads) per column for dense patterns (n p >> 32): 1024
// candidate gaps per round, block-wide prefix sum, first invalid candidate found
// with a block min.  Same draws and the same rows as k_iid_walk.
template <int MODE>
__global__ void __launch_bounds__(1024) k_iid_walk_cta(int kind, PhiloxKey key, uint32_t blk, int64_t n,
                                                       double denom, double scale, double shift, int* counts,
                                                       const int* col_ptr, int* row_idx, double* values,
                                                       double* dense, int64_t ld, unsigned* status) {
    FQB_PDL_ENTRY();
    __shared__ long long warp_tot[32];
    __shared__ int first_bad_s;
    __shared__ long long row_s;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int col = blockIdx.x;
    long long row = -1;
    uint64_t t_base = 0;
    const int base_out = MODE == kFillCsc ? col_ptr[col] : 0;
    const double nd = double(n);
    for (;;) {
        const uint64_t t = t_base + tid;
        const double u = stream_unit(key, blk, uint32_t(col), gap_unit(kind, t));
        const double ratio = log(u) / denom;
        const bool stop = ratio >= nd;
        const long long gap = stop ? (long long)n : 1 + (long long)ratio;
        long long x = warp_incl_scan(gap, lane);
        if (lane == 31) warp_tot[warp] = x;
        if (tid == 0) first_bad_s = 1024;
        __syncthreads();
        if (warp == 0) {
            long long w = warp_tot[lane];
            w = warp_incl_scan(w, lane);
            warp_tot[lane] = w;
        }
        __syncthreads();
        const long long r = row + x + (warp > 0 ? warp_tot[warp - 1] : 0);
        const bool bad = stop || r >= n;
        if (bad) atomicMin(&first_bad_s, tid);
        __syncthreads();
        const int first_bad = first_bad_s;
        if (tid < first_bad && MODE != kCount) {
            double v;
            if (!nonzero_value(kind, key, blk, uint32_t(col), t, scale, v)) atomicOr(status, kGenZeroGaussian);
            if (MODE == kFillCsc) {
                row_idx[base_out + t] = int(r);
                values[base_out + t] = v;
            } else {
                dense[int64_t(col) * ld + r] = v - shift;
            }
        }
        if (first_bad < 1024) {
            if (MODE == kCount && tid == 0) counts[col] = int(t_base + first_bad);
            return;
        }
        if (tid == 1023) row_s = r;
        __syncthreads();
        row = row_s;
        t_base += 1024;
        __syncthreads();
    }
}

__global__ void k_philox_u32(PhiloxKey key, uint32_t blk, uint32_t col, int count, uint32_t* out) {
    FQB_PDL_ENTRY();
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < count) out[i] = philox_word(key, blk, col, uint64_t(i));
}

// one thread per (pair, column): gaussians 2k and 2k+1 of the column
__global__ void k_gaussian_dense(PhiloxKey key, uint32_t blk, int64_t n, int l, double* out,
                                 int64_t ld, unsigned* status) {
    FQB_PDL_ENTRY();
    const int64_t pairs = (n + 1) >> 1;
    const int64_t idx = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    const int col = blockIdx.y;
    if (idx >= pairs || col >= l) return;
    const uint4 o = philox_block(key, blk, uint32_t(col), uint64_t(idx));
    double z0, z1;
    box_muller(unit_from_words(o.x, o.y), unit_from_words(o.z, o.w), z0, z1);
    double* c = out + int64_t(col) * ld;
    const int64_t i = 2 * idx;
    c[i] = z0;
    if (i + 1 < n) c[i + 1] = z1;
    if (z0 == 0.0 || (i + 1 < n && z1 == 0.0)) atomicOr(status, kGenZeroGaussian);
}

constexpr int kMaxZeta = 256;

// one thread per column; exactly zeta nonzeros
__global__ void k_zeta_fill(int kind, PhiloxKey key, uint32_t blk, int64_t n, int l, int zeta,
                            double scale, int* col_ptr, int* row_idx, double* values,
                            unsigned* status) {
    FQB_PDL_ENTRY();
    const int col = blockIdx.x * blockDim.x + threadIdx.x;
    if (col > l) return;
    col_ptr[col] = col * zeta;
    if (col == l) return;
    int rows[kMaxZeta];
    double vals[kMaxZeta];
    PhiloxStream rng(key, blk, uint32_t(col));
    int have = 0;
    while (have < zeta) {
        const uint32_t w = rng.next_u32();
        const int r = int((uint64_t(w) * uint64_t(n)) >> 32);
        bool dup = false;
        for (int t = 0; t < have; ++t) dup |= rows[t] == r;
        if (!dup) rows[have++] = r;
    }
    for (int t = 0; t < zeta; ++t) {
        if (kind == kSparseSign) {
            vals[t] = (rng.next_u32() & 0x80000000u) ? -scale : scale;
        } else {
            double g;
            if (!rng.next_gaussian<true>(g)) atomicOr(status, kGenZeroGaussian);
            vals[t] = g * scale;
        }
    }
    for (int t = 1; t < zeta; ++t) {
        const int kr = rows[t];
        const double kv = vals[t];
        int s = t - 1;
        while (s >= 0 && rows[s] > kr) {
            rows[s + 1] = rows[s];
            vals[s + 1] = vals[s];
            --s;
        }
        rows[s + 1] = kr;
        vals[s + 1] = kv;
    }
    int64_t base = int64_t(col) * zeta;
    for (int t = 0; t < zeta; ++t) {
        row_idx[base + t] = rows[t];
        values[base + t] = vals[t];
    }
}

// single-CTA exclusive scan (l is at most a few thousand)
__global__ void k_exclusive_scan(const int* counts, int l, int* col_ptr) {
    FQB_PDL_ENTRY();
    __shared__ int carry;
    __shared__ int warp_sums[32];
    if (threadIdx.x == 0) carry = 0;
    __syncthreads();
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (int base = 0; base < l; base += blockDim.x) {
        const int i = base + threadIdx.x;
        int v = i < l ? counts[i] : 0;
        int x = v;
#pragma unroll
        for (int off = 1; off < 32; off <<= 1) {
            const int y = __shfl_up_sync(0xffffffffu, x, off);
            if (lane >= off) x += y;
        }
        if (lane == 31) warp_sums[warp] = x;
        __syncthreads();
        if (warp == 0) {
            int ws = lane < int(blockDim.x >> 5) ? warp_sums[lane] : 0;
#pragma unroll
            for (int off = 1; off < 32; off <<= 1) {
                const int y = __shfl_up_sync(0xffffffffu, ws, off);
                if (lane >= off) ws += y;
            }
            warp_sums[lane] = ws;
        }
        __syncthreads();
        const int prefix = carry + (warp > 0 ? warp_sums[warp - 1] : 0) + x - v;
        if (i < l) col_ptr[i] = prefix;
        __syncthreads();
        if (threadIdx.x == blockDim.x - 1) carry = prefix + v;
        __syncthreads();
    }
    if (threadIdx.x == 0) col_ptr[l] = carry;
}

__global__ void k_fill_const(double* out, int64_t rows, int cols, int64_t ld, double v) {
    FQB_PDL_ENTRY();
    const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    const int c = blockIdx.y;
    if (i < rows && c < cols) out[int64_t(c) * ld + i] = v;
}

__global__ void k_scatter(const int* col_ptr, const int* row_idx, const double* values, int l,
                          double shift, double* out, int64_t ld) {
    FQB_PDL_ENTRY();
    const int c = blockIdx.x;
    for (int idx = col_ptr[c] + threadIdx.x; idx < col_ptr[c + 1]; idx += blockDim.x)
        out[int64_t(c) * ld + row_idx[idx]] = values[idx] - shift;
}

}  // namespace

void launch_philox_u32(uint64_t seed, uint32_t block_id, uint32_t column, int count, uint32_t* out,
                       cudaStream_t s, LaunchCounter& lc) {
    if (count <= 0) return;
    launch_k(k_philox_u32, unsigned(ceil_div(count, 256)), 256, 0, s, philox_key(seed), block_id, column,
                                                                count, out);
    FQB_LAUNCHED();
    lc.bump();
}

void launch_gaussian_dense(uint64_t seed, int block_id, int64_t n, int l, double* out, int64_t ld,
                           unsigned* status, cudaStream_t s, LaunchCounter& lc) {
    const int64_t pairs = (n + 1) / 2;
    dim3 grid(unsigned(ceil_div(pairs, 256)), unsigned(l));
    launch_k(k_gaussian_dense, grid, 256, 0, s, philox_key(seed), uint32_t(block_id), n, l, out, ld, status);
    FQB_LAUNCHED();
    lc.bump();
}

// expected nonzeros per column from the walk's own constant denom = log1p(-p)
static bool dense_columns(int64_t n, double denom) { return double(n) * -std::expm1(denom) > 256.0; }

void launch_iid_count(int kind, uint64_t seed, int block_id, int64_t n, int l, double denom,
                      int* counts, cudaStream_t s, LaunchCounter& lc) {
    if (dense_columns(n, denom)) {
        launch_k(k_iid_walk_cta<kCount>, unsigned(l), 1024, 0, s, kind, philox_key(seed), uint32_t(block_id), n, denom,
                                                          0.0, 0.0, counts, nullptr, nullptr, nullptr, nullptr, 0,
                                                          nullptr);
        FQB_LAUNCHED();
        lc.bump();
        return;
    }
    launch_k(k_iid_walk<kCount>, unsigned(ceil_div(l, 8)), 256, 0, s, 
        kind, philox_key(seed), uint32_t(block_id), n, l, denom, 0.0, 0.0, counts, nullptr, nullptr,
        nullptr, nullptr, 0, nullptr);
    FQB_LAUNCHED();
    lc.bump();
}

void launch_iid_fill_csc(int kind, uint64_t seed, int block_id, int64_t n, int l, double denom,
                         double scale, const int* col_ptr, int* row_idx, double* values,
                         unsigned* status, cudaStream_t s, LaunchCounter& lc) {
    if (dense_columns(n, denom)) {
        launch_k(k_iid_walk_cta<kFillCsc>, unsigned(l), 1024, 0, s, kind, philox_key(seed), uint32_t(block_id), n, denom,
                                                            scale, 0.0, nullptr, col_ptr, row_idx, values, nullptr,
                                                            0, status);
        FQB_LAUNCHED();
        lc.bump();
        return;
    }
    launch_k(k_iid_walk<kFillCsc>, unsigned(ceil_div(l, 8)), 256, 0, s, 
        kind, philox_key(seed), uint32_t(block_id), n, l, denom, scale, 0.0, nullptr, col_ptr,
        row_idx, values, nullptr, 0, status);
    FQB_LAUNCHED();
    lc.bump();
}

void launch_iid_fill_dense(int kind, uint64_t seed, int block_id, int64_t n, int l, double denom,
                           double scale, double shift, double* out, int64_t ld, unsigned* status,
                           cudaStream_t s, LaunchCounter& lc) {
    dim3 g0(unsigned(ceil_div(n, 256)), unsigned(l));
    launch_k(k_fill_const, g0, 256, 0, s, out, n, l, ld, -shift);
    FQB_LAUNCHED();
    if (dense_columns(n, denom)) {
        launch_k(k_iid_walk_cta<kFillDense>, unsigned(l), 1024, 0, s, kind, philox_key(seed), uint32_t(block_id), n,
                                                              denom, scale, shift, nullptr, nullptr, nullptr,
                                                              nullptr, out, ld, status);
        FQB_LAUNCHED();
        lc.bump(2);
        return;
    }
    launch_k(k_iid_walk<kFillDense>, unsigned(ceil_div(l, 8)), 256, 0, s, 
        kind, philox_key(seed), uint32_t(block_id), n, l, denom, scale, shift, nullptr, nullptr,
        nullptr, nullptr, out, ld, status);
    FQB_LAUNCHED();
    lc.bump(2);
}

void launch_zeta_fill(int kind, uint64_t seed, int block_id, int64_t n, int l, int zeta,
                      double scale, int* col_ptr, int* row_idx, double* values, unsigned* status,
                      cudaStream_t s, LaunchCounter& lc) {
    if (zeta > kMaxZeta) throw Error(kStatusConfig, "zeta exceeds 256");
    launch_k(k_zeta_fill, unsigned(ceil_div(l + 1, 64)), 64, 0, s, kind, philox_key(seed), uint32_t(block_id),
                                                             n, l, zeta, scale, col_ptr, row_idx,
                                                             values, status);
    FQB_LAUNCHED();
    lc.bump();
}

void launch_exclusive_scan(const int* counts, int l, int* col_ptr, cudaStream_t s, LaunchCounter& lc) {
    launch_k(k_exclusive_scan, 1, 1024, 0, s, counts, l, col_ptr);
    FQB_LAUNCHED();
    lc.bump();
}

void launch_densify(const int* col_ptr, const int* row_idx, const double* values, int64_t n, int l,
                    double shift, double* out, int64_t ld, cudaStream_t s, LaunchCounter& lc) {
    dim3 g0(unsigned(ceil_div(n, 256)), unsigned(l));
    launch_k(k_fill_const, g0, 256, 0, s, out, n, l, ld, -shift);
    FQB_LAUNCHED();
    launch_k(k_scatter, unsigned(l), 128, 0, s, col_ptr, row_idx, values, l, shift, out, ld);
    FQB_LAUNCHED();
    lc.bump(2);
}

}  // namespace farqb
