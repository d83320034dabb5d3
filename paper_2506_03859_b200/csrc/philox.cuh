// philox.cuh -- counter-based Philox4x32-10 on the device.
//
// Same bijection, key and counter layout as the reference generator
// (/root/reference/proj/include/rsvd/rng.hpp:15-88): key = seed, counter =
// {draw lo, draw hi, column, block_id}.  Because the generator is counter
// based, the k-th 128-bit output of any stream is computed directly from
// (seed, block_id, column, k): the sketch kernels below never walk a stream
// sequentially unless the draw order itself is data dependent.
#pragma once

#include <cstdint>

#include "../../include/farqb/detmath.h"

namespace farqb {

struct PhiloxKey {
    uint32_t k0, k1;
};

__host__ __device__ __forceinline__ PhiloxKey philox_key(uint64_t seed) {
    return {uint32_t(seed), uint32_t(seed >> 32)};
}

// Ten rounds (rng.hpp:64-80).  __umulhi gives the high word of the 32x32 product.
__device__ __forceinline__ uint4 philox10(uint4 c, PhiloxKey k) {
    uint32_t k0 = k.k0, k1 = k.k1;
#pragma unroll
    for (int r = 0; r < 10; ++r) {
        const uint32_t hi0 = __umulhi(0xD2511F53u, c.x), lo0 = 0xD2511F53u * c.x;
        const uint32_t hi1 = __umulhi(0xCD9E8D57u, c.z), lo1 = 0xCD9E8D57u * c.z;
        c = make_uint4(hi1 ^ c.y ^ k0, lo1, hi0 ^ c.w ^ k1, lo0);
        k0 += 0x9E3779B9u;
        k1 += 0xBB67AE85u;
    }
    return c;
}

// 128-bit output number `ctr` of stream (block_id, column).
__device__ __forceinline__ uint4 philox_block(PhiloxKey key, uint32_t block_id, uint32_t column,
                                              uint64_t ctr) {
    return philox10(make_uint4(uint32_t(ctr), uint32_t(ctr >> 32), column, block_id), key);
}

// u32 word number `w` of the stream.
__device__ __forceinline__ uint32_t philox_word(PhiloxKey key, uint32_t block_id, uint32_t column,
                                                uint64_t w) {
    const uint4 o = philox_block(key, block_id, column, w >> 2);
    switch (w & 3) {
        case 0: return o.x;
        case 1: return o.y;
        case 2: return o.z;
        default: return o.w;
    }
}

// (u64 >> 11 + 0.5) 2^-53, low word first (rng.hpp:26-35).  Exact arithmetic,
// identical on host and device.
__device__ __forceinline__ double unit_from_words(uint32_t lo, uint32_t hi) {
    const uint64_t v = uint64_t(lo) | (uint64_t(hi) << 32);
    return (double(v >> 11) + 0.5) * 0x1p-53;
}

// Box-Muller on one pair of units (rng.hpp:44-55); z0 is the cosine branch.
__device__ __forceinline__ void box_muller(double u1, double u2, double& z0, double& z1) {
    const double r = sqrt(-2.0 * log(u1));
    const double a = 6.283185307179586476925286766559 * u2;
    double s, c;
    sincos(a, &s, &c);
    z0 = r * c;
    z1 = r * s;
}

// The same pair on the libm-free Box-Muller of include/farqb/detmath.h: bit-identical
// to the host (fixed-zeta sparse-Gaussian values, a kind the reference lacks).
__device__ __forceinline__ void box_muller_det(double u1, double u2, double& z0, double& z1) {
    fqd_box_muller(u1, u2, &z0, &z1);
}

// Sequential view of one stream, for the few generators whose draw order is
// data dependent (fixed-zeta duplicate rejection).  Mirrors the reference's
// buffered next_u32 / next_unit / next_gaussian (rng.hpp:21-56).
struct PhiloxStream {
    PhiloxKey key;
    uint32_t block_id, column;
    uint64_t ctr = 0;
    uint4 buf;
    int pos = 4;
    double spare = 0.0;
    bool have_spare = false;

    __device__ PhiloxStream(PhiloxKey k, uint32_t b, uint32_t c) : key(k), block_id(b), column(c) {}

    __device__ __forceinline__ uint32_t next_u32() {
        if (pos == 4) {
            buf = philox_block(key, block_id, column, ctr++);
            pos = 0;
        }
        const uint32_t v = pos == 0 ? buf.x : pos == 1 ? buf.y : pos == 2 ? buf.z : buf.w;
        ++pos;
        return v;
    }
    __device__ __forceinline__ double next_unit() {
        const uint32_t lo = next_u32();
        const uint32_t hi = next_u32();
        return unit_from_words(lo, hi);
    }
    // Returns false if the reference would have redrawn on an exact zero
    // (probability ~2^-52 per draw); callers flag that as an internal error.
    template <bool kDet = false>
    __device__ __forceinline__ bool next_gaussian(double& out) {
        if (have_spare) {
            have_spare = false;
            if (spare != 0.0) {
                out = spare;
                return true;
            }
            return false;
        }
        const double u1 = next_unit();
        const double u2 = next_unit();
        double z0, z1;
        if (kDet)
            box_muller_det(u1, u2, z0, z1);
        else
            box_muller(u1, u2, z0, z1);
        spare = z1;
        have_spare = true;
        out = z0;
        return z0 != 0.0;
    }
};

}  // namespace farqb
