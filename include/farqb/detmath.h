/*
 * detmath.h -- bit-reproducible log / sincos / Box-Muller for host and device.
 *
 * Every result here is a fixed sequence of IEEE-754 round-to-nearest operations
 * (+, -, *, /, sqrt, fused multiply-add), which both gcc (x86-64 SSE2, fma(),
 * -ffp-contract=off) and nvcc (__dadd_rn / __dmul_rn / __fma_rn, which are never
 * contracted) evaluate identically.  So a value drawn from Philox and pushed
 * through fqd_box_muller() has the same bits on the B200 and on the host --
 * unlike the libm Box-Muller of the reference generator (rng.hpp:44-55), whose
 * CUDA and glibc results differ by a few ulp.
 *
 * Users:
 *   - the fixed-zeta sparse-Gaussian test matrices (BASELINE configs 4 and 5;
 *     a kind the reference does not have), so the device draws the
 *     same Omega values as the host generator for a given seed;
 *   - the deterministic low-rank generator (csrc/detgen.cu and its host twin
 *     oracle/detgen.c) that makes config 3/4-sized matrices bit-identically on
 *     the GPU and on the CPU, so the reference can be run on the same A.
 *
 * Accuracy: ~2-3 ulp (log), ~2 ulp (sin/cos); the point is reproducibility, not
 * correct rounding.
 */
#ifndef FARQB_DETMATH_H
#define FARQB_DETMATH_H

#include <stdint.h>

#if defined(__CUDACC__)
#define FQD_FN __host__ __device__ __forceinline__
#if defined(__CUDA_ARCH__)
#define FQD_ADD(a, b) __dadd_rn((a), (b))
#define FQD_SUB(a, b) __dsub_rn((a), (b))
#define FQD_MUL(a, b) __dmul_rn((a), (b))
#define FQD_FMA(a, b, c) __fma_rn((a), (b), (c))
#define FQD_DIV(a, b) __ddiv_rn((a), (b))
#define FQD_SQRT(a) __dsqrt_rn((a))
#define FQD_BITS(x) ((uint64_t)__double_as_longlong(x))
#define FQD_FROM_BITS(u) __longlong_as_double((long long)(u))
#endif
#else
#include <math.h>
#include <string.h>
#define FQD_FN static inline
#endif

#if !defined(FQD_ADD)
/* host: plain IEEE double arithmetic; the including translation unit must be
 * compiled with -ffp-contract=off (gcc's default in ISO C mode) so that no a*b+c
 * is fused behind our back; fma() is the correctly rounded fused operation. */
#define FQD_ADD(a, b) ((a) + (b))
#define FQD_SUB(a, b) ((a) - (b))
#define FQD_MUL(a, b) ((a) * (b))
#define FQD_FMA(a, b, c) fma((a), (b), (c))
#define FQD_DIV(a, b) ((a) / (b))
#define FQD_SQRT(a) sqrt((a))
FQD_FN uint64_t fqd_bits_(double x) { uint64_t u; memcpy(&u, &x, sizeof u); return u; }
FQD_FN double fqd_from_bits_(uint64_t u) { double x; memcpy(&x, &u, sizeof x); return x; }
#define FQD_BITS(x) fqd_bits_(x)
#define FQD_FROM_BITS(u) fqd_from_bits_(u)
#endif

/* Natural log of a positive normal x: x = 2^e m, m in [sqrt(1/2), sqrt(2)),
 * log m = 2 atanh(s), s = (m - 1) / (m + 1), |s| <= 0.1716, 11 odd terms. */
FQD_FN double fqd_log(double x) {
    uint64_t u = FQD_BITS(x);
    int e = (int)((u >> 52) & 0x7ff) - 1023;
    double m = FQD_FROM_BITS((u & 0x000fffffffffffffULL) | 0x3ff0000000000000ULL);
    if (m > 1.4142135623730951) {
        m = FQD_MUL(m, 0.5);
        e += 1;
    }
    const double f = FQD_SUB(m, 1.0);                 /* exact (Sterbenz) */
    const double s = FQD_DIV(f, FQD_ADD(2.0, f));
    const double z = FQD_MUL(s, s);
    /* p(z) = sum_{k=1..11} 2/(2k+1) z^(k-1) */
    double p = 2.0 / 23.0;
    p = FQD_FMA(p, z, 2.0 / 21.0);
    p = FQD_FMA(p, z, 2.0 / 19.0);
    p = FQD_FMA(p, z, 2.0 / 17.0);
    p = FQD_FMA(p, z, 2.0 / 15.0);
    p = FQD_FMA(p, z, 2.0 / 13.0);
    p = FQD_FMA(p, z, 2.0 / 11.0);
    p = FQD_FMA(p, z, 2.0 / 9.0);
    p = FQD_FMA(p, z, 2.0 / 7.0);
    p = FQD_FMA(p, z, 2.0 / 5.0);
    p = FQD_FMA(p, z, 2.0 / 3.0);
    const double lm = FQD_FMA(FQD_MUL(s, z), p, FQD_MUL(2.0, s));
    const double de = (double)e;
    const double ln2_hi = 6.93147180369123816490e-01; /* 0x3fe62e42fee00000: e * ln2_hi exact */
    const double ln2_lo = 1.90821492927058770002e-10;
    return FQD_FMA(de, ln2_hi, FQD_FMA(de, ln2_lo, lm));
}

/* sin and cos of x, |x| <= pi/4, Taylor to x^17 / x^18 */
FQD_FN void fqd_sincos_small(double x, double* s, double* c) {
    const double y = FQD_MUL(x, x);
    double ps = -1.0 / 355687428096000.0;              /* -1/17! */
    ps = FQD_FMA(ps, y, 1.0 / 1307674368000.0);        /* 1/15! */
    ps = FQD_FMA(ps, y, -1.0 / 6227020800.0);          /* -1/13! */
    ps = FQD_FMA(ps, y, 1.0 / 39916800.0);             /* 1/11! */
    ps = FQD_FMA(ps, y, -1.0 / 362880.0);              /* -1/9! */
    ps = FQD_FMA(ps, y, 1.0 / 5040.0);                 /* 1/7! */
    ps = FQD_FMA(ps, y, -1.0 / 120.0);                 /* -1/5! */
    ps = FQD_FMA(ps, y, 1.0 / 6.0);                    /* 1/3! (subtracted below) */
    /* sin x = x - x y (1/6 - y/120 + ...) */
    *s = FQD_FMA(-FQD_MUL(x, y), ps, x);
    double pc = 1.0 / 6402373705728000.0;              /* 1/18! */
    pc = FQD_FMA(pc, y, -1.0 / 20922789888000.0);      /* -1/16! */
    pc = FQD_FMA(pc, y, 1.0 / 87178291200.0);          /* 1/14! */
    pc = FQD_FMA(pc, y, -1.0 / 479001600.0);           /* -1/12! */
    pc = FQD_FMA(pc, y, 1.0 / 3628800.0);              /* 1/10! */
    pc = FQD_FMA(pc, y, -1.0 / 40320.0);               /* -1/8! */
    pc = FQD_FMA(pc, y, 1.0 / 720.0);                  /* 1/6! */
    pc = FQD_FMA(pc, y, -1.0 / 24.0);                  /* -1/4! */
    pc = FQD_FMA(pc, y, 0.5);                          /* 1/2! (subtracted below) */
    /* cos x = 1 - y (1/2 - y/24 + ...) */
    *c = FQD_FMA(-y, pc, 1.0);
}

/* sin(2 pi u), cos(2 pi u) for u in [0, 1): quadrant from 4u (exact), the rest
 * reduced to [0, pi/4] by the complement r -> 1 - r (exact for r in (1/2, 1)). */
FQD_FN void fqd_sincos_2pi(double u, double* s, double* c) {
    const double t = FQD_MUL(u, 4.0);
    const int q = (int)t;
    double r = FQD_SUB(t, (double)q);
    const int flip = r > 0.5;
    if (flip) r = FQD_SUB(1.0, r);
    double sa, ca;
    fqd_sincos_small(FQD_MUL(r, 1.5707963267948966), &sa, &ca);
    double sp = flip ? ca : sa, cp = flip ? sa : ca;   /* sin, cos of (r pi/2) before the flip */
    switch (q & 3) {
        case 0: *s = sp; *c = cp; break;
        case 1: *s = cp; *c = -sp; break;
        case 2: *s = -sp; *c = -cp; break;
        default: *s = -cp; *c = sp; break;
    }
}

/* Box-Muller on one pair of units in (0, 1) (the shape of rng.hpp:44-55):
 * z0 = sqrt(-2 log u1) cos(2 pi u2), z1 = ... sin(2 pi u2). */
FQD_FN void fqd_box_muller(double u1, double u2, double* z0, double* z1) {
    const double r = FQD_SQRT(FQD_MUL(-2.0, fqd_log(u1)));
    double s, c;
    fqd_sincos_2pi(u2, &s, &c);
    *z0 = FQD_MUL(r, c);
    *z1 = FQD_MUL(r, s);
}

#endif /* FARQB_DETMATH_H */
