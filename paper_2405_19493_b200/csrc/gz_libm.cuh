/*
 * gz_libm.cuh -- exp/log that reproduce the host glibc results bit for bit.
 *
 * Why: the reference evaluates the ziggurat wedge test `y < exp(-0.5*x*x)`
 * (samplers.py:113, samplers.py:164, engine.py:106, engine.py:145), the tail
 * `-log(u)` (samplers.py:53-54, engine.py:95-96, engine.py:134-135) and the polar
 * multiplier `sqrt(-2*log(s)/s)` (samplers.py:189, engine.py:171) with CPython /
 * numba `math.exp` / `math.log`, i.e. with the host glibc libm.  CUDA's own
 * `exp`/`log` are not bit-identical to glibc, so a decision or an output could
 * differ by an ulp.  These functions restate glibc's (>= 2.28) table-driven
 * algorithms -- the FMA ifunc variants that an x86-64 host with FMA/AVX2 runs --
 * with the same operation order and the same fused multiply-adds as the
 * compiled library (read from its disassembly),
 * and the library's own table/coefficient data (gz_libm_consts.h).
 *
 * Compiled both for the device (nvcc, explicit __fma_rn/__dmul_rn/... so that
 * no contraction can change an operation) and for the host (gcc/g++ with
 * -ffp-contract=off, fma() from <math.h>), so the restatement is sweep-checked
 * against the real libm on the CPU without a GPU (tests/test_host_api.py, the
 * host sweep; tests/test_gpu_parity.py test_device_libm_bit_exact_sweep on the device).
 * Table and coefficient data: glibc (LGPL-2.1+; the optimized-routines exp/log,
 * MIT/Apache-2.0 upstream) -- see NOTICE.
 */
#pragma once
#include <stdint.h>
#include "gz_libm_consts.h"

#if defined(__CUDACC__)
#define GZ_HD __host__ __device__ __forceinline__
#else
#include <math.h>
#include <string.h>
#define GZ_HD static inline
#endif

#if defined(__CUDA_ARCH__)
#define GZ_FMA(a, b, c) __fma_rn((a), (b), (c))
#define GZ_MUL(a, b) __dmul_rn((a), (b))
#define GZ_ADD(a, b) __dadd_rn((a), (b))
#define GZ_SUB(a, b) __dsub_rn((a), (b))
#define GZ_DBL(u) __longlong_as_double((long long)(u))
#define GZ_BITS(d) ((uint64_t)__double_as_longlong(d))
#else
#define GZ_FMA(a, b, c) fma((a), (b), (c))
#define GZ_MUL(a, b) ((a) * (b))
#define GZ_ADD(a, b) ((a) + (b))
#define GZ_SUB(a, b) ((a) - (b))
GZ_HD double gz_host_dbl(uint64_t u) { double d; memcpy(&d, &u, 8); return d; }
GZ_HD uint64_t gz_host_bits(double d) { uint64_t u; memcpy(&u, &d, 8); return u; }
#define GZ_DBL(u) gz_host_dbl(u)
#define GZ_BITS(d) gz_host_bits(d)
#endif

/* Scalar coefficients: in the constant bank on the device (so DFMA takes them
 * as c[][] operands instead of re-materialising 64-bit immediates), literal
 * bit patterns on the host.  The 256-entry tables are passed by pointer (the
 * kernels keep a shared-memory copy). */
#if defined(__CUDACC__)
static __constant__ double gzk_EXP_INVLN2N = GZ_EXP_INVLN2N_F;
static __constant__ double gzk_EXP_SHIFT = GZ_EXP_SHIFT_F;
static __constant__ double gzk_EXP_NEGLN2HIN = GZ_EXP_NEGLN2HIN_F;
static __constant__ double gzk_EXP_NEGLN2LON = GZ_EXP_NEGLN2LON_F;
static __constant__ double gzk_EXP_C2 = GZ_EXP_C2_F;
static __constant__ double gzk_EXP_C3 = GZ_EXP_C3_F;
static __constant__ double gzk_EXP_C4 = GZ_EXP_C4_F;
static __constant__ double gzk_EXP_C5 = GZ_EXP_C5_F;
static __constant__ double gzk_LOG_LN2HI = GZ_LOG_LN2HI_F;
static __constant__ double gzk_LOG_LN2LO = GZ_LOG_LN2LO_F;
static __constant__ double gzk_LOG_A0 = GZ_LOG_A0_F;
static __constant__ double gzk_LOG_A1 = GZ_LOG_A1_F;
static __constant__ double gzk_LOG_A2 = GZ_LOG_A2_F;
static __constant__ double gzk_LOG_A3 = GZ_LOG_A3_F;
static __constant__ double gzk_LOG_A4 = GZ_LOG_A4_F;
static __constant__ double gzk_LOG_B0 = GZ_LOG_B0_F;
static __constant__ double gzk_LOG_B1 = GZ_LOG_B1_F;
static __constant__ double gzk_LOG_B2 = GZ_LOG_B2_F;
static __constant__ double gzk_LOG_B3 = GZ_LOG_B3_F;
static __constant__ double gzk_LOG_B4 = GZ_LOG_B4_F;
static __constant__ double gzk_LOG_B5 = GZ_LOG_B5_F;
static __constant__ double gzk_LOG_B6 = GZ_LOG_B6_F;
static __constant__ double gzk_LOG_B7 = GZ_LOG_B7_F;
static __constant__ double gzk_LOG_B8 = GZ_LOG_B8_F;
static __constant__ double gzk_LOG_B9 = GZ_LOG_B9_F;
static __constant__ double gzk_LOG_B10 = GZ_LOG_B10_F;
#endif
#if defined(__CUDA_ARCH__)
#define GZ_K(name) (gzk_##name)
#else
#define GZ_K(name) GZ_DBL(GZ_##name)
#endif

static const uint64_t gz_exp_tab_host[256] = GZ_EXP_TAB_INIT;
static const uint64_t gz_log_tab_host[256] = GZ_LOG_TAB_INIT;

/* exp(x): glibc's exp (FMA variant).  `tab` is the 256-entry GZ_EXP_TAB. */
GZ_HD double gz_exp_t(double x, const uint64_t* __restrict__ tab)
{
    uint64_t ix = GZ_BITS(x);
    uint32_t abstop = (uint32_t)(ix >> 52) & 0x7ff;
    int special = 0;
    if (abstop - 0x3c9u >= 0x3fu) {
        if ((int32_t)(abstop - 0x3c9u) < 0)
            return GZ_ADD(1.0, x);                 /* |x| < 2^-54 (incl. 0, subnormals) */
        if (abstop >= 0x409u) {                    /* |x| >= 1024, inf, nan */
            if (ix == 0xfff0000000000000ULL) return 0.0;
            if (abstop >= 0x7ffu) return GZ_ADD(1.0, x);
            return (ix >> 63) ? 0.0 : GZ_DBL(0x7ff0000000000000ULL);
        }
        special = 1;                               /* 512 <= |x| < 1024 */
    }
    double kd = GZ_FMA(x, GZ_K(EXP_INVLN2N), GZ_K(EXP_SHIFT));
    uint64_t ki = GZ_BITS(kd);
    kd = GZ_SUB(kd, GZ_K(EXP_SHIFT));
    double r = GZ_FMA(kd, GZ_K(EXP_NEGLN2HIN), x);
    r = GZ_FMA(kd, GZ_K(EXP_NEGLN2LON), r);
    uint32_t idx = 2u * (uint32_t)(ki & 127u);
    uint64_t top = ki << 45;
    double tail = GZ_DBL(tab[idx]);
    uint64_t sbits = tab[idx + 1] + top;
    double p23 = GZ_FMA(r, GZ_K(EXP_C3), GZ_K(EXP_C2));
    double tr = GZ_ADD(r, tail);
    double r2 = GZ_MUL(r, r);
    double p45 = GZ_FMA(r, GZ_K(EXP_C5), GZ_K(EXP_C4));
    double t = GZ_FMA(p23, r2, tr);
    double r4 = GZ_MUL(r2, r2);
    double tmp = GZ_FMA(r4, p45, t);
    if (!special) {
        double scale = GZ_DBL(sbits);
        return GZ_FMA(scale, tmp, scale);
    }
    /* exponent of scale may have over/underflowed: glibc's specialcase */
    if ((ki & 0x80000000ULL) == 0) {
        sbits -= 1009ULL << 52;
        double scale = GZ_DBL(sbits);
        return GZ_MUL(GZ_DBL(0x7f00000000000000ULL) /* 0x1p1009 */, GZ_FMA(scale, tmp, scale));
    }
    sbits += 1022ULL << 52;
    double scale = GZ_DBL(sbits);
    double st = GZ_MUL(scale, tmp);                /* not fused in the library here */
    double y = GZ_ADD(scale, st);
    if (y < 1.0) {
        /* round y + 1 correctly in the subnormal range; library operation order */
        double hi = GZ_ADD(y, 1.0);
        double lo = GZ_ADD(GZ_SUB(scale, y), st);
        lo = GZ_ADD(GZ_ADD(GZ_SUB(1.0, hi), y), lo);
        y = GZ_SUB(GZ_ADD(lo, hi), 1.0);
        if (y == 0.0) y = 0.0;
    }
    return GZ_MUL(y, GZ_DBL(0x0010000000000000ULL) /* 0x1p-1022 */);
}

GZ_HD double gz_log_core(uint64_t ix, const uint64_t* __restrict__ tab);

/* log(x): glibc's log (FMA variant).  `tab` is the 256-entry GZ_LOG_TAB. */
GZ_HD double gz_log_t(double x, const uint64_t* __restrict__ tab)
{
    uint64_t ix = GZ_BITS(x);
    if (ix - 0x3fee000000000000ULL <= 0x308ffffffffffULL) {
        /* x in [1 - 2^-4, 1 + 0x1.09p-4): degree-11 polynomial around 1 */
        if (ix == 0x3ff0000000000000ULL) return 0.0;
        double r = GZ_SUB(x, 1.0);
        double r2 = GZ_MUL(r, r);
        double r3 = GZ_MUL(r, r2);
        double p1 = GZ_FMA(r2, GZ_K(LOG_B3), GZ_FMA(r, GZ_K(LOG_B2), GZ_K(LOG_B1)));
        double p2 = GZ_FMA(r2, GZ_K(LOG_B6), GZ_FMA(r, GZ_K(LOG_B5), GZ_K(LOG_B4)));
        double p3 = GZ_FMA(r3, GZ_K(LOG_B10),
                           GZ_FMA(r2, GZ_K(LOG_B9), GZ_FMA(r, GZ_K(LOG_B8), GZ_K(LOG_B7))));
        double q = GZ_FMA(p3, r3, p2);
        q = GZ_FMA(q, r3, p1);
        double t = GZ_FMA(r, 134217728.0, r);          /* r + r*2^27 */
        double rhi = GZ_FMA(-134217728.0, r, t);       /* t - r*2^27 */
        double rhi2 = GZ_MUL(rhi, rhi);
        double rlo = GZ_SUB(r, rhi);
        double hi = GZ_FMA(rhi2, GZ_K(LOG_B0), r);
        double lo = GZ_FMA(rhi2, GZ_K(LOG_B0), GZ_SUB(r, hi));
        double rr = GZ_ADD(r, rhi);
        double c = GZ_MUL(GZ_K(LOG_B0), rlo);
        lo = GZ_FMA(c, rr, lo);
        double y = GZ_FMA(q, r3, lo);
        return GZ_ADD(hi, y);
    }
    uint32_t top = (uint32_t)(ix >> 48);
    if (top - 0x0010u >= 0x7ff0u - 0x0010u) {
        if ((ix << 1) == 0) return GZ_DBL(0xfff0000000000000ULL);    /* log(+-0) = -inf */
        if (ix == 0x7ff0000000000000ULL) return x;                   /* log(inf) = inf */
        if ((top & 0x8000u) || (top & 0x7ff0u) == 0x7ff0u)
            return GZ_DBL(0x7ff8000000000000ULL);                     /* negative or nan */
        /* subnormal: normalise */
        ix = GZ_BITS(GZ_MUL(x, 4503599627370496.0 /* 2^52 */)) - (52ULL << 52);
    }
    return gz_log_core(ix, tab);
}

/* glibc log's table path for the bit pattern of a positive normal x outside the
   near-1 interval (the tail of gz_log_t, callable directly when the caller
   already knows the branch) */
GZ_HD double gz_log_core(uint64_t ix, const uint64_t* __restrict__ tab)
{
    uint64_t tmp = ix - 0x3fe6000000000000ULL;
    uint32_t i = (uint32_t)(tmp >> 45) & 127u;
    int32_t k = (int32_t)((int64_t)tmp >> 52);
    uint64_t iz = ix - (tmp & 0xfff0000000000000ULL);
    double invc = GZ_DBL(tab[2 * i]);
    double logc = GZ_DBL(tab[2 * i + 1]);
    double z = GZ_DBL(iz);
    double kd = (double)k;
    double w = GZ_FMA(kd, GZ_K(LOG_LN2HI), logc);
    double r = GZ_FMA(z, invc, -1.0);
    double a12 = GZ_FMA(r, GZ_K(LOG_A2), GZ_K(LOG_A1));
    double hi = GZ_ADD(r, w);
    double r2 = GZ_MUL(r, r);
    double lo = GZ_ADD(GZ_SUB(w, hi), r);
    lo = GZ_FMA(kd, GZ_K(LOG_LN2LO), lo);
    double r3 = GZ_MUL(r, r2);
    double a34 = GZ_FMA(r, GZ_K(LOG_A4), GZ_K(LOG_A3));
    double t = GZ_FMA(r2, GZ_K(LOG_A0), lo);
    double a = GZ_FMA(a34, r2, a12);
    double y = GZ_FMA(r3, a, t);
    return GZ_ADD(y, hi);
}
