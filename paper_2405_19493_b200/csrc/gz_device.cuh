/*
 * gz_device.cuh -- per-lane PRNG steps, jump-ahead and small helpers shared by
 * the sm_100a kernels of gz_engine.cu.
 *
 * Sources restated (bit for bit):
 *   Lcg48      sources.py:56-80  (state <- (0x5DEECE66D*state + 0xB) mod 2^48;
 *              one u64 = top 32 bits of two consecutive states, high first,
 *              unsigned OR) -- engine.py:52-58 `_lcg_step`
 *   SplitMix64 sources.py:100-116 (state += gamma; out = mix64(state)) --
 *              engine.py:60-66 `_sm_step`; mix64 sources.py:83-87
 *   unit       sources.py:45-47 ((u >> 11) * 2^-53, exact)
 *
 * Jump-ahead: a warp decodes one stream with lane j evaluating draw k+j of a
 * 32*D-draw window.  SplitMix64's state after n draws is s0 + n*gamma; the
 * LCG's is A_n*s0 + C_n (mod 2^48) with (A_n, C_n) the n-fold composition,
 * precomputed on the host into c_lcgA/c_lcgC.
 */
#pragma once
#include <stdint.h>

#define GZ_FULL 0xffffffffu
#define GZ_MASK48 ((1ULL << 48) - 1ULL)
#define GZ_LCG_A 0x5DEECE66DULL
#define GZ_LCG_C 0xBULL
#define GZ_GOLDEN_GAMMA 0x9E3779B97F4A7C15ULL
#define GZ_LCG_JUMP_MAX 260

/* (A_n, C_n): state after n single LCG steps = A_n*s + C_n mod 2^48, stored in
 * __constant__ c_lcgA / c_lcgC (gz_engine.cu) for n < GZ_LCG_JUMP_MAX. */

/* 32-bit multiply-add and register-pair moves spelled out, so that the cross terms of a
   64-bit product ride on the wide product's high word as a chain of two IMADs: written as
   a sum, the compiler computes them beside the product and joins the two with one more
   add (4 instructions per 64 x 64 -> 64 multiply by a constant instead of 3). */
__device__ __forceinline__ uint32_t mad_lo32(uint32_t a, uint32_t b, uint32_t c)
{
    uint32_t r;
    asm("mad.lo.u32 %0, %1, %2, %3;" : "=r"(r) : "r"(a), "r"(b), "r"(c));
    return r;
}
__device__ __forceinline__ void u64_halves(uint64_t v, uint32_t& lo, uint32_t& hi)
{
    asm("mov.b64 {%0, %1}, %2;" : "=r"(lo), "=r"(hi) : "l"(v));
}
template <uint64_t CC>
__device__ __forceinline__ uint64_t gz_mul64c(uint64_t z)
{
    constexpr uint32_t clo = (uint32_t)CC, chi = (uint32_t)(CC >> 32);
    uint32_t zl, zh, pl, ph;
    u64_halves(z, zl, zh);
    u64_halves((uint64_t)zl * clo, pl, ph);
    uint64_t r;
    asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "r"(pl), "r"(mad_lo32(zl, chi, mad_lo32(zh, clo, ph))));
    return r;
}

/* sources.py:83-88 (mix64, the SplitMix64 finaliser) */
__device__ __forceinline__ uint64_t gz_mix64(uint64_t z)
{
    /* plain products: with gz_mul64c (3 instead of 4 instructions each) config 3 ran 465
       G/s against 481 -- the two multiplies are in series and the longer chain costs more
       than the two instructions save */
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}

__device__ __forceinline__ uint64_t gz_lcg_mad(uint64_t a, uint64_t s, uint64_t c)
{
    return (a * s + c) & GZ_MASK48;
}

/* u64 from the two LCG states t1 (first step) and t2 (second step) */
__device__ __forceinline__ uint64_t gz_lcg_u64(uint64_t t1, uint64_t t2)
{
    return ((t1 >> 16) << 32) | (t2 >> 16);
}

/* (u >> 11) * 2^-53: exact (53-bit integer, power-of-two scale) */
__device__ __forceinline__ double gz_unit53(uint64_t u)
{
    return __dmul_rn(__ull2double_rn(u >> 11), 1.1102230246251565e-16);
}

/* 2*unit - 1, exact: the polar method's v = 2.0 * next_f64_unit() - 1.0
 * (samplers.py:185-186) is exact in binary64, so one rounding suffices. */
__device__ __forceinline__ double gz_unit53_pm1(uint64_t u)
{
    return __fma_rn(__ull2double_rn(u >> 11), 2.220446049250313e-16, -1.0);
}

__device__ __forceinline__ uint32_t gz_bitrange(int b, int n)
{
    return n >= 32 ? GZ_FULL : (((1u << n) - 1u) << b);
}

/* sequential single-stream draw (used by the rare tail / window-extension paths) */
template <int SRC>
__device__ __forceinline__ uint64_t gz_next_seq(uint64_t& st, uint64_t gamma)
{
    if constexpr (SRC == 0) {
        uint64_t t1 = gz_lcg_mad(GZ_LCG_A, st, GZ_LCG_C);
        uint64_t t2 = gz_lcg_mad(GZ_LCG_A, t1, GZ_LCG_C);
        st = t2;
        return gz_lcg_u64(t1, t2);
    } else {
        st += gamma;
        return gz_mix64(st);
    }
}
