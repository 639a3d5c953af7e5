/*
 * gz_k_tma.cuh -- k_zig_tma: the lane-per-stream ziggurat for many streams
 * (configs 3 and 4 and any launch of >= 32768 streams with 16-byte-aligned
 * rows), built on the Blackwell data path.
 *
 * Not a standalone header: included by gz_engine.cu inside its anonymous
 * namespace, after the shared device globals and helpers it uses.
 *
 * Work split: a lane owns one stream and steps it exactly like the reference's
 * per-stream loop (engine.py:75-112 original, 114-151 modified ziggurat; the
 * attempt is ZigguratSampler._draw, samplers.py:95-115 / 144-165).  A warp owns
 * 32 consecutive streams = 32 rows of the output.
 *
 * Fast path without divergence.  Each lane makes TMA_K attempts per round with
 * no branch: the draw chain (LCG48 double step or SplitMix64 increment) runs
 * unconditionally, the layer row {ktab, wtab} comes from shared memory (8
 * replicas, one per 16-byte bank group, so a quarter-warp's gathers never
 * conflict), and a fast accept is committed by predicated instructions: the
 * deviate goes to the lane's ring slot, the per-row witnesses (xor checksum
 * bits, power sums) are folded in registers in deviate order.  The first
 * attempt that is not a fast accept (a wedge candidate, 2.7 % of attempts, or
 * a tail entry, 0.06 %) FREEZES the lane for the rest of the round: its state
 * stays after that attempt's draw, and later attempts of the round are not
 * committed.  After the round the warp resolves the frozen lanes together
 * (one pass: recover the attempt's draw from the state, draw the wedge's
 * uniform, float pre-filter and the exact glibc exp near the boundary, or the
 * tail loop), so the slow path costs one pass per round instead of one per
 * attempt that any lane of the warp needs it.  Per stream the draws, the
 * accept/reject decisions and the order of the deviates are exactly the
 * reference's.
 *
 * Output by TMA.  The ring of a warp is NT tiles of 32 rows x 16 deviates
 * (4 KiB, the SWIZZLE_128B layout a TMA tensor box expects: the 16-byte chunk c
 * of row r sits at chunk c ^ (r & 7)).  When every lane of the warp has
 * produced 32 more deviates, one lane issues two tensor stores
 * (cp.async.bulk.tensor.2d, SASS UTMASTG) of 16 columns each: 256-byte row
 * segments, which calibration (tools/calib/calib_tma.cu) measured at 6.2 TB/s
 * against 5.0 TB/s for lane STG.128 of 128-byte segments.  The tensor map
 * clips rows beyond n_streams and columns beyond n_per.
 */
#pragma once

constexpr int TMA_TILE_BYTES = 32 * 128;
constexpr int TMA_REP = 8;             /* replicas of the layer rows */
constexpr uint64_t GZ_LCG_AINV = 0xDFE05BCB1365ULL;   /* 0x5DEECE66D^-1 mod 2^48 */
constexpr size_t TMA_SMEM_MAX = 232448;   /* sm_100 opt-in dynamic shared memory per block */

/* dynamic shared memory of k_zig_tma without the ring alignment slack */
__host__ __device__ constexpr size_t tma_smem_core(int NW, int NT, int NL, int K, bool lcg) { return (size_t)NW * NT * TMA_TILE_BYTES + (size_t)NL * 16 * TMA_REP + (size_t)NL * 8 + (lcg ? 16 * (size_t)(K + 1) : 0); }
/* a power-of-two ring whose base fits 16 KiB alignment: a slot address is one LOP3 */
__host__ __device__ constexpr bool tma_align16(int NW, int NT, int NL, int K, bool lcg, bool mut) { return !mut && (NT & (NT - 1)) == 0 && tma_smem_core(NW, NT, NL, K, lcg) + 16384 <= TMA_SMEM_MAX; }
__host__ __device__ constexpr size_t tma_smem_bytes(int NW, int NT, int NL, int K, bool lcg, bool mut) { return tma_smem_core(NW, NT, NL, K, lcg) + (tma_align16(NW, NT, NL, K, lcg, mut) ? 16384 : 1024); }

#ifndef TMA_CHV
#define TMA_CHV 1
#endif

__device__ __forceinline__ void tma_store_tile(const CUtensorMap* tm, uint32_t src, int c0, int r0)
{
    asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%1, %2}], [%3];" ::"l"(tm), "r"(c0),
                 "r"(r0), "r"(src)
                 : "memory");
}

/* TMA tensor load of one box into shared memory, completing on an mbarrier */
__device__ __forceinline__ void tma_load_tile(const CUtensorMap* tm, uint32_t dst, uint32_t mbar, int c0, int r0)
{
    asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
                 ::"r"(dst), "l"(tm), "r"(c0), "r"(r0), "r"(mbar)
                 : "memory");
}
__device__ __forceinline__ void mbar_init(uint32_t mbar, uint32_t count)
{
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(mbar), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint32_t mbar, uint32_t bytes)
{
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(mbar), "r"(bytes) : "memory");
}
__device__ __forceinline__ bool mbar_try_wait(uint32_t mbar, uint32_t parity)
{
    uint32_t ok;
    asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
                 : "=r"(ok)
                 : "r"(mbar), "r"(parity)
                 : "memory");
    return ok != 0;
}
/* all but the N most recent bulk groups of this thread have completed (writes performed) */
template <int N>
__device__ __forceinline__ void tma_wait_done_but() { asm volatile("cp.async.bulk.wait_group %0;" ::"n"(N) : "memory"); }

__device__ __forceinline__ void tma_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
__device__ __forceinline__ void tma_wait_read_all() { asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory"); }
__device__ __forceinline__ void tma_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }
__device__ __forceinline__ void fence_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

__device__ __forceinline__ void lds_u64x2_v(uint32_t a, uint64_t& x, uint64_t& y)
{
    asm volatile("ld.shared.v2.u64 {%0, %1}, [%2];" : "=l"(x), "=l"(y) : "r"(a));
}
/* a gather from a read-only table (layer rows, jump constants): not volatile, so the
   compiler may hoist it past the ring stores of earlier attempts */
__device__ __forceinline__ void lds_tab(uint32_t a, uint64_t& x, uint64_t& y)
{
    asm("ld.shared.v2.u64 {%0, %1}, [%2];" : "=l"(x), "=l"(y) : "r"(a));
}

/* one draw of the stream: `t` is the draw cursor (LCG: the unmasked 48-bit
   state, bits above 47 are don't-care; SplitMix64: the state), advanced
   unconditionally; returns the u64 of engine.py:52-58 / 60-66 */
template <int SRC>
__device__ __forceinline__ uint64_t tma_draw(uint64_t& t, uint64_t gam)
{
    if constexpr (SRC == 0) {
        const uint64_t t1 = t * GZ_LCG_A + GZ_LCG_C;
        const uint64_t t2 = t1 * GZ_LCG_A + GZ_LCG_C;
        t = t2;
        return ((uint64_t)(uint32_t)(t1 >> 16) << 32) | (uint32_t)(t2 >> 16);
    } else {
        t += gam;
        return gz_mix64(t);
    }
}

/* the draw that produced state S (S = the cursor right after it) */
template <int SRC>
__device__ __forceinline__ uint64_t tma_recover(uint64_t S)
{
    if constexpr (SRC == 0) {
        const uint64_t t1 = (S - GZ_LCG_C) * GZ_LCG_AINV;   /* the previous state, mod 2^48 */
        return ((uint64_t)(uint32_t)(t1 >> 16) << 32) | (uint32_t)(S >> 16);
    } else {
        return gz_mix64(S);
    }
}

/* layer index, mantissa and sign bit of an attempt (samplers.py:96-99 / 145-148) */
template <bool MOD>
__device__ __forceinline__ void tma_split(uint64_t u, uint32_t& i, uint64_t& m, uint64_t& sgn)
{
    if constexpr (MOD) {
        i = (uint32_t)u & 255u;
        m = u >> 9;
        sgn = (u >> 8) << 63;
    } else {
        i = (uint32_t)(u >> 56) & 127u;
        m = u & 0x00ffffffffffffffULL;
        sgn = u & 0x8000000000000000ULL;
    }
}

/* one LCG48 step on 32-bit halves, (h:l) <- A*(h:l) + C mod 2^64 (only bits 0..47
   matter): IMAD.WIDE.U32 of the low words with the increment, two IMADs for the
   cross terms (A = 0x5_DEECE66D) */
/* The cross terms ride on the product's high word as a chain of two IMADs (mad.lo.u32
   spelled out, the halves taken by a register-pair move): written as a sum, the compiler
   computes them beside the wide product and joins the two with an extra 3-input add on
   the ALU pipe (8 instructions per two steps instead of 6). */
/* (mad_lo32 and u64_halves: gz_device.cuh) */
__device__ __forceinline__ void lcg_step32(uint32_t l, uint32_t h, uint32_t& ol, uint32_t& oh, uint64_t inc)
{
    uint32_t ph;
    u64_halves((uint64_t)l * 0xDEECE66Du + inc, ol, ph);
    oh = mad_lo32(l, 5u, mad_lo32(h, 0xDEECE66Du, ph));
}
/* two steps at once, (A^2, A C + C): the same shape */
__device__ __forceinline__ void lcg_step32x2(uint32_t l, uint32_t h, uint32_t& ol, uint32_t& oh, uint64_t inc2)
{
    uint32_t ph;
    u64_halves((uint64_t)l * 0xB4600A69u + inc2, ol, ph);
    oh = mad_lo32(l, 0xBB20u, mad_lo32(h, 0xB4600A69u, ph));
}

/* the draw cursor of one round.  LCG48: 32-bit halves of the unmasked state (bits
   above 47 are don't-care: they only reach bits >= 48 of later products); one
   u64 = two steps t1 = A*t + C, t2 = A*t1 + C, each one IMAD.WIDE.U32 and two
   IMADs (A = 0x5_DEECE66D), and the draw's halves are bits 16..47 of t1 and t2
   (engine.py:52-58, unsigned OR).  SplitMix64: t += gamma, mix64 (engine.py:60-66). */
template <int SRC>
struct TmaCursor {
    uint32_t lo, hi;
    __device__ __forceinline__ TmaCursor() : lo(0), hi(0) {}
    __device__ __forceinline__ explicit TmaCursor(uint64_t s) : lo((uint32_t)s), hi((uint32_t)(s >> 32)) {}
    __device__ __forceinline__ uint64_t state() const { return ((uint64_t)hi << 32) | lo; }
    __device__ __forceinline__ void draw(uint64_t gam, uint64_t inc2, uint32_t& uhi, uint32_t& ulo)
    {
        if constexpr (SRC == 0) {
            uint32_t t1l, t1h, t2l, t2h;
            lcg_step32(lo, hi, t1l, t1h, gam);   /* gam carries the increment 0xB for the LCG */
            /* the second state straight from the first (A^2, A*C + C): the two steps
               do not wait for each other */
            lcg_step32x2(lo, hi, t2l, t2h, inc2);
            uhi = __funnelshift_r(t1l, t1h, 16);
            ulo = __funnelshift_r(t2l, t2h, 16);
            lo = t2l;
            hi = t2h;
        } else {
            const uint64_t s = state() + gam;
            lo = (uint32_t)s;
            hi = (uint32_t)(s >> 32);
            const uint64_t u = gz_mix64(s);
            uhi = (uint32_t)(u >> 32);
            ulo = (uint32_t)u;
        }
    }
};

/* byte offset of the layer row (x 128: 8 replicas of 16 B), mantissa halves and
   the sign (bit 31 of the high word) of an attempt (samplers.py:96-99 / 145-148) */
template <bool MOD>
__device__ __forceinline__ void tma_split32(uint32_t uhi, uint32_t ulo, uint32_t& ioff, uint32_t& mhi, uint32_t& mlo,
                                            uint32_t& sgn)
{
    if constexpr (MOD) {
        ioff = (ulo & 255u) << 7;
        mlo = __funnelshift_r(ulo, uhi, 9);
        mhi = uhi >> 9;
        sgn = (ulo << 23) & 0x80000000u;
    } else {
        ioff = (uhi >> 17) & 0x3f80u;
        mhi = uhi & 0x00ffffffu;
        mlo = ulo;
        sgn = uhi & 0x80000000u;
    }
}

/* ring slot of deviate w of this lane's row: tile (w / 16) mod NT, 16-byte
   chunk ((w mod 16) / 2) ^ (row mod 8) (SWIZZLE_128B), 8-byte half w mod 2 */
/* Ring position counter.  Deviate w of a lane's row lives in ring tile
   (w / 16) mod NT, 16-byte chunk ((w mod 16) / 2) ^ (row mod 8) (SWIZZLE_128B) and
   8-byte half w mod 2.  The lane keeps
       C(w) = (w / 16) << 12 | 0xF80 | (w mod 16) << 3
   whose bits 7..11 are always ones, so C + 8 carries from the column bits straight
   into the tile bits: advancing is one add and one OR, and the slot address is one
   LOP3 ((C & tile|column mask) ^ row swizzle) plus the row base.  C is monotone in
   w, so limits and the warp minimum compare C directly. */
__device__ __forceinline__ uint32_t tma_cenc(int w) { return ((uint32_t)(w >> 4) << 12) | 0xF80u | ((uint32_t)(w & 15) << 3); }
__device__ __forceinline__ int tma_cdec(uint32_t c) { return (int)(((c >> 12) << 4) | ((c >> 3) & 15u)); }
__device__ __forceinline__ uint32_t tma_cinc(uint32_t c) { return (c + 8u) | 0xF80u; }
template <int NT>
__device__ __forceinline__ uint32_t tma_caddr(uint32_t my_row, uint32_t lx, uint32_t c)
{
    return my_row + ((c & (((NT - 1u) << 12) | 0x78u)) ^ lx);
}

/* per-row witnesses, in deviate order: xor of the bit patterns (bench.py:174-175)
   and the power sums the moments are merged from (stats.py:232-259) */
__device__ __forceinline__ void tma_fold_fp(uint64_t zb, double& a1, double& a2, double& a3, double& a4)
{
    const double z = __longlong_as_double((long long)zb);
    const double z2 = __dmul_rn(z, z);
    a1 = __dadd_rn(a1, z);
    a2 = __dadd_rn(a2, z2);
    a3 = __fma_rn(z2, z, a3);
    a4 = __fma_rn(z2, z2, a4);
}

__device__ __forceinline__ void tma_fold(uint64_t zb, uint64_t& ck, double& a1, double& a2, double& a3, double& a4)
{
    const double z = __longlong_as_double((long long)zb);
    ck ^= zb;
    const double z2 = __dmul_rn(z, z);
    a1 = __dadd_rn(a1, z);
    a2 = __dadd_rn(a2, z2);
    a3 = __fma_rn(z2, z, a3);
    a4 = __fma_rn(z2, z2, a4);
}

/*
 * EPI_MUTATE (config 5, x += sigma * z over every gene of `generations`
 * generations, samplers.py:195-200): the ring tiles are first filled with x by TMA
 * tensor LOADS (an mbarrier per ring slot; a lane writes a tile only after the
 * warp has seen its load complete), a commit replaces the slot's x with
 * x + sigma * z (two roundings), and the flush stores the tile back.  A row of the
 * warp's column sequence is generations x n_genes columns; generation g + 1 reads
 * a gene block that generation g stored n_genes/16 tiles earlier, so before every
 * load the lane that issues them waits until all but its 7 most recent stores have
 * completed (needs n_genes >= 16 (NT + 8)).
 */
template <int SRC, bool MOD, bool STATS, int NW, int NT, int FL, int TMA_K, int EPI = EPI_STORE>
__global__ void __launch_bounds__(NW * 32, 1) k_zig_tma(const __grid_constant__ LaneParams p,
                                                        const __grid_constant__ CUtensorMap tm)
{
    constexpr int NL = MOD ? 256 : 128;
    constexpr bool MUT = EPI == EPI_MUTATE;
    static_assert(!MUT || (SRC == 1 && !MOD && !STATS && FL == 1), "mutation: SplitMix64, original ziggurat");
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    const uint32_t raw_sh = sh_addr(smem_raw);
    /* SWIZZLE_128B tiles: 1 KiB aligned; the UNCOND rounds need the ring 16 KiB aligned */
    constexpr bool ALIGN16 = tma_align16(NW, NT, NL, TMA_K, SRC == 0, MUT);
    const uint32_t base_sh = ALIGN16 ? ((raw_sh + 16383u) & ~16383u) : ((raw_sh + 1023u) & ~1023u);
    unsigned char* base = smem_raw + (base_sh - raw_sh);
    constexpr uint32_t RING = NW * NT * TMA_TILE_BYTES;
    const uint32_t kw_sh = base_sh + RING;
    ulonglong2* s_kw = reinterpret_cast<ulonglong2*>(base + RING);
    float2* s_yf = reinterpret_cast<float2*>(base + RING + NL * 16 * TMA_REP);
    ulonglong2* s_jump = reinterpret_cast<ulonglong2*>(base + RING + NL * 16 * TMA_REP + NL * 8);
    /* EPI_MUTATE: one mbarrier per ring slot of each warp, after the tables */
    const uint32_t mbar_sh = base_sh + RING + NL * 16 * TMA_REP + NL * 8;
    for (int j = threadIdx.x; j < NL * TMA_REP; j += blockDim.x) s_kw[j] = p.kw[j / TMA_REP];
    for (int j = threadIdx.x; j < NL; j += blockDim.x) s_yf[j] = p.yf[j];
    /* LCG: (A, C) of 2n steps, n <= TMA_K (the state after n draws from a round's start) */
    if (SRC == 0 && threadIdx.x <= TMA_K) s_jump[threadIdx.x] = make_ulonglong2(c_lcgA[2 * threadIdx.x], c_lcgC[2 * threadIdx.x]);
    if (MUT && threadIdx.x < NW * NT) mbar_init(mbar_sh + 8 * threadIdx.x, 1);
    if constexpr (MUT) asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    __syncthreads();

    const int lane = threadIdx.x & 31;
    const int wib = threadIdx.x >> 5;
    const uint32_t wring = base_sh + wib * NT * TMA_TILE_BYTES;
    const uint32_t my_row = wring + lane * 128;
    const uint32_t lx = (uint32_t)(lane & 7) << 4;                  /* the row's swizzle */
    /* UNCOND rounds: with the ring base 16 KiB aligned (ALIGN16) my_row has no bit in the
       tile|column mask, so a slot address is ((C & mask) ^ rowx), one LOP3 */
    constexpr bool UNCOND = !MUT && (NT & (NT - 1)) == 0;
    const uint32_t rowx = my_row ^ lx;
    const uint32_t my_kw = kw_sh + lx;                              /* replica lane & 7 */
    const uint32_t yf_sh = sh_addr(s_yf);
    const uint32_t jump_sh = sh_addr(s_jump);
    /* LCG: the increments of one and two steps as opaque register pairs (an immediate
       addend would split every IMAD.WIDE.U32 into a multiply and a 64-bit add) */
    const uint64_t lcg_inc = SRC == 0 ? ld_keep(&c_lcgC[1]) : 0;
    const uint64_t lcg_inc2 = SRC == 0 ? ld_keep(&c_lcgC[2]) : 0;
    /* LCG draw chains of the UNCOND rounds: (A, C) of 2 (TMA_K / CH) j steps */
    uint64_t jA[TMA_CHV > 1 ? TMA_CHV : 1], jC[TMA_CHV > 1 ? TMA_CHV : 1];
#pragma unroll
    for (int j = 0; j < (TMA_CHV > 1 ? TMA_CHV : 1); ++j) {
        jA[j] = (SRC == 0 && j > 0) ? ld_keep(&c_lcgA[2 * (TMA_K / TMA_CHV) * j]) : 0;
        jC[j] = (SRC == 0 && j > 0) ? ld_keep(&c_lcgC[2 * (TMA_K / TMA_CHV) * j]) : 0;
    }
    const int n_per = p.n_per;
    const uint32_t guard32 = p.guard > 0xffffffffll ? 0xffffffffu : (uint32_t)p.guard;
    const int64_t n_streams = p.n_streams;
    const int64_t n_groups = (n_streams + 31) >> 5;
    const int64_t gstride = (int64_t)gridDim.x * NW;
    constexpr int FB = FL * 16;                                    /* columns per flush */
    constexpr int SLACK = (NT - FL) * 16;                          /* columns writable past the flushed ones */
    static_assert(((NT & (NT - 1)) == 0 || NT == 3) && FL <= NT / 2, "ring: 3 or a power of two tiles, at most half in flight");
    /* ring slot of a tile (a power-of-two ring: mask; three tiles: the lane tracks its
       tile's byte offset tb, advanced when the column bits of C wrap) */
    auto slot_of = [](int tile) { return (NT & (NT - 1)) == 0 ? (tile & (NT - 1)) : tile % NT; };

    /* The warp's rows (32 streams each: groups g0, g0 + gstride, ...) are one
       continuous sequence of ring columns, rowlen = n_per rounded up to a tile per
       row, so a lane that finishes a row starts its next row at once instead of
       waiting at the row end for the slowest lane of the warp. */
    const int64_t g0 = (int64_t)blockIdx.x * NW + wib;
    const uint32_t my_mbar = mbar_sh + 8 * NT * wib;
    if (g0 < n_groups) {
        /* a mutation row is every generation of one individual (n_per % 16 == 0) */
        const int rowlen = MUT ? n_per * p.generations : (n_per + 15) & ~15;
        const int n_row = MUT ? rowlen : n_per;       /* deviates per row */
        const int ng = (int)((n_groups - g0 + gstride - 1) / gstride);
        const int wtot = ng * rowlen;                 /* ring columns of this warp */
        const uint32_t c_end = tma_cenc(wtot);

        int k = -1;                   /* this lane's current row */
        int64_t sid = 0;
        bool valid = false, failed = false;
        uint64_t S = 0, gam = lcg_inc;
        uint32_t C = tma_cenc(0), c_rowend = tma_cenc(0);
        uint32_t tb = 0;              /* NT == 3: byte offset of C's ring tile */
        uint32_t rej = 0, c_rej = 0xffffffffu;
        int flushed = 0;                                          /* columns handed to TMA (warp-uniform) */
        int fk = 0, fcol = 0, fgene = 0;                          /* the flush position: row, column, gene */
        uint32_t c_lim = tma_cenc(min(wtot, NT * 16));            /* nothing in flight yet: the whole ring */
        uint32_t c_limr = 0;                                      /* min(c_lim, c_rowend) */
        uint32_t c_ring = tma_cenc(NT * 16);                      /* UNCOND: ring room, not capped at wtot */
        uint64_t ck = 0;
        double a1 = 0.0, a2 = 0.0, a3 = 0.0, a4 = 0.0;
        double sig = 0.0;                                         /* EPI_MUTATE: the row's sigma */
        /* EPI_MUTATE: x tiles loaded ahead (issued / seen complete by every lane) and the
           load position (row, gene column) of the next one */
        int ld_issued = 0, ld_ready = 0, lk = 0, lcol = 0, lgene = 0;
        bool just_flushed = false;   /* a store left this round: its slot is reloaded next round */
        auto issue_loads = [&](int upto) {
            /* lane 0 only: loads of tiles [ld_issued, upto) into their (free) ring slots */
            while (ld_issued < upto && ld_issued * 16 < wtot) {
                tma_wait_done_but<7>();   /* the previous generation's store of this gene block */
                asm volatile("fence.proxy.async.global;" ::: "memory");
                const int sl = slot_of(ld_issued);
                mbar_expect_tx(my_mbar + 8 * sl, TMA_TILE_BYTES);
                tma_load_tile(&tm, wring + sl * TMA_TILE_BYTES, my_mbar + 8 * sl, lgene,
                              (int)((g0 + (int64_t)lk * gstride) * 32));
                ++ld_issued;
                lgene += 16;
                if (lgene >= n_per) lgene = 0;
                lcol += 16;
                if (lcol >= rowlen) {
                    lcol = 0;
                    ++lk;
                }
            }
        };
        if constexpr (MUT) {
            if (lane == 0) issue_loads(NT);
            __syncwarp();
        }

        /* row transitions (divergent, once per row and lane): store the finished
           row's state, load the next row's */
        auto next_rows = [&]() {
            while (C >= c_rowend && k < ng) {
                if (valid && !failed) {
                    if constexpr (SRC == 0) {
                        p.state_out[sid] = S & GZ_MASK48;
                    } else {
                        p.state_out[2 * sid] = S;
                        p.state_out[2 * sid + 1] = gam;
                    }
                }
                ++k;
                failed = false;
                if (k < ng) {
                    sid = (g0 + k * gstride) * 32 + lane;
                    valid = sid < n_streams;
                    if (valid) {
                        if constexpr (SRC == 0) {
                            S = p.state_in[sid];
                        } else {
                            S = p.state_in[2 * sid];
                            gam = p.state_in[2 * sid + 1];
                        }
                        C = tma_cenc(k * rowlen);
                        c_rowend = tma_cenc(k * rowlen + n_row);
                        if constexpr (MUT) sig = p.sigma[sid];
                        if constexpr (NT == 3) tb = (uint32_t)slot_of((k * rowlen) >> 4) * TMA_TILE_BYTES;
                    } else {
                        C = c_rowend = tma_cenc((k + 1) * rowlen);   /* no stream: skip the row */
                    }
                } else {
                    valid = false;
                    C = c_end;
                }
            }
            c_limr = min(c_lim, c_rowend);
        };
        next_rows();
        /* EPI_MUTATE: tiles whose x load every lane has seen complete */
        auto poll_loads = [&]() {
            /* loads go only into slots whose store has been read, so the loaded tiles are
               exactly the writable ones */
            if (lane == 0 && !just_flushed && ld_issued < (flushed >> 4) + NT && ld_issued * 16 < wtot) {
                tma_wait_read_all();   /* the last store (issued a round ago) has been read */
                issue_loads((flushed >> 4) + NT);
            }
            ld_issued = __shfl_sync(GZ_FULL, ld_issued, 0);
            lk = __shfl_sync(GZ_FULL, lk, 0);
            lcol = __shfl_sync(GZ_FULL, lcol, 0);
            lgene = __shfl_sync(GZ_FULL, lgene, 0);
            int r = ld_ready;
            while (r < ld_issued && mbar_try_wait(my_mbar + 8 * slot_of(r), (uint32_t)(r / NT) & 1u)) ++r;
            ld_ready = (int)__reduce_min_sync(GZ_FULL, (unsigned)r);
            c_lim = tma_cenc(min(wtot, 16 * ld_ready));
            c_limr = min(c_lim, c_rowend);
        };
        if constexpr (MUT) poll_loads();

        while (true) {
            /* ---- one round: TMA_K attempts per lane, no branches ---- */
            bool frozen = false;
            const uint32_t C0 = C;
            TmaCursor<SRC> t(S);
            if constexpr (UNCOND) {
                /* every attempt's deviate goes to slot C0 + k unconditionally (the slots past the
                   committed prefix are rewritten later); the committed attempts are the leading
                   fast accepts, capped at the row end.  A lane writes only when the whole round
                   fits the ring room (act), so no slot of a tile in flight is touched. */
                const bool act = C0 < c_rowend && ((C0 + 8u * TMA_K) | 0xF80u) <= c_ring;
                uint32_t fm = 0;
                /* LCG: CH independent draw chains (chain j starts 2 KC j steps ahead by one jump),
                   so the attempts of different chains do not wait for each other */
                constexpr int CH = (SRC == 0 && TMA_K % TMA_CHV == 0) ? TMA_CHV : 1, KC = TMA_K / CH;
                static_assert(TMA_K % CH == 0, "chains split the round evenly");
                TmaCursor<SRC> tcs[CH] = {t};
#pragma unroll
                for (int j = 1; j < CH; ++j) tcs[j] = TmaCursor<SRC>(S * jA[j] + jC[j]);
                /* stores after the last attempt (see k_zig_lst: a table gather may not pass a
                   shared store in program order) */
                uint64_t zbs[TMA_K];
#pragma unroll
                for (int kk2 = 0; kk2 < TMA_K; ++kk2) {
                    uint32_t uhi, ulo;
                    tcs[kk2 / KC].draw(gam, lcg_inc2, uhi, ulo);
                    uint32_t ioff, mhi, mlo, sgn;
                    tma_split32<MOD>(uhi, ulo, ioff, mhi, mlo, sgn);
                    uint64_t kk, wb;
                    lds_tab(my_kw + ioff, kk, wb);
                    const uint64_t m = ((uint64_t)mhi << 32) | mlo;
                    const double x = __dmul_rn(__ull2double_rn(m), __longlong_as_double((long long)wb));
                    if (m < kk) fm |= 1u << kk2;
                    zbs[kk2] = (uint64_t)__double_as_longlong(x) ^ ((uint64_t)sgn << 32);
                    GZ_CHECK(ioff < NL * 128u, ioff);
                }
                if (act) {
#pragma unroll
                    for (int kk2 = 0; kk2 < TMA_K; ++kk2) {
                        const uint32_t cm = (C0 + 8u * kk2) & (((NT - 1u) << 12) | 0x78u);
                        const uint32_t a = ALIGN16 ? (cm ^ rowx) : (my_row + (cm ^ lx));
                        GZ_CHECK(a == tma_caddr<NT>(my_row, lx, (C0 + 8u * kk2) | 0xF80u), a);
                        asm volatile("st.shared.u64 [%0], %1;" ::"r"(a), "l"(zbs[kk2]) : "memory");
                    }
                }
                const int lead = __ffs(~fm) - 1;   /* leading fast accepts (fm < 2^TMA_K) */
                const uint32_t C_lead = (C0 + 8u * (uint32_t)lead) | 0xF80u;
                if (act) {
                    C = min(C_lead, c_rowend);
                    frozen = C_lead < c_rowend && lead < TMA_K;
                }
                GZ_CHECK(!act || tma_cdec(C) <= flushed + SLACK + FB, tma_cdec(C) - flushed);
            } else {
#pragma unroll
            for (int kk2 = 0; kk2 < TMA_K; ++kk2) {
                const bool live = !frozen && C < c_limr;
                uint32_t uhi, ulo;
                t.draw(gam, lcg_inc2, uhi, ulo);
                uint32_t ioff, mhi, mlo, sgn;
                tma_split32<MOD>(uhi, ulo, ioff, mhi, mlo, sgn);
                uint64_t kk, wb;
                lds_tab(my_kw + ioff, kk, wb);
                const uint64_t m = ((uint64_t)mhi << 32) | mlo;
                const double x = __dmul_rn(__ull2double_rn(m), __longlong_as_double((long long)wb));
                const bool ok = m < kk;
                const bool commit = live && ok;
                frozen = frozen || (live && !ok);
                const uint64_t zb = (uint64_t)__double_as_longlong(x) ^ ((uint64_t)sgn << 32);
                const uint32_t a = NT == 3 ? my_row + tb + ((C & 0x78u) ^ lx) : tma_caddr<NT>(my_row, lx, C);
                GZ_CHECK(ioff < NL * 128u, ioff);
                GZ_CHECK(!commit || (a >= wring && a < wring + NT * TMA_TILE_BYTES), a - wring);
                GZ_CHECK(!commit || tma_cdec(C) < flushed + SLACK + FB, tma_cdec(C) - flushed);
                /* EPI_MUTATE: the slot's x is read whether or not the attempt commits (the
                   address is inside the ring either way), so only the store is predicated */
                uint64_t sv = zb;
                if constexpr (MUT) {
                    double xo;
                    asm("ld.shared.f64 %0, [%1];" : "=d"(xo) : "r"(a));
                    sv = (uint64_t)__double_as_longlong(__dadd_rn(xo, __dmul_rn(sig, __longlong_as_double((long long)zb))));
                }
                if (commit) asm volatile("st.shared.u64 [%0], %1;" ::"r"(a), "l"(sv) : "memory");
                if constexpr (NT == 3) {
                    /* three tiles: advance the tile offset (branch-free) when the column wraps */
                    const uint32_t cn = tma_cinc(C);
                    const uint32_t tn = tb == 2u * TMA_TILE_BYTES ? 0u : tb + TMA_TILE_BYTES;
                    tb = (commit && (cn & 0x78u) == 0) ? tn : tb;
                    C = commit ? cn : C;
                } else {
                    C = commit ? tma_cinc(C) : C;
                }
            }
            }
            /* the live attempts are a prefix of the round: the committed ones plus a
               frozen one; the state after them by jump-ahead from the round's start */
            {
                const uint32_t n_live = (uint32_t)(tma_cdec(C) - tma_cdec(C0)) + (frozen ? 1u : 0u);
                GZ_CHECK(n_live <= (uint32_t)TMA_K, n_live);
                if constexpr (SRC == 0) {
                    uint64_t ja, jc;
                    lds_tab(jump_sh + 16 * n_live, ja, jc);
                    S = S * ja + jc;
                } else {
                    S += (uint64_t)n_live * gam;
                }
            }
            /* ---- the frozen lanes' slow attempts, resolved together ---- */
            if (__any_sync(GZ_FULL, frozen)) {
                if (frozen) {
                    const uint64_t u = tma_recover<SRC>(S);
                    uint32_t i;
                    uint64_t m, sgn;
                    tma_split<MOD>(u, i, m, sgn);
                    uint64_t kk, wb;
                    lds_tab(my_kw + (i << 7), kk, wb);
                    double x = __dmul_rn(__ull2double_rn(m), __longlong_as_double((long long)wb));
                    bool ok;
                    if (i != 0) {
                        /* wedge: the next draw is its uniform, whatever the outcome */
                        const uint64_t u2 = tma_draw<SRC>(S, gam);
                        ok = wedge_accept_f(u2, x, p.yd + i, lds_f32x2(yf_sh + 8 * i));
                        if (!ok) {
                            rej = (C == c_rej) ? rej + 1 : 1;   /* consecutive rejections */
                            c_rej = C;
                            if (rej >= guard32) {
                                failed = true;
                                gz_raise(GZ_ERR_GUARD, sid);
                                C = c_rowend;
                            }
                        }
                    } else {
                        const TailOut to = tail_seq<SRC>(S & (SRC == 0 ? GZ_MASK48 : ~0ULL), gam, p.r, p.guard);
                        S = to.st;
                        x = to.v;
                        ok = to.k >= 0;
                        if (!ok) {
                            failed = true;
                            gz_raise(GZ_ERR_GUARD, sid);
                            C = c_rowend;
                        }
                    }
                    GZ_CHECK(i < (uint32_t)NL, i);
                    if (ok) {
                        GZ_CHECK(C < c_limr, tma_cdec(C));
                        const uint64_t zb = (uint64_t)__double_as_longlong(x) ^ sgn;
                        const uint32_t a = NT == 3 ? my_row + tb + ((C & 0x78u) ^ lx) : tma_caddr<NT>(my_row, lx, C);
                        if constexpr (MUT) {
                            double xo;
                            asm volatile("ld.shared.f64 %0, [%1];" : "=d"(xo) : "r"(a) : "memory");
                            const double xn = __dadd_rn(xo, __dmul_rn(sig, __longlong_as_double((long long)zb)));
                            asm volatile("st.shared.f64 [%0], %1;" ::"r"(a), "d"(xn) : "memory");
                        } else if (!UNCOND || i == 0) {
                            /* (UNCOND: a wedge's slot already holds x, written in the round) */
                            asm volatile("st.shared.u64 [%0], %1;" ::"r"(a), "l"(zb) : "memory");
                        }
                        C = tma_cinc(C);
                        if constexpr (NT == 3) {
                            if ((C & 0x78u) == 0) tb = tb == 2u * TMA_TILE_BYTES ? 0u : tb + TMA_TILE_BYTES;
                        }
                    }
                }
            }
            next_rows();
            /* ---- hand complete blocks of FB columns to TMA ---- */
            const int minw = tma_cdec(__reduce_min_sync(GZ_FULL, C));
            just_flushed = false;
            while (minw - flushed >= FB || (minw >= wtot && flushed < wtot)) {
                const int cnt = min(FB, wtot - flushed);
                GZ_CHECK(cnt > 0 && flushed + cnt <= minw && fk < ng && fcol < rowlen, fcol);
                GZ_CHECK(fk * rowlen + fcol == flushed, flushed);
                if constexpr (STATS) {
                    /* per-row witnesses, folded in deviate order from this lane's row of
                       the tiles (stats.py:232-259 power sums, bench.py:174-175 xor) */
#pragma unroll
                    for (int j = 0; j < FL; ++j) {
                        if (16 * j < cnt) {
                            const int col = fcol + 16 * j;   /* FL > 1 needs rowlen % (16 FL) == 0 */
                            const uint32_t trow =
                                wring + slot_of((flushed >> 4) + j) * TMA_TILE_BYTES + lane * 128;
                            if (col + 16 <= n_per) {
#pragma unroll
                                for (int c2 = 0; c2 < 8; ++c2) {
                                    uint64_t v0, v1;
                                    lds_u64x2_v(trow + (((uint32_t)c2 << 4) ^ lx), v0, v1);
                                    ck ^= v0 ^ v1;
                                    tma_fold_fp(v0, a1, a2, a3, a4);
                                    tma_fold_fp(v1, a1, a2, a3, a4);
                                }
                            } else {
                                for (int c2 = 0; c2 < 8; ++c2) {
                                    uint64_t v0, v1;
                                    lds_u64x2_v(trow + (((uint32_t)c2 << 4) ^ lx), v0, v1);
                                    if (col + 2 * c2 < n_per) tma_fold(v0, ck, a1, a2, a3, a4);
                                    if (col + 2 * c2 + 1 < n_per) tma_fold(v1, ck, a1, a2, a3, a4);
                                }
                            }
                            if (col + 16 >= n_per) {
                                /* the row's last tile: its witnesses are complete */
                                const int64_t tsid = (g0 + (int64_t)fk * gstride) * 32 + lane;
                                if (tsid < n_streams) {
                                    if (p.checksum) p.checksum[tsid] = ck;
                                    if (p.psum) {
                                        p.psum[4 * tsid + 0] = a1;
                                        p.psum[4 * tsid + 1] = a2;
                                        p.psum[4 * tsid + 2] = a3;
                                        p.psum[4 * tsid + 3] = a4;
                                    }
                                }
                                ck = 0;
                                a1 = a2 = a3 = a4 = 0.0;
                            }
                        }
                    }
                }
                fence_async_smem();
                __syncwarp();
                if (lane == 0) {
                    tma_wait_read_all();   /* the previous block (issued >= FB columns ago) */
#pragma unroll
                    for (int j = 0; j < FL; ++j) {
                        if (16 * j < cnt)
                            tma_store_tile(&tm, wring + slot_of((flushed >> 4) + j) * TMA_TILE_BYTES,
                                           (MUT ? fgene : fcol) + 16 * j, (int)((g0 + (int64_t)fk * gstride) * 32));
                    }
                    tma_commit();
                }
                __syncwarp();
                flushed += cnt;
                fcol += cnt;
                if (fcol >= rowlen) {
                    fcol = 0;
                    ++fk;
                }
                if constexpr (MUT) {
                    fgene += cnt;
                    if (fgene >= n_per) fgene = 0;
                    just_flushed = true;
                } else {
                    c_lim = tma_cenc(min(wtot, flushed + SLACK));   /* the tiles of the block just freed */
                    c_ring = tma_cenc(flushed + SLACK);
                    c_limr = min(c_lim, c_rowend);
                }
            }
            if constexpr (MUT) poll_loads();
            if (minw >= wtot) break;   /* every row complete and handed to TMA */
        }
        if (lane == 0) tma_wait_all();
    }
}

