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
 * Output by TMA.  The ring of a warp is TMA_NT tiles of 32 rows x 16 deviates
 * (4 KiB, the SWIZZLE_128B layout a TMA tensor box expects: the 16-byte chunk c
 * of row r sits at chunk c ^ (r & 7)).  When every lane of the warp has
 * produced 32 more deviates, one lane issues two tensor stores
 * (cp.async.bulk.tensor.2d, SASS UTMASTG) of 16 columns each: 256-byte row
 * segments, which calibration (tools/calib/calib_tma.cu) measured at 6.2 TB/s
 * against 5.0 TB/s for lane STG.128 of 128-byte segments.  The tensor map
 * clips rows beyond n_streams and columns beyond n_per.
 */
#pragma once

constexpr int TMA_K = 8;               /* attempts per lane per round */
constexpr int TMA_NT = 4;              /* ring tiles per warp (power of two) */
constexpr int TMA_TILE_BYTES = 32 * 128;
constexpr int TMA_REP = 8;             /* replicas of the layer rows */
constexpr uint64_t GZ_LCG_AINV = 0xDFE05BCB1365ULL;   /* 0x5DEECE66D^-1 mod 2^48 */

__device__ __forceinline__ void tma_store_tile(const CUtensorMap* tm, uint32_t src, int c0, int r0)
{
    asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%1, %2}], [%3];" ::"l"(tm), "r"(c0),
                 "r"(r0), "r"(src)
                 : "memory");
}

__device__ __forceinline__ void tma_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
__device__ __forceinline__ void tma_wait_read_all() { asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory"); }
__device__ __forceinline__ void tma_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }
__device__ __forceinline__ void fence_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

__device__ __forceinline__ void lds_u64x2_v(uint32_t a, uint64_t& x, uint64_t& y)
{
    asm volatile("ld.shared.v2.u64 {%0, %1}, [%2];" : "=l"(x), "=l"(y) : "r"(a));
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

/* the draw cursor of one round.  LCG48: 32-bit halves of the unmasked state (bits
   above 47 are don't-care: they only reach bits >= 48 of later products); one
   u64 = two steps t1 = A*t + C, t2 = A*t1 + C, each one IMAD.WIDE.U32 and two
   IMADs (A = 0x5_DEECE66D), and the draw's halves are bits 16..47 of t1 and t2
   (engine.py:52-58, unsigned OR).  SplitMix64: t += gamma, mix64 (engine.py:60-66). */
template <int SRC>
struct TmaCursor {
    uint32_t lo, hi;
    __device__ __forceinline__ explicit TmaCursor(uint64_t s) : lo((uint32_t)s), hi((uint32_t)(s >> 32)) {}
    __device__ __forceinline__ uint64_t state() const { return ((uint64_t)hi << 32) | lo; }
    __device__ __forceinline__ void draw(uint64_t gam, uint32_t& uhi, uint32_t& ulo)
    {
        if constexpr (SRC == 0) {
            const uint64_t p1 = (uint64_t)lo * 0xDEECE66Du + 0xBu;
            const uint32_t t1l = (uint32_t)p1;
            const uint32_t t1h = (uint32_t)(p1 >> 32) + hi * 0xDEECE66Du + lo * 5u;
            const uint64_t p2 = (uint64_t)t1l * 0xDEECE66Du + 0xBu;
            const uint32_t t2l = (uint32_t)p2;
            const uint32_t t2h = (uint32_t)(p2 >> 32) + t1h * 0xDEECE66Du + t1l * 5u;
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

/* ring slot of deviate w of this lane's row: tile (w / 16) mod TMA_NT, 16-byte
   chunk ((w mod 16) / 2) ^ (row mod 8) (SWIZZLE_128B), 8-byte half w mod 2 */
__device__ __forceinline__ uint32_t tma_slot(uint32_t my_row, uint32_t lx, int w)
{
    return my_row + (((uint32_t)w << 8) & ((TMA_NT - 1) << 12)) + ((((uint32_t)w << 3) & 0x78u) ^ lx);
}

/* per-row witnesses, in deviate order: xor of the bit patterns (bench.py:174-175)
   and the power sums the moments are merged from (stats.py:232-259) */
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

template <int SRC, bool MOD, bool STATS, int NW>
__global__ void __launch_bounds__(NW * 32, 1) k_zig_tma(const __grid_constant__ LaneParams p,
                                                        const __grid_constant__ CUtensorMap tm)
{
    constexpr int NL = MOD ? 256 : 128;
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    const uint32_t raw_sh = sh_addr(smem_raw);
    const uint32_t base_sh = (raw_sh + 1023u) & ~1023u;            /* SWIZZLE_128B tiles: 1 KiB aligned */
    unsigned char* base = smem_raw + (base_sh - raw_sh);
    const uint32_t kw_sh = base_sh + NW * TMA_NT * TMA_TILE_BYTES;
    ulonglong2* s_kw = reinterpret_cast<ulonglong2*>(base + NW * TMA_NT * TMA_TILE_BYTES);
    float2* s_yf = reinterpret_cast<float2*>(base + NW * TMA_NT * TMA_TILE_BYTES + NL * 16 * TMA_REP);
    for (int j = threadIdx.x; j < NL * TMA_REP; j += blockDim.x) s_kw[j] = p.kw[j / TMA_REP];
    for (int j = threadIdx.x; j < NL; j += blockDim.x) s_yf[j] = p.yf[j];
    __syncthreads();

    const int lane = threadIdx.x & 31;
    const int wib = threadIdx.x >> 5;
    const uint32_t wring = base_sh + wib * TMA_NT * TMA_TILE_BYTES;
    const uint32_t my_row = wring + lane * 128;
    const uint32_t lx = (uint32_t)(lane & 7) << 4;                  /* the row's swizzle */
    const uint32_t my_kw = kw_sh + lx;                              /* replica lane & 7 */
    const uint32_t yf_sh = sh_addr(s_yf);
    const int total = p.n_per;
    const uint32_t guard32 = p.guard > 0xffffffffll ? 0xffffffffu : (uint32_t)p.guard;
    const int64_t n_streams = p.n_streams;
    const int64_t n_groups = (n_streams + 31) >> 5;
    const int64_t gstride = (int64_t)gridDim.x * NW;
    constexpr int SLACK = (TMA_NT - 2) * 16;                       /* columns writable past the flushed ones */

    for (int64_t grp = (int64_t)blockIdx.x * NW + wib; grp < n_groups; grp += gstride) {
        const int64_t row0 = grp * 32;
        const int64_t sid = row0 + lane;
        const bool valid = sid < n_streams;
        uint64_t S = 0, gam = 0;
        if (valid) {
            if constexpr (SRC == 0) {
                S = p.state_in[sid];
            } else {
                S = p.state_in[2 * sid];
                gam = p.state_in[2 * sid + 1];
            }
        }
        int w = valid ? 0 : total;     /* deviates produced */
        int flushed = 0;               /* columns handed to TMA (warp-uniform) */
        int lim = min(total, TMA_NT * 16);   /* nothing in flight yet: the whole ring */
        uint32_t rej = 0;
        int w_rej = -1;
        bool failed = false;
        uint64_t ck = 0;
        double a1 = 0.0, a2 = 0.0, a3 = 0.0, a4 = 0.0;

        while (true) {
            /* ---- one round: TMA_K attempts per lane, no branches ---- */
            bool frozen = false;
            TmaCursor<SRC> t(S);
#pragma unroll
            for (int k = 0; k < TMA_K; ++k) {
                const bool live = !frozen && w < lim;
                uint32_t uhi, ulo;
                t.draw(gam, uhi, ulo);
                if (live) S = t.state();
                uint32_t ioff, mhi, mlo, sgn;
                tma_split32<MOD>(uhi, ulo, ioff, mhi, mlo, sgn);
                uint64_t kk, wb;
                lds_u64x2_v(my_kw + ioff, kk, wb);
                const uint64_t m = ((uint64_t)mhi << 32) | mlo;
                const double x = __dmul_rn(__ull2double_rn(m), __longlong_as_double((long long)wb));
                const bool ok = m < kk;
                const bool commit = live && ok;
                frozen = frozen || (live && !ok);
                /* the commit is predicated, not branched: a skipped attempt folds +0.0 into
                   the witnesses, which leaves every sum (never -0.0) and the xor unchanged */
                const uint64_t zb = commit ? ((uint64_t)__double_as_longlong(x) ^ ((uint64_t)sgn << 32)) : 0ull;
                const uint32_t a = tma_slot(my_row, lx, w);
                if (commit) asm volatile("st.shared.u64 [%0], %1;" ::"r"(a), "l"(zb) : "memory");
                if constexpr (STATS) tma_fold(zb, ck, a1, a2, a3, a4);
                w += commit ? 1 : 0;
            }
            /* ---- the frozen lanes' slow attempts, resolved together ---- */
            if (__any_sync(GZ_FULL, frozen)) {
                if (frozen) {
                    const uint64_t u = tma_recover<SRC>(S);
                    uint32_t i;
                    uint64_t m, sgn;
                    tma_split<MOD>(u, i, m, sgn);
                    uint64_t kk, wb;
                    lds_u64x2_v(my_kw + (i << 7), kk, wb);
                    double x = __dmul_rn(__ull2double_rn(m), __longlong_as_double((long long)wb));
                    bool ok;
                    if (i != 0) {
                        /* wedge: the next draw is its uniform, whatever the outcome */
                        const uint64_t u2 = tma_draw<SRC>(S, gam);
                        ok = wedge_accept_f(u2, x, p.yd + i, lds_f32x2(yf_sh + 8 * i));
                        if (!ok) {
                            rej = (w == w_rej) ? rej + 1 : 1;   /* consecutive rejections */
                            w_rej = w;
                            if (rej >= guard32) {
                                failed = true;
                                w = total;
                            }
                        }
                    } else {
                        const TailOut to = tail_seq<SRC>(S & (SRC == 0 ? GZ_MASK48 : ~0ULL), gam, p.r, p.guard);
                        S = to.st;
                        x = to.v;
                        ok = to.k >= 0;
                        if (!ok) {
                            failed = true;
                            w = total;
                        }
                    }
                    if (ok) {
                        const uint64_t zb = (uint64_t)__double_as_longlong(x) ^ sgn;
                        asm volatile("st.shared.u64 [%0], %1;" ::"r"(tma_slot(my_row, lx, w)), "l"(zb) : "memory");
                        if constexpr (STATS) tma_fold(zb, ck, a1, a2, a3, a4);
                        ++w;
                    }
                }
            }
            /* ---- hand complete 32-column blocks to TMA ---- */
            const int minw = (int)__reduce_min_sync(GZ_FULL, (unsigned)w);
            while (minw - flushed >= 32 || (minw >= total && flushed < total)) {
                const int cnt = min(32, total - flushed);
                fence_async_smem();
                __syncwarp();
                if (lane == 0) {
                    tma_wait_read_all();   /* the previous block (issued >= 32 columns ago) */
                    const int tile = (flushed >> 4) & (TMA_NT - 1);
                    tma_store_tile(&tm, wring + tile * TMA_TILE_BYTES, flushed, (int)row0);
                    if (cnt > 16)
                        tma_store_tile(&tm, wring + ((tile + 1) & (TMA_NT - 1)) * TMA_TILE_BYTES, flushed + 16,
                                       (int)row0);
                    tma_commit();
                }
                __syncwarp();
                flushed += cnt;
                lim = min(total, flushed + SLACK);   /* the tiles of the block just freed */
            }
            if (minw >= total) break;   /* every row complete and handed to TMA */
        }
        if (valid) {
            if (failed) {
                gz_raise(GZ_ERR_GUARD, sid);
            } else {
                if constexpr (SRC == 0) {
                    p.state_out[sid] = S & GZ_MASK48;
                } else {
                    p.state_out[2 * sid] = S;
                    p.state_out[2 * sid + 1] = gam;
                }
                if constexpr (STATS) {
                    if (p.checksum) p.checksum[sid] = ck;
                    if (p.psum) {
                        p.psum[4 * sid + 0] = a1;
                        p.psum[4 * sid + 1] = a2;
                        p.psum[4 * sid + 2] = a3;
                        p.psum[4 * sid + 3] = a4;
                    }
                }
            }
        }
        /* the ring is reused by the next group: its last blocks must have been read */
        if (lane == 0) tma_wait_read_all();
        __syncwarp();
    }
    if (lane == 0) tma_wait_all();
}
