/*
 * gz_k_lane.cuh -- the lane-per-stream kernels (k_zig_lane incl. the fused mutation, k_polar_lane, k_polar_lqd).
 *
 * Not a standalone header: included by gz_engine.cu inside its anonymous
 * namespace, after the shared device globals and helpers it uses.
 */
#pragma once

/* ------------------------------------------------- lane-per-stream kernels */

/*
 * For launches with many streams (configs 2-4: >= 2^20 streams) one LANE owns
 * one stream and steps it sequentially, exactly like the reference loop
 * (engine.py:75-112, 114-151, 153-181); no jump-ahead or parse is needed.  A
 * warp's 32 rows are staged through a shared-memory ring (LRING deviates per
 * lane) and flushed LK columns at a time as 128-byte row segments, so global
 * stores stay coalesced although every lane writes a different row.  Lanes
 * drift apart by their rejections; the ring absorbs the drift.
 */
constexpr int LK = 16;           /* flush width (deviates per row per flush) */
constexpr int LRING = 2 * LK;    /* ring capacity per lane (power of two) */
constexpr int LSTRIDE = LRING + 1;
constexpr int LANE_THREADS = 256;
constexpr int LANE_WARPS = LANE_THREADS / 32;

struct LaneParams {
    int64_t n_streams, ld;
    int n_per;
    const uint64_t* state_in;
    uint64_t* state_out;
    const double* spare_in;
    const uint8_t* has_in;
    double* spare_out;
    uint8_t* has_out;
    double* out;
    uint64_t* checksum;
    double* psum;
    const ulonglong2* kw;
    const double2* yd;
    const float2* yf;
    int n_layers, index_bits;
    double r;
    int64_t guard;
    int vec_ok;
    const double* sigma;    /* EPI_MUTATE: per-row step sizes */
    int generations;        /* EPI_MUTATE */
};

/* write ring slots [f, f + cnt) of the warp's 32 rows to out columns [col, col + cnt) */
__device__ __forceinline__ void lane_flush(const double* ring, double* out, int64_t ld, int64_t row0, int64_t n_rows,
                                           int f, int64_t col, int cnt, bool vec, int lane)
{
    const int c0 = f & (LRING - 1);
    if (vec && cnt == LK) {
        const int q = lane & 7;         /* 16-byte piece of a 128-byte row segment */
        const int rq = lane >> 3;
        double* base = out + (row0 + rq) * ld + col + 2 * q;
        const int64_t step = 4 * ld;
        const double* src = ring + rq * LSTRIDE + c0 + 2 * q;
        if (row0 + 32 <= n_rows) {
            /* a full group of 32 rows: no per-row bounds checks */
#pragma unroll
            for (int it = 0; it < 8; ++it)
                *reinterpret_cast<double2*>(base + it * step) =
                    make_double2(src[it * 4 * LSTRIDE], src[it * 4 * LSTRIDE + 1]);
        } else {
#pragma unroll
            for (int it = 0; it < 8; ++it) {
                if (row0 + it * 4 + rq < n_rows)
                    *reinterpret_cast<double2*>(base + it * step) =
                        make_double2(src[it * 4 * LSTRIDE], src[it * 4 * LSTRIDE + 1]);
            }
        }
    } else {
        for (int rr = 0; rr < 32; ++rr) {
            if (lane < cnt && row0 + rr < n_rows) out[(row0 + rr) * ld + col + lane] = ring[rr * LSTRIDE + c0 + lane];
        }
    }
}

/* the inverse of lane_flush for LK columns: read x columns [col, col + LK) of the
   warp's 32 rows into ring slots [f, f + LK) (EPI_MUTATE) */
__device__ __forceinline__ void lane_fetch(double* ring, const double* x, int64_t ld, int64_t row0, int64_t n_rows,
                                           int f, int64_t col, bool vec, int lane)
{
    const int c0 = f & (LRING - 1);
    if (vec) {
        const int q = lane & 7;
        const int rq = lane >> 3;
        const double* base = x + (row0 + rq) * ld + col + 2 * q;
        double* dst = ring + rq * LSTRIDE + c0 + 2 * q;
#pragma unroll
        for (int it = 0; it < 8; ++it) {
            if (row0 + it * 4 + rq < n_rows) {
                const double2 v = *reinterpret_cast<const double2*>(base + (int64_t)(it * 4) * ld);
                dst[it * 4 * LSTRIDE] = v.x;
                dst[it * 4 * LSTRIDE + 1] = v.y;
            }
        }
    } else {
        for (int rr = 0; rr < 32; ++rr) {
            if (lane < LK && row0 + rr < n_rows) ring[rr * LSTRIDE + c0 + lane] = x[(row0 + rr) * ld + col + lane];
        }
    }
}

/* per-row witnesses over columns [f, f + cnt) of this lane's ring row */
__device__ __forceinline__ void lane_stats(const double* myring, int f, int cnt, uint64_t& ck, double& a1, double& a2,
                                           double& a3, double& a4)
{
    for (int c = 0; c < cnt; ++c) {
        const double v = myring[(f + c) & (LRING - 1)];
        ck ^= (uint64_t)__double_as_longlong(v);
        const double v2 = __dmul_rn(v, v);
        a1 = __dadd_rn(a1, v);
        a2 = __dadd_rn(a2, v2);
        a3 = __fma_rn(v2, v, a3);
        a4 = __fma_rn(v2, v2, a4);
    }
}

/* lane_fetch split in two for 16-byte-aligned rows: issue the loads of a chunk one
   flush early into registers, land them in the ring at the next flush */
__device__ __forceinline__ void lane_fetch_issue(double2 (&pf)[8], const double* x, int64_t ld, int64_t row0,
                                                 int64_t n_rows, int64_t col, int lane)
{
    const int q = lane & 7;
    const int rq = lane >> 3;
    const double* base = x + (row0 + rq) * ld + col + 2 * q;
    const int64_t step = 4 * ld;
    const bool full = row0 + 32 <= n_rows;
#pragma unroll
    for (int it = 0; it < 8; ++it)
        if (full || row0 + it * 4 + rq < n_rows) pf[it] = *reinterpret_cast<const double2*>(base + it * step);
}

__device__ __forceinline__ void lane_fetch_land(double* ring, const double2 (&pf)[8], int64_t row0, int64_t n_rows,
                                                int f, int lane)
{
    const int q = lane & 7;
    const int rq = lane >> 3;
    double* dst = ring + rq * LSTRIDE + (f & (LRING - 1)) + 2 * q;
    const bool full = row0 + 32 <= n_rows;
#pragma unroll
    for (int it = 0; it < 8; ++it) {
        if (full || row0 + it * 4 + rq < n_rows) {
            dst[it * 4 * LSTRIDE] = pf[it].x;
            dst[it * 4 * LSTRIDE + 1] = pf[it].y;
        }
    }
}

template <int SRC>
__device__ __forceinline__ uint64_t lane_next(uint64_t& S, uint64_t gam)
{
    if constexpr (SRC == 0) {
        /* the reference's independent double step (engine.py:42-43, 52-58) */
        const uint64_t t1 = gz_lcg_mad(GZ_LCG_A, S, GZ_LCG_C);
        const uint64_t t2 = gz_lcg_mad(0xBB20B4600A69ULL, S, 0x40942DE6BAULL);
        S = t2;
        return gz_lcg_u64(t1, t2);
    } else {
        S += gam;
        return gz_mix64(S);
    }
}

/* SplitMix64: the draw after state S, mixed one attempt ahead (off the critical
   path).  The LCG's double step is cheap and stays in place (measured slower
   when pipelined). */
template <int SRC>
__device__ __forceinline__ void lane_pend(uint64_t S, uint64_t gam, uint64_t& nxt)
{
    if constexpr (SRC == 1) nxt = gz_mix64(S + gam);
}

/* consume the next draw (and, for SplitMix64, mix the one after it) */
template <int SRC>
__device__ __forceinline__ uint64_t lane_take(uint64_t& S, uint64_t gam, uint64_t& nxt)
{
    if constexpr (SRC == 0) {
        return lane_next<SRC>(S, gam);
    } else {
        const uint64_t u = nxt;
        S += gam;
        lane_pend<SRC>(S, gam, nxt);
        return u;
    }
}

template <int SRC>
__device__ __forceinline__ void lane_load_state(const LaneParams& p, int64_t sid, bool valid, uint64_t& S, uint64_t& gam)
{
    S = 0;
    gam = 0;
    if (valid) {
        if constexpr (SRC == 0) {
            S = p.state_in[sid];
        } else {
            S = p.state_in[2 * sid];
            gam = p.state_in[2 * sid + 1];
        }
    }
}

template <int SRC>
__device__ __forceinline__ void lane_store_state(const LaneParams& p, int64_t sid, uint64_t S, uint64_t gam)
{
    if constexpr (SRC == 0) {
        p.state_out[sid] = S;
    } else {
        p.state_out[2 * sid] = S;
        p.state_out[2 * sid + 1] = gam;
    }
}

/* explicit shared-window addressing for the lane loop: 32-bit shared addresses
   computed once (generic pointers into dynamic shared memory cost a window-base
   computation per access on sm_100) */
__device__ __forceinline__ uint32_t sh_addr(const void* ptr)
{
    return (uint32_t)__cvta_generic_to_shared(ptr);
}

__device__ __forceinline__ ulonglong2 lds_u64x2(uint32_t a)
{
    ulonglong2 v;
    asm("ld.shared.v2.u64 {%0, %1}, [%2];" : "=l"(v.x), "=l"(v.y) : "r"(a));
    return v;
}

__device__ __forceinline__ float2 lds_f32x2(uint32_t a)
{
    float2 v;
    asm("ld.shared.v2.f32 {%0, %1}, [%2];" : "=f"(v.x), "=f"(v.y) : "r"(a));
    return v;
}

__device__ __forceinline__ double lds_f64(uint32_t a)
{
    double v;
    asm volatile("ld.shared.f64 %0, [%1];" : "=d"(v) : "r"(a) : "memory");
    return v;
}

__device__ __forceinline__ void sts_f64(uint32_t a, double v)
{
    asm volatile("st.shared.f64 [%0], %1;" ::"r"(a), "d"(v) : "memory");
}

/* lane_stats over a full group: cnt == LK and f a multiple of LK, so the LK values
   are contiguous in the ring (same order, same roundings as lane_stats) */
__device__ __forceinline__ void lane_stats_full(uint32_t myring_sh, int f, uint64_t& ck, double& a1, double& a2,
                                                double& a3, double& a4)
{
    const uint32_t base = myring_sh + 8 * (f & (LRING - 1));
#pragma unroll
    for (int c = 0; c < LK; ++c) {
        const double v = lds_f64(base + 8 * c);
        ck ^= (uint64_t)__double_as_longlong(v);
        const double v2 = __dmul_rn(v, v);
        a1 = __dadd_rn(a1, v);
        a2 = __dadd_rn(a2, v2);
        a3 = __fma_rn(v2, v, a3);
        a4 = __fma_rn(v2, v2, a4);
    }
}

template <int SRC, int IBT, bool MOD, bool STATS, int EPI = EPI_STORE>
__global__ void __launch_bounds__(LANE_THREADS, EPI == EPI_MUTATE ? 2 : 3) k_zig_lane(const __grid_constant__ LaneParams p)
{
    extern __shared__ __align__(16) unsigned char smem[];
    const int nl = IBT ? (1 << IBT) : p.n_layers;
    ulonglong2* s_kw = reinterpret_cast<ulonglong2*>(smem);
    float2* s_yf = reinterpret_cast<float2*>(smem + 16 * nl);
    /* the double wedge rows are read only near the accept boundary: global memory,
       except for the (occupancy-limited, 2-warp-block) mutation launches */
    constexpr bool YD_SMEM = EPI == EPI_MUTATE;
    double2* s_yd = reinterpret_cast<double2*>(smem + 24 * nl);
    double* s_ring = reinterpret_cast<double*>(smem + (YD_SMEM ? 40 : 24) * nl);
    for (int i = threadIdx.x; i < nl; i += blockDim.x) {
        s_kw[i] = p.kw[i];
        s_yf[i] = p.yf[i];
        if constexpr (YD_SMEM) s_yd[i] = p.yd[i];
    }
    __syncthreads();
    const int lane = threadIdx.x & 31;
    const int wib = threadIdx.x >> 5;
    double* ring = s_ring + wib * 32 * LSTRIDE;
    double* myring = ring + lane * LSTRIDE;
    const uint32_t kw_sh = sh_addr(s_kw), yf_sh = sh_addr(s_yf), myring_sh = sh_addr(myring);
    const int ib = IBT ? IBT : p.index_bits;
    const uint32_t imask = (uint32_t)nl - 1u;
    const int mbits = 63 - ib;
    const uint64_t mmask = (1ULL << mbits) - 1ULL;
    const double r = p.r;
    const int n_per = p.n_per;
    /* EPI_MUTATE walks the row `generations` times: deviate w updates column w mod n_per */
    const int total = EPI == EPI_MUTATE ? n_per * p.generations : n_per;
    const int64_t guard = p.guard;
    /* consecutive wedge rejections are counted in 32 bits: a guard above
       2^32 - 1 behaves as 2^32 - 1 (4e9 consecutive rejections) */
    const uint32_t guard32 = guard > 0xffffffffll ? 0xffffffffu : (uint32_t)guard;
    const int64_t n_streams = p.n_streams;
    const int64_t n_groups = (n_streams + 31) >> 5;
    const int nwb = (int)(blockDim.x >> 5);
    const int64_t gstride = (int64_t)gridDim.x * nwb;

    for (int64_t grp = (int64_t)blockIdx.x * nwb + wib; grp < n_groups; grp += gstride) {
        const int64_t row0 = grp * 32;
        const int64_t sid = row0 + lane;
        const bool valid = sid < n_streams;
        uint64_t S, gam;
        lane_load_state<SRC>(p, sid, valid, S, gam);
        uint64_t nxt = 0;
        lane_pend<SRC>(S, gam, nxt);
        int w = valid ? 0 : total;       /* deviates produced by this lane */
        int flushed = 0;                 /* warp-uniform */
        int fcol = 0;                    /* row column of slot `flushed` */
        double sig = 0.0;
        double2 pf[8];                   /* EPI_MUTATE: the next refill chunk in flight */
        if constexpr (EPI == EPI_MUTATE) {
            if (valid) sig = p.sigma[sid];
            lane_fetch(ring, p.out, p.ld, row0, n_streams, 0, 0, p.vec_ok, lane);
            lane_fetch(ring, p.out, p.ld, row0, n_streams, LK, LK, p.vec_ok, lane);
            if (p.vec_ok) lane_fetch_issue(pf, p.out, p.ld, row0, n_streams, 2 * LK, lane);
            __syncwarp();
        }
        bool failed = false;
        uint32_t rej = 0;
        uint64_t ck = 0;
        double a1 = 0.0, a2 = 0.0, a3 = 0.0, a4 = 0.0;

        while (true) {
            const int lim = min(total, flushed + LRING);
#pragma unroll 4
            for (int it = 0; it < LK; ++it) {
                if (w < lim) {
                    /* one attempt of ZigguratSampler._draw (samplers.py:95-115) */
                    const uint64_t u = lane_take<SRC>(S, gam, nxt);
                    uint32_t i;
                    uint64_t m, sgn;
                    if constexpr (MOD) {
                        i = (uint32_t)u & imask;
                        m = u >> (ib + 1);
                        sgn = (u >> ib) << 63;
                    } else {
                        i = (uint32_t)(u >> mbits) & imask;
                        m = u & mmask;
                        sgn = u & 0x8000000000000000ULL;
                    }
                    const ulonglong2 kw = lds_u64x2(kw_sh + 16 * i);
                    double x = __dmul_rn(__ull2double_rn(m), __longlong_as_double((long long)kw.y));
                    bool ok = m < kw.x;
                    if (!ok) {
                        if (i != 0) {
                            /* wedge: the next draw is its uniform */
                            const uint64_t u2 = lane_take<SRC>(S, gam, nxt);
                            ok = wedge_accept_f(u2, x, YD_SMEM ? s_yd + i : p.yd + i, lds_f32x2(yf_sh + 8 * i));
                            if (!ok && ++rej >= guard32) {
                                failed = true;
                                w = total;
                            }
                        } else {
                            /* r and the guard loaded here (volatile asm on the __grid_constant__
                               block): otherwise their loads are hoisted into the fast path */
                            double tr = r;
                            int64_t tg = guard;
                            if constexpr (EPI != EPI_MUTATE) {
                                asm volatile("ld.f64 %0, [%1];" : "=d"(tr) : "l"(&p.r));
                                asm volatile("ld.s64 %0, [%1];" : "=l"(tg) : "l"(&p.guard));
                            }
                            const TailOut to = tail_seq<SRC>(S, gam, tr, tg);
                            S = to.st;
                            lane_pend<SRC>(S, gam, nxt);
                            x = to.v;
                            ok = to.k >= 0;
                            if (!ok) {
                                failed = true;
                                w = total;
                            }
                        }
                    }
                    if (ok) {
                        rej = 0;
                        /* sign by bit flip: identical to the reference's negation */
                        const double z = __longlong_as_double((long long)((uint64_t)__double_as_longlong(x) ^ sgn));
                        const uint32_t slot = myring_sh + 8 * (w & (LRING - 1));
                        GZ_CHECK(w < lim && w - flushed < LRING, w - flushed);
                        if constexpr (EPI == EPI_MUTATE) {
                            sts_f64(slot, __dadd_rn(lds_f64(slot), __dmul_rn(sig, z)));
                        } else {
                            sts_f64(slot, z);
                        }
                        ++w;
                    }
                }
            }
            const int lag = (int)__reduce_min_sync(GZ_FULL, (unsigned)(w - flushed));
            const bool done = __all_sync(GZ_FULL, w >= total);
            const int cnt = lag >= LK ? LK : (done ? total - flushed : 0);
            GZ_CHECK(cnt >= 0 && cnt <= LK && fcol >= 0, cnt);
            if (cnt > 0) {
                __syncwarp();
                if constexpr (STATS) {
                    if (cnt == LK) lane_stats_full(myring_sh, flushed, ck, a1, a2, a3, a4);
                    else lane_stats(myring, flushed, cnt, ck, a1, a2, a3, a4);
                }
                lane_flush(ring, p.out, p.ld, row0, n_streams, flushed, fcol, cnt, p.vec_ok, lane);
                flushed += cnt;
                if constexpr (EPI == EPI_MUTATE) {
                    /* cnt == LK here: n_per is a multiple of LK (>= 4 LK); refill the freed
                       slots with the columns of deviates [flushed + LK, flushed + 2 LK),
                       loaded at the previous flush, and put the next chunk in flight */
                    fcol += cnt;
                    if (fcol >= n_per) fcol -= n_per;
                    if (flushed + LK < total) {
                        __syncwarp();
                        int nc = fcol + LK;
                        if (nc >= n_per) nc -= n_per;
                        if (p.vec_ok) {
                            lane_fetch_land(ring, pf, row0, n_streams, flushed + LK, lane);
                            if (flushed + 2 * LK < total) {
                                int pc = nc + LK;
                                if (pc >= n_per) pc -= n_per;
                                lane_fetch_issue(pf, p.out, p.ld, row0, n_streams, pc, lane);
                            }
                        } else {
                            lane_fetch(ring, p.out, p.ld, row0, n_streams, flushed + LK, nc, false, lane);
                        }
                    }
                } else {
                    fcol += cnt;
                }
                __syncwarp();
            }
            if (done && flushed >= total) break;
        }
        if (valid) {
            if (failed) {
                gz_raise(GZ_ERR_GUARD, sid);
            } else {
                lane_store_state<SRC>(p, sid, S, gam);
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
        __syncwarp();
    }
}

/*
 * Polar, one lane per stream.  Every iteration each lane makes one attempt
 * (two draws).  Accepted pairs whose s takes glibc log's main branch are
 * transformed at once; the ~6% whose s lies in [1 - 2^-4, 1) (log's
 * near-1 polynomial) reserve their two ring slots and wait in a per-warp
 * shared-memory queue that is transformed 32 at a time, so neither log branch
 * diverges inside a warp.
 */
constexpr int PQ = 64;           /* near-1 queue capacity (entries) */

struct PolarQueue {
    double v1[PQ], v2[PQ], s[PQ];
    int meta[PQ];                /* owner lane | ring slot << 5 | spare << 10 */
};

__device__ __forceinline__ void polar_finish(double v1, double v2, double s, double L, double& o1, double& o2)
{
    const double mul = sqrt_rn_nb(div_rn_nb(__dmul_rn(-2.0, L), s));
    o1 = __dmul_rn(v1, mul);
    o2 = __dmul_rn(v2, mul);
}

/* transform queue entries [0, n) and move [n, cnt) to the front; returns cnt - n */
__device__ __forceinline__ int polar_drain(PolarQueue& q, int cnt, int n, double* ring, const uint64_t* s_log,
                                           double* spare_out, int64_t row0, int lane)
{
    if (lane < n) {
        const double s = q.s[lane];
        const int meta = q.meta[lane];
        double o1, o2;
        polar_finish(q.v1[lane], q.v2[lane], s, gz_log_t(s, s_log), o1, o2);
        const int owner = meta & 31;
        const int slot = (meta >> 5) & 31;
        double* orow = ring + owner * LSTRIDE;
        orow[slot] = o1;
        if (meta >> 10) {
            if (spare_out) spare_out[row0 + owner] = o2;
        } else {
            orow[(slot + 1) & (LRING - 1)] = o2;
        }
    }
    const int rest = cnt - n;
    double a = 0.0, b = 0.0, c = 0.0;
    int m = 0;
    if (lane < rest) {
        a = q.v1[n + lane]; b = q.v2[n + lane]; c = q.s[n + lane]; m = q.meta[n + lane];
    }
    __syncwarp();
    if (lane < rest) {
        q.v1[lane] = a; q.v2[lane] = b; q.s[lane] = c; q.meta[lane] = m;
    }
    __syncwarp();
    return rest;
}

template <int SRC, bool STATS>
__global__ void __launch_bounds__(LANE_THREADS, 2) k_polar_lane(const LaneParams p)
{
    extern __shared__ __align__(16) unsigned char smem[];
    uint64_t* s_log = reinterpret_cast<uint64_t*>(smem);
    double* s_ring = reinterpret_cast<double*>(smem + 256 * 8);
    PolarQueue* s_q = reinterpret_cast<PolarQueue*>(smem + 256 * 8 + LANE_WARPS * 32 * LSTRIDE * 8);
    for (int i = threadIdx.x; i < 256; i += blockDim.x) s_log[i] = g_log_tab[i];
    __syncthreads();
    const int lane = threadIdx.x & 31;
    const uint32_t lt = (1u << lane) - 1u;
    const int wib = threadIdx.x >> 5;
    double* ring = s_ring + wib * 32 * LSTRIDE;
    double* myring = ring + lane * LSTRIDE;
    PolarQueue& qb = s_q[wib];
    const int n_per = p.n_per;
    const int64_t guard = p.guard;
    const int64_t n_streams = p.n_streams;
    const int64_t n_groups = (n_streams + 31) >> 5;
    const int64_t gstride = (int64_t)gridDim.x * LANE_WARPS;

    for (int64_t grp = (int64_t)blockIdx.x * LANE_WARPS + wib; grp < n_groups; grp += gstride) {
        const int64_t row0 = grp * 32;
        const int64_t sid = row0 + lane;
        const bool valid = sid < n_streams;
        uint64_t S, gam;
        lane_load_state<SRC>(p, sid, valid, S, gam);
        int has = 0, spare_here = 0;   /* spare_here: the spare's value is in `spare` */
        double spare = 0.0;
        if (valid && p.has_in && p.has_in[sid]) {
            has = 1;
            spare_here = 1;
            spare = p.spare_in[sid];
        }
        int w = valid ? 0 : n_per;
        int flushed = 0, nb = 0;
        bool failed = false;
        int64_t rej = 0;
        uint64_t ck = 0;
        double a1 = 0.0, a2 = 0.0, a3 = 0.0, a4 = 0.0;
        if (has && w < n_per) {   /* the cached deviate comes first (samplers.py:182-184) */
            myring[0] = spare;
            w = 1;
            has = 0;
        }

        while (true) {
            const int lim = min(n_per, flushed + LRING);
#pragma unroll 1
            for (int it = 0; it < LK / 2; ++it) {
                bool near1 = false;
                double v1 = 0.0, v2 = 0.0, s = 2.0;
                const int need = (w + 1 < n_per) ? 2 : 1;
                if (w + need <= lim) {
                    v1 = gz_unit53_pm1(lane_next<SRC>(S, gam));
                    v2 = gz_unit53_pm1(lane_next<SRC>(S, gam));
                    s = __dadd_rn(__dmul_rn(v1, v1), __dmul_rn(v2, v2));
                    if (s > 0.0 && s < 1.0) {
                        rej = 0;
                        near1 = (uint64_t)__double_as_longlong(s) >= 0x3fee000000000000ULL;
                        if (!near1) {
                            /* main branch of glibc log: transform now */
                            double o1, o2;
                            polar_finish(v1, v2, s, gz_log_t(s, s_log), o1, o2);
                            myring[w & (LRING - 1)] = o1;
                            if (need == 2) myring[(w + 1) & (LRING - 1)] = o2;
                            else { spare = o2; has = 1; spare_here = 1; }
                            w += need;
                        }
                    } else if (++rej >= guard) {
                        failed = true;
                        w = n_per;
                    }
                }
                const uint32_t mb = __ballot_sync(GZ_FULL, near1);
                if (mb) {
                    if (near1) {
                        const int pos = nb + __popc(mb & lt);
                        qb.v1[pos] = v1;
                        qb.v2[pos] = v2;
                        qb.s[pos] = s;
                        qb.meta[pos] = lane | ((w & (LRING - 1)) << 5) | ((need == 2 ? 0 : 1) << 10);
                        if (need == 1) { has = 1; spare_here = 0; }
                        w += need;
                    }
                    nb += __popc(mb);
                    __syncwarp();
                    if (nb >= 32) nb = polar_drain(qb, nb, 32, ring, s_log, p.spare_out, row0, lane);
                }
            }
            const int lag = (int)__reduce_min_sync(GZ_FULL, (unsigned)(w - flushed));
            const bool done = __all_sync(GZ_FULL, w >= n_per);
            const int cnt = lag >= LK ? LK : (done ? n_per - flushed : 0);
            if (cnt > 0) {
                /* every reserved slot must hold its deviate before the flush */
                if (nb) nb = polar_drain(qb, nb, nb, ring, s_log, p.spare_out, row0, lane);
                __syncwarp();
                if constexpr (STATS) lane_stats(myring, flushed, cnt, ck, a1, a2, a3, a4);
                lane_flush(ring, p.out, p.ld, row0, n_streams, flushed, flushed, cnt, p.vec_ok, lane);
                __syncwarp();
                flushed += cnt;
            }
            if (done && flushed >= n_per) break;
        }
        if (nb) nb = polar_drain(qb, nb, nb, ring, s_log, p.spare_out, row0, lane);
        __syncwarp();
        if (valid) {
            if (failed) {
                gz_raise(GZ_ERR_GUARD, sid);
            } else {
                lane_store_state<SRC>(p, sid, S, gam);
                /* a queued final pair wrote its spare in polar_drain */
                if (p.spare_out && (!has || spare_here)) p.spare_out[sid] = has ? spare : 0.0;
                if (p.has_out) p.has_out[sid] = (uint8_t)has;
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
        __syncwarp();
    }
}

/*
 * Polar, one lane per stream, queued transforms (the polar lane kernel without
 * fused witnesses).  Every lane makes one attempt per iteration; an accepted
 * pair reserves its two row slots and joins one of two per-warp shared-memory
 * queues by glibc log branch.  The main-branch queue is transformed 64 entries
 * at a time (two independent log/divide/sqrt chains per lane), the near-1 queue
 * 32 at a time, so the transform always runs on full warps.  The drains store
 * each pair straight to its row (16 bytes per lane; the halves of a 32-byte
 * sector written a few iterations apart merge in L2), so there is no ring, no
 * flush bookkeeping and no lane waits for the slowest lane until the rows end.
 */
template <int CAP>
struct LaneQueue {
    double v1[CAP], v2[CAP], s[CAP];
    int meta[CAP];            /* owner lane | spare << 5 | row slot << 6 */
};

__device__ __forceinline__ double lq_mul(double s, const uint64_t* s_log, bool near)
{
    const double L = near ? gz_log_t(s, s_log) : gz_log_core((uint64_t)__double_as_longlong(s), s_log);
    return sqrt_rn_nb(div_rn_nb(__dmul_rn(-2.0, L), s));
}

/* move entries [n, cnt) (fewer than 32) to the front */
template <int CAP>
__device__ __forceinline__ int lq_shift(LaneQueue<CAP>& q, int cnt, int n, int lane)
{
    const int rest = cnt - n;
    double a = 0.0, b = 0.0, c = 0.0;
    int m = 0;
    if (lane < rest) {
        a = q.v1[n + lane]; b = q.v2[n + lane]; c = q.s[n + lane]; m = q.meta[n + lane];
    }
    __syncwarp();
    if (lane < rest) {
        q.v1[lane] = a; q.v2[lane] = b; q.s[lane] = c; q.meta[lane] = m;
    }
    __syncwarp();
    return rest;
}

struct LqDirect {
    double* out;
    int64_t ld, row0;
    double* spare_out;
};

__device__ __forceinline__ void lqd_put(const LqDirect& o, int meta, double v1, double v2, double mul)
{
    const double o1 = __dmul_rn(v1, mul), o2 = __dmul_rn(v2, mul);
    const int owner = meta & 31;
    const int w = meta >> 6;
    double* d = o.out + (o.row0 + owner) * o.ld + w;
    if (meta & 32) {
        d[0] = o1;
        if (o.spare_out) o.spare_out[o.row0 + owner] = o2;
    } else {
        pair_store(d, o1, o2);
    }
}

template <int CAP>
__device__ __forceinline__ int lqd_drain64(LaneQueue<CAP>& q, int cnt, const LqDirect& o, const uint64_t* s_log, int lane)
{
    const double sA = q.s[lane], sB = q.s[lane + 32];
    const double mA = lq_mul(sA, s_log, false);
    const double mB = lq_mul(sB, s_log, false);
    lqd_put(o, q.meta[lane], q.v1[lane], q.v2[lane], mA);
    lqd_put(o, q.meta[lane + 32], q.v1[lane + 32], q.v2[lane + 32], mB);
    return lq_shift(q, cnt, 64, lane);
}

template <int CAP>
__device__ __forceinline__ int lqd_drain32(LaneQueue<CAP>& q, int cnt, int n, const LqDirect& o, const uint64_t* s_log,
                                           bool near, int lane)
{
    if (lane < n) lqd_put(o, q.meta[lane], q.v1[lane], q.v2[lane], lq_mul(q.s[lane], s_log, near));
    return lq_shift(q, cnt, n, lane);
}

template <int CAP>
__device__ __forceinline__ void lqd_drain_all(LaneQueue<CAP>& q, int cnt, const LqDirect& o, const uint64_t* s_log,
                                              bool near, int lane)
{
    for (int b = 0; b < cnt; b += 32) {
        const int i = b + lane;
        if (i < cnt) lqd_put(o, q.meta[i], q.v1[i], q.v2[i], lq_mul(q.s[i], s_log, near));
    }
    __syncwarp();
}

constexpr int LQD_MAIN = 96;    /* < 64 left after a drain + 32 pushed */
constexpr int LQD_NEAR = 64;    /* < 32 left + 32 pushed */
constexpr size_t LQD_WARP_BYTES = sizeof(LaneQueue<LQD_MAIN>) + sizeof(LaneQueue<LQD_NEAR>);

template <int SRC>
__global__ void __launch_bounds__(LANE_THREADS, 3) k_polar_lqd(const LaneParams p)
{
    extern __shared__ __align__(16) unsigned char smem[];
    uint64_t* s_log = reinterpret_cast<uint64_t*>(smem);
    for (int i = threadIdx.x; i < 256; i += blockDim.x) s_log[i] = g_log_tab[i];
    __syncthreads();
    const int lane = threadIdx.x & 31;
    const uint32_t lt = (1u << lane) - 1u;
    const int wib = threadIdx.x >> 5;
    unsigned char* wbase = smem + 256 * 8 + (size_t)wib * LQD_WARP_BYTES;
    LaneQueue<LQD_MAIN>& qm = *reinterpret_cast<LaneQueue<LQD_MAIN>*>(wbase);
    LaneQueue<LQD_NEAR>& qn = *reinterpret_cast<LaneQueue<LQD_NEAR>*>(wbase + sizeof(LaneQueue<LQD_MAIN>));
    const int n_per = p.n_per;
    const uint32_t guard32 = p.guard > 0xffffffffll ? 0xffffffffu : (uint32_t)p.guard;
    const int64_t n_streams = p.n_streams;
    const int64_t n_groups = (n_streams + 31) >> 5;
    const int64_t gstride = (int64_t)gridDim.x * LANE_WARPS;

    for (int64_t grp = (int64_t)blockIdx.x * LANE_WARPS + wib; grp < n_groups; grp += gstride) {
        const int64_t row0 = grp * 32;
        const int64_t sid = row0 + lane;
        const bool valid = sid < n_streams;
        const LqDirect o{p.out, p.ld, row0, p.spare_out};
        uint64_t S, gam;
        lane_load_state<SRC>(p, sid, valid, S, gam);
        int has = 0, spare_here = 0;   /* spare_here: the spare's value is in `spare` */
        double spare = 0.0;
        if (valid && p.has_in && p.has_in[sid]) {
            has = 1;
            spare_here = 1;
            spare = p.spare_in[sid];
        }
        int w = valid ? 0 : n_per;
        int nm = 0, nn = 0;
        bool failed = false;
        uint32_t rej = 0;
        if (has && w < n_per) {   /* the cached deviate comes first (samplers.py:182-184) */
            p.out[sid * p.ld] = spare;
            w = 1;
            has = 0;
            spare_here = 0;
        }

        do {
#pragma unroll 1
            for (int it = 0; it < 8; ++it) {
                bool acc = false, near1 = false;
                double v1 = 0.0, v2 = 0.0, s = 2.0;
                if (w < n_per) {
                    /* one attempt of PolarSampler (samplers.py:185-192) */
                    v1 = gz_unit53_pm1(lane_next<SRC>(S, gam));
                    v2 = gz_unit53_pm1(lane_next<SRC>(S, gam));
                    s = __dadd_rn(__dmul_rn(v1, v1), __dmul_rn(v2, v2));
                    if (s > 0.0 && s < 1.0) {
                        rej = 0;
                        acc = true;
                        near1 = (uint64_t)__double_as_longlong(s) >= 0x3fee000000000000ULL;
                    } else if (++rej >= guard32) {
                        failed = true;
                        w = n_per;
                    }
                }
                const uint32_t mm = __ballot_sync(GZ_FULL, acc && !near1);
                const uint32_t mn = __ballot_sync(GZ_FULL, near1);
                if (acc) {
                    const int last = w + 1 >= n_per;   /* one slot left: o2 becomes the spare */
                    const int meta = lane | (last ? 32 : 0) | (w << 6);
                    if (near1) {
                        const int pos = nn + __popc(mn & lt);
                        qn.v1[pos] = v1; qn.v2[pos] = v2; qn.s[pos] = s; qn.meta[pos] = meta;
                    } else {
                        const int pos = nm + __popc(mm & lt);
                        qm.v1[pos] = v1; qm.v2[pos] = v2; qm.s[pos] = s; qm.meta[pos] = meta;
                    }
                    has = last;
                    w += 2;
                }
                nm += __popc(mm);
                nn += __popc(mn);
                if (nm >= 64) {
                    __syncwarp();
                    nm = lqd_drain64(qm, nm, o, s_log, lane);
                }
                if (nn >= 32) {
                    __syncwarp();
                    nn = lqd_drain32(qn, nn, 32, o, s_log, true, lane);
                }
            }
        } while (!__all_sync(GZ_FULL, w >= n_per));
        __syncwarp();
        if (nm) lqd_drain_all(qm, nm, o, s_log, false, lane);
        if (nn) lqd_drain_all(qn, nn, o, s_log, true, lane);
        if (valid) {
            if (failed) {
                gz_raise(GZ_ERR_GUARD, sid);
            } else {
                lane_store_state<SRC>(p, sid, S, gam);
                if (p.spare_out && (!has || spare_here)) p.spare_out[sid] = has ? spare : 0.0;
                if (p.has_out) p.has_out[sid] = (uint8_t)has;
            }
        }
        __syncwarp();
    }
}
