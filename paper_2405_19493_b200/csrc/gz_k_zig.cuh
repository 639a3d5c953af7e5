/*
 * gz_k_zig.cuh -- the wedge test, the sequential tail and the warp-per-stream ziggurat kernel k_zig.
 *
 * Not a standalone header: included by gz_engine.cu inside its anonymous
 * namespace, after the shared device globals and helpers it uses.
 */
#pragma once

/* ------------------------------------------------------------ wedge test */

/* Exact glibc exp, out of line: reached only when the cheap filters below are
 * ambiguous (|y/exp(t) - 1| < 2^-15, about one wedge test in ten thousand). */
__device__ __noinline__ bool wedge_exact(double y, double t)
{
    return y < gz_exp_t(t, g_exp_tab);
}

/*
 * Decide `y < exp(t)` exactly as the reference does with glibc exp
 * (samplers.py:113, engine.py:106).  t = -0.5*x*x lies in (-7, 0].  A single
 * precision exp (__expf of float(t): relative error < 2^-19.6 for |t| < 8.2,
 * CUDA's 2 + 1.16|t| ulp bound plus the conversion of t) settles every case
 * farther than 2^-15 from the boundary; the rest use the bit-exact
 * restatement of glibc's exp.  The decision is therefore identical to the
 * reference's in every case.
 */
__device__ __forceinline__ bool wedge_accept(double y, double t)
{
    const double e = (double)__expf((float)t);
    if (y < __dmul_rn(e, 1.0 - 0x1p-15)) return true;
    if (y > __dmul_rn(e, 1.0 + 0x1p-15)) return false;
    return wedge_exact(y, t);
}

/*
 * The same decision with a single-precision pre-filter: y and exp(t) are
 * approximated in float and the exact double path runs only within 2^-15 of the
 * boundary.  Error budget (every table n = 8..1024): y from float copies of
 * ytab[i] and dy = ytab[i+1]-ytab[i] and the top 24 bits of the uniform draw,
 * |y_f/y - 1| <= 2^-24 (2 + 2 max dy/ytab) < 2^-21.8 (max dy/ytab[i] = 1.16 at
 * n = 8); ex2.approx of t = -x^2/(2 ln 2) >= -11.8 computed in float, argument
 * error <= 6 * 2^-24 * 11.8 -> |e_f/e - 1| < 2^-18.2 plus ex2's 2 ulp.  The band
 * 2^-15 leaves a factor 8 of margin.  u2 is the wedge's uniform draw, ydp/yf
 * the layer's table rows.
 */
__device__ __forceinline__ bool wedge_accept_f(uint64_t u2, double x, const double2* ydp, float2 yf)
{
    const float y = __fmaf_rn(__uint2float_rn((uint32_t)(u2 >> 40)), yf.y, yf.x);
    const float xf = __double2float_rn(x);
    float e;   /* 2^t, t = -x^2 / (2 ln 2) >= -12: no range reduction needed */
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(e) : "f"(-0.72134752044448170f * xf * xf));
    if (y < e * (1.0f - 0x1p-15f)) return true;
    if (y > e * (1.0f + 0x1p-15f)) return false;
    const double2 yd = *ydp;   /* only near the boundary: the double rows stay in global memory */
    const double yy = __dadd_rn(yd.x, __dmul_rn(gz_unit53(u2), yd.y));
    return wedge_exact(yy, __dmul_rn(__dmul_rn(-0.5, x), x));
}

/*
 * tail_sample (samplers.py:40-57; engine.py:89-103) run sequentially by one
 * lane from the stream state `st` (the state after the attempt's draw).
 * Returns the number of (u1, u2) pairs consumed, or -1 when the guard trips;
 * *val = r + x; st is advanced past the consumed draws.
 */
struct TailOut {
    uint64_t st;   /* state after the consumed draws */
    double v;      /* r + x */
    int k;         /* (u1, u2) pairs consumed, -1 when the guard tripped */
};

template <int SRC>
__device__ __noinline__ TailOut tail_seq(uint64_t st, uint64_t gamma, double r, int64_t guard)
{
    TailOut o;
    o.v = 0.0;
    o.k = -1;
    for (int64_t k = 0; k < guard; ++k) {
        const double u1 = gz_unit53(gz_next_seq<SRC>(st, gamma));
        const double u2 = gz_unit53(gz_next_seq<SRC>(st, gamma));
        if (u1 <= 0.0 || u2 <= 0.0) continue;
        const double x = __ddiv_rn(-gz_log_t(u1, g_log_tab), r);
        const double y = -gz_log_t(u2, g_log_tab);
        if (__dmul_rn(2.0, y) > __dmul_rn(x, x)) {
            o.v = __dadd_rn(r, x);
            o.k = (int)(k + 1);
            break;
        }
    }
    o.st = st;
    return o;
}

/* ------------------------------------------------------------ ziggurat */

struct ZigParams {
    int64_t n_streams, n_per, ld;
    const uint64_t* state_in;
    uint64_t* state_out;
    double* out;            /* EPI_STORE: deviates; EPI_MUTATE: x (in/out) */
    const double* sigma;    /* EPI_MUTATE */
    uint64_t* checksum;     /* optional */
    double* psum;           /* optional [n_streams][4] */
    const ulonglong2* kw;   /* {ktab[i], bits(wtab[i])} */
    const double2* yd;      /* {ytab[i], ytab[i+1] - ytab[i]} */
    int n_layers, index_bits;
    double r;
    int64_t guard;
    int generations;
};

/* per-lane LCG jump constants of the warp-per-stream windows: draw 32d + j of a
   window is lane j's steps 2j+1, 2j+2 from the sub-round base; AW/CW jump 64 steps */
struct ZigLaneConsts {
    uint64_t A1, C1, A2, C2, AW, CW;
};

template <int SRC>
__device__ __forceinline__ ZigLaneConsts zig_lane_consts(int lane)
{
    ZigLaneConsts k{0, 0, 0, 0, 0, 0};
    if constexpr (SRC == 0) {
        k.A1 = ld_keep(&c_lcgA[2 * lane + 1]); k.C1 = ld_keep(&c_lcgC[2 * lane + 1]);
        k.A2 = ld_keep(&c_lcgA[2 * lane + 2]); k.C2 = ld_keep(&c_lcgC[2 * lane + 2]);
        k.AW = ld_keep(&c_lcgA[64]); k.CW = ld_keep(&c_lcgC[64]);
    }
    return k;
}

/* one window of W = 32*D draws from state S (the state before the window's first
   draw): lane j of sub-round d holds draw 32d + j -- its value as a fast-path
   deviate, the masks of non-fast (nf) and tail (tl) draws, the wedge decisions of
   every wedge candidate (am), the lane's state after its draw (st) and, for a wedge
   candidate in the window's last draw, the state after its uniform (extw) */
template <int D>
struct ZigWindow {
    uint64_t st[D];
    double val[D];
    uint32_t nf[D], tl[D], am[D];
    uint64_t extw;
};

template <int SRC, bool MOD, int D>
__device__ __forceinline__ void zig_window(ZigWindow<D>& w, uint64_t S, uint64_t gam, uint64_t gl, uint64_t g32,
                                           const ZigLaneConsts& kc, const ulonglong2* s_kw, const double2* s_yd,
                                           int ib, uint32_t imask, int mbits, uint64_t mmask, int lane)
{
    /* ---- draws: lane j of sub-round d holds draw 32d + j ---- */
    uint64_t u[D];
    if constexpr (SRC == 0) {
        uint64_t Sb = S;
#pragma unroll
        for (int d = 0; d < D; ++d) {
            if (d) Sb = gz_lcg_mad(kc.AW, Sb, kc.CW);
            const uint64_t t1 = gz_lcg_mad(kc.A1, Sb, kc.C1);
            w.st[d] = gz_lcg_mad(kc.A2, Sb, kc.C2);
            u[d] = gz_lcg_u64(t1, w.st[d]);
        }
    } else {
#pragma unroll
        for (int d = 0; d < D; ++d) {
            w.st[d] = S + gl + (uint64_t)d * g32;
            u[d] = gz_mix64(w.st[d]);
        }
    }
    /* ---- fast-path classification ---- */
    uint32_t li[D];
#pragma unroll
    for (int d = 0; d < D; ++d) {
        const uint64_t uu = u[d];
        uint32_t i, neg;
        uint64_t m;
        if constexpr (MOD) {
            i = (uint32_t)uu & imask;
            m = uu >> (ib + 1);
            neg = (uint32_t)(uu >> ib) & 1u;
        } else {
            i = (uint32_t)(uu >> mbits) & imask;
            m = uu & mmask;
            neg = (uint32_t)(uu >> 63);
        }
        const ulonglong2 kw = s_kw[i];
        const bool fast = m < kw.x;
        const double x = __dmul_rn(__ull2double_rn(m), __longlong_as_double((long long)kw.y));
        w.val[d] = neg ? -x : x;
        li[d] = i;
        w.nf[d] = __ballot_sync(GZ_FULL, !fast);
        w.tl[d] = __ballot_sync(GZ_FULL, !fast && i == 0);
    }
    /* ---- wedge decisions for every candidate lane, once per window ---- */
    w.extw = 0;
    uint32_t anyw = 0;
#pragma unroll
    for (int d = 0; d < D; ++d) {
        w.am[d] = 0;
        anyw |= w.nf[d] & ~w.tl[d];
    }
    if (anyw) {
#pragma unroll
        for (int d = 0; d < D; ++d) {
            const uint32_t wm = w.nf[d] & ~w.tl[d];
            if (wm) {
                double un = __shfl_down_sync(GZ_FULL, gz_unit53(u[d]), 1);
                if (d + 1 < D) {
                    const double n0 = __shfl_sync(GZ_FULL, gz_unit53(u[(d + 1) % D]), 0);
                    if (lane == 31) un = n0;
                }
                const bool cand = (wm >> lane) & 1u;
                if (d == D - 1 && lane == 31 && cand) {
                    /* the wedge's uniform is the first draw after the window */
                    uint64_t e = w.st[d];
                    un = gz_unit53(gz_next_seq<SRC>(e, gam));
                    w.extw = e;
                }
                bool acc = false;
                if (cand) {
                    const double2 yy = s_yd[li[d]];
                    const double y = __dadd_rn(yy.x, __dmul_rn(un, yy.y));
                    const double x = fabs(w.val[d]);
                    const double t = __dmul_rn(__dmul_rn(-0.5, x), x);
                    acc = wedge_accept(y, t);
                }
                w.am[d] = __ballot_sync(GZ_FULL, acc);
            }
        }
    }
}

/*
 * One stream by one warp: windows of W = 32*D draws (zig_window), a warp-uniform
 * parse that restores the sequential attempt order, and the emit.  SRC: 0 LCG48,
 * 1 SplitMix64.  MOD: modified ziggurat bit layout (samplers.py:128-133 vs 79-84).
 * EPI: store deviates, or fuse x += sigma*z (config 5).  STATS: fuse the per-row
 * xor checksum and power sums (config 4).
 */
template <int SRC, bool MOD, int D, int EPI, bool STATS>
__device__ __forceinline__ void zig_warp_stream(const ZigParams& p, int64_t sid, const ulonglong2* s_kw,
                                                const double2* s_yd, const ZigLaneConsts& kc, int lane)
{
    constexpr int W = 32 * D;
    const uint32_t lt = (1u << lane) - 1u;
    const int ib = p.index_bits;
    const uint32_t imask = (uint32_t)p.n_layers - 1u;
    const int mbits = 63 - ib;
    const uint64_t mmask = (1ULL << mbits) - 1ULL;
    const double r = p.r;
    const int64_t total = p.n_per * (int64_t)(EPI == EPI_MUTATE ? p.generations : 1);

    uint64_t S, gam = 0, gl = 0, g32 = 0;
    if constexpr (SRC == 0) {
        S = p.state_in[sid];
    } else {
        S = p.state_in[2 * sid];
        gam = p.state_in[2 * sid + 1];
        gl = (uint64_t)(lane + 1) * gam;
        g32 = gam << 5;
    }
    double* row = p.out + sid * p.ld;
    const double sig = (EPI == EPI_MUTATE) ? p.sigma[sid] : 0.0;
    int64_t produced = 0, rej_run = 0, jrow = 0;
    uint64_t ck = 0;
    double a1 = 0.0, a2 = 0.0, a3 = 0.0, a4 = 0.0;
    bool failed = false;

    while (produced < total) {
        ZigWindow<D> w;
        zig_window<SRC, MOD, D>(w, S, gam, gl, g32, kc, s_kw, s_yd, ib, imask, mbits, mmask, lane);
        /* ---- warp-uniform parse: which draws start attempts, which emit ---- */
        const int64_t remL = total - produced;
        const int rem = remL > W ? W + 1 : (int)remL;
        int q = 0, cnt = 0, ext_lane = 0, ext_kind = 0;
        bool stop = false;
        uint64_t ext_t = 0;
        uint32_t em[D];
        int eb[D];
#pragma unroll
        for (int d = 0; d < D; ++d) {
            em[d] = 0;
            eb[d] = cnt;
            if (stop || q >= 32 * (d + 1)) continue;
            int b = q - 32 * d;
            const uint32_t nfd = w.nf[d];
            while (true) {
                const uint32_t pend = nfd & (GZ_FULL << b);
                const int f = pend ? (__ffs(pend) - 1) : 32;
                const int nF = f - b;
                if (cnt + nF >= rem) {
                    const int take = rem - cnt;
                    em[d] |= gz_bitrange(b, take);
                    cnt = rem;
                    q = 32 * d + b + take;
                    stop = true;
                    break;
                }
                em[d] |= gz_bitrange(b, nF);
                cnt += nF;
                /* the guard counts the rejections of one call: a fast-path deviate ends it */
                if (nF > 0) rej_run = 0;
                if (f == 32) {
                    q = 32 * (d + 1);
                    break;
                }
                const int pos = 32 * d + f;
                if ((w.tl[d] >> f) & 1u) {
                    int tt = 0;
                    if (lane == f) {
                        const TailOut to = tail_seq<SRC>(w.st[d], gam, r, p.guard);
                        tt = to.k;
                        ext_t = to.st;
                        w.val[d] = signbit(w.val[d]) ? -to.v : to.v;
                    }
                    tt = __shfl_sync(GZ_FULL, tt, f);
                    if (tt < 0) {
                        failed = true;
                        stop = true;
                        break;
                    }
                    em[d] |= 1u << f;
                    ++cnt;
                    rej_run = 0;
                    q = pos + 1 + 2 * tt;
                    ext_kind = 1;
                    ext_lane = f;
                } else {
                    if ((w.am[d] >> f) & 1u) {
                        em[d] |= 1u << f;
                        ++cnt;
                        rej_run = 0;
                    } else if (++rej_run >= p.guard) {
                        failed = true;
                        stop = true;
                        break;
                    }
                    q = pos + 2;
                    ext_kind = 2;
                }
                if (cnt >= rem) {
                    stop = true;
                    break;
                }
                if (q >= 32 * (d + 1)) break;
                b = q - 32 * d;
            }
        }
        if (failed) break;
        /* ---- emit: the window's deviates go to consecutive slots ---- */
#pragma unroll
        for (int d = 0; d < D; ++d) {
            if ((em[d] >> lane) & 1u) {
                const int rel = eb[d] + __popc(em[d] & lt);
                const double v = w.val[d];
                if constexpr (EPI == EPI_STORE) {
                    row[produced + rel] = v;
                } else {
                    int64_t j = jrow + rel;
                    if (j >= p.n_per) j -= p.n_per;
                    row[j] = __dadd_rn(row[j], __dmul_rn(sig, v));
                }
                if constexpr (STATS) {
                    ck ^= (uint64_t)__double_as_longlong(v);
                    const double v2 = __dmul_rn(v, v);
                    a1 = __dadd_rn(a1, v);
                    a2 = __dadd_rn(a2, v2);
                    a3 = __fma_rn(v2, v, a3);
                    a4 = __fma_rn(v2, v2, a4);
                }
            }
        }
        if constexpr (EPI == EPI_MUTATE) {
            jrow += cnt;
            if (jrow >= p.n_per) jrow -= p.n_per;
            __syncwarp();
        }
        produced += cnt;
        /* ---- advance the stream state past the consumed draws ---- */
        if constexpr (SRC == 1) {
            S += (uint64_t)q * gam;
        } else {
            if (q <= W) {
                const int pq = q - 1;
                uint64_t sel = w.st[0];
#pragma unroll
                for (int d = 1; d < D; ++d)
                    if ((pq >> 5) == d) sel = w.st[d];
                S = __shfl_sync(GZ_FULL, sel, pq & 31);
            } else if (ext_kind == 1) {
                S = __shfl_sync(GZ_FULL, ext_t, ext_lane);
            } else {
                S = __shfl_sync(GZ_FULL, w.extw, 31);
            }
        }
    }
    if (failed) {
        if (lane == 0) gz_raise(GZ_ERR_GUARD, sid);
        return;
    }
    if (lane == 0) {
        if constexpr (SRC == 0) {
            p.state_out[sid] = S;
        } else {
            p.state_out[2 * sid] = S;
            p.state_out[2 * sid + 1] = gam;
        }
    }
    if constexpr (STATS) {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            ck ^= __shfl_xor_sync(GZ_FULL, ck, o);
            a1 = __dadd_rn(a1, __shfl_xor_sync(GZ_FULL, a1, o));
            a2 = __dadd_rn(a2, __shfl_xor_sync(GZ_FULL, a2, o));
            a3 = __dadd_rn(a3, __shfl_xor_sync(GZ_FULL, a3, o));
            a4 = __dadd_rn(a4, __shfl_xor_sync(GZ_FULL, a4, o));
        }
        if (lane == 0) {
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

/* one warp per stream (persistent grid-stride over streams) */
template <int SRC, bool MOD, int D, int EPI, bool STATS>
__global__ void __launch_bounds__(256) k_zig(const ZigParams p)
{
    extern __shared__ __align__(16) unsigned char smem[];
    const int nl = p.n_layers;
    ulonglong2* s_kw = reinterpret_cast<ulonglong2*>(smem);
    double2* s_yd = reinterpret_cast<double2*>(smem + 16 * nl);
    for (int i = threadIdx.x; i < nl; i += blockDim.x) {
        s_kw[i] = p.kw[i];
        s_yd[i] = p.yd[i];
    }
    __syncthreads();
    const int lane = threadIdx.x & 31;
    const ZigLaneConsts kc = zig_lane_consts<SRC>(lane);
    const int64_t w0 = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t sid = w0; sid < p.n_streams; sid += nw)
        zig_warp_stream<SRC, MOD, D, EPI, STATS>(p, sid, s_kw, s_yd, kc, lane);
}
