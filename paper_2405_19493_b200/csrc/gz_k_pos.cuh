/*
 * gz_k_pos.cuh -- the ziggurats over FEW long streams, decoded by draw POSITION
 * (included by gz_engine.cu after gz_k_seg.cuh).
 *
 * A stream's draws are position-addressable (SplitMix64: state s0 + n*gamma; LCG48:
 * (A_2n, C_2n) jump-ahead), and an attempt of the original or modified ziggurat
 * (samplers.py:95-115 / 144-165, engine.py:75-151) consumes one draw unless its first
 * draw is not a fast accept: a wedge candidate consumes exactly one more draw (its
 * uniform, samplers.py:111-114) and a tail entry 2t more (samplers.py:40-57).  So the
 * sequential loop over one stream is recovered from three data-parallel steps:
 *
 *   1. classify: every draw position p of the pass is evaluated AS IF an attempt
 *      started there (fast accept and its signed deviate; 97-98 % of positions).  A
 *      position that is not a fast accept ("non-fast", 2-3 %) is resolved on the spot
 *      by its lane -- wedge test with the next position's draw (the right neighbour
 *      lane's, by shuffle), or the tail loop -- and queued in per-warp entry lists in
 *      position order: {p, draws consumed, accepted, value}.
 *   2. parse (one warp): only the non-fast positions can consume more than their own
 *      draw, so the attempt starts are fixed by a scan over the SPARSE entry list
 *      (about 60 per pass of 2176 positions): an entry is a start unless an earlier
 *      start's draws cover it (pos_parse: alternating runs by bit operations, a
 *      sequential walk for chunks with tails reaching further or possible rejection
 *      runs).  The parse rewrites the position array -- an accepted non-fast start
 *      gets its deviate, the further draws of a start are marked -- counts the
 *      positions per warp region that are not accepted starts, carries the guard's
 *      consecutive-rejection run (engine.py:37, samplers.py:27,32-33) and finds the
 *      position after the row's last deviate (the final state).
 *   3. emit: the positions still holding values are exactly the accepted starts, in
 *      order: a ballot compaction per 32-position window, coalesced stores.
 *
 * Same draws, same decisions, same order as the sequential loop.  Anything unusual
 * (an entry list overflow, a guard trip, a tail longer than 2^28 pairs) hands the
 * whole stream to the exact warp-per-stream loop (zig_warp_stream), which also raises
 * the guard status.  One block of POS_NW warps per stream, small enough (24-27 KiB of
 * shared memory) that 8 blocks share an SM: config 1's 1024 streams run in one wave.
 *
 * Opt-in (GZ_POS=1): bit-exact on every test, but on config 1 it runs 56.8 us against
 * 47.2 us for k_zig_lseg -- 22.2 M warp-instructions (classify 44 per 32-position
 * window plus 48 in the 60 % of windows with a non-fast position, emit 24) against
 * 24.7 M, and the two block barriers around the one-warp parse per pass are the top
 * stall.
 */
#pragma once

constexpr int POS_NW = 4;      /* warps per block; a block decodes one stream at a time */
constexpr int POS_J = 17;      /* 32-position windows per warp per pass */
constexpr int POS_PP = 32 * POS_NW * POS_J;   /* positions per full pass (2176) */
constexpr int POS_ECAP = 64;   /* non-fast entries per warp per pass (mean 15 at J = 17) */
constexpr uint64_t POS_MARK = 0xFFF8000000000001ULL;   /* NaN: "not a fast accept" */

struct PosShared {
    int cnt[POS_NW];    /* entries per warp this pass (-1: overflow / guard in the tail loop) */
    int nacc[POS_NW];   /* positions of each warp region that are not accepted starts */
    int carry;          /* positions of the next pass covered by this pass's last start */
    int run;            /* consecutive rejections carried into the next pass */
    int bad;            /* hand the stream to the exact loop */
};

/* the stream state after `draws` draws from s0 */
template <int SRC>
__device__ __forceinline__ uint64_t pos_state_at(uint64_t s0, uint64_t gam, uint64_t draws)
{
    if constexpr (SRC == 0) {
        uint64_t n = 2 * draws, S = s0;
        while (n) {
            const int b = __ffsll((long long)n) - 1;
            n &= n - 1;
            S = (c_lcgP2A[b] * S + c_lcgP2C[b]) & GZ_MASK48;
        }
        return S;
    } else {
        return s0 + draws * gam;
    }
}

__host__ __device__ constexpr size_t pos_smem_bytes(int nl)
{
    return 24 * (size_t)nl + ((sizeof(PosShared) + 15) & ~(size_t)15) + 8 * (size_t)POS_PP +
           (size_t)POS_NW * POS_ECAP * (8 + 4 + 4);
}

/* the whole stream through the exact warp-per-stream loop (out of line: it is rare) */
template <int SRC, bool MOD>
__device__ __noinline__ void pos_fallback(const LaneParams& p, int64_t sid, int nl, int ib, int lane)
{
    ZigParams zp;
    zp.n_streams = p.n_streams; zp.n_per = p.n_per; zp.ld = p.ld;
    zp.state_in = p.state_in; zp.state_out = p.state_out; zp.out = p.out;
    zp.sigma = nullptr; zp.checksum = nullptr; zp.psum = nullptr;
    zp.kw = p.kw; zp.yd = p.yd; zp.n_layers = nl; zp.index_bits = ib; zp.r = p.r; zp.guard = p.guard;
    zp.generations = 1;
    const ZigLaneConsts kc = zig_lane_consts<SRC>(lane);
    zig_warp_stream<SRC, MOD, 4, EPI_STORE, false>(zp, sid, p.kw, p.yd, kc, lane);
}

__device__ __forceinline__ int pos_region(int x, int RW)
{
    static_assert(POS_NW == 4, "pos_region assumes 4 warp regions");
    return (x >= RW) + (x >= 2 * RW) + (x >= 3 * RW);
}

/* the shared slot of entry g of the pass (entries of warp region v at v * POS_ECAP) */
__device__ __forceinline__ int pos_slot(int g, int c1, int c2, int c3)
{
    const int v = (g >= c1) + (g >= c2) + (g >= c3);
    const int base = v == 0 ? 0 : v == 1 ? c1 : v == 2 ? c2 : c3;
    return v * POS_ECAP + (g - base);
}

/* a start's effect on the position array: its deviate at q when accepted, its further
   draws marked (they are not attempt starts); every position of the pass that is not an
   accepted start is counted in its warp region's nacc */
__device__ __forceinline__ void pos_apply(PosShared& sh, uint32_t xb, int q, int len, int acc, double ev, int PP, int RW)
{
    if (acc) sts_u64(xb + 8 * q, (uint64_t)__double_as_longlong(ev));
    else atomicAdd(&sh.nacc[pos_region(q, RW)], 1);
    const int ce = min(q + len, PP);
    for (int x = q + 1; x < ce; ++x) {
        sts_u64(xb + 8 * x, POS_MARK);
        atomicAdd(&sh.nacc[pos_region(x, RW)], 1);
    }
}

/*
 * The parse of one pass, by one warp, 32 entries at a time.  Entry k (position q_k,
 * draws len_k, accepted acc_k) is an attempt start unless an earlier start covers it.
 * Fast path: when no entry can be reached by any start other than its predecessor
 * (q_k >= q_{k-2} + len_{k-2}, and the incoming coverage reaches at most the chunk's
 * first entry), c_k = "q_k < q_{k-1} + len_{k-1}" says k is covered iff k-1 is a start,
 * so inside a run of set c bits the starts alternate: start_k = !c_k || (k - a) odd, a
 * the run's first index.  The row offsets come from an exclusive scan of the skipped
 * positions (len - 1 + rejected) and the coverage before each entry from a max-scan of
 * the starts' ends.  A chunk with a rejected start right after the previous start's
 * last draw (a possible rejection run) or with a longer reach (tails) is walked
 * sequentially by lane 0 -- the same rules one entry at a time.
 */
template <int SRC>
__device__ __noinline__ void pos_parse(const LaneParams& p, PosShared& sh, uint64_t* s_x, const int* s_eq, const int* s_ela,
                                       const double* s_ev, int PP, int RW, int64_t need, int carry, int run, uint64_t S0,
                                       uint64_t gam, int64_t passB, int64_t sid, int lane, bool force_serial)
{
    const uint32_t xb = sh_addr(s_x);
    const uint32_t lt = (1u << lane) - 1u;
    int b = 0, c1, c2, c3, total;
    {
        const int n0 = sh.cnt[0], n1 = sh.cnt[1], n2 = sh.cnt[2], n3 = sh.cnt[3];
        b = (n0 | n1 | n2 | n3) < 0;
        c1 = max(n0, 0);
        c2 = c1 + max(n1, 0);
        c3 = c2 + max(n2, 0);
        total = c3 + max(n3, 0);
    }
    if (lane < POS_NW) sh.nacc[lane] = 0;
    __syncwarp();
    const int t = need <= PP ? (int)need - 1 : -1;   /* the row's last deviate, pass-relative */
    int cov = carry, D = carry, r = run, fin = -1;  /* warp-uniform */
    for (int x = lane; x < min(carry, PP); x += 32) {
        sts_u64(xb + 8 * x, POS_MARK);
        atomicAdd(&sh.nacc[pos_region(x, RW)], 1);
    }
    for (int g0 = 0; g0 < total && !b; g0 += 32) {
        const int g = g0 + lane;
        const bool in = g < total;
        int q = 0x7fffffff, len = 1, acc = 1;
        double ev = 0.0;
        if (in) {
            const int slot = pos_slot(g, c1, c2, c3);
            q = s_eq[slot];
            const int la = s_ela[slot];
            len = la >> 1;
            acc = la & 1;
            ev = s_ev[slot];
        }
        const int qp = __shfl_up_sync(GZ_FULL, q, 1), ep = qp + __shfl_up_sync(GZ_FULL, len, 1);
        const int qpp = __shfl_up_sync(GZ_FULL, q, 2), epp = qpp + __shfl_up_sync(GZ_FULL, len, 2);
        const bool c = lane == 0 ? q < cov : q < ep;
        const bool far = in && ((lane == 1 && q < cov) || (lane >= 2 && q < epp));
        const uint32_t C = __ballot_sync(GZ_FULL, c && in);
        const uint32_t Z = ~C & ((lane == 31 ? GZ_FULL : (2u << lane) - 1u));
        const int a = Z ? 32 - __clz(Z) : 0;
        const bool st = in && (!c || ((lane - a) & 1));
        /* skipped positions before each entry, coverage before each entry */
        const int d = st ? len - 1 + (acc ^ 1) : 0;
        int ds = d, em = st ? q + len : cov;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int y = __shfl_up_sync(GZ_FULL, ds, o), z = __shfl_up_sync(GZ_FULL, em, o);
            if (lane >= o) {
                ds += y;
                em = max(em, z);
            }
        }
        const int Dk = D + ds - d;
        int covb = __shfl_up_sync(GZ_FULL, em, 1);
        if (lane == 0) covb = cov;
        covb = max(covb, cov);
        const bool adj = st && !acc && q == covb;
        if (__any_sync(GZ_FULL, far || adj || force_serial)) {
            /* the sequential walk of this chunk (lane 0) */
            if (lane == 0) {
                const int ge = min(total, g0 + 32);
                for (int k = g0; k < ge; ++k) {
                    const int slot = pos_slot(k, c1, c2, c3);
                    const int qk = s_eq[slot];
                    if (qk < cov) continue;
                    const int la = s_ela[slot], lk = la >> 1, ak = la & 1;
                    if (fin < 0 && t >= 0) {
                        if (t < qk - D) fin = t + D + 1;
                        else if (ak && t == qk - D) fin = qk + lk;
                    }
                    if (qk != cov) r = 0;
                    if (ak) r = 0;
                    else if ((int64_t)++r >= p.guard) b = 1;
                    pos_apply(sh, xb, qk, lk, ak, s_ev[slot], PP, RW);
                    D += lk - 1 + (ak ^ 1);
                    cov = qk + lk;
                }
            }
            cov = __shfl_sync(GZ_FULL, cov, 0);
            D = __shfl_sync(GZ_FULL, D, 0);
            r = __shfl_sync(GZ_FULL, r, 0);
            fin = __shfl_sync(GZ_FULL, fin, 0);
            b = __shfl_sync(GZ_FULL, b, 0);
            continue;
        }
        if (st) {
            int f = -1;
            if (t >= 0) {
                if (t >= covb - Dk && t < q - Dk) f = t + Dk + 1;
                else if (acc && t == q - Dk) f = q + len;
            }
            if (f >= 0) fin = f;   /* at most one lane */
            pos_apply(sh, xb, q, len, acc, ev, PP, RW);
            if (!acc && p.guard <= 1) b = 1;
        }
        fin = __reduce_max_sync(GZ_FULL, (unsigned)(fin + 1)) - 1;
        b = __any_sync(GZ_FULL, b) ? 1 : 0;
        const uint32_t S = __ballot_sync(GZ_FULL, st);
        if (S) {
            const int ls = 31 - __clz(S);
            const int qs = __shfl_sync(GZ_FULL, q, ls), lsn = __shfl_sync(GZ_FULL, len, ls),
                      as = __shfl_sync(GZ_FULL, acc, ls);
            r = as ? 0 : 1;
            cov = qs + lsn;
        }
        D = __shfl_sync(GZ_FULL, D + ds, 31);
    }
    /* after the last start: accepted fast starts up to the pass end */
    if (fin < 0 && t >= 0 && t + D < PP) fin = t + D + 1;
    if (lane == 0) {
        const int over = cov > PP ? cov - PP : 0;
        sh.carry = over;
        sh.run = cov < PP ? 0 : r;
        sh.bad = b;
        if (!b && fin >= 0) {
            const uint64_t s_end = pos_state_at<SRC>(S0, gam, (uint64_t)(passB + fin));
            if constexpr (SRC == 0) {
                p.state_out[sid] = s_end;
            } else {
                p.state_out[2 * sid] = s_end;
                p.state_out[2 * sid + 1] = gam;
            }
        }
    }
}

template <int SRC, int IBT, bool MOD>
__global__ void __launch_bounds__(32 * POS_NW, 8) k_zig_pos(const __grid_constant__ LaneParams p, const float dpv,
                                                            const int mode)
{
    extern __shared__ __align__(16) unsigned char smem[];
    const int nl = IBT ? (1 << IBT) : p.n_layers;
    ulonglong2* s_kw = reinterpret_cast<ulonglong2*>(smem);
    float2* s_yf = reinterpret_cast<float2*>(smem + 16 * nl);
    PosShared& sh = *reinterpret_cast<PosShared*>(smem + 24 * nl);
    uint64_t* s_x = reinterpret_cast<uint64_t*>(smem + 24 * nl + ((sizeof(PosShared) + 15) & ~(size_t)15));
    double* s_ev = reinterpret_cast<double*>(s_x + POS_PP);
    int* s_eq = reinterpret_cast<int*>(s_ev + POS_NW * POS_ECAP);
    int* s_ela = s_eq + POS_NW * POS_ECAP;
    for (int i = threadIdx.x; i < nl; i += blockDim.x) {
        s_kw[i] = p.kw[i];
        s_yf[i] = p.yf[i];
    }
    __syncthreads();
    const int lane = threadIdx.x & 31;
    const int w = threadIdx.x >> 5;
    const uint32_t lt = (1u << lane) - 1u;
    const uint32_t kw_sh = sh_addr(s_kw), yf_sh = sh_addr(s_yf);
    const int ib = IBT ? IBT : p.index_bits;
    const uint32_t imask = (uint32_t)nl - 1u;
    const int mbits = 63 - ib;
    const uint64_t mmask = (1ULL << mbits) - 1ULL;
    uint64_t AW = 0, CW = 0;   /* LCG: 32 draws = 64 steps */
    if constexpr (SRC == 0) {
        AW = ld_keep(&c_lcgA[64]);
        CW = ld_keep(&c_lcgC[64]);
    }
    int* const my_eq = s_eq + w * POS_ECAP;
    int* const my_ela = s_ela + w * POS_ECAP;
    double* const my_ev = s_ev + w * POS_ECAP;

    for (int64_t sid = blockIdx.x; sid < p.n_streams; sid += gridDim.x) {
        uint64_t S0, gam = 0;
        if constexpr (SRC == 0) {
            S0 = p.state_in[sid];
        } else {
            S0 = p.state_in[2 * sid];
            gam = p.state_in[2 * sid + 1];
        }
        const uint64_t g32 = 32 * gam;
        double* const row = p.out + sid * p.ld;
        int64_t need = p.n_per, produced = 0, passB = 0;
        int carry = 0, run = 0;
        bool bad = mode == 1;   /* test knobs: 1 every stream to the exact loop, 2 sequential parse */
        while (need > 0 && !bad) {
            const float fneed = (float)need;
            int Jp = (int)ceilf((fneed * dpv + 6.0f * sqrtf(fneed * 0.06f) + 32.0f) / (32.0f * POS_NW));
            Jp = max(1, min(Jp, POS_J));
            const int PP = 32 * POS_NW * Jp;
            const int R = w * 32 * Jp;
            /* 1. classify every position of the warp's region; resolve the non-fast ones */
            uint64_t S = pos_state_at<SRC>(S0, gam, (uint64_t)(passB + R + lane));
            int cnt = 0;
            bool ovf = false;
            uint32_t xa = sh_addr(s_x) + 8 * (R + lane);
#pragma unroll 1
            for (int j = 0; j < Jp; ++j, xa += 256) {
                uint64_t St = S;
                const uint64_t u = lane_next<SRC>(St, gam);   /* St: the state after this draw */
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
                const double x = __dmul_rn(__ull2double_rn(m), __longlong_as_double((long long)kw.y));
                const bool fast = m < kw.x;
                const int pr = R + 32 * j + lane;
                const uint64_t xs = (uint64_t)__double_as_longlong(x) ^ sgn;
                sts_u64(xa, fast ? xs : POS_MARK);
                const uint32_t nfb = __ballot_sync(GZ_FULL, !fast);
                if (nfb) {
                    uint64_t u2 = __shfl_down_sync(GZ_FULL, u, 1);   /* the draw at p + 1 */
                    if (!fast) {
                        const int slot = cnt + __popc(nfb & lt);
                        uint64_t v = xs;
                        int la;
                        if (i != 0) {
                            if (lane == 31) {
                                uint64_t S2 = St;
                                u2 = lane_next<SRC>(S2, gam);
                            }
                            la = 4 + (wedge_accept_f(u2, x, p.yd + i, lds_f32x2(yf_sh + 8 * i)) ? 1 : 0);
                        } else {
                            const TailOut to = tail_seq<SRC>(St, gam, p.r, p.guard);
                            if (to.k < 0 || to.k >= (1 << 28)) ovf = true;
                            la = 2 * (1 + 2 * to.k) + 1;
                            v = (uint64_t)__double_as_longlong(to.v) ^ sgn;
                        }
                        if (slot < POS_ECAP) {
                            my_eq[slot] = pr;
                            my_ela[slot] = la;
                            my_ev[slot] = __longlong_as_double((long long)v);
                        } else {
                            ovf = true;
                        }
                    }
                    cnt += __popc(nfb);
                }
                if constexpr (SRC == 0) S = gz_lcg_mad(AW, S, CW);
                else S += g32;
            }
            ovf = __any_sync(GZ_FULL, ovf);
            if (lane == 0) sh.cnt[w] = (ovf || cnt > POS_ECAP) ? -1 : cnt;
            __syncthreads();
            /* 2. parse the sparse entry list in position order (warp 0; pos_parse) */
            if (w == 0) pos_parse<SRC>(p, sh, s_x, s_eq, s_ela, s_ev, PP, 32 * Jp, need, carry, run, S0, gam, passB, sid, lane,
                                        mode == 2);
            __syncthreads();
            if (sh.bad) {
                bad = true;
                break;
            }
            /* 3. emit: the positions holding values are the accepted starts, in order:
               a ballot compaction per 32-position window, coalesced stores */
            {
                int base = 0;
                for (int v = 0; v < w; ++v) base += 32 * Jp - sh.nacc[v];   /* accepted starts before the region */
                const int lim = need < PP ? (int)need : PP;   /* deviates still wanted */
                double* const dst = row + produced;
                uint32_t xa = sh_addr(s_x) + 8 * (R + lane);
#pragma unroll 1
                for (int j = 0; j < Jp; ++j, xa += 256) {
                    const uint64_t val = lds_u64(xa);
                    const bool keep = (uint32_t)(val >> 32) != (uint32_t)(POS_MARK >> 32);
                    const uint32_t bal = __ballot_sync(GZ_FULL, keep);
                    const int gi = base + __popc(bal & lt);
                    if (keep && gi < lim) dst[gi] = __longlong_as_double((long long)val);
                    base += __popc(bal);
                }
            }
            __syncthreads();   /* sh.nacc read below; s_x and the entries are rewritten next pass */
            int c = PP;
            for (int v = 0; v < POS_NW; ++v) c -= sh.nacc[v];
            produced += c;
            need -= c;
            passB += PP;
            carry = sh.carry;
            run = sh.run;
        }
        if (bad) {
            /* the exact sequential loop decides (and raises a guard trip) */
            if (w == 0) pos_fallback<SRC, MOD>(p, sid, nl, ib, lane);
        } else if (p.n_per == 0 && threadIdx.x == 0) {
            if constexpr (SRC == 0) {
                p.state_out[sid] = S0;
            } else {
                p.state_out[2 * sid] = S0;
                p.state_out[2 * sid + 1] = gam;
            }
        }
        __syncthreads();
    }
}
