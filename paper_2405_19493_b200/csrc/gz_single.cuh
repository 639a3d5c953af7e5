/*
 * gz_single.cuh -- one long stream decoded by the whole GPU (included by
 * gz_engine.cu after its kernels and DevCtx).
 *
 * The reference's own API fills ONE stream per call (engine.fill_gaussians,
 * engine.py:235-270; bench.py:201-215 times exactly that).  A warp per stream
 * decodes about 0.1 G variates/s there, slower than the reference's CPU loop,
 * so calls with one stream and many variates take this path instead:
 *
 *   polar  attempt j always consumes draws 2j and 2j+1 (samplers.py:185-192),
 *          so the attempts are independent: count accepted attempts per block,
 *          exclusive-scan the counts, and let every block transform and store
 *          its accepted pairs at their prefix rank (stream compaction).
 *   ziggurat  an attempt consumes 1 draw (fast path), 2 (wedge: the next draw
 *          is its uniform) or 1 + 2t (tail, t pairs); which draws start attempts
 *          is a chain 0 -> 0 + len(0) -> ...  Every draw position is classified
 *          as if it started an attempt (len, accepted, value: independent), each
 *          chunk of positions is walked from every possible entry offset
 *          0..SZ_E-1 (the previous chunk's last attempt may overhang), the chunk
 *          entries are linked in a prefix over chunks, and every chunk re-walks
 *          from its true entry and stores its deviates at their prefix rank.
 *
 * Results are identical to the sequential loop by construction (same draws, same
 * decisions, same order); tests compare them with the oracle and the golden
 * fixtures.  Rare shapes this path does not cover (a tail overhanging more than
 * SZ_E - 1 draws into the next chunk, a chunk with no accepted attempt, guards
 * below SINGLE_MIN_GUARD) fall back to the warp-per-stream kernels.
 */
#pragma once

constexpr int64_t SINGLE_MIN_N = 1 << 15;       /* below this the warp kernel is faster */
constexpr int64_t SINGLE_MIN_GUARD = 1 << 13;   /* a guard trip needs a whole rejected chunk */
constexpr int SP_T = 256;                       /* polar: attempts per block */
constexpr int CL_J = 8;                         /* ziggurat classify: positions per thread */
constexpr uint64_t CL_A512 = 0x94fba1cf4801ULL, CL_C512 = 0x9e1922a97200ULL;   /* 512 LCG steps */
constexpr int SZ_L = 1024;                      /* ziggurat: draw positions per chunk (= 32 bitmap words) */
constexpr int SZ_E = 8;                         /* ziggurat: entry offsets walked per chunk */

/* (A, C) of n LCG steps (state -> A*state + C mod 2^48), by squaring */
__device__ __forceinline__ void lcg_jump_n(uint64_t n, uint64_t& A, uint64_t& C)
{
    uint64_t a = GZ_LCG_A, c = GZ_LCG_C;
    A = 1;
    C = 0;
    while (n) {
        if (n & 1) {
            C = (a * C + c) & GZ_MASK48;
            A = (a * A) & GZ_MASK48;
        }
        c = (a * c + c) & GZ_MASK48;
        a = (a * a) & GZ_MASK48;
        n >>= 1;
    }
}

/* the stream state after `draws` u64 draws from s0 (LCG: 2 steps per draw) */
template <int SRC>
__device__ __forceinline__ uint64_t single_state_at(uint64_t s0, uint64_t gam, uint64_t draws)
{
    if constexpr (SRC == 0) {
        uint64_t A, C;
        lcg_jump_n(2 * draws, A, C);
        return (A * s0 + C) & GZ_MASK48;
    } else {
        return s0 + draws * gam;
    }
}

/* ------------------------------------------------------------------ polar */

/* SP_K consecutive attempts per thread: the per-thread jump and the block's base jump
   are paid once per SP_K attempts */
constexpr int SP_K = 8;
constexpr int SP_BLOCK = SP_T * SP_K;   /* attempts per block */

/* the state before attempt jb + SP_K*t of the block (thread 0 jumps to the block
   base, every thread jumps 4*SP_K*t LCG steps / 2*SP_K*t draws from it) */
template <int SRC>
__device__ __forceinline__ uint64_t polar_single_state(const uint64_t* st0, uint64_t& gam, int64_t jb, uint64_t* s_base)
{
    const int t = threadIdx.x;
    const uint64_t s0 = st0[0];
    if constexpr (SRC == 0) {
        gam = 0;
        if (t == 0) *s_base = single_state_at<0>(s0, 0, 2 * (uint64_t)jb);
        __syncthreads();
        uint64_t A, C;
        lcg_jump_n(4 * (uint64_t)SP_K * t, A, C);
        return (A * *s_base + C) & GZ_MASK48;
    } else {
        gam = st0[1];
        return s0 + (uint64_t)(2 * (jb + (int64_t)SP_K * t)) * gam;
    }
}

/* one polar attempt from state S (the state before its first draw): v1, v2, s; S
   advances past its two draws */
template <int SRC>
__device__ __forceinline__ bool polar_single_attempt(uint64_t& S, uint64_t gam, double& v1, double& v2, double& s)
{
    const uint64_t ua = gz_next_seq<SRC>(S, gam);
    const uint64_t ub = gz_next_seq<SRC>(S, gam);
    v1 = gz_unit53_pm1(ua);
    v2 = gz_unit53_pm1(ub);
    s = __dadd_rn(__dmul_rn(v1, v1), __dmul_rn(v2, v2));
    return s > 0.0 && s < 1.0;
}

/* this thread's SP_K attempts: bit k of the result = attempt k accepted */
template <int SRC>
__device__ __forceinline__ uint32_t polar_single_mask(uint64_t S, uint64_t gam, int64_t first, int64_t end)
{
    uint32_t m = 0;
#pragma unroll
    for (int k = 0; k < SP_K; ++k) {
        double v1, v2, s;
        const bool acc = polar_single_attempt<SRC>(S, gam, v1, v2, s);
        if (acc && first + k < end) m |= 1u << k;
    }
    return m;
}

/* pass 1: accepted attempts per block for attempts [j0, j0 + n_att) */
template <int SRC>
__global__ void __launch_bounds__(SP_T) k_polar_single_count(const uint64_t* st0, int64_t j0, int64_t n_att, int* cnt)
{
    __shared__ uint64_t s_base;
    __shared__ int s_c[SP_T / 32];
    const int64_t jb = j0 + (int64_t)blockIdx.x * SP_BLOCK;
    uint64_t gam;
    const uint64_t S = polar_single_state<SRC>(st0, gam, jb, &s_base);
    const int64_t first = jb + (int64_t)SP_K * threadIdx.x;
    const int c = __popc(polar_single_mask<SRC>(S, gam, first, j0 + n_att));
    const int wc = __reduce_add_sync(GZ_FULL, (unsigned)c);
    if ((threadIdx.x & 31) == 0) s_c[threadIdx.x >> 5] = wc;
    __syncthreads();
    if (threadIdx.x == 0) {
        int tot = 0;
        for (int w = 0; w < SP_T / 32; ++w) tot += s_c[w];
        cnt[blockIdx.x] = tot;
    }
}

struct PolarSingleOut {
    double* out;           /* deviate 0 of the call (after a cached spare) */
    int64_t pairs_done;    /* pairs stored by earlier segments */
    int64_t np;            /* pairs the call needs */
    bool odd;              /* the last pair's second value is the new spare */
    double* spare_out;
    uint64_t* state_out;
};

/* store pair k of the call (the odd call's last pair: one deviate + the spare) */
__device__ __forceinline__ void polar_single_store(const PolarSingleOut& o, int64_t k, double v1, double v2, double mul)
{
    const double o1 = __dmul_rn(v1, mul), o2 = __dmul_rn(v2, mul);
    if (o.odd && k == o.np - 1) {
        o.out[2 * k] = o1;
        if (o.spare_out) o.spare_out[0] = o2;
    } else {
        pair_store(o.out + 2 * k, o1, o2);
    }
}

/*
 * pass 2: every thread regenerates its SP_K attempts and writes its accepted pairs,
 * in attempt order, to a block queue in shared memory; the block then transforms
 * the queue with all threads -- glibc log's main branch at once, the near-1 pairs
 * (s >= 1 - 2^-4) compacted into a list and transformed after -- and stores pair q
 * of the queue at its prefix rank (coalesced).
 */
template <int SRC>
__global__ void __launch_bounds__(SP_T) k_polar_single_emit(const uint64_t* st0, int64_t j0, int64_t n_att,
                                                            const int* prefix, PolarSingleOut o)
{
    __shared__ uint64_t s_base;
    __shared__ int s_c[SP_T / 32];
    __shared__ uint64_t s_log[256];
    __shared__ double2 s_q[SP_BLOCK];
    __shared__ short s_near[SP_BLOCK];
    __shared__ int s_nn;
    const int64_t pre = prefix[blockIdx.x];
    const int64_t need = o.np - o.pairs_done;
    if (pre >= need) return;   /* block-uniform */
    for (int i = threadIdx.x; i < 256; i += SP_T) s_log[i] = g_log_tab[i];
    if (threadIdx.x == 0) s_nn = 0;
    const int64_t jb = j0 + (int64_t)blockIdx.x * SP_BLOCK;
    uint64_t gam;
    const uint64_t S0 = polar_single_state<SRC>(st0, gam, jb, &s_base);
    const int64_t first = jb + (int64_t)SP_K * threadIdx.x, end = j0 + n_att;
    const uint32_t m = polar_single_mask<SRC>(S0, gam, first, end);
    /* block exclusive scan of the per-thread counts */
    const int c = __popc(m);
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    int incl = c;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        const int t = __shfl_up_sync(GZ_FULL, incl, d);
        if (lane >= d) incl += t;
    }
    if (lane == 31) s_c[wid] = incl;
    __syncthreads();
    int wbase = 0;
    for (int w = 0; w < wid; ++w) wbase += s_c[w];
    int nq = 0;
    for (int w = 0; w < SP_T / 32; ++w) nq += s_c[w];
    int q = wbase + incl - c;
    /* regenerate and queue the accepted pairs; the attempt of the call's last pair
       leaves the stream state */
    {
        uint64_t S = S0;
#pragma unroll
        for (int k = 0; k < SP_K; ++k) {
            double v1, v2, s;
            polar_single_attempt<SRC>(S, gam, v1, v2, s);
            if ((m >> k) & 1u) {
                s_q[q] = make_double2(v1, v2);
                if (pre + q == need - 1) {
                    if constexpr (SRC == 0) {
                        o.state_out[0] = S & GZ_MASK48;
                    } else {
                        o.state_out[0] = S;
                        o.state_out[1] = gam;
                    }
                }
                ++q;
            }
        }
    }
    __syncthreads();
    const int nkeep = (int)(need - pre < nq ? need - pre : nq);
    /* main branch: all threads; near-1 pairs are listed for the second pass */
    for (int i = threadIdx.x; i < nkeep; i += SP_T) {
        const double2 v = s_q[i];
        const double s = __dadd_rn(__dmul_rn(v.x, v.x), __dmul_rn(v.y, v.y));
        const bool near = (uint64_t)__double_as_longlong(s) >= 0x3fee000000000000ULL;
        if (!near) {
            const double mul = sqrt_rn_nb(div_rn_nb(__dmul_rn(-2.0, gz_log_core((uint64_t)__double_as_longlong(s), s_log)), s));
            polar_single_store(o, o.pairs_done + pre + i, v.x, v.y, mul);
        }
        const uint32_t nb = __ballot_sync(__activemask(), near);
        if (near) {
            const int leader = __ffs(nb) - 1;
            int base = 0;
            if (lane == leader) base = atomicAdd(&s_nn, __popc(nb));
            base = __shfl_sync(nb, base, leader);
            s_near[base + __popc(nb & ((1u << lane) - 1u))] = (short)i;
        }
    }
    __syncthreads();
    const int nn = s_nn;
    for (int t = threadIdx.x; t < nn; t += SP_T) {
        const int i = s_near[t];
        const double2 v = s_q[i];
        const double s = __dadd_rn(__dmul_rn(v.x, v.x), __dmul_rn(v.y, v.y));
        polar_single_store(o, o.pairs_done + pre + i, v.x, v.y, polar_mul(s, s_log));
    }
}

/* ------------------------------------------------------------------ ziggurat */

/* a position classified as an attempt start: draws consumed, accepted, value */
struct ZigPos {
    uint16_t len;          /* 1 fast, 2 wedge, 1 + 2t tail; 0: tail guard tripped */
    uint8_t acc;
    uint8_t pad;
};

template <int SRC, bool MOD>
__global__ void __launch_bounds__(256) k_zig_single_classify(const uint64_t* st0, int64_t p0, int64_t n_pos,
                                                             const ulonglong2* kw, const double2* yd, const float2* yf,
                                                             int n_layers, double r, int64_t guard, ZigPos* pos,
                                                             double* val)
{
    __shared__ uint64_t s_base;
    /* a block classifies CL_J * 256 positions: thread t takes pb + t + 256 j, j < CL_J,
       so the per-thread jump is paid once and the next position is a constant jump of
       512 LCG steps (coalesced stores at every j) */
    const int64_t pb = p0 + (int64_t)blockIdx.x * (256 * CL_J);
    const int t = threadIdx.x;
    uint64_t s0 = st0[0], gam = 0;
    if constexpr (SRC == 1) gam = st0[1];
    uint64_t St;   /* the state before position pb + t + 256 j's draw */
    if constexpr (SRC == 0) {
        if (t == 0) s_base = single_state_at<0>(s0, 0, (uint64_t)pb);
        __syncthreads();
        uint64_t A, C;
        lcg_jump_n(2 * (uint64_t)t, A, C);
        St = (A * s_base + C) & GZ_MASK48;
    } else {
        St = s0 + (uint64_t)(pb + t) * gam;
    }
    int ib = 0;
    while ((1 << (ib + 1)) <= n_layers) ++ib;
    const uint32_t imask = (uint32_t)n_layers - 1u;
    const int mbits = 63 - ib;
    const uint64_t mmask = (1ULL << mbits) - 1ULL;
    for (int jj = 0; jj < CL_J; ++jj) {
        const int64_t k = pb + t + 256 * jj;
        if (k >= p0 + n_pos) break;
        uint64_t S = St;
        if constexpr (SRC == 0) St = (CL_A512 * St + CL_C512) & GZ_MASK48;
        else St += 256 * gam;
        /* ZigguratSampler._draw one attempt (samplers.py:95-115 / 144-165) */
        const uint64_t u = gz_next_seq<SRC>(S, gam);
        uint32_t i;
        uint64_t m;
        bool neg;
        if constexpr (MOD) {
            i = (uint32_t)u & imask;
            m = u >> (ib + 1);
            neg = (u >> ib) & 1;
        } else {
            i = (uint32_t)(u >> mbits) & imask;
            m = u & mmask;
            neg = u >> 63;
        }
        const ulonglong2 kk = kw[i];
        double x = __dmul_rn(__ull2double_rn(m), __longlong_as_double((long long)kk.y));
        ZigPos zp{1, 1, 0};
        if (m >= kk.x) {
            if (i != 0) {
                const uint64_t u2 = gz_next_seq<SRC>(S, gam);
                zp.len = 2;
                /* the float pre-filter settles all but the cases within 2^-15 of the boundary */
                zp.acc = wedge_accept_f(u2, x, yd + i, yf[i]) ? 1 : 0;
            } else {
                const TailOut to = tail_seq<SRC>(S, gam, r, guard);
                if (to.k < 0 || 1 + 2 * (int64_t)to.k > 65535) {
                    zp.len = 0;   /* guard tripped or an overlong tail: the caller falls back */
                    zp.acc = 0;
                } else {
                    zp.len = (uint16_t)(1 + 2 * to.k);
                    x = to.v;
                }
            }
        }
        pos[k - p0] = zp;
        val[k - p0] = neg ? -x : x;
    }
}

/* per chunk and entry offset e: where the walk leaves the chunk and what it found */
struct ZigExit {
    int32_t exit;          /* next attempt start - chunk end (>= 0) */
    int32_t cnt;           /* accepted attempts started in the chunk */
    int32_t bad;           /* a zero-length position (guard / overlong tail) on the walk */
    int32_t pad;
};

/* walk every entry offset 0..SZ_E-1 of chunk blockIdx.x through the chunk (one warp
   per chunk) and leave, per entry, where the walk leaves the chunk, its accepted
   count and the bitmap of its accepted attempt starts (SZ_L bits), so the emit pass
   needs no walk.  The chunk is cut into SZ_S sub-chunks walked at once from every
   entry (lane = SZ_E * sub-chunk + entry), and the sub-chunk walks are composed per
   chunk entry by shuffles: the serial chain a lane follows is SZ_L / SZ_S positions
   long, not SZ_L.  A walk that leaves a sub-chunk SZ_E or more positions past its end
   (a long tail attempt) has no precomputed continuation: that chunk entry is walked
   through the whole chunk by one lane instead (same result). */
constexpr int SZ_W = SZ_L / 32;   /* bitmap words per chunk and entry */
static_assert(SZ_W == 32, "the emit pass maps one bitmap word per lane");
constexpr int SZ_S = 32 / SZ_E;   /* sub-chunks per chunk */
constexpr int SZ_SL = SZ_L / SZ_S;   /* positions per sub-chunk */
constexpr int SZ_SW = SZ_SL / 32;    /* bitmap words per sub-chunk and entry */
static_assert(SZ_S * SZ_E == 32 && SZ_SL % 32 == 0, "one lane per (sub-chunk, entry)");

/* walk positions [p, end) of the packed chunk pk from p, setting the accepted starts in
   the bitmap words bmw[(q - w0) >> 5] (q: chunk position); returns the position where
   the walk leaves [.., end) and adds the accepted count; bad on a zero-length position */
__device__ __forceinline__ int zig_walk(const uint16_t* pk, int p, int end, int w0, uint32_t* bmw, int& cnt,
                                        int& bad)
{
    int cw = p >> 5;
    uint32_t word = 0;   /* bitmap word cw, stored when the walk leaves it */
    while (p < end) {
        const uint32_t v = pk[p];
        const int l = (int)(v & 0x7FFFu);
        if (l == 0) {
            bad = 1;
            break;
        }
        const uint32_t acc = v >> 15;
        cnt += (int)acc;
        if ((p >> 5) != cw) {
            bmw[cw - w0] = word;
            cw = p >> 5;
            word = 0;
        }
        word |= acc << (p & 31);
        p += l;
    }
    if (cw - w0 < (end - (w0 << 5) + 31) >> 5) bmw[cw - w0] = word;
    return p;
}

__global__ void __launch_bounds__(32) k_zig_single_exits(const ZigPos* pos, int64_t n_pos, int n_chunks, ZigExit* ex,
                                                         uint32_t* bm)
{
    __shared__ uint16_t s_pk[SZ_L + 16];
    __shared__ uint32_t s_sb[SZ_S][SZ_E][SZ_SW + 1];   /* sub-chunk bitmaps */
    __shared__ uint32_t s_out[SZ_E][SZ_W + 1];         /* chunk bitmaps per entry */
    const int lane = threadIdx.x;
    const int c = blockIdx.x;
    if (c >= n_chunks) return;
    const int64_t c0 = (int64_t)c * SZ_L;
    const int nl = (int)(n_pos - c0 < SZ_L ? n_pos - c0 : SZ_L);
    if (nl == SZ_L) {
        /* 16-byte loads: four positions per lane and step */
        const uint4* src = reinterpret_cast<const uint4*>(pos + c0);
#pragma unroll
        for (int it = 0; it < SZ_L / 4 / 32; ++it) {
            const int q = it * 32 + lane;
            const uint4 v = src[q];
            const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                const uint32_t len = w[k] & 0xFFFFu, acc = (w[k] >> 16) & 0xFFu;
                s_pk[4 * q + k] = (uint16_t)(len > 0x7FFFu ? 0u : (len | (acc ? 0x8000u : 0u)));
            }
        }
    } else {
        for (int i = lane; i < nl; i += 32) {
            const ZigPos zp = pos[c0 + i];
            s_pk[i] = (uint16_t)(zp.len > 0x7FFF ? 0 : (zp.len | (zp.acc ? 0x8000 : 0)));
        }
    }
    {
        uint32_t* sb = &s_sb[0][0][0];
        for (int i = lane; i < SZ_S * SZ_E * (SZ_SW + 1); i += 32) sb[i] = 0u;
        uint32_t* so = &s_out[0][0];
        for (int i = lane; i < SZ_E * (SZ_W + 1); i += 32) so[i] = 0u;
    }
    __syncwarp();
    /* lane = SZ_E * g + e walks entry e of sub-chunk g */
    const int g = lane / SZ_E, e = lane % SZ_E;
    const int sbeg = g * SZ_SL;
    const int send = min(sbeg + SZ_SL, nl);
    int cnt = 0, bad = 0, xo = 0;
    if (sbeg < nl) {
        const int p = zig_walk(s_pk, sbeg + e, send, sbeg >> 5, s_sb[g][e], cnt, bad);
        xo = bad ? 0 : p - send;
    }
    __syncwarp();
    /* compose the sub-chunk walks for chunk entry e = lane (lanes >= SZ_E follow along) */
    int en = lane < SZ_E ? lane : 0, tot = 0, cbad = 0, slow = 0;
    int ent[SZ_S];
#pragma unroll
    for (int gg = 0; gg < SZ_S; ++gg) {
        ent[gg] = en;
        const int src = SZ_E * gg + (en < SZ_E ? en : 0);
        const int x_ = __shfl_sync(GZ_FULL, xo, src);
        const int c_ = __shfl_sync(GZ_FULL, cnt, src);
        const int b_ = __shfl_sync(GZ_FULL, bad, src);
        if (gg * SZ_SL < nl && !slow && !cbad) {
            if (en >= SZ_E) {
                slow = 1;          /* overhang past the precomputed entries */
            } else {
                tot += c_;
                cbad |= b_;
                en = x_;
            }
        }
    }
    if (lane < SZ_E) {
        ZigExit x;
        if (slow) {
            /* the whole chunk from entry `lane` by this lane */
            int sc = 0, sbd = 0;
            const int p = zig_walk(s_pk, lane, nl, 0, s_out[lane], sc, sbd);
            x.exit = sbd ? 0 : p - nl;
            x.cnt = sc;
            x.bad = sbd;
        } else {
#pragma unroll
            for (int gg = 0; gg < SZ_S; ++gg) {
                if (gg * SZ_SL >= nl || cbad) break;
#pragma unroll
                for (int w = 0; w < SZ_SW; ++w) s_out[lane][gg * SZ_SW + w] = s_sb[gg][ent[gg]][w];
            }
            x.exit = cbad ? 0 : en;
            x.cnt = tot;
            x.bad = cbad;
        }
        x.pad = 0;
        ex[(int64_t)c * SZ_E + lane] = x;
    }
    __syncwarp();
    uint32_t* dst = bm + (int64_t)c * SZ_E * SZ_W;
#pragma unroll
    for (int e2 = 0; e2 < SZ_E; ++e2) dst[e2 * SZ_W + lane] = s_out[e2][lane];
}

/* the chunk chain, three levels: lb <= LINK_B chunks per block composed for every entry
   (the host picks lb near sqrt(chunks): both serial chains stay short),
   blocks linked by one thread, chunk entries/bases expanded per block */
constexpr int LINK_B = 128;

struct ZigLinkF {
    int32_t exit, bad;     /* bad: an entry >= SZ_E, a zero-count chunk or a bad walk on the way */
    int64_t cnt;
};

__global__ void __launch_bounds__(32) k_zig_single_link_blocks(const ZigExit* ex, int n_chunks, int lb, ZigLinkF* fb)
{
    __shared__ ZigExit s_ex[LINK_B * SZ_E];
    const int b = blockIdx.x;
    const int c0 = b * lb, c1 = min(c0 + lb, n_chunks);
    for (int i = threadIdx.x; i < (c1 - c0) * SZ_E; i += 32) s_ex[i] = ex[(int64_t)c0 * SZ_E + i];
    __syncwarp();
    const int e0 = threadIdx.x;
    if (e0 >= SZ_E) return;
    int e = e0, bad = 0;
    int64_t cnt = 0;
    for (int c = c0; c < c1; ++c) {
        if (e >= SZ_E) {
            bad = 1;
            break;
        }
        const ZigExit x = s_ex[(c - c0) * SZ_E + e];
        if (x.bad || x.cnt == 0) bad = 1;
        cnt += x.cnt;
        e = x.exit;
    }
    ZigLinkF f;
    f.exit = e;
    f.bad = bad;
    f.cnt = cnt;
    fb[(int64_t)b * SZ_E + e0] = f;
}

struct ZigLinkTop {
    int64_t total;         /* accepted attempts of the whole segment from entry 0 */
    int32_t exit;          /* next attempt start - segment end */
    int32_t bad;
};

/* one block: the blocks' composed functions staged in shared memory, linked by one thread */
__global__ void __launch_bounds__(256) k_zig_single_link_top(const ZigLinkF* fb, int n_blocks, int* b_entry,
                                                             int64_t* b_base, ZigLinkTop* top)
{
    extern __shared__ ZigLinkF s_fb[];
    for (int i = threadIdx.x; i < n_blocks * SZ_E; i += blockDim.x) s_fb[i] = fb[i];
    __syncthreads();
    if (threadIdx.x != 0) return;
    int e = 0, bad = 0;
    int64_t base = 0;
    for (int b = 0; b < n_blocks; ++b) {
        b_entry[b] = e;
        b_base[b] = base;
        if (e >= SZ_E) {
            bad = 1;
            break;
        }
        const ZigLinkF f = s_fb[b * SZ_E + e];
        bad |= f.bad;
        base += f.cnt;
        e = f.exit;
    }
    top->total = base;
    top->exit = e;
    top->bad = bad;
}

__global__ void __launch_bounds__(32) k_zig_single_link_expand(const ZigExit* ex, int n_chunks, int lb,
                                                               const int* b_entry, const int64_t* b_base, int* entry,
                                                               int64_t* base)
{
    __shared__ ZigExit s_ex[LINK_B * SZ_E];
    const int b = blockIdx.x;
    const int c0 = b * lb, c1 = min(c0 + lb, n_chunks);
    for (int i = threadIdx.x; i < (c1 - c0) * SZ_E; i += 32) s_ex[i] = ex[(int64_t)c0 * SZ_E + i];
    __syncwarp();
    if (threadIdx.x != 0) return;
    int e = b_entry[b];
    int64_t bs = b_base[b];
    for (int c = c0; c < c1; ++c) {
        entry[c] = e < SZ_E ? e : -1;
        base[c] = bs;
        if (e >= SZ_E) {
            e = SZ_E;
            continue;
        }
        const ZigExit x = s_ex[(c - c0) * SZ_E + e];
        bs += x.cnt;
        e = x.exit;
    }
}

struct ZigSingleOut {
    double* out;           /* output index 0 of this segment */
    int64_t need;          /* deviates this segment must still produce */
    int64_t p0;            /* first draw position of the segment (absolute) */
    uint64_t* state_out;   /* written by the block holding the last needed deviate */
};

/* chunk c stores the values of its accepted attempt starts (the bitmap of its true
   entry) from output index base[c] on; one warp per chunk, one bitmap word per lane */
template <int SRC>
__global__ void __launch_bounds__(32) k_zig_single_emit(const ZigPos* pos, const double* val, int64_t n_pos,
                                                        const uint32_t* bm, const int* entry, const int64_t* base,
                                                        const uint64_t* st0, const ZigLinkTop* top, ZigSingleOut o)
{
    const int c = blockIdx.x;
    const int64_t b0 = base[c];
    const int e = entry[c];
    /* warp-uniform; a bad segment writes nothing (the caller reruns the call on the
       warp kernel) */
    if (b0 >= o.need || e < 0 || top->bad) return;
    const int64_t c0 = (int64_t)c * SZ_L;
    const int lane = threadIdx.x;
    const int nl = (int)(n_pos - c0 < SZ_L ? n_pos - c0 : SZ_L);
    /* the chunk's values staged in shared memory by coalesced loads (one double of
       padding per 32: a lane's run of 32 positions starts in its own bank pair) */
    __shared__ double s_v[SZ_L + SZ_L / 32];
    __shared__ double s_o[SZ_L];
    if (nl == SZ_L) {
        const double2* src = reinterpret_cast<const double2*>(val + c0);
#pragma unroll 4
        for (int it = 0; it < SZ_L / 64; ++it) {
            const int q = it * 32 + lane;
            const double2 v = src[q];
            s_v[2 * q + (q >> 4)] = v.x;
            s_v[2 * q + 1 + (q >> 4)] = v.y;
        }
    } else {
        for (int i = lane; i < nl; i += 32) s_v[i + (i >> 5)] = val[c0 + i];
    }
    const uint32_t word = bm[((int64_t)c * SZ_E + e) * SZ_W + lane];
    const int mine = __popc(word);
    int incl = mine;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
        const int v = __shfl_up_sync(GZ_FULL, incl, off);
        if (lane >= off) incl += v;
    }
    const int r0 = incl - mine;                      /* rank of this lane's first value in the chunk */
    const int cnt = __shfl_sync(GZ_FULL, incl, 31);
    __syncwarp();
    /* compact the accepted starts' values in order */
    {
        uint32_t w = word;
        int r = r0;
        const double* sv = s_v + 33 * lane;
        while (w) {
            const int bit = __ffs(w) - 1;
            w &= w - 1;
            s_o[r++] = sv[bit];
        }
    }
    __syncwarp();
    const int lim = (int)(o.need - b0 < (int64_t)cnt ? o.need - b0 : (int64_t)cnt);
    double* const dst = o.out + b0;
    for (int i = lane; i < lim; i += 32) dst[i] = s_o[i];
    /* the segment's last needed deviate: the stream continues after it */
    const int64_t k = o.need - 1 - b0;           /* its rank in this chunk */
    if (k >= r0 && k < r0 + mine) {
        uint32_t w = word;
        for (int t = 0; t < (int)(k - r0); ++t) w &= w - 1;
        const int64_t p = c0 + 32 * lane + (__ffs(w) - 1);
        const uint64_t s0 = st0[0];
        const uint64_t gam = SRC == 1 ? st0[1] : 0;
        const uint64_t draws = (uint64_t)(o.p0 + p + pos[p].len);
        o.state_out[0] = single_state_at<SRC>(s0, gam, draws);
        if (SRC == 1) o.state_out[1] = gam;
    }
}

/* ------------------------------------------------------------------ fill_u64 */

/* u64 draws [0, n) of one stream (engine.fill_u64 on one source, engine.py:224-232),
   one thread per draw: draw k is independent given the state after k draws */
template <int SRC>
__global__ void __launch_bounds__(256) k_u64_single(const uint64_t* st0, int64_t n, uint64_t* out)
{
    __shared__ uint64_t s_base;
    const int64_t kb = (int64_t)blockIdx.x * 256;
    const int t = threadIdx.x;
    const uint64_t s0 = st0[0];
    uint64_t S, gam = 0;
    if constexpr (SRC == 0) {
        if (t == 0) s_base = single_state_at<0>(s0, 0, (uint64_t)kb);
        __syncthreads();
        uint64_t A, C;
        lcg_jump_n(2 * (uint64_t)t, A, C);
        S = (A * s_base + C) & GZ_MASK48;
    } else {
        gam = st0[1];
        S = s0 + (uint64_t)(kb + t) * gam;
    }
    if (kb + t < n) out[kb + t] = gz_next_seq<SRC>(S, gam);
}

/* the state after n draws (a separate launch: state_out may alias the input) */
template <int SRC>
__global__ void k_u64_single_state(const uint64_t* st0, int64_t n, uint64_t* state_out)
{
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    const uint64_t gam = SRC == 1 ? st0[1] : 0;
    state_out[0] = single_state_at<SRC>(st0[0], gam, (uint64_t)n);
    if (SRC == 1) state_out[1] = gam;
}
