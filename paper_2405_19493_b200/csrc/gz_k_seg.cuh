/*
 * gz_k_seg.cuh -- the ziggurats over FEW long streams (included by gz_engine.cu
 * after gz_single.cuh).
 *
 * With fewer streams than the GPU holds warps (config 1: 1024 streams), a warp per
 * stream leaves most of the machine idle and every warp walks its whole row.  Here
 * a row's draws are cut into segments decoded in parallel from GUESSED entries.  An
 * attempt that starts in segment k-1 may overhang into segment k (wedge: 2 draws,
 * tail: 1 + 2t), so the true entry e of segment k is the exit of segment k-1.
 * Decoding is deterministic from an attempt start, so if the guessed decode has an
 * attempt start at e, both decodes agree from there on: its deviates from e are the
 * true ones and its exit is the true exit.  Almost always the guess synchronises
 * within a few draws (a fast-path attempt consumes exactly one draw); when it does
 * not, the segment is re-decoded from e.  Same draws, same decisions, same order as
 * the sequential loop.
 *
 * Guard: used only when the guard exceeds any rejection run two segments can hold;
 * a segment with no deviate after its entry, or a tail that exhausts its guard,
 * hands the whole stream to the exact warp-per-stream loop (zig_warp_stream).
 * (A first form with one WARP per segment, decoding with the window parse, ran
 * config 1 in 66 us; this lane form runs it in 51 us.)
 */
#pragma once

/*
 * Lane-segment form (k_zig_lseg, the default): a block of P warps per stream, one
 * LANE per segment.  Each round cuts the row's next 32*P*L draws into 32*P segments
 * of L draws; lane k of warp w decodes segment 32w + k with the lane kernel's
 * sequential attempt loop (k_zig_lane) from a guessed entry (segment 0: the known
 * entry), staging its deviates in shared memory ([value][segment], padded rows) and
 * their attempt ends in an L2 scratch.  Links inside a warp are resolved with
 * shuffles (a lane whose guess did not synchronise re-decodes from its true entry),
 * links between warps in warp order at block barriers; offsets by a warp scan plus
 * a prefix over the warps.  A warp's segments are consecutive, so its deviates form
 * one contiguous run of the row, stored coalesced (each lane finds its source
 * segment by a binary search over the offsets).  Per deviate it executes the lane
 * kernel's instructions instead of the window parse's.
 */
struct LsegParams {
    double* scr_v;      /* unused (deviates are staged in shared memory) */
    uint32_t* scr_e;    /* [warps][lcap][32] */
    int lcap;           /* max draws per segment (>= every round's L) */
    float dpv;          /* expected draws per deviate */
    int guess;          /* entry guessed by lanes 1..31 */
    int force_fallback;
};

struct LsegOut {
    int cnt, exit, bad;
    uint32_t sm0, em0;
};

/* lane-sequential decode of one segment from position e0 (S: the state before it) */
template <int SRC, int IBT, bool MOD>
__device__ __forceinline__ LsegOut lseg_decode(uint64_t S, uint64_t gam, int e0, int L, const LaneParams& p,
                                               uint32_t kw_sh, uint32_t yf_sh, int ib, uint32_t imask, int mbits,
                                               uint64_t mmask, double* sv, int vstride, uint32_t* se, int lane)
{
    LsegOut o;
    o.cnt = 0; o.bad = 0; o.sm0 = 0; o.em0 = 0;
    const bool rec = e0 == 0;
    const uint32_t guard32 = p.guard > 0xffffffffll ? 0xffffffffu : (uint32_t)p.guard;
    uint64_t nxt = 0;
    lane_pend<SRC>(S, gam, nxt);
    uint32_t rej = 0;
    int q = e0, cnt = 0;
    while (q < L) {
        const int start = q;
        const uint64_t u = lane_take<SRC>(S, gam, nxt);
        ++q;
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
                const uint64_t u2 = lane_take<SRC>(S, gam, nxt);
                ++q;
                ok = wedge_accept_f(u2, x, p.yd + i, lds_f32x2(yf_sh + 8 * i));
                if (!ok && ++rej >= guard32) {
                    o.bad = 1;
                    break;
                }
            } else {
                double tr = p.r;
                int64_t tg = p.guard;
                asm volatile("ld.f64 %0, [%1];" : "=d"(tr) : "l"(&p.r));
                asm volatile("ld.s64 %0, [%1];" : "=l"(tg) : "l"(&p.guard));
                const TailOut to = tail_seq<SRC>(S, gam, tr, tg);
                S = to.st;
                lane_pend<SRC>(S, gam, nxt);
                x = to.v;
                ok = to.k >= 0;
                if (!ok) {
                    o.bad = 1;
                    break;
                }
                q += 2 * to.k;
            }
        }
        if (rec && start < 32) {
            o.sm0 |= 1u << start;
            if (ok) o.em0 |= 1u << start;
        }
        if (ok) {
            rej = 0;
            sv[cnt * vstride] = __longlong_as_double((long long)((uint64_t)__double_as_longlong(x) ^ sgn));
            se[(size_t)cnt * 32] = (uint32_t)q;
            ++cnt;
        }
    }
    o.cnt = cnt;
    o.exit = q;
    return o;
}

/* link the lanes of one warp: lane 0's true entry is ek0; every other lane's is its
   left neighbour's exit.  A lane whose decode has no attempt start at its true entry
   re-decodes from it (left to right).  Returns this lane's true entry. */
template <int SRC, int IBT, bool MOD>
__device__ __forceinline__ int lseg_link(LsegOut& o, int& e0, int ek0, int L, uint64_t S0, uint64_t gam, int64_t seg_base,
                                         const LaneParams& p, uint32_t kw_sh, uint32_t yf_sh, int ib, uint32_t imask,
                                         int mbits, uint64_t mmask, double* sv, int vstride, uint32_t* se, int lane)
{
    int ek = __shfl_up_sync(GZ_FULL, o.exit, 1) - L;
    if (lane == 0) ek = ek0;
    bool cov = lane == 0 || ek == e0 || (e0 == 0 && ek < 32 && ((o.sm0 >> ek) & 1u));
    uint32_t unc = __ballot_sync(GZ_FULL, !cov);
    while (unc) {
        const int ks = __ffs(unc) - 1;
        if (lane == ks) {
            e0 = ek;
            o = lseg_decode<SRC, IBT, MOD>(single_state_at<SRC>(S0, gam, (uint64_t)(seg_base + e0)), gam, e0, L, p,
                                           kw_sh, yf_sh, ib, imask, mbits, mmask, sv, vstride, se, lane);
        }
        const int ex = __shfl_up_sync(GZ_FULL, o.exit, 1) - L;
        if (lane > ks) ek = ex;
        cov = lane <= ks || ek == e0 || (e0 == 0 && ek < 32 && ((o.sm0 >> ek) & 1u));
        unc = __ballot_sync(GZ_FULL, !cov);
    }
    return ek;
}

constexpr int LSEG_MAXP = 8;

struct LsegShared {
    int exit31[LSEG_MAXP];      /* each warp's last segment exit */
    int total[LSEG_MAXP];       /* valid deviates per warp */
    int64_t woff[LSEG_MAXP];    /* row offset of each warp's first deviate (this round) */
    int64_t kept;               /* deviates kept this round */
};

template <int SRC, int IBT, bool MOD>
#ifndef LSEG_MINB1
#define LSEG_MINB1 3   /* blocks per SM the SplitMix64 form is compiled for */
#endif
__global__ void __launch_bounds__(32 * LSEG_MAXP, SRC == 1 ? LSEG_MINB1 : 2) k_zig_lseg(const __grid_constant__ LaneParams p, const LsegParams sp)
{
    extern __shared__ __align__(16) unsigned char smem[];
    const int nl = IBT ? (1 << IBT) : p.n_layers;
    ulonglong2* s_kw = reinterpret_cast<ulonglong2*>(smem);
    float2* s_yf = reinterpret_cast<float2*>(smem + 16 * nl);
    LsegShared& sh = *reinterpret_cast<LsegShared*>(smem + 24 * nl);
    /* deviates staged in shared memory, [value][segment] with a padded row: the decode
       writes a row per attempt, the copy reads a column per lane, both conflict-free */
    double* s_val = reinterpret_cast<double*>(smem + 24 * nl + ((sizeof(LsegShared) + 15) & ~(size_t)15));
    for (int i = threadIdx.x; i < nl; i += blockDim.x) {
        s_kw[i] = p.kw[i];
        s_yf[i] = p.yf[i];
    }
    __syncthreads();
    const int lane = threadIdx.x & 31;
    const int w = threadIdx.x >> 5;
    const int P = blockDim.x >> 5;
    const int g = threadIdx.x;               /* segment index within the round */
    const uint32_t kw_sh = sh_addr(s_kw), yf_sh = sh_addr(s_yf);
    const int ib = IBT ? IBT : p.index_bits;
    const uint32_t imask = (uint32_t)nl - 1u;
    const int mbits = 63 - ib;
    const uint64_t mmask = (1ULL << mbits) - 1ULL;
    const int64_t wg = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int vstride = 32 * P + 1;
    double* const sv = s_val + g;
    uint32_t* const se = sp.scr_e + (size_t)wg * sp.lcap * 32 + lane;

    for (int64_t sid = blockIdx.x; sid < p.n_streams; sid += gridDim.x) {
        uint64_t S0, gam = 0;
        if constexpr (SRC == 0) {
            S0 = p.state_in[sid];
        } else {
            S0 = p.state_in[2 * sid];
            gam = p.state_in[2 * sid + 1];
        }
        double* row = p.out + sid * p.ld;
        int64_t need = p.n_per, produced = 0, base = 0;
        int entry = 0;
        bool anomaly = sp.force_fallback != 0;
        while (need > 0 && !anomaly) {
            /* draws for `need` deviates with a 6-sigma margin, over 32P segments */
            const float fneed = (float)need;
            int L = (int)ceilf((fneed * sp.dpv + 6.0f * sqrtf(fneed * 0.06f) + 32.0f) / (float)(32 * P));
            L = max(16, min(L, sp.lcap));
            const int64_t seg_base = base + (int64_t)g * L;
            int e0 = g == 0 ? entry : sp.guess;
            LsegOut o = lseg_decode<SRC, IBT, MOD>(single_state_at<SRC>(S0, gam, (uint64_t)(seg_base + e0)), gam, e0, L, p,
                                                   kw_sh, yf_sh, ib, imask, mbits, mmask, sv, vstride, se, lane);
            /* lanes 1..31 of every warp; lane 0 provisionally at its own entry */
            int ek = lseg_link<SRC, IBT, MOD>(o, e0, e0, L, S0, gam, seg_base, p, kw_sh, yf_sh, ib, imask, mbits,
                                              mmask, sv, vstride, se, lane);
            if (lane == 31) sh.exit31[w] = o.exit;
            __syncthreads();
            /* links between warps, in order: warp v's lane 0 starts where warp v-1's lane 31
               ends; a warp whose lane-0 guess missed re-decodes it and relinks its lanes */
            if (w == 0 && lane == 0) ek = entry;
            for (int v = 1; v < P; ++v) {
                __syncthreads();
                if (w == v) {
                    const int e = sh.exit31[v - 1] - L;
                    const int e_own = __shfl_sync(GZ_FULL, e0, 0);
                    const uint32_t sm_own = __shfl_sync(GZ_FULL, o.sm0, 0);
                    const bool cov = e == e_own || (e_own == 0 && e < 32 && ((sm_own >> e) & 1u));
                    if (!cov) {
                        if (lane == 0) {
                            e0 = e;
                            o = lseg_decode<SRC, IBT, MOD>(single_state_at<SRC>(S0, gam, (uint64_t)(seg_base + e0)), gam,
                                                           e0, L, p, kw_sh, yf_sh, ib, imask, mbits, mmask, sv, vstride,
                                                           se, lane);
                        }
                        ek = lseg_link<SRC, IBT, MOD>(o, e0, e, L, S0, gam, seg_base, p, kw_sh, yf_sh, ib, imask, mbits,
                                                      mmask, sv, vstride, se, lane);
                        if (lane == 31) sh.exit31[w] = o.exit;
                    }
                    if (lane == 0) ek = e;
                }
            }
            const int skip = ek == e0 ? 0 : __popc(o.em0 & ((1u << ek) - 1u));
            const int valid = o.cnt - skip;
            if (__syncthreads_or(o.bad || valid <= 0)) {
                anomaly = true;
                break;
            }
            /* offsets: warp scan, then a prefix over the warps */
            int off = valid;
#pragma unroll
            for (int d = 1; d < 32; d <<= 1) {
                const int t = __shfl_up_sync(GZ_FULL, off, d);
                if (lane >= d) off += t;
            }
            if (lane == 31) sh.total[w] = off;
            off -= valid;
            __syncthreads();
            if (threadIdx.x == 0) {
                int64_t acc = 0;
                for (int v = 0; v < P; ++v) {
                    sh.woff[v] = acc;
                    acc += sh.total[v];
                }
                sh.kept = acc > need ? need : acc;   /* deviates kept this round */
            }
            __syncthreads();
            const int64_t goff = sh.woff[w] + off;
            const int64_t kept = sh.kept;
            const int64_t room = need - goff;
            const int take = room <= 0 ? 0 : (int)(room < valid ? room : valid);
            {
                /* the warp's segments are consecutive, so its deviates form one contiguous
                   run of the row: lane t of each pass finds its segment by a binary search
                   over the offsets and stores coalesced */
                const int wlen = (int)__reduce_add_sync(GZ_FULL, (unsigned)take);
                double* dst = row + produced + sh.woff[w];
                const double* wval = s_val + 32 * w;
                for (int t0 = 0; t0 < wlen; t0 += 32) {
                    const int t = t0 + lane;
                    int src = 0;
#pragma unroll
                    for (int step = 16; step > 0; step >>= 1) {
                        const int cand = src + step;
                        if (__shfl_sync(GZ_FULL, off, cand) <= t) src = cand;
                    }
                    const int o_s = __shfl_sync(GZ_FULL, off, src);
                    const int k_s = __shfl_sync(GZ_FULL, skip, src);
                    if (t < wlen) dst[t] = wval[(k_s + t - o_s) * vstride + src];
                }
            }
            if (kept == need) {
                if (take > 0 && goff + take == need) {
                    const uint32_t end = se[(size_t)(skip + take - 1) * 32];
                    const uint64_t s_end = single_state_at<SRC>(S0, gam, (uint64_t)(seg_base + end));
                    if constexpr (SRC == 0) {
                        p.state_out[sid] = s_end;
                    } else {
                        p.state_out[2 * sid] = s_end;
                        p.state_out[2 * sid + 1] = gam;
                    }
                }
                need = 0;
            } else {
                need -= kept;
                produced += kept;
                entry = sh.exit31[P - 1] - L;
                base += (int64_t)32 * P * L;
            }
            __syncthreads();
        }
        if (anomaly) {
            /* the exact sequential loop decides (and raises a guard trip) */
            if (w == 0) {
                ZigParams zp;
                zp.n_streams = p.n_streams; zp.n_per = p.n_per; zp.ld = p.ld;
                zp.state_in = p.state_in; zp.state_out = p.state_out; zp.out = p.out;
                zp.sigma = nullptr; zp.checksum = nullptr; zp.psum = nullptr;
                zp.kw = p.kw; zp.yd = p.yd; zp.n_layers = nl; zp.index_bits = ib; zp.r = p.r; zp.guard = p.guard;
                zp.generations = 1;
                const ZigLaneConsts kc = zig_lane_consts<SRC>(lane);
                zig_warp_stream<SRC, MOD, 4, EPI_STORE, false>(zp, sid, p.kw, p.yd, kc, lane);
            }
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
