/*
 * gz_k_seg.cuh -- the ziggurats over FEW long streams: G warps per stream
 * (included by gz_engine.cu after gz_single.cuh).
 *
 * With fewer streams than the GPU holds warps (config 1: 1024 streams), a warp per
 * stream leaves most of the machine idle and every warp walks its whole row.  Here
 * a block of G warps owns one stream.  Per round, the row's next draws are cut into
 * G segments of L draws; warp k decodes segment k with the warp-per-stream window
 * (zig_window) from a GUESSED entry -- warp 0 from the known one, the others from
 * the segment's first draw -- into a scratch buffer (values and each value's
 * attempt end).  An attempt that starts in segment k-1 may overhang into segment k
 * (wedge: 2 draws, tail: 1 + 2t), so the true entry e of segment k is the exit of
 * segment k-1.  Decoding is deterministic from an attempt start, so if the guessed
 * decode has an attempt start at e, both decodes agree from there on: its values
 * from e are the true ones and its exit is the true exit.  Almost always the guess
 * synchronises within a few draws (a fast-path attempt consumes exactly one draw);
 * when it does not, the warp re-decodes from e.  Thread 0 links the segments in
 * order, the warps copy their values to the row at their prefix offsets, and the
 * final state is the stream state after the last stored deviate's attempt.
 *
 * Same draws, same decisions, same order as the sequential loop.  Guard: used only
 * when the guard exceeds any rejection run two segments can hold; a segment with no
 * deviate after its entry, or a tail that exhausts its guard, hands the whole stream
 * to the exact warp-per-stream loop (zig_warp_stream) in the same block.
 */
#pragma once

constexpr int SEG_MAXG = 5;   /* block <= 160 threads */
#ifndef SEG_MINB
#define SEG_MINB 4   /* __launch_bounds__(160, 4): at most 96 registers (5 -> 72 with spills: slower) */
#endif

struct SegOut {
    int cnt;        /* deviates emitted by attempts starting in [entry, L) */
    int exit;       /* the first attempt start >= L (segment-relative) */
    uint32_t sm0;   /* decodes from entry 0: attempt starts among positions 0..31 */
    uint32_t em0;   /* ... and those of them that emitted a deviate */
    int bad;        /* a tail exhausted its guard / the rejection run reached it */
    int entry;      /* the entry this decode started from */
};

struct SegShared {
    SegOut so[SEG_MAXG];
    int skip[SEG_MAXG], take[SEG_MAXG];
    int64_t off[SEG_MAXG];
    int redo, redo_entry, anomaly, e_after, final_k, got;
};

struct SegParams {
    double* scr_v;      /* [grid][G][lcap] deviates */
    uint32_t* scr_e;    /* [grid][G][lcap] attempt ends (segment-relative) */
    int lcap;           /* segment length cap (draws) */
    float dpv;          /* draws per deviate used to size a round (with a margin) */
    int guess;          /* entry guessed by warps 1..G-1 (0; tests use 1 to force re-decodes) */
    int force_fallback; /* tests: every stream through zig_warp_stream */
};

/* decode one segment: attempts starting at segment positions [entry, L); S is the
   stream state before the draw at position `entry` */
template <int SRC, bool MOD, int D>
__device__ __forceinline__ SegOut zig_seg_decode(uint64_t S, uint64_t gam, int entry, int L, const ZigParams& p,
                                                 const ulonglong2* s_kw, const double2* s_yd,
                                                 const ZigLaneConsts& kc, double* vb, uint32_t* ve, int lane)
{
    constexpr int W = 32 * D;
    const uint32_t lt = (1u << lane) - 1u;
    const int ib = p.index_bits;
    const uint32_t imask = (uint32_t)p.n_layers - 1u;
    const int mbits = 63 - ib;
    const uint64_t mmask = (1ULL << mbits) - 1ULL;
    const double r = p.r;
    uint64_t gl = 0, g32 = 0;
    if constexpr (SRC == 1) {
        gl = (uint64_t)(lane + 1) * gam;
        g32 = gam << 5;
    }
    SegOut o;
    o.cnt = 0; o.exit = entry; o.sm0 = 0; o.em0 = 0; o.bad = 0; o.entry = entry;
    int q0 = entry;        /* segment position of the window's first draw (an attempt start) */
    int cnt = 0;
    int64_t rej_run = 0;
    bool first = entry == 0;
    while (q0 < L) {
        ZigWindow<D> w;
        zig_window<SRC, MOD, D>(w, S, gam, gl, g32, kc, s_kw, s_yd, ib, imask, mbits, mmask, lane);
        const int lim = L - q0;    /* window positions >= lim start no attempt of this segment */
        int q = 0, c = 0, ext_lane = 0, ext_kind = 0;
        bool stop = false;
        uint64_t ext_t = 0;
        uint32_t em[D], sm_first = 0;
        int ebase[D], tlen[D];
#pragma unroll
        for (int d = 0; d < D; ++d) {
            em[d] = 0;
            ebase[d] = c;
            tlen[d] = 0;
            if (stop || q >= 32 * (d + 1)) continue;
            int b = q - 32 * d;
            const int limd = lim - 32 * d;   /* > b */
            const uint32_t nfd = w.nf[d];
            while (true) {
                const uint32_t pend = nfd & (GZ_FULL << b);
                const int f = pend ? (__ffs(pend) - 1) : 32;
                if (limd <= f) {
                    /* the fast run reaches the segment end: its last attempt starts at lim - 1 */
                    em[d] |= gz_bitrange(b, limd - b);
                    if (first && d == 0) sm_first |= gz_bitrange(b, limd - b);
                    c += limd - b;
                    rej_run = 0;
                    q = lim;
                    stop = true;
                    break;
                }
                em[d] |= gz_bitrange(b, f - b);
                if (first && d == 0) sm_first |= gz_bitrange(b, f - b);
                c += f - b;
                if (f > b) rej_run = 0;
                if (f == 32) {
                    q = 32 * (d + 1);
                    break;
                }
                const int pos = 32 * d + f;
                if (first && d == 0) sm_first |= 1u << f;
                if ((w.tl[d] >> f) & 1u) {
                    int tt = 0;
                    if (lane == f) {
                        const TailOut to = tail_seq<SRC>(w.st[d], gam, r, p.guard);
                        tt = to.k;
                        ext_t = to.st;
                        w.val[d] = signbit(w.val[d]) ? -to.v : to.v;
                        tlen[d] = 1 + 2 * to.k;
                    }
                    tt = __shfl_sync(GZ_FULL, tt, f);
                    if (tt < 0) {
                        o.bad = 1;
                        stop = true;
                        break;
                    }
                    em[d] |= 1u << f;
                    ++c;
                    rej_run = 0;
                    q = pos + 1 + 2 * tt;
                    ext_kind = 1;
                    ext_lane = f;
                } else {
                    if ((w.am[d] >> f) & 1u) {
                        em[d] |= 1u << f;
                        ++c;
                        rej_run = 0;
                    } else if (++rej_run >= p.guard) {
                        o.bad = 1;
                        stop = true;
                        break;
                    }
                    q = pos + 2;
                    ext_kind = 2;
                }
                if (q >= lim) {
                    stop = true;
                    break;
                }
                if (q >= 32 * (d + 1)) break;
                b = q - 32 * d;
            }
        }
        if (o.bad) break;
        /* ---- emit into the scratch row: deviate and its attempt's end position ---- */
#pragma unroll
        for (int d = 0; d < D; ++d) {
            if ((em[d] >> lane) & 1u) {
                const int rel = cnt + ebase[d] + __popc(em[d] & lt);
                vb[rel] = w.val[d];
                const uint32_t nfb = (w.nf[d] >> lane) & 1u, tlb = (w.tl[d] >> lane) & 1u;
                const int len = nfb ? (tlb ? tlen[d] : 2) : 1;
                ve[rel] = (uint32_t)(q0 + 32 * d + lane + len);
            }
        }
        if (first) {
            o.sm0 = sm_first;
            o.em0 = em[0];
            first = false;
        }
        cnt += c;
        /* ---- advance past the consumed draws ---- */
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
        q0 += q;
        if (stop) break;
    }
    o.cnt = cnt;
    o.exit = q0;
    return o;
}

template <int SRC, bool MOD, int D>
__global__ void __launch_bounds__(32 * SEG_MAXG, SEG_MINB) k_zig_seg(const ZigParams p, const SegParams sp)
{
    extern __shared__ __align__(16) unsigned char smem[];
    const int nl = p.n_layers;
    ulonglong2* s_kw = reinterpret_cast<ulonglong2*>(smem);
    double2* s_yd = reinterpret_cast<double2*>(smem + 16 * nl);
    SegShared& sh = *reinterpret_cast<SegShared*>(smem + 32 * nl);
    for (int i = threadIdx.x; i < nl; i += blockDim.x) {
        s_kw[i] = p.kw[i];
        s_yd[i] = p.yd[i];
    }
    __syncthreads();
    const int G = (int)(blockDim.x >> 5);
    const int k = (int)(threadIdx.x >> 5);
    const int lane = threadIdx.x & 31;
    const ZigLaneConsts kc = zig_lane_consts<SRC>(lane);
    double* vb = sp.scr_v + ((int64_t)blockIdx.x * G + k) * sp.lcap;
    uint32_t* ve = sp.scr_e + ((int64_t)blockIdx.x * G + k) * sp.lcap;

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
            const int Lr = min(sp.lcap, (int)ceilf((float)need * sp.dpv / (float)G) + 32);
            {
                const int e0 = k == 0 ? entry : sp.guess;
                const SegOut o = zig_seg_decode<SRC, MOD, D>(single_state_at<SRC>(S0, gam, (uint64_t)(base + (int64_t)k * Lr + e0)),
                                                             gam, e0, Lr, p, s_kw, s_yd, kc, vb, ve, lane);
                if (lane == 0) sh.so[k] = o;
            }
            __syncthreads();
            /* link the segments in order; re-decode a segment whose guess did not synchronise */
            int from = 0, e = entry;
            while (true) {
                if (threadIdx.x == 0) {
                    sh.redo = -1;
                    sh.anomaly = 0;
                    for (int j = from; j < G; ++j) {
                        const SegOut& oj = sh.so[j];
                        int skip;
                        if (oj.entry == e) {
                            skip = 0;
                        } else if (oj.entry == 0 && e < 32 && ((oj.sm0 >> e) & 1u)) {
                            skip = __popc(oj.em0 & ((1u << e) - 1u));
                        } else {
                            sh.redo = j;
                            sh.redo_entry = e;
                            break;
                        }
                        if (oj.bad || oj.cnt - skip <= 0) {
                            sh.anomaly = 1;
                            break;
                        }
                        sh.skip[j] = skip;
                        e = oj.exit - Lr;
                    }
                    sh.e_after = e;
                }
                __syncthreads();
                if (sh.anomaly || sh.redo < 0) break;
                from = sh.redo;
                e = sh.redo_entry;
                if (k == from) {
                    const SegOut o = zig_seg_decode<SRC, MOD, D>(single_state_at<SRC>(S0, gam, (uint64_t)(base + (int64_t)k * Lr + e)),
                                                                 gam, e, Lr, p, s_kw, s_yd, kc, vb, ve, lane);
                    if (lane == 0) sh.so[k] = o;
                }
                __syncthreads();
            }
            if (sh.anomaly) {
                anomaly = true;
                break;
            }
            /* offsets and counts; the round that completes the row finds the last attempt */
            if (threadIdx.x == 0) {
                int64_t off = produced, left = need;
                sh.final_k = -1;
                for (int j = 0; j < G; ++j) {
                    const int valid = sh.so[j].cnt - sh.skip[j];
                    const int take = left <= 0 ? 0 : (int)(left < (int64_t)valid ? left : (int64_t)valid);
                    sh.take[j] = take;
                    sh.off[j] = off;
                    off += take;
                    left -= take;
                    if (left == 0 && take > 0 && sh.final_k < 0) sh.final_k = j;
                }
                sh.got = (int)(need - left);
            }
            __syncthreads();
            {
                /* scratch (L2) -> row: eight loads in flight per lane before the stores */
                const int take = sh.take[k], skip = sh.skip[k];
                double* dst = row + sh.off[k];
                const double* src = vb + skip;
                for (int i0 = 0; i0 < take; i0 += 256) {
                    double v[8];
#pragma unroll
                    for (int u = 0; u < 8; ++u) {
                        const int i = i0 + 32 * u + lane;
                        v[u] = i < take ? __ldcg(src + i) : 0.0;
                    }
#pragma unroll
                    for (int u = 0; u < 8; ++u) {
                        const int i = i0 + 32 * u + lane;
                        if (i < take) dst[i] = v[u];
                    }
                }
            }
            const int got = sh.got;
            if (need - got == 0 && k == sh.final_k && lane == 0) {
                const uint32_t end = ve[sh.skip[k] + sh.take[k] - 1];
                const uint64_t s_end = single_state_at<SRC>(S0, gam, (uint64_t)(base + (int64_t)k * Lr + end));
                if constexpr (SRC == 0) {
                    p.state_out[sid] = s_end;
                } else {
                    p.state_out[2 * sid] = s_end;
                    p.state_out[2 * sid + 1] = gam;
                }
            }
            need -= got;
            produced += got;
            base += (int64_t)G * Lr;
            entry = sh.e_after;
            __syncthreads();
        }
        if (anomaly) {
            /* the exact sequential loop decides (and raises a guard trip) */
            if (k == 0) zig_warp_stream<SRC, MOD, D, EPI_STORE, false>(p, sid, s_kw, s_yd, kc, lane);
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
