/*
 * gz_k_lst.cuh -- k_zig_lst: the lane-per-stream ziggurat with lane-private
 * output staging and 256-bit row stores (configs 3 and 4: the auto choice for
 * >= 32768 streams with the standard 128/256-layer tables, 32-byte aligned
 * rows and a row stride that is a multiple of 4 deviates).
 *
 * Not a standalone header: included by gz_engine.cu inside its anonymous
 * namespace, after gz_k_tma.cuh (whose draw, split, recover and fold helpers
 * it uses).
 *
 * A lane owns one stream at a time and steps it exactly as the reference's
 * per-stream loop (engine.py:75-112 original, 114-151 modified ziggurat; the
 * attempt is ZigguratSampler._draw, samplers.py:95-115 / 144-165).  Rounds of
 * TMA_K attempts run without branches, as in k_zig_tma: every attempt's
 * deviate is written to the lane's next staging slot unconditionally, the
 * committed attempts are the leading fast accepts, and the first attempt that
 * is not a fast accept freezes the lane for the rest of the round; the frozen
 * lanes of a warp then resolve their wedge / tail attempts together (one pass
 * per round: recover the draw from the state, draw the wedge's uniform, float
 * pre-filter and the exact glibc exp near the boundary, or the tail loop).
 *
 * Output: each lane stages its row in a private 16-slot ring in shared memory
 * (128 bytes, the 16-byte chunks XOR-swizzled by lane & 7) and, after every
 * round, writes each complete 4-deviate chunk to its row with one 32-byte
 * store (STG.E.256: a full L2 sector).  Lanes never wait for each other: no
 * warp-wide flush, no ring-room stalls, so there is no cross-lane drift, and a
 * warp needs 4 KiB of shared memory instead of 16 KiB -- 20 warps per SM.
 * Rows of a lane follow each other (lane l of warp g takes the streams
 * (g + k * warps) * 32 + l); the next row's state is loaded when a row starts.
 *
 * Fused witnesses (STATS): the per-row xor checksum (bench.py:174-175) and
 * power sums (stats.py:232-259) are folded from each stored chunk in deviate
 * order -- the order of k_zig_tma and of the oracle's default digest.
 */
#pragma once

/* staging slots per lane (8 bytes each): a round writes TMA_K of them past <= 3 unstored */
__host__ __device__ constexpr int lst_slots(int k) { return k <= 12 ? 16 : 32; }
#ifndef LST_EXP
#define LST_EXP 0
#endif
#ifndef LST_CVT
#define LST_CVT 0
#endif

/* (double)m for m = mhi * 2^32 + mlo < 2^56, rounded to nearest even: the classic
   two-constant conversion -- (2^84 + mhi 2^32) - (2^84 + 2^52) is exact, and the
   final add of 2^52 + mlo rounds once -- so it equals __ull2double_rn(m) with two
   fixed-latency DADDs instead of the variable-latency I2F.F64.U64 */
__device__ __forceinline__ double lst_u56_to_f64(uint32_t mhi, uint32_t mlo)
{
    if constexpr (LST_CVT) {
        const double h = __hiloint2double(0x45300000, (int)mhi);
        const double l = __hiloint2double(0x43300000, (int)mlo);
        return __dadd_rn(__dsub_rn(h, 19342813118337666422669312.0 /* 2^84 + 2^52 */), l);
    } else {
        return __ull2double_rn(((uint64_t)mhi << 32) | mlo);
    }
}

template <int SRC, bool MOD, bool STATS, int NW, int TMA_K>
__global__ void __launch_bounds__(NW * 32, 1) k_zig_lst(const __grid_constant__ LaneParams p)
{
    constexpr int NL = MOD ? 256 : 128;
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    const uint32_t base_sh = sh_addr(smem_raw);
    constexpr int SL = lst_slots(TMA_K);
    constexpr uint32_t SMASK = (SL - 1) << 3;   /* slot bits of a byte offset */
    constexpr uint32_t RING = NW * 32 * SL * 8;
    ulonglong2* s_kw = reinterpret_cast<ulonglong2*>(smem_raw + RING);
    float2* s_yf = reinterpret_cast<float2*>(smem_raw + RING + NL * 16 * TMA_REP);
    ulonglong2* s_jump = reinterpret_cast<ulonglong2*>(smem_raw + RING + NL * 16 * TMA_REP + NL * 8);
    for (int j = threadIdx.x; j < NL * TMA_REP; j += blockDim.x) s_kw[j] = p.kw[j / TMA_REP];
    for (int j = threadIdx.x; j < NL; j += blockDim.x) s_yf[j] = p.yf[j];
    /* LCG: (A, C) of 2n steps, n <= TMA_K (the state after n draws from a round's start) */
    if (SRC == 0 && threadIdx.x <= TMA_K) s_jump[threadIdx.x] = make_ulonglong2(c_lcgA[2 * threadIdx.x], c_lcgC[2 * threadIdx.x]);
    __syncthreads();

    const int lane = threadIdx.x & 31;
    const int wib = threadIdx.x >> 5;
    const uint32_t lx = (uint32_t)(lane & 7) << 4;
    /* the lane's ring: 128-byte aligned, so slot s is at ((8 s) & 0x78) ^ rowx */
    const uint32_t rowx = (base_sh + (uint32_t)threadIdx.x * (SL * 8)) ^ lx;
    const uint32_t my_kw = base_sh + RING + lx;   /* replica lane & 7 of the layer rows */
    const uint32_t yf_sh = sh_addr(s_yf);
    const uint32_t jump_sh = sh_addr(s_jump);
    const uint64_t lcg_inc = SRC == 0 ? ld_keep(&c_lcgC[1]) : 0;
    const uint64_t lcg_inc2 = SRC == 0 ? ld_keep(&c_lcgC[2]) : 0;
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
    const int64_t g0 = (int64_t)blockIdx.x * NW + wib;
    const int ng = g0 < n_groups ? (int)((n_groups - g0 + gstride - 1) / gstride) : 0;

    /* the lane's rows: k = 0 .. ng-1, stream (g0 + k gstride) * 32 + lane (if < n_streams) */
    int k = -1;
    int64_t sid = 0;
    bool valid = false, failed = false;
    uint64_t S = 0, gam = lcg_inc;
    uint64_t S_next = 0, gam_next = lcg_inc;   /* the next row's state, loaded a row ahead */
    uint32_t C = 0;          /* deviates committed by this lane (all rows; slot = C mod 16) */
    uint32_t c_row0 = 0;     /* C at the start of the current row */
    uint32_t c_rowend = 0;   /* C at its end */
    uint32_t f = 0;          /* deviates stored */
    uint32_t rej = 0, c_rej = 0xffffffffu;
    double* rowp = nullptr;
    uint64_t ck = 0;
    double a1 = 0.0, a2 = 0.0, a3 = 0.0, a4 = 0.0;

    /* consecutive rows of a lane are sstride streams apart: stream, row and state
       pointers advance by constant strides (no 64-bit multiplies per row) */
    const int64_t sstride = gstride * 32;
    const int64_t last = n_streams - 1;
    sid = g0 * 32 + lane - sstride;
    double* rowp_next = p.out + (g0 * 32 + lane) * p.ld;
    const int64_t rstride = sstride * p.ld;
    /* the next row's state, loaded a row ahead (clamped to a valid stream, so the load is
       unconditional and lands in its own registers) */
    auto load_state = [&](int64_t q, uint64_t& s, uint64_t& g) {
        if (q > last) q = last;
        if constexpr (SRC == 0) {
            s = ld_keep(p.state_in + q);
        } else {
            s = ld_keep(p.state_in + 2 * q);
            g = ld_keep(p.state_in + 2 * q + 1);
        }
    };
    /* the row transition (divergent: once per row and lane): finish the row, start the next */
    auto next_row = [&]() {
        while (C >= c_rowend && k < ng) {
            if (valid && !failed) {
                if (n_per & 3) {
                    /* the row's last partial chunk */
                    for (; f < c_rowend; ++f) {
                        uint64_t v;
                        asm volatile("ld.shared.u64 %0, [%1];" : "=l"(v) : "r"(((f << 3) & SMASK) ^ rowx));
                        rowp[f - c_row0] = __longlong_as_double((long long)v);
                        if constexpr (STATS) tma_fold(v, ck, a1, a2, a3, a4);
                    }
                }
                /* its witnesses and its final state */
                if constexpr (STATS) {
                    if (p.checksum) p.checksum[sid] = ck;
                    if (p.psum) {
                        double* ps = p.psum + 4 * sid;   /* 16-byte aligned (lst_eligible) */
                        asm volatile("st.global.v2.f64 [%0], {%1, %2};" ::"l"(ps), "d"(a1), "d"(a2) : "memory");
                        asm volatile("st.global.v2.f64 [%0], {%1, %2};" ::"l"(ps + 2), "d"(a3), "d"(a4) : "memory");
                    }
                }
                if constexpr (SRC == 0) {
                    p.state_out[sid] = S & GZ_MASK48;
                } else {
                    asm volatile("st.global.v2.u64 [%0], {%1, %2};" ::"l"(p.state_out + 2 * sid), "l"(S), "l"(gam) : "memory");
                }
            }
            ++k;
            failed = false;
            if constexpr (STATS) {
                ck = 0;
                a1 = a2 = a3 = a4 = 0.0;
            }
            /* rows start on a chunk boundary */
            if (n_per & 3) C = (C + 3u) & ~3u;
            f = C;
            c_row0 = C;
            sid += sstride;
            rowp = rowp_next;
            rowp_next += rstride;
            valid = k < ng && sid < n_streams;
            S = S_next;
            gam = gam_next;
            load_state(sid + sstride, S_next, gam_next);
            c_rowend = valid ? C + (uint32_t)n_per : C;   /* no stream: skip the row */
        }
    };
    if (ng > 0) load_state(sid + sstride, S_next, gam_next);
    next_row();

    while (__any_sync(GZ_FULL, k < ng)) {
        /* ---- one round: TMA_K attempts per lane, no branches ---- */
        const bool act = C < c_rowend;
        const uint32_t C0 = C;
        /* LCG: CH independent draw chains (chain j starts 2 KC j steps ahead by one jump) */
        constexpr int CH = (SRC == 0 && TMA_K % TMA_CHV == 0) ? TMA_CHV : 1, KC = TMA_K / CH;
        TmaCursor<SRC> tcs[CH] = {TmaCursor<SRC>(S)};
#pragma unroll
        for (int j = 1; j < CH; ++j) tcs[j] = TmaCursor<SRC>(S * jA[j] + jC[j]);
        uint32_t fm = 0;
        /* the deviates are kept in registers and stored after the last attempt: a table
           gather may not pass a shared store in program order (ptxas cannot tell that
           they never alias), so storing inside the loop would serialise the attempts */
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
            const double x = __dmul_rn(lst_u56_to_f64(mhi, mlo), __longlong_as_double((long long)wb));
            if (m < kk) fm |= 1u << kk2;
            zbs[kk2] = (uint64_t)__double_as_longlong(x) ^ ((uint64_t)sgn << 32);
            GZ_CHECK(ioff < NL * 128u, ioff);
        }
        if (act) {
#pragma unroll
            for (int kk2 = 0; kk2 < TMA_K; ++kk2) {
                const uint32_t a = (((C0 + (uint32_t)kk2) << 3) & SMASK) ^ rowx;
                asm volatile("st.shared.u64 [%0], %1;" ::"r"(a), "l"(zbs[kk2]) : "memory");
            }
        }
        bool frozen = false;
        if (act) {
            const int lead = __ffs(~fm) - 1;   /* leading fast accepts */
            const uint32_t C_lead = C0 + (uint32_t)lead;
            C = min(C_lead, c_rowend);
            frozen = C_lead < c_rowend && lead < TMA_K;
        }
        /* the live attempts are a prefix of the round: the committed ones plus a frozen
           one; the state after them by jump-ahead from the round's start */
        {
            const uint32_t n_live = (C - C0) + (frozen ? 1u : 0u);
            GZ_CHECK(n_live <= (uint32_t)TMA_K, n_live);
            if constexpr (SRC == 0 && (LST_EXP & 4)) {
                S = tcs[CH - 1].state();   /* timing experiment: no jump (wrong results) */
            } else if constexpr (SRC == 0) {
                uint64_t ja, jc;
                lds_tab(jump_sh + 16 * n_live, ja, jc);
                S = S * ja + jc;
            } else {
                S += (uint64_t)n_live * gam;
            }
        }
        /* ---- the frozen lanes' slow attempts, resolved together ---- */
        /* LST_EXP (timing experiments only, wrong results): 1 no frozen pass, 2 no row stores, 3 neither */
        if ((LST_EXP & 1) == 0 && __any_sync(GZ_FULL, frozen)) {
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
                    /* wedge: the next draw is its uniform, whatever the outcome; an accepted
                       wedge's slot already holds x (written in the round) */
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
                    if (ok) {
                        const uint64_t zb = (uint64_t)__double_as_longlong(x) ^ sgn;
                        asm volatile("st.shared.u64 [%0], %1;" ::"r"(((C << 3) & SMASK) ^ rowx), "l"(zb) : "memory");
                    } else {
                        failed = true;
                        gz_raise(GZ_ERR_GUARD, sid);
                        C = c_rowend;
                    }
                }
                GZ_CHECK(i < (uint32_t)NL, i);
                if (ok) ++C;
            }
        }
        /* ---- complete 4-deviate chunks to the row: one 32-byte store each ---- */
        auto store_chunk = [&]() {
            const uint32_t a = ((f << 3) & SMASK) ^ rowx;   /* slots f .. f+3: two 16-byte chunks */
            uint64_t v0, v1, v2, v3;
            lds_u64x2_v(a, v0, v1);
            lds_u64x2_v(a ^ 0x10u, v2, v3);
            double* dst = rowp + (f - c_row0);
            if ((LST_EXP & 2) == 0 || (v0 ^ v1 ^ v2 ^ v3) == 0x123456789ULL)
                asm volatile("st.global.v4.b64 [%0], {%1, %2, %3, %4};" ::"l"(dst), "l"(v0), "l"(v1), "l"(v2), "l"(v3)
                             : "memory");
            if constexpr (STATS) {
                ck ^= v0 ^ v1 ^ v2 ^ v3;
                tma_fold_fp(v0, a1, a2, a3, a4);
                tma_fold_fp(v1, a1, a2, a3, a4);
                tma_fold_fp(v2, a1, a2, a3, a4);
                tma_fold_fp(v3, a1, a2, a3, a4);
            }
            f += 4u;
        };
        if (!failed) {
            while (C - f >= 4u) store_chunk();
        }
        if (C >= c_rowend) next_row();
    }
}
