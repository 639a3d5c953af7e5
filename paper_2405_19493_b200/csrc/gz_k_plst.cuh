/*
 * gz_k_plst.cuh -- k_polar_lst: the polar method, one lane per stream, with the
 * k_zig_lst output path (config 2: the auto choice for >= 32768 polar streams
 * without fused witnesses, 32-byte aligned rows and a row stride that is a
 * multiple of 4 deviates).
 *
 * Not a standalone header: included by gz_engine.cu inside its anonymous
 * namespace, after gz_k_polar.cuh and gz_k_lst.cuh (whose divide / sqrt, shared
 * memory and staging helpers it uses).
 *
 * A lane owns one stream at a time and steps it exactly as the reference
 * (PolarSampler.next_gaussian, samplers.py:168-192; engine.py:154-196): an attempt
 * always consumes two draws, v = 2 u - 1 (exact), s = v1 v1 + v2 v2 (two products
 * and a sum, each rounded), accepted when 0 < s < 1, and an accepted attempt emits
 * v1 * mul and then its spare v2 * mul, mul = sqrt(-2 log(s) / s) with glibc's log
 * and correctly rounded divide and square root.  Because every attempt consumes
 * exactly two draws there is nothing to freeze: a round of K attempts runs with no
 * branch, every attempt is transformed by glibc log's table path, and its two
 * outputs are staged at the next free pair of slots (a rejected attempt's outputs
 * land where the next accepted attempt's go and are overwritten).  The rare
 * accepted attempts with s in glibc's near-1 interval [1 - 2^-4, 1) (6.25 % of
 * them) join a per-warp queue (ballot rank) and are recomputed by the whole warp
 * with the degree-11 branch after the round, written over their staged outputs.
 *
 * Rows: a row that starts with a cached spare stages it first; the attempt that
 * completes a row ends the lane's live attempts (the state is one jump-ahead from
 * the round's start), and when the row is one deviate short of a pair the pair's
 * second output becomes the row's spare.  Guards count consecutive rejections
 * (each accept resets: the reference's guard is per next_gaussian call).
 * Output: slot-major staging and 32-byte row stores exactly as k_zig_lst.
 */
#pragma once

constexpr uint64_t PLST_NEAR1 = 0x3fee000000000000ULL;   /* glibc log's near-1 interval starts at 1 - 2^-4 */

/* bytes of dynamic shared memory: the log table, the jump table, per warp the staging
   (16 slots x 32 lanes x 8 B) and a near-1 queue of 32 K entries x 32 B */
__host__ __device__ constexpr uint32_t plst_smem_bytes(int NW, int K)
{
    return 2048u + 16u * (uint32_t)(K + 1) + (uint32_t)NW * (LST_RING + 32u * 32u * (uint32_t)K + 32u * 16u) + 1024u;
}

/* one u64 of the stream from the draw cursor (LCG48 in the shifted domain of k_zig_lst,
   T = state << 16: bits 16..47 of a step are T's high word; two steps, the second
   straight from the cursor by (A^2, AC + C); SplitMix64: t += gamma, mix64) */
template <int SRC>
__device__ __forceinline__ uint64_t plst_draw(uint32_t& sl, uint32_t& sh, uint64_t gam, uint64_t inc1, uint64_t inc2)
{
    if constexpr (SRC == 0) {
        uint32_t t1l, t1h;
        lcg_step32(sl, sh, t1l, t1h, inc1);
        uint32_t t2l, t2h;
        lcg_step32x2(sl, sh, t2l, t2h, inc2);
        sl = t2l;
        sh = t2h;
        return ((uint64_t)t1h << 32) | t2h;
    } else {
        const uint64_t t = (((uint64_t)sh << 32) | sl) + gam;
        sl = (uint32_t)t;
        sh = (uint32_t)(t >> 32);
        return gz_mix64(t);
    }
}

/* v = 2 next_f64_unit() - 1 = (u >> 11) 2^-52 - 1, exact (samplers.py:185-186), computed as
   (u & ~2047) 2^-63 - 1: the same 53-bit integer scaled, one mask instead of a 64-bit shift */
__device__ __forceinline__ double plst_pm1(uint64_t u)
{
    return __fma_rn(__ull2double_rn(u & ~2047ULL), 0x1p-63, -1.0);
}

template <int SRC, int NW, int K>
__global__ void __launch_bounds__(NW * 32, 1) k_polar_lst(const __grid_constant__ LaneParams p)
{
    static_assert(2 * K + 3 <= LST_SLOTS, "a round's outputs and the unstored deviates share the staging slots");
    constexpr uint32_t QB = 32u * 32u * K;   /* near-1 queue bytes per warp: every attempt of a round */
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    uint64_t* s_log = reinterpret_cast<uint64_t*>(smem_raw);
    const uint32_t base = sh_addr(smem_raw);
    const uint32_t jump_sh = base + 2048u;
    const uint32_t warps_sh = (jump_sh + 16u * (K + 1) + 1023u) & ~1023u;
    for (int j = threadIdx.x; j < 256; j += blockDim.x) s_log[j] = g_log_tab[j];
    /* LCG: (A, C) of 4n steps, n <= K (the state after n attempts from a round's start) */
    if (SRC == 0 && threadIdx.x <= K)
        asm volatile("st.shared.v2.u64 [%0], {%1, %2};" ::"r"(jump_sh + 16 * threadIdx.x), "l"(c_lcgA[4 * threadIdx.x]),
                     "l"(c_lcgC[4 * threadIdx.x] << 16)
                     : "memory");
    __syncthreads();

    const int lane = threadIdx.x & 31;
    const uint32_t lt = (1u << lane) - 1u;
    const uint32_t wib = threadIdx.x >> 5;
    const uint32_t wsh = warps_sh + wib * (LST_RING + QB);
    const uint32_t ringl = wsh + (uint32_t)lane * 8;   /* staging slot s of this lane at ringl + 256 s */
    const uint32_t q_sh = wsh + LST_RING;             /* near-1 queue: {v1, v2, s, staging address} */
    const uint32_t stslot = warps_sh + NW * (LST_RING + QB) + (uint32_t)threadIdx.x * 16u;   /* next row's state */
    const uint64_t inc1 = SRC == 0 ? ld_keep(&c_lcgC[1]) << 16 : 0, inc2 = SRC == 0 ? ld_keep(&c_lcgC[2]) << 16 : 0;
    const int n_per = p.n_per;
    const uint32_t guard32 = p.guard > 0xffffffffll ? 0xffffffffu : (uint32_t)p.guard;
    const uint32_t n_streams = (uint32_t)p.n_streams;   /* < 2^31 (plst_eligible) */
    const uint32_t n_groups = (uint32_t)(((int64_t)p.n_streams + 31) >> 5);
    const uint32_t gstride = gridDim.x * NW;
    const uint32_t g0 = blockIdx.x + wib * gridDim.x;   /* round-robin over the blocks */
    const int ng = g0 < n_groups ? (int)((n_groups - g0 + gstride - 1) / gstride) : 0;

    int k = -1;
    bool valid = false, failed = false;
    uint64_t S = 0, gam = 0;
    uint32_t C = 0, c_row0 = 0, c_rowend = 0, f = 0;
    uint32_t rej = 0;
    int has = 0;          /* the finished row left a spare */
    double spare = 0.0;
    const uint32_t sstride = gstride * 32;
    const uint32_t last = n_streams - 1;
    uint32_t sid = g0 * 32 + (uint32_t)lane - sstride;
    const int64_t rstride = (int64_t)sstride * p.ld;
    double* rowp = p.out + (int64_t)(g0 * 32 + (uint32_t)lane) * p.ld - rstride;
    /* the next row's state, copied global -> shared by cp.async (as k_zig_lst) */
    auto prefetch_state = [&](uint32_t q) {
        q = min(q, last);
        if constexpr (SRC == 0) {
            lst_cp8(stslot, p.state_in + q);
        } else {
            lst_cp8(stslot, p.state_in + 2 * (int64_t)q);
            lst_cp8(stslot + 8, p.state_in + 2 * (int64_t)q + 1);
        }
        asm volatile("cp.async.commit_group;" ::: "memory");
    };
    auto take_state = [&](uint64_t& s, uint64_t& g) {
        asm volatile("cp.async.wait_group 0;" ::: "memory");
        s = lds_u64(stslot);
        if constexpr (SRC == 0) s <<= 16;   /* the shifted domain */
        if constexpr (SRC == 1) g = lds_u64(stslot + 8);
    };
    /* the row transition (divergent: once per row and lane) */
    auto next_row = [&]() {
        if (valid) {
            if (failed) {
                gz_raise(GZ_ERR_GUARD, sid);
            } else {
                /* the row's last partial chunk (slots 0 .. c_rowend - f - 1) */
                for (uint32_t q = 0; q < c_rowend - f; ++q) rowp[f + q - c_row0] = __longlong_as_double((long long)lds_u64(ringl + 256 * q));
                if constexpr (SRC == 0) {
                    p.state_out[sid] = S >> 16;
                } else {
                    asm volatile("st.global.v2.u64 [%0], {%1, %2};" ::"l"(p.state_out + 2 * (int64_t)sid), "l"(S), "l"(gam)
                                 : "memory");
                }
                if (p.spare_out) p.spare_out[sid] = has ? spare : 0.0;
                if (p.has_out) p.has_out[sid] = (uint8_t)has;
            }
        }
        ++k;
        failed = false;
        has = 0;
        rej = 0;
        /* rows start on a chunk boundary, with nothing unstored */
        C = (C + 3u) & ~3u;
        f = C;
        c_row0 = C;
        sid += sstride;
        rowp += rstride;
        valid = k < ng && sid < n_streams;
        take_state(S, gam);
        prefetch_state(sid + sstride);
        c_rowend = valid ? C + (uint32_t)n_per : C;
        if (valid && n_per > 0 && p.has_in && p.has_in[sid]) {
            /* the cached deviate comes first (samplers.py:182-184) */
            sts_u64(ringl, (uint64_t)__double_as_longlong(p.spare_in[sid]));
            C += 1;
        }
    };
    if (ng > 0) prefetch_state(sid + sstride);
    next_row();

    while (__any_sync(GZ_FULL, k < ng)) {
        /* ---- one round: K attempts per lane, no branches ---- */
        const bool act = C < c_rowend;
        const uint32_t C0 = C;
        GZ_CHECK(C0 - f <= 3u, C0 - f);   /* the unstored deviates sit at slots 0..2 */
        const uint32_t wb = ringl + (C0 - f) * 256;   /* slot of deviate C0 */
        uint32_t sl = (uint32_t)S, sh = (uint32_t)(S >> 32);
        uint32_t am = 0, cnt = 0, qn = 0;
#pragma unroll
        for (int j = 0; j < K; ++j) {
            const double v1 = plst_pm1(plst_draw<SRC>(sl, sh, gam, inc1, inc2));
            const double v2 = plst_pm1(plst_draw<SRC>(sl, sh, gam, inc1, inc2));
            const double s = __dadd_rn(__dmul_rn(v1, v1), __dmul_rn(v2, v2));
            const uint64_t sb = (uint64_t)__double_as_longlong(s);
            const bool acc = s > 0.0 && s < 1.0;
            /* glibc log's table path for every attempt (samplers.py:189) */
            const double mul = sqrt_rn_nb(div_rn_nb(__dmul_rn(-2.0, gz_log_core(sb, s_log)), s));
            const uint32_t a = wb + cnt * 512u;
            if (act) {
                sts_u64(a, (uint64_t)__double_as_longlong(__dmul_rn(v1, mul)));
                sts_u64(a + 256, (uint64_t)__double_as_longlong(__dmul_rn(v2, mul)));
            }
            /* near-1 accepted attempts: queued for the exact branch */
            const bool nr = act && acc && sb >= PLST_NEAR1;
            const uint32_t mn = __ballot_sync(GZ_FULL, nr);
            if (nr) {
                const uint32_t e = q_sh + (qn + __popc(mn & lt)) * 32u;
                asm volatile("st.shared.v2.f64 [%0], {%1, %2};" ::"r"(e), "d"(v1), "d"(v2) : "memory");
                asm volatile("st.shared.v2.u64 [%0], {%1, %2};" ::"r"(e + 16), "l"(sb), "l"((uint64_t)a) : "memory");
            }
            qn += __popc(mn);
            am |= (acc ? 1u : 0u) << j;
            cnt += acc ? 1u : 0u;
        }
        /* ---- the live attempts and the row's progress ---- */
        uint32_t n_live = K;
        bool row_spare = false;
        if (act) {
            const uint32_t need = (c_rowend - C0 + 1) >> 1;   /* pairs that complete the row */
            if (cnt >= need) {
                /* the row completes at the need-th accepted attempt */
                uint32_t m = am;
                for (uint32_t i = 1; i < need; ++i) m &= m - 1;
                n_live = (uint32_t)__ffs(m);
                row_spare = ((c_rowend - C0) & 1u) != 0;
                C = c_rowend;
            } else {
                C = C0 + 2 * cnt;
            }
            /* consecutive rejections over the live attempts (each accept resets) */
            const uint32_t lm = am & ((2u << (n_live - 1)) - 1u);
            const uint32_t lead = lm ? (uint32_t)__ffs(lm) - 1 : n_live;
            bool trip = rej + lead >= guard32;
            if (guard32 <= (uint32_t)K && !trip && lm) {
                /* a run between two accepts can trip a small guard */
                uint32_t run = 0;
                for (uint32_t i = 0; i < n_live; ++i) {
                    run = ((lm >> i) & 1u) ? 0 : run + 1;
                    trip |= run >= guard32;
                }
            }
            rej = lm ? n_live - (32u - (uint32_t)__clz(lm)) : rej + n_live;
            if (trip) {
                failed = true;
                C = c_rowend;
                row_spare = false;
            }
        } else {
            n_live = 0;
        }
        if constexpr (SRC == 0) {
            uint64_t ja, jc;
            lds_tab(jump_sh + 16 * n_live, ja, jc);
            S = S * ja + jc;
        } else {
            S += (uint64_t)(2 * n_live) * gam;
        }
        /* ---- near-1 attempts of the round, by the whole warp (glibc's degree-11 branch) ---- */
        if (qn != 0) {
            __syncwarp();
            for (uint32_t e0 = 0; e0 < qn; e0 += 32) {
                if (e0 + (uint32_t)lane < qn) {
                    const uint32_t e = q_sh + (e0 + (uint32_t)lane) * 32u;
                    double v1, v2;
                    uint64_t sb, a;
                    asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(v1), "=d"(v2) : "r"(e));
                    asm volatile("ld.shared.v2.u64 {%0, %1}, [%2];" : "=l"(sb), "=l"(a) : "r"(e + 16));
                    const double s = __longlong_as_double((long long)sb);
                    const double mul = sqrt_rn_nb(div_rn_nb(__dmul_rn(-2.0, gz_log_t(s, s_log)), s));
                    sts_u64((uint32_t)a, (uint64_t)__double_as_longlong(__dmul_rn(v1, mul)));
                    sts_u64((uint32_t)a + 256, (uint64_t)__double_as_longlong(__dmul_rn(v2, mul)));
                }
            }
            __syncwarp();
        }
        /* the completed row's spare: the second output of its last pair */
        GZ_CHECK(qn <= 32u * K, qn);
        if (row_spare) {
            GZ_CHECK(c_rowend - f < (uint32_t)LST_SLOTS, c_rowend - f);
            has = 1;
            spare = __longlong_as_double((long long)lds_u64(ringl + (c_rowend - f) * 256));
        }
        /* ---- complete 4-deviate chunks to the row (slots 0, 4, 8, 12) ---- */
        if (!failed) {
            const uint32_t pend = C - f;   /* <= 2 K + 3 */
            GZ_CHECK(pend <= 2u * K + 3u, pend);
            double* dst = rowp + (f - c_row0);
            uint32_t nst = 0;
#pragma unroll
            for (int q = 0; q < (2 * K + 3) / 4; ++q) {
                if (pend >= 4u * (q + 1)) {
                    const uint32_t ph = ringl + 1024u * q;
                    const uint64_t v0 = lds_u64(ph), v1 = lds_u64(ph + 256), v2 = lds_u64(ph + 512), v3 = lds_u64(ph + 768);
                    asm volatile("st.global.v4.b64 [%0], {%1, %2, %3, %4};" ::"l"(dst + 4 * q), "l"(v0), "l"(v1), "l"(v2),
                                 "l"(v3)
                                 : "memory");
                    nst = q + 1;
                }
            }
            if (nst != 0) {
                const uint32_t ph = ringl + 1024u * nst;
                const uint64_t w0 = lds_u64(ph), w1 = lds_u64(ph + 256), w2 = lds_u64(ph + 512);
                sts_u64(ringl, w0);
                sts_u64(ringl + 256, w1);
                sts_u64(ringl + 512, w2);
                f += 4u * nst;
            }
        }
        if (C >= c_rowend && k < ng) next_row();
    }
}
