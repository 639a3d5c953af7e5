/*
 * gz_k_lst.cuh -- k_zig_lst: the lane-per-stream ziggurat with lane-private
 * output staging and 256-bit row stores (configs 3 and 4: the auto choice for
 * >= 32768 streams with the standard 128/256-layer tables, 32-byte aligned
 * rows and a row stride that is a multiple of 4 deviates).
 *
 * Not a standalone header: included by gz_engine.cu inside its anonymous
 * namespace, after gz_k_tma.cuh (whose recover and fold helpers it uses).
 *
 * A lane owns one stream at a time and steps it exactly as the reference's
 * per-stream loop (engine.py:75-112 original, 114-151 modified ziggurat; the
 * attempt is ZigguratSampler._draw, samplers.py:95-115 / 144-165).  Rounds of
 * K attempts run without branches: every attempt's deviate is staged
 * unconditionally, the committed attempts are the leading fast accepts, and
 * the first attempt that is not a fast accept freezes the lane for the rest of
 * the round; the frozen lanes of a warp then resolve their wedge / tail
 * attempts together (one pass per round: the staged x, the recovered layer,
 * the wedge's uniform, float pre-filter and the exact glibc exp near the
 * boundary, or the tail loop).
 *
 * Shared memory, laid out for the bank structure (all addresses are 32-bit
 * shared-window offsets computed once):
 *  - layer rows: a 64 KiB-aligned table of 256 entries x 256 bytes, entry e =
 *    layer e mod n (the original ziggurat indexes it with the draw's top byte,
 *    sign included: entries e and e + 128 hold the same layer), 8 replicas of
 *    the 16-byte row {ktab, bits(wtab)} per entry, lane & 7 reading its own.
 *    The gather address is ONE byte permute: the draw's index byte dropped into
 *    byte 1 of (table base | replica offset).
 *  - staging: per warp 16 slots x 32 lanes x 8 bytes, slot-major (slot s of lane
 *    l at s * 256 + l * 8), so every lane owns one bank pair and the per-slot
 *    stores and chunk loads of a half-warp never conflict whatever the lanes'
 *    positions.  The slots are a ring: deviate d of a lane (counted over all its
 *    rows) sits at slot d mod 16; the warp's block is 4 KiB aligned, so the slot
 *    number is bits 8..11 of the address and a slot address is one AND-OR on
 *    d << 8.  A round writes its K candidates behind the <= 3 unstored deviates,
 *    complete 4-deviate chunks leave with one 32-byte store each (STG.E.256: a
 *    full L2 sector; a chunk starts at a multiple of 4, so it never wraps), and
 *    what is left over stays where it is.  (Until round 2's last pass the
 *    unstored deviates were moved back to slot 0 every round: 3 loads and 3
 *    stores per lane -- ncu showed the L1TEX LSU data pipe, which carries the
 *    shared-memory wavefronts AND the lane-private sector stores, at 93.7 % of
 *    its peak, so those 12 wavefronts per round were worth 4 % of the kernel.)
 *    Lanes never wait for each other: no warp-wide flush, no cross-lane drift.
 * Rows of a lane follow each other (lane l of warp g takes the streams
 * (g + k * warps) * 32 + l); the next row's state is loaded when a row starts.
 *
 * Fused witnesses (STATS): the per-row xor checksum (bench.py:174-175) and
 * power sums (stats.py:232-259) are folded from each stored chunk in deviate
 * order -- the order of k_zig_tma and of the oracle's default digest.
 *
 * EPI_MUTATE (config 5, x += sigma * z over every gene of `generations`
 * generations, samplers.py:195-200 with mu = x): a lane's row is one individual,
 * generations x n_genes deviates long; a chunk of 4 deviates updates 4 genes
 * (x + sigma z, two roundings) with one 32-byte load and one 32-byte store.  Every
 * round loads the x of the next two chunks into the same registers (the next round
 * stores at most two; a register shift of in-flight loads would wait for them) and
 * prefetches the LST_XPF chunks after them into L1; generation g + 1
 * reads genes that generation g stored n_genes deviates earlier, in the same thread.
 * Warps take their groups round-robin over the blocks (g = block + warp * blocks),
 * so a launch with fewer groups than warp slots still spreads over every SM.
 */
#pragma once

constexpr int LST_SLOTS = 16;                       /* staging slots per lane */
constexpr uint32_t LST_RING = LST_SLOTS * 256;      /* staging bytes per warp */
constexpr uint32_t LST_TAB = 0x10000;               /* the layer-row table (64 KiB) */
/* dynamic shared memory of k_zig_lst for NW warps, n layers and K attempts per round,
   given the dynamic window's offset (0x400 on sm_100 without clusters; the kernel
   re-derives the layout from the real base and fails loudly if it does not fit) */
__host__ __device__ constexpr uint32_t lst_smem_bytes(int NW, int NL, int K, uint32_t base = 0x400)
{
    const uint32_t tab = (base + 0xFFFFu) & ~0xFFFFu;
    const uint32_t r0 = (base + LST_RING - 1u) & ~(LST_RING - 1u);   /* rings are 4 KiB aligned */
    const uint32_t na = (tab - r0) / LST_RING < (uint32_t)NW ? (tab - r0) / LST_RING : (uint32_t)NW;
    return tab + LST_TAB + ((uint32_t)NW - na) * LST_RING + (uint32_t)NL * 8 + 16u * (uint32_t)(K + 1) + 16u +
           (uint32_t)NW * 32u * 16u - base;
}

/* the next row's state, copied global -> shared without a register (cp.async): a state
   loaded into a register a row ahead would be copied between registers by the compiler
   at the loop's back edge, i.e. waited for right after its load was issued */
__device__ __forceinline__ void lst_cp8(uint32_t dst, const void* src)
{
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(dst), "l"(src) : "memory");
}

__device__ __forceinline__ uint64_t lds_u64(uint32_t a)
{
    uint64_t v;
    asm volatile("ld.shared.u64 %0, [%1];" : "=l"(v) : "r"(a));
    return v;
}
__device__ __forceinline__ void sts_u64(uint32_t a, uint64_t v)
{
    asm volatile("st.shared.u64 [%0], %1;" ::"r"(a), "l"(v) : "memory");
}

/* the staging slot of deviate d of a lane (d counts the lane's deviates over all its rows):
   slot d mod 16 of the lane's column.  The warp's staging block is 4 KiB aligned, so the
   slot number is bits 8..11 of the address: one AND-OR on (d << 8). */
__device__ __forceinline__ uint32_t lst_slot(uint32_t ringl, uint32_t d256)
{
    return ringl | (d256 & (LST_RING - 256u));
}

#ifndef LST_XPF
#define LST_XPF 4   /* EPI_MUTATE: prefetch window beyond the two loaded x chunks (L1; 2: 244, 4: 248, 6: 247.5 G/s on c5) */
#endif
#ifndef LST_XPF_L2
#define LST_XPF_L2 0
#endif
/* EPI_MUTATE helpers: four genes in with one 32-byte load, x + sigma z */
__device__ __forceinline__ void ldg_x4(const double* a, uint64_t (&v)[4])
{
    asm volatile("ld.global.v4.b64 {%0, %1, %2, %3}, [%4];" : "=l"(v[0]), "=l"(v[1]), "=l"(v[2]), "=l"(v[3]) : "l"(a));
}
__device__ __forceinline__ uint64_t mut_x(uint64_t x, double sig, uint64_t zb)
{
    return (uint64_t)__double_as_longlong(
        __dadd_rn(__longlong_as_double((long long)x), __dmul_rn(sig, __longlong_as_double((long long)zb))));
}

/* (double)m for m = mhi * 2^32 + mlo (< 2^56, or m * 512 < 2^64 for the modified ziggurat), rounded to nearest even */
__device__ __forceinline__ double lst_u56_to_f64(uint32_t mhi, uint32_t mlo)
{
    return __ull2double_rn(((uint64_t)mhi << 32) | mlo);
}

template <int SRC, bool MOD, bool STATS, int NW, int TMA_K, int EPI = EPI_STORE>
__global__ void __launch_bounds__(NW * 32, 1) k_zig_lst(const __grid_constant__ LaneParams p)
{
    static_assert(TMA_K + 3 <= LST_SLOTS, "a round's candidates and the unstored deviates share the staging slots");
    constexpr bool MUT = EPI == EPI_MUTATE;
    static_assert(!MUT || (!STATS && TMA_K <= 8), "the mutation keeps the x of two chunks in registers");
    constexpr int NL = MOD ? 256 : 128;
    /* the mutation epilogue keeps the first unstored deviate at slot 0 (it waits on the x
       loads, not on the LSU pipe: the ring's address arithmetic cost it 1.5 %) */
    constexpr bool RING = !MUT;
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    const uint32_t base = sh_addr(smem_raw);
    uint32_t dyn;
    asm("mov.u32 %0, %%dynamic_smem_size;" : "=r"(dyn));
    /* the layout of lst_smem_bytes from the real window offset */
    const uint32_t tab = (base + 0xFFFFu) & ~0xFFFFu;
    const uint32_t r0 = (base + LST_RING - 1u) & ~(LST_RING - 1u);
    const uint32_t na = min((uint32_t)NW, (tab - r0) / LST_RING);
    const uint32_t after = tab + LST_TAB;
    const uint32_t yf_sh = after + ((uint32_t)NW - na) * LST_RING;
    const uint32_t jump_sh = yf_sh + NL * 8;
    /* per thread 16 bytes: the next row's state (and gamma) */
    const uint32_t stslot = ((jump_sh + 16u * (TMA_K + 1) + 15u) & ~15u) + (uint32_t)threadIdx.x * 16u;
    if (stslot + 16u * (NW * 32 - threadIdx.x) > base + dyn) {
        if (threadIdx.x == 0) gz_raise(GZ_ERR_CHECK, __LINE__);
        return;
    }
    for (int j = threadIdx.x; j < 256 * TMA_REP; j += blockDim.x) {
        ulonglong2 v = p.kw[(j / TMA_REP) & (NL - 1)];
        if constexpr (!MOD) {
            /* entries 128..255 are the same layers with the sign bit set: a negative wtab
               there makes m * wtab the signed deviate (negation is exact) */
            if (j / TMA_REP >= 128) v.y ^= 0x8000000000000000ULL;
        }
        if constexpr (MOD) {
            /* the modified ziggurat's mantissa is u >> 9: with ktab << 9 and wtab * 2^-9 the
               attempt compares and converts u & ~511 = m * 512 instead (m < k exactly when
               m * 512 < k * 512; (double)(m * 512) * (w / 512) rounds as (double)m * w) */
            v.x <<= 9;
            v.y = (unsigned long long)__double_as_longlong(__dmul_rn(__longlong_as_double((long long)v.y), 0x1p-9));
        }
        asm volatile("st.shared.v2.u64 [%0], {%1, %2};" ::"r"(tab + (uint32_t)(j / TMA_REP) * 256 + (uint32_t)(j % TMA_REP) * 16),
                     "l"(v.x), "l"(v.y)
                     : "memory");
    }
    for (int j = threadIdx.x; j < NL; j += blockDim.x) {
        const float2 v = p.yf[j];
        asm volatile("st.shared.v2.f32 [%0], {%1, %2};" ::"r"(yf_sh + 8 * j), "f"(v.x), "f"(v.y) : "memory");
    }
    /* LCG: (A, C) of 2n steps, n <= K (the state after n draws from a round's start) */
    if (SRC == 0 && threadIdx.x <= TMA_K)
        asm volatile("st.shared.v2.u64 [%0], {%1, %2};" ::"r"(jump_sh + 16 * threadIdx.x), "l"(c_lcgA[2 * threadIdx.x]),
                     "l"(c_lcgC[2 * threadIdx.x] << 16)
                     : "memory");
    __syncthreads();

    const int lane = threadIdx.x & 31;
    const uint32_t wib = threadIdx.x >> 5;
    /* the lane's staging column (slot s at ringl + 256 s) and its replica of the layer rows */
    const uint32_t ringl = (wib < na ? r0 + wib * LST_RING : after + (wib - na) * LST_RING) + (uint32_t)lane * 8;
    const uint32_t kwl = tab | ((uint32_t)(lane & 7) << 4);
    const int n_per = p.n_per;
    /* the increments of one and two LCG steps, C and A C + C, held in registers */
    /* LCG48 in the shifted domain: the lane keeps T = state * 2^16 mod 2^64, which obeys
       T' = A T + (C << 16) mod 2^64, so a step's output bits 16..47 are T's high word --
       no funnel shift -- and the jump, inverse and increments carry C << 16 */
    const uint64_t inc1 = SRC == 0 ? ld_keep(&c_lcgC[1]) << 16 : 0, inc2 = SRC == 0 ? ld_keep(&c_lcgC[2]) << 16 : 0;
    const uint32_t guard32 = p.guard > 0xffffffffll ? 0xffffffffu : (uint32_t)p.guard;
    /* stream ids in 32 bits: n_streams < 2^31 (lst_eligible), so id + 2 * sstride < 2^32 */
    const uint32_t n_streams = (uint32_t)p.n_streams;
    const uint32_t n_groups = (uint32_t)(((int64_t)p.n_streams + 31) >> 5);
    const uint32_t gstride = gridDim.x * NW;
    const uint32_t g0 = blockIdx.x + wib * gridDim.x;   /* round-robin over the blocks */
    const int ng = g0 < n_groups ? (int)((n_groups - g0 + gstride - 1) / gstride) : 0;

    /* the lane's rows: k = 0 .. ng-1, stream (g0 + k gstride) * 32 + lane (if < n_streams) */
    int k = -1;
    bool valid = false, failed = false;
    uint64_t S = 0, gam = 0;
    uint32_t C = 0;          /* deviates committed by this lane (all rows) */
    uint32_t c_row0 = 0;     /* C at the start of the current row */
    uint32_t c_rowend = 0;   /* C at its end */
    uint32_t f = 0;          /* deviates stored; the unstored ones C - f <= 3 sit at slots 0.. */
    uint32_t rej = 0, c_rej = 0xffffffffu;
    uint64_t ck = 0;
    double a1 = 0.0, a2 = 0.0, a3 = 0.0, a4 = 0.0;
    /* EPI_MUTATE: the row length, the gene of deviate f, the row's sigma and the x of the
       chunks at genes gpos and gpos + 4 (loaded a round ahead) */
    const uint32_t rowlen = MUT ? (uint32_t)n_per * (uint32_t)p.generations : (uint32_t)n_per;
    uint32_t gpos = 0;
    double sig = 0.0;
    uint64_t xa[2][4] = {};

    /* consecutive rows of a lane are sstride streams apart */
    const uint32_t sstride = gstride * 32;
    const uint32_t last = n_streams - 1;
    uint32_t sid = g0 * 32 + (uint32_t)lane - sstride;   /* modular: the first row adds sstride back */
    const int64_t rstride = (int64_t)sstride * p.ld;
    double* rowp = p.out + (int64_t)(g0 * 32 + (uint32_t)lane) * p.ld - rstride;
    auto prefetch_state = [&](uint32_t q) {
        q = min(q, last);   /* clamped: the copy is unconditional */
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
        if constexpr (SRC == 0) s <<= 16;
        if constexpr (SRC == 1) g = lds_u64(stslot + 8);
    };
    /* the row transition (divergent: once per row and lane, called when C >= c_rowend and
       k < ng): finish the row, start the next (at most one per round) */
    auto next_row = [&]() {
        {
            if (valid && !failed) {
                if (n_per & 3) {
                    /* the row's last partial chunk (deviates f .. c_rowend - 1 of the ring) */
                    for (uint32_t q = 0; q < c_rowend - f; ++q) {
                        const uint64_t v = lds_u64(lst_slot(ringl, (f + q) << 8));   /* (never a mutation row: genes % 4 == 0) */
                        rowp[f + q - c_row0] = __longlong_as_double((long long)v);
                        if constexpr (STATS) tma_fold(v, ck, a1, a2, a3, a4);
                    }
                }
                /* its witnesses and its final state */
                if constexpr (STATS) {
                    if (p.checksum) p.checksum[sid] = ck;
                    if (p.psum) {
                        double* ps = p.psum + 4 * (int64_t)sid;   /* 16-byte aligned (lst_eligible) */
                        asm volatile("st.global.v2.f64 [%0], {%1, %2};" ::"l"(ps), "d"(a1), "d"(a2) : "memory");
                        asm volatile("st.global.v2.f64 [%0], {%1, %2};" ::"l"(ps + 2), "d"(a3), "d"(a4) : "memory");
                    }
                }
                if constexpr (SRC == 0) {
                    p.state_out[sid] = S >> 16;
                } else {
                    asm volatile("st.global.v2.u64 [%0], {%1, %2};" ::"l"(p.state_out + 2 * (int64_t)sid), "l"(S), "l"(gam)
                                 : "memory");
                }
            }
            ++k;
            failed = false;
            if constexpr (STATS) {
                ck = 0;
                a1 = a2 = a3 = a4 = 0.0;
            }
            /* rows start on a chunk boundary, with nothing unstored */
            if (n_per & 3) C = (C + 3u) & ~3u;
            f = C;
            c_row0 = C;
            sid += sstride;
            rowp += rstride;
            valid = k < ng && sid < n_streams;
            take_state(S, gam);
            prefetch_state(sid + sstride);
            c_rowend = valid ? C + rowlen : C;   /* no stream: skip the row */
            if constexpr (MUT) {
                if (valid) {
                    gpos = 0;
                    sig = p.sigma[sid];
                    ldg_x4(rowp, xa[0]);
                    ldg_x4(rowp + 4, xa[1]);
                }
            }
        }
    };
    if (ng > 0) prefetch_state(sid + sstride);
    next_row();

    while (__any_sync(GZ_FULL, k < ng)) {
        /* ---- one round: TMA_K attempts per lane, no branches ---- */
        const bool act = C < c_rowend;
        const uint32_t C0 = C;
        GZ_CHECK(C0 - f <= 3u, C0 - f);   /* at most 3 unstored deviates (ring: at slots f mod 16 ..; mutation: at slots 0..2) */
        /* the leading fast accepts, counted as they come: the running AND rides in the
           compare's predicate slot, the count is one predicated add per attempt */
        bool fast = true;
        uint32_t lead = 0;
        /* the deviates stay in registers until the last attempt: a table gather may not
           pass a shared store in program order (ptxas cannot tell that they never alias) */
        uint64_t zbs[TMA_K];
        uint32_t sl = (uint32_t)S, sh = (uint32_t)(S >> 32);
#pragma unroll
        for (int kk2 = 0; kk2 < TMA_K; ++kk2) {
            uint32_t uhi, ulo;
            if constexpr (SRC == 0) {
                /* u64 = two steps, t1 = A t + C and t2 = A^2 t + (A C + C) straight from t
                   (engine.py:52-58: bits 16..47 of each state) */
                uint32_t t1l, t1h, t2l, t2h;
                lcg_step32(sl, sh, t1l, t1h, inc1);
                lcg_step32x2(sl, sh, t2l, t2h, inc2);
                uhi = t1h;
                ulo = t2h;
                sl = t2l;
                sh = t2h;
            } else {
                const uint64_t t = (((uint64_t)sh << 32) | sl) + gam;
                sl = (uint32_t)t;
                sh = (uint32_t)(t >> 32);
                const uint64_t u = gz_mix64(t);
                uhi = (uint32_t)(u >> 32);
                ulo = (uint32_t)u;
            }
            uint32_t mhi, mlo, sgn, row;
            if constexpr (MOD) {
                row = __byte_perm(ulo, kwl, 0x7604);   /* layer = low byte */
                mlo = ulo & ~511u;                     /* m * 512 (see the table fill) */
                mhi = uhi;
                sgn = (ulo << 23) & 0x80000000u;
            } else {
                row = __byte_perm(uhi, kwl, 0x7634);   /* sign and layer = top byte */
                mhi = uhi & 0x00ffffffu;
                mlo = ulo;
                sgn = uhi & 0x80000000u;
            }
            uint64_t kk, wb;
            lds_tab(row, kk, wb);
            const uint64_t m = ((uint64_t)mhi << 32) | mlo;
            const double x = __dmul_rn(lst_u56_to_f64(mhi, mlo), __longlong_as_double((long long)wb));
            fast = fast && m < kk;
            /* (spelled as a predicated add: from `lead += fast` the compiler makes an add
               and a predicated move) */
            asm("{\n\t.reg .pred q;\n\tsetp.ne.u32 q, %1, 0;\n\t@q add.u32 %0, %0, 1;\n\t}" : "+r"(lead) : "r"((uint32_t)fast));
            /* the original ziggurat's sign is in the table row (see the fill) */
            zbs[kk2] = MOD ? (uint64_t)__double_as_longlong(x) ^ ((uint64_t)sgn << 32) : (uint64_t)__double_as_longlong(x);
        }
        const uint32_t c0s = (RING ? C0 : C0 - f) << 8;   /* deviate C0 + j goes to slot (C0 + j) mod 16 */
        if (act) {
#pragma unroll
            for (int kk2 = 0; kk2 < TMA_K; ++kk2)
                asm volatile("st.shared.u64 [%0], %1;" ::"r"(RING ? lst_slot(ringl, c0s + 256u * kk2) : ringl + c0s + 256u * kk2),
                             "l"(zbs[kk2])
                             : "memory");
        }
        bool frozen = false;
        if (act) {
            const uint32_t C_lead = C0 + lead;
            C = min(C_lead, c_rowend);
            frozen = C_lead < c_rowend && lead < (uint32_t)TMA_K;
        }
        /* the live attempts are a prefix of the round: the committed ones plus a frozen
           one; the state after them by jump-ahead from the round's start */
        {
            const uint32_t n_live = (C - C0) + (frozen ? 1u : 0u);
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
                const uint32_t slot = RING ? lst_slot(ringl, C << 8) : ringl + ((C - f) << 8);   /* the frozen attempt's staged x */
                GZ_CHECK(C - f < (uint32_t)LST_SLOTS, C - f);
                uint64_t u;
                if constexpr (SRC == 0) {
                    /* the draw that produced T: the previous T by the inverse step mod 2^64 */
                    const uint64_t t1 = (S - inc1) * 0x7B13DFE05BCB1365ULL;   /* A^-1 mod 2^64 */
                    u = (t1 & 0xffffffff00000000ULL) | (S >> 32);
                } else {
                    u = tma_recover<SRC>(S);
                }
                uint32_t i;
                uint64_t m_unused, sgn;
                tma_split<MOD>(u, i, m_unused, sgn);
                double x = __longlong_as_double((long long)(lds_u64(slot) & 0x7fffffffffffffffULL));
                bool ok;
                if (i != 0) {
                    /* wedge: the next draw is its uniform, whatever the outcome; an accepted
                       wedge's slot already holds x */
                    uint64_t u2;
                    if constexpr (SRC == 0) {
                        const uint64_t t1 = S * GZ_LCG_A + inc1, t2 = t1 * GZ_LCG_A + inc1;
                        S = t2;
                        u2 = (t1 & 0xffffffff00000000ULL) | (t2 >> 32);
                    } else {
                        u2 = tma_draw<SRC>(S, gam);
                    }
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
                    const TailOut to = tail_seq<SRC>(SRC == 0 ? S >> 16 : S, gam, p.r, p.guard);
                    S = SRC == 0 ? to.st << 16 : to.st;
                    x = to.v;
                    ok = to.k >= 0;
                    if (ok) {
                        const uint64_t zb = (uint64_t)__double_as_longlong(x) ^ sgn;
                        asm volatile("st.shared.u64 [%0], %1;" ::"r"(slot), "l"(zb) : "memory");
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
        /* ---- complete 4-deviate chunks to the row: one 32-byte store each, from slots
           0, 4, 8 (straight-line, at most (K + 3) / 4 of them); the <= 3 left over move
           back to slot 0 ---- */
        if (!failed) {
            const uint32_t pend = C - f;   /* <= K + 3 */
            GZ_CHECK(pend <= (uint32_t)TMA_K + 3u, pend);
            double* dst = rowp + (MUT ? gpos : f - c_row0);
            uint32_t nst = 0;
#pragma unroll
            for (int q = 0; q < (TMA_K + 3) / 4; ++q) {
                if (pend >= 4u * (q + 1)) {
                    /* f is a multiple of 4: no wrap inside a chunk */
                    const uint32_t ph = RING ? lst_slot(ringl, (f << 8) + 1024u * q) : ringl + 1024u * q;
                    uint64_t v0 = lds_u64(ph), v1 = lds_u64(ph + 256), v2 = lds_u64(ph + 512), v3 = lds_u64(ph + 768);
                    if constexpr (MUT) {
                        /* x + sigma z (gaussian_affine with mu = x: two roundings) */
                        v0 = mut_x(xa[q][0], sig, v0);
                        v1 = mut_x(xa[q][1], sig, v1);
                        v2 = mut_x(xa[q][2], sig, v2);
                        v3 = mut_x(xa[q][3], sig, v3);
                        /* genes gpos + 4 q .. + 3 of the row; gpos + 4 wraps to gene 0 */
                        if (q == 1 && gpos + 4u == (uint32_t)n_per) dst -= n_per;
                    }
                    asm volatile("st.global.v4.b64 [%0], {%1, %2, %3, %4};" ::"l"(dst + 4 * q), "l"(v0), "l"(v1), "l"(v2),
                                 "l"(v3)
                                 : "memory");
                    if constexpr (STATS) {
                        ck ^= v0 ^ v1 ^ v2 ^ v3;
                        tma_fold_fp(v0, a1, a2, a3, a4);
                        tma_fold_fp(v1, a1, a2, a3, a4);
                        tma_fold_fp(v2, a1, a2, a3, a4);
                        tma_fold_fp(v3, a1, a2, a3, a4);
                    }
                    nst = q + 1;
                }
            }
            if (nst != 0) {
                if constexpr (!RING) {
                    /* the <= 3 left over move back to slot 0 */
                    const uint32_t ph = ringl + 1024u * nst;
                    const uint64_t w0 = lds_u64(ph), w1 = lds_u64(ph + 256), w2 = lds_u64(ph + 512);
                    sts_u64(ringl, w0);
                    sts_u64(ringl + 256, w1);
                    sts_u64(ringl + 512, w2);
                }
                f += 4u * nst;   /* RING: the <= 3 left over stay where they are, slots f mod 16 .. */
                if constexpr (MUT) {
                    gpos += 4u * nst;
                    if (gpos >= (uint32_t)n_per) gpos -= (uint32_t)n_per;
                }
            }
            if constexpr (MUT) {
                /* the x of the next two chunks, a round ahead, always into the same registers
                   (a conditional shift of the in-flight registers would make the compiler copy
                   them and wait for the loads); past the row's end they reread this row */
                if (valid) {
                    uint32_t g1 = gpos + 4u;
                    if (g1 == (uint32_t)n_per) g1 = 0;
                    ldg_x4(rowp + gpos, xa[0]);
                    ldg_x4(rowp + g1, xa[1]);
                    /* the chunks that entered the prefetch window [gpos, gpos + 4 (2 + XPF)) */
#pragma unroll
                    for (int j = 0; j < 2; ++j) {
                        if ((uint32_t)j < nst) {
                            uint32_t g = gpos + 4u * (2 + LST_XPF - nst + j);
                            if (g >= (uint32_t)n_per) g -= (uint32_t)n_per;
                            if (LST_XPF_L2) asm volatile("prefetch.global.L2 [%0];" ::"l"(rowp + g));
                            else asm volatile("prefetch.global.L1 [%0];" ::"l"(rowp + g));
                        }
                    }
                }
            }
        }
        if (C >= c_rowend && k < ng) next_row();
    }
}
