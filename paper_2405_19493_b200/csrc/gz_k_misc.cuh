/*
 * gz_k_misc.cuh -- fill_u64, device seeding, affine uniforms, reductions, layer occupancy, libm evaluation.
 *
 * Not a standalone header: included by gz_engine.cu inside its anonymous
 * namespace, after the shared device globals and helpers it uses.
 */
#pragma once

/* -------------------------------------------------------------- fill_u64 */

template <int SRC>
__global__ void __launch_bounds__(256) k_u64(int64_t n_streams, int64_t n_per, int64_t ld, const uint64_t* state_in,
                                             uint64_t* state_out, uint64_t* out)
{
    const int lane = threadIdx.x & 31;
    const int64_t w0 = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    uint64_t A1 = 0, C1 = 0, A2 = 0, C2 = 0;
    if constexpr (SRC == 0) {
        A1 = ld_keep(&c_lcgA[2 * lane + 1]); C1 = ld_keep(&c_lcgC[2 * lane + 1]);
        A2 = ld_keep(&c_lcgA[2 * lane + 2]); C2 = ld_keep(&c_lcgC[2 * lane + 2]);
    }
    for (int64_t sid = w0; sid < n_streams; sid += nw) {
        uint64_t S, gam = 0, gl = 0;
        if constexpr (SRC == 0) {
            S = state_in[sid];
        } else {
            S = state_in[2 * sid];
            gam = state_in[2 * sid + 1];
            gl = (uint64_t)(lane + 1) * gam;
        }
        uint64_t* row = out + sid * ld;
        for (int64_t b = 0; b < n_per; b += 32) {
            uint64_t u, stv;
            if constexpr (SRC == 0) {
                const uint64_t t1 = gz_lcg_mad(A1, S, C1);
                stv = gz_lcg_mad(A2, S, C2);
                u = gz_lcg_u64(t1, stv);
            } else {
                stv = S + gl;
                u = gz_mix64(stv);
            }
            const int64_t take = min((int64_t)32, n_per - b);
            if (lane < take) row[b + lane] = u;
            if constexpr (SRC == 0) S = __shfl_sync(GZ_FULL, stv, (int)take - 1);
            else S += (uint64_t)take * gam;
        }
        if (lane == 0) {
            if constexpr (SRC == 0) {
                state_out[sid] = S;
            } else {
                state_out[2 * sid] = S;
                state_out[2 * sid + 1] = gam;
            }
        }
    }
}

/* ------------------------------------------------------------- seeding */

__global__ void k_seed(int scheme, uint64_t master, int64_t first, int64_t count, uint64_t* out)
{
    for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < count; k += (int64_t)gridDim.x * blockDim.x) {
        const uint64_t id = (uint64_t)(first + k);
        switch (scheme) {
        case GZ_SEED_LCG_MASTER_PLUS_ID:
            out[k] = ((master + id) ^ GZ_LCG_A) & GZ_MASK48;
            break;
        case GZ_SEED_SM_OUTPUT_OF_MASTER:
            out[2 * k] = gz_mix64(master + (id + 1) * GZ_GOLDEN_GAMMA);
            out[2 * k + 1] = GZ_GOLDEN_GAMMA;
            break;
        case GZ_SEED_SM_ID_XOR_MASTER:
            out[2 * k] = id ^ master;
            out[2 * k + 1] = GZ_GOLDEN_GAMMA;
            break;
        default:
            out[2 * k] = master + id;
            out[2 * k + 1] = GZ_GOLDEN_GAMMA;
            break;
        }
    }
}

/* out[j] = a + b*unit(draw j) of one stream (jump-ahead per element) */
template <int SRC>
__global__ void k_unit_affine(const uint64_t* state, int64_t n, double a, double b, double* out)
{
    const uint64_t S = state[0];
    const uint64_t gam = SRC ? state[1] : 0;
    for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < n; j += (int64_t)gridDim.x * blockDim.x) {
        uint64_t u;
        if constexpr (SRC == 1) {
            u = gz_mix64(S + (uint64_t)(j + 1) * gam);
        } else {
            /* state after 2j steps via binary powering of the LCG map */
            uint64_t A = 1, C = 0, pa = GZ_LCG_A, pc = GZ_LCG_C;
            for (uint64_t e = (uint64_t)(2 * j); e; e >>= 1) {
                if (e & 1) { C = gz_lcg_mad(pa, C, pc); A = (A * pa) & GZ_MASK48; }
                pc = gz_lcg_mad(pa, pc, pc);
                pa = (pa * pa) & GZ_MASK48;
            }
            uint64_t s0 = gz_lcg_mad(A, S, C);
            const uint64_t t1 = gz_lcg_mad(GZ_LCG_A, s0, GZ_LCG_C);
            const uint64_t t2 = gz_lcg_mad(GZ_LCG_A, t1, GZ_LCG_C);
            u = gz_lcg_u64(t1, t2);
        }
        out[j] = __dadd_rn(a, __dmul_rn(b, gz_unit53(u)));
    }
}

__global__ void k_unit_affine_state(int src, uint64_t* state, int64_t n)
{
    if (threadIdx.x == 0 && blockIdx.x == 0) {
        if (src == 1) {
            state[0] += (uint64_t)n * state[1];
        } else {
            uint64_t st = state[0];
            /* jump 2n steps */
            uint64_t A = 1, C = 0, pa = GZ_LCG_A, pc = GZ_LCG_C;
            for (uint64_t e = (uint64_t)(2 * n); e; e >>= 1) {
                if (e & 1) { C = gz_lcg_mad(pa, C, pc); A = (A * pa) & GZ_MASK48; }
                pc = gz_lcg_mad(pa, pc, pc);
                pa = (pa * pa) & GZ_MASK48;
            }
            state[0] = gz_lcg_mad(A, st, C);
        }
    }
}

/* ------------------------------------------------------------- reductions */

#define RED_CHUNK 2048
/* stage 1: block b reduces rows [b*RED_CHUNK, ...) in a fixed tree order */
__global__ void __launch_bounds__(256) k_psum_stage1(const double* psum, int64_t n_rows, double* part)
{
    __shared__ double sh[4][256];
    const int64_t r0 = (int64_t)blockIdx.x * RED_CHUNK;
    double acc[4] = {0.0, 0.0, 0.0, 0.0};
    for (int k = threadIdx.x; k < RED_CHUNK; k += 256) {
        const int64_t rr = r0 + k;
        if (rr < n_rows)
            for (int c = 0; c < 4; ++c) acc[c] = __dadd_rn(acc[c], psum[4 * rr + c]);
    }
    for (int c = 0; c < 4; ++c) sh[c][threadIdx.x] = acc[c];
    __syncthreads();
    for (int w = 128; w > 0; w >>= 1) {
        if (threadIdx.x < w)
            for (int c = 0; c < 4; ++c) sh[c][threadIdx.x] = __dadd_rn(sh[c][threadIdx.x], sh[c][threadIdx.x + w]);
        __syncthreads();
    }
    if (threadIdx.x == 0)
        for (int c = 0; c < 4; ++c) part[4 * blockIdx.x + c] = sh[c][0];
}

__global__ void k_psum_stage2(const double* part, int64_t n_part, double n_values, double* out5)
{
    __shared__ double sh[4][256];
    double acc[4] = {0.0, 0.0, 0.0, 0.0};
    for (int64_t k = threadIdx.x; k < n_part; k += 256)
        for (int c = 0; c < 4; ++c) acc[c] = __dadd_rn(acc[c], part[4 * k + c]);
    for (int c = 0; c < 4; ++c) sh[c][threadIdx.x] = acc[c];
    __syncthreads();
    for (int w = 128; w > 0; w >>= 1) {
        if (threadIdx.x < w)
            for (int c = 0; c < 4; ++c) sh[c][threadIdx.x] = __dadd_rn(sh[c][threadIdx.x], sh[c][threadIdx.x + w]);
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        const double n = n_values, S1 = sh[0][0], S2 = sh[1][0], S3 = sh[2][0], S4 = sh[3][0];
        const double mean = S1 / n;
        const double m2 = S2 - S1 * mean;
        const double m3 = S3 - 3.0 * mean * S2 + 2.0 * n * mean * mean * mean;
        const double m4 = S4 - 4.0 * mean * S3 + 6.0 * mean * mean * S2 - 3.0 * n * mean * mean * mean * mean;
        out5[0] = n; out5[1] = mean; out5[2] = m2; out5[3] = m3; out5[4] = m4;
    }
}

/* power sums of a raw buffer: block b reduces values [b*POW_CHUNK, ...) in a fixed
   tree order (deterministic for a given n), one psum row per block */
#define POW_CHUNK 8192
__global__ void __launch_bounds__(256) k_pow_stage1(const double* x, int64_t n, double* part)
{
    __shared__ double sh[4][256];
    const int64_t v0 = (int64_t)blockIdx.x * POW_CHUNK;
    double acc[4] = {0.0, 0.0, 0.0, 0.0};
    for (int k = threadIdx.x; k < POW_CHUNK; k += 256) {
        const int64_t vv = v0 + k;
        if (vv < n) {
            const double v = x[vv];
            const double v2 = __dmul_rn(v, v);
            acc[0] = __dadd_rn(acc[0], v);
            acc[1] = __dadd_rn(acc[1], v2);
            acc[2] = __fma_rn(v2, v, acc[2]);
            acc[3] = __fma_rn(v2, v2, acc[3]);
        }
    }
    for (int c = 0; c < 4; ++c) sh[c][threadIdx.x] = acc[c];
    __syncthreads();
    for (int w = 128; w > 0; w >>= 1) {
        if (threadIdx.x < w)
            for (int c = 0; c < 4; ++c) sh[c][threadIdx.x] = __dadd_rn(sh[c][threadIdx.x], sh[c][threadIdx.x + w]);
        __syncthreads();
    }
    if (threadIdx.x < 4) part[4 * blockIdx.x + threadIdx.x] = sh[threadIdx.x][0];
}

/*
 * Layer occupancy of one stream (the reference's sample_with_occupancy,
 * samplers.py:89-115 / 138-165): n_calls sequential calls of the ziggurat by
 * one thread, counting the layer index of every attempt.  A verification
 * utility (cli.py verify, 10^5 calls), not a throughput path.
 */
template <int SRC, bool MOD>
__global__ void k_zig_occupancy(const uint64_t* state_in, uint64_t* state_out, int64_t n_calls, double* out,
                                unsigned long long* counts, const ulonglong2* kw, const double2* yd, int n_layers,
                                double r, int64_t guard)
{
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    uint64_t st = state_in[0];
    const uint64_t gam = SRC == 1 ? state_in[1] : 0;
    int ib = 0;
    while ((1 << (ib + 1)) <= n_layers) ++ib;
    const uint32_t imask = (uint32_t)n_layers - 1u;
    const int mbits = 63 - ib;
    const uint64_t mmask = (1ULL << mbits) - 1ULL;
    for (int64_t c = 0; c < n_calls; ++c) {
        bool done = false;
        double v = 0.0;
        for (int64_t a = 0; a < guard && !done; ++a) {
            const uint64_t u = gz_next_seq<SRC>(st, gam);
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
            counts[i] += 1;
            const ulonglong2 k = kw[i];
            double x = __dmul_rn(__ull2double_rn(m), __longlong_as_double((long long)k.y));
            if (m < k.x) {
                done = true;
            } else if (i == 0) {
                const TailOut to = tail_seq<SRC>(st, gam, r, guard);
                st = to.st;
                if (to.k < 0) {
                    gz_raise(GZ_ERR_GUARD, 0);
                    return;
                }
                x = to.v;
                done = true;
            } else {
                const double U = gz_unit53(gz_next_seq<SRC>(st, gam));
                const double y = __dadd_rn(yd[i].x, __dmul_rn(U, yd[i].y));
                done = wedge_exact(y, __dmul_rn(__dmul_rn(-0.5, x), x));
            }
            v = neg ? -x : x;
        }
        if (!done) {
            gz_raise(GZ_ERR_GUARD, 0);
            return;
        }
        if (out) out[c] = v;
    }
    state_out[0] = st;
    if (SRC == 1) state_out[1] = gam;
}

__global__ void k_xor_reduce(const uint64_t* in, int64_t n, unsigned long long* out)
{
    uint64_t acc = 0;
    for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < n; k += (int64_t)gridDim.x * blockDim.x)
        acc ^= in[k];
    for (int o = 16; o > 0; o >>= 1) acc ^= __shfl_xor_sync(GZ_FULL, acc, o);
    if ((threadIdx.x & 31) == 0 && acc) atomicXor(out, (unsigned long long)acc);
}

__global__ void k_libm_eval(int fn, const double* in, double* out, int64_t n)
{
    for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < n; k += (int64_t)gridDim.x * blockDim.x)
        out[k] = fn == 0 ? gz_exp_t(in[k], g_exp_tab) : gz_log_t(in[k], g_log_tab);
}

/* one tail_sample call (samplers.py:40-57) on one stream, by one thread */
template <int SRC>
__global__ void k_tail_sample(uint64_t* state, double r, int64_t guard, double* out)
{
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    const uint64_t gam = SRC == 1 ? state[1] : 0;
    const TailOut to = tail_seq<SRC>(state[0], gam, r, guard);
    if (to.k < 0) {
        gz_raise(GZ_ERR_GUARD, 0);
        return;
    }
    state[0] = SRC == 0 ? (to.st & GZ_MASK48) : to.st;
    out[0] = to.v;
}

/* ------------------------------------------------------ scripted sources */

/* a scripted word stream on the device: words[cursor++], exhaustion flagged */
struct ScriptDraws {
    const uint64_t* w;
    int64_t n, pos;
    bool out;   /* read past the end */
    __device__ __forceinline__ uint64_t next()
    {
        if (pos >= n) {
            out = true;
            return 0;
        }
        return w[pos++];
    }
    __device__ __forceinline__ double unit() { return gz_unit53(next()); }
};

/* samplers.py:95-115 / 144-165 (ziggurats) and 179-192 (polar), call after call,
   over scripted words, by one thread */
__global__ void k_scripted(int alg, const ulonglong2* kw, const double2* yd, int n_layers, double r,
                           const uint64_t* words, int64_t n_words, int64_t* cursor, int64_t n, double* out,
                           const double* spare_in, const uint8_t* has_in, double* spare_out, uint8_t* has_out,
                           int64_t guard)
{
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    ScriptDraws d{words, n_words, *cursor, false};
    int ib = 0;
    while (alg != GZ_ALG_POLAR && alg != 3 && (1 << (ib + 1)) <= n_layers) ++ib;
    const uint32_t imask = (uint32_t)n_layers - 1u;
    const int mbits = 63 - ib;
    const uint64_t mmask = (alg == 1 || alg == 2) ? (1ULL << mbits) - 1ULL : 0;
    bool has = alg == GZ_ALG_POLAR && has_in && has_in[0];
    double spare = has ? spare_in[0] : 0.0;
    int code = 0;
    for (int64_t c = 0; c < n && !code; ++c) {
        double v = 0.0;
        bool done = false;
        if (alg == 3) {
            /* tail_sample(src, r) calls (samplers.py:40-57) */
            for (int64_t t = 0; t < guard && !done; ++t) {
                const double u1 = d.unit(), u2 = d.unit();
                if (d.out) break;
                if (u1 <= 0.0 || u2 <= 0.0) continue;
                const double xt = __ddiv_rn(-gz_log_t(u1, g_log_tab), r);
                const double yt = -gz_log_t(u2, g_log_tab);
                if (__dmul_rn(2.0, yt) > __dmul_rn(xt, xt)) {
                    v = __dadd_rn(r, xt);
                    done = true;
                }
            }
        } else if (alg == GZ_ALG_POLAR) {
            if (has) {
                has = false;
                v = spare;
                done = true;
            }
            for (int64_t a = 0; a < guard && !done; ++a) {
                const double v1 = __fma_rn(2.0, d.unit(), -1.0);
                const double v2 = __fma_rn(2.0, d.unit(), -1.0);
                if (d.out) break;
                const double s = __dadd_rn(__dmul_rn(v1, v1), __dmul_rn(v2, v2));
                if (s > 0.0 && s < 1.0) {
                    const double mul = polar_mul(s, g_log_tab);
                    v = __dmul_rn(v1, mul);
                    spare = __dmul_rn(v2, mul);
                    has = true;
                    done = true;
                }
            }
        } else {
            const bool mod = alg == GZ_ALG_MODIFIED_ZIGGURAT;
            for (int64_t a = 0; a < guard && !done; ++a) {
                const uint64_t u = d.next();
                if (d.out) break;
                uint32_t i;
                uint64_t m;
                bool neg;
                if (mod) {
                    i = (uint32_t)u & imask;
                    m = u >> (ib + 1);
                    neg = (u >> ib) & 1;
                } else {
                    i = (uint32_t)(u >> mbits) & imask;
                    m = u & mmask;
                    neg = u >> 63;
                }
                const ulonglong2 k = kw[i];
                double x = __dmul_rn(__ull2double_rn(m), __longlong_as_double((long long)k.y));
                bool ok = m < k.x;
                if (!ok && i == 0) {
                    /* tail_sample (samplers.py:40-57) */
                    for (int64_t t = 0; t < guard && !ok; ++t) {
                        const double u1 = d.unit(), u2 = d.unit();
                        if (d.out) break;
                        if (u1 <= 0.0 || u2 <= 0.0) continue;
                        const double xt = __ddiv_rn(-gz_log_t(u1, g_log_tab), r);
                        const double yt = -gz_log_t(u2, g_log_tab);
                        if (__dmul_rn(2.0, yt) > __dmul_rn(xt, xt)) {
                            x = __dadd_rn(r, xt);
                            ok = true;
                        }
                    }
                    if (!ok && !d.out) {
                        code = GZ_ERR_GUARD;
                        break;
                    }
                } else if (!ok) {
                    const double y = __dadd_rn(yd[i].x, __dmul_rn(d.unit(), yd[i].y));
                    if (d.out) break;
                    ok = wedge_exact(y, __dmul_rn(__dmul_rn(-0.5, x), x));
                }
                if (ok) {
                    v = neg ? -x : x;
                    done = true;
                }
            }
        }
        if (d.out) code = GZ_ERR_EXHAUSTED;
        else if (!done && !code) code = GZ_ERR_GUARD;
        if (!code) out[c] = v;
    }
    if (code) gz_raise(code, 0);
    *cursor = d.pos;
    if (alg == GZ_ALG_POLAR) {
        if (spare_out) spare_out[0] = has ? spare : 0.0;
        if (has_out) has_out[0] = has ? 1 : 0;
    }
}

