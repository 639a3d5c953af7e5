/*
 * gz_b200.h -- C ABI of the B200 Gaussian variate engine (libgzb200.so).
 *
 * This is the drop-in boundary for the reference's batch engine
 * (/root/reference/pkg/src/gausszig/engine.py).  Plain pointers and sizes only;
 * no torch types.  Every entry point returns an int status:
 *
 *   GZ_OK (0)           success
 *   GZ_ERR_GUARD (1)    a rejection loop ran `guard` times without accepting
 *                       (engine.py:102,111,141,150,178 RuntimeError /
 *                        samplers.py:32-33 RejectionLoopExceeded)
 *   GZ_ERR_INVALID (2)  invalid argument (engine.py:209,269 TypeError /
 *                        tables.py:109-110 ValueError)
 *   GZ_ERR_CUDA (3)     CUDA runtime error (no device, launch failure, ...)
 *   GZ_ERR_EXHAUSTED (4) a scripted source ran out of words (sources.py
 *                       ScriptExhausted)
 *
 * gz_last_error() returns a message for the last non-zero status of the calling
 * thread.  "Device" pointers are CUDA device (or managed) memory of the current
 * device; "host" pointers are CPU memory (pinned for full PCIe speed).
 *
 * Stream state layout (engine.py:204-209 `_state_array`):
 *   GZ_SRC_LCG48     uint64_t state[n_streams]            (48-bit LCG state)
 *   GZ_SRC_SPLITMIX  uint64_t state[n_streams][2]         ({state, gamma})
 * Output layout: row s of `out` (row stride `ld` elements, ld >= n_per) holds
 * exactly what engine.fill_gaussians(sampler_s, source_s, row) produces for a
 * fresh call on stream s, and state_out/spare_out hold what that call writes
 * back (engine.py:212-213, 248-253).  state_out may alias state_in.
 */
#ifndef GZ_B200_H
#define GZ_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define GZ_OK 0
#define GZ_ERR_GUARD 1
#define GZ_ERR_INVALID 2
#define GZ_ERR_CUDA 3
#define GZ_ERR_EXHAUSTED 4

/* samplers.py:225-237 SAMPLER_IDS */
#define GZ_ALG_POLAR 0
#define GZ_ALG_ZIGGURAT 1
#define GZ_ALG_MODIFIED_ZIGGURAT 2
/* sources.py:154-163 SOURCE_IDS */
#define GZ_SRC_LCG48 0
#define GZ_SRC_SPLITMIX 1

/* gz_seed_streams schemes (the five BASELINE configs) */
#define GZ_SEED_LCG_MASTER_PLUS_ID 0   /* Lcg48(master + id)                     (C2, C4) */
#define GZ_SEED_SM_OUTPUT_OF_MASTER 1  /* SplitMix64(id-th output of SplitMix64(master)) (C1, C3) */
#define GZ_SEED_SM_ID_XOR_MASTER 2     /* SplitMix64(id ^ master)                  (C5) */
#define GZ_SEED_SM_MASTER_PLUS_ID 3    /* SplitMix64(master + id)                          */

#define GZ_MAX_TABLE_SLOTS 16
#define GZ_DEFAULT_GUARD 1000000       /* samplers.py:27 LOOP_GUARD, engine.py:37 _GUARD */

/* Library version (major*10000 + minor*100 + patch). */
int gz_version(void);
/* Message for the last non-zero status returned on this thread. */
const char* gz_last_error(void);
/* Number of visible CUDA devices (0 when none); never fails. */
int gz_device_count(void);
/*
 * Kernel family for gz_fill_gaussians on the current device: 0 = automatic
 * (one lane per stream from 32768 streams up, one warp per stream below),
 * 1 = always one warp per stream (jump-ahead decode), 2 = always one lane per
 * stream (ziggurat rows leave through lane-private 32-byte stores where the row
 * layout allows, else TMA tensor stores), 3 = one lane per stream with the
 * shared-ring lane stores only, 4 = one lane per stream with TMA tensor stores.
 * Results are identical; this only selects the schedule.
 */
int gz_set_kernel_policy(int policy);
/* Select the CUDA device used by subsequent calls from this thread. */
int gz_set_device(int device);

/*
 * Upload ziggurat tables into slot `slot` (0 <= slot < GZ_MAX_TABLE_SLOTS) of the
 * current device.  Host arrays: ktab[n], wtab[n], ytab[n+1], boundary r -- the
 * fields of tables.ZigguratTables (tables.py:38-64), built by
 * build_ziggurat_tables (tables.py:107-131).  Replaces engine.py:216-221
 * `_table_arrays`.  n must be a power of two in [8, 1024].
 */
int gz_tables_upload(int slot, int n, const uint64_t* ktab, const double* wtab, const double* ytab, double r);

/*
 * Batch Gaussian fill over many independent streams (device pointers).
 * Replaces engine.fill_gaussians (engine.py:235-270) applied to each stream.
 *   alg         GZ_ALG_*; ziggurats read tables from `table_slot`
 *   src         GZ_SRC_*
 *   spare_in, has_spare_in, spare_out, has_spare_out: polar only (else NULL): the cached second deviate per
 *               stream, in and out (engine.py:249-253); NULL in = no spare.
 *   checksum_out  optional u64[n_streams]: xor of the raw bit patterns of the
 *               row (bench.py:174-175 `_checksum_fold`), fused into the fill
 *   psum_out    optional f64[n_streams][4]: per-row power sums
 *               {sum x, sum x^2, sum x^3, sum x^4} for gz_moments_reduce
 *   guard       rejection-loop guard (GZ_DEFAULT_GUARD in the reference)
 *   cuda_stream cudaStream_t (NULL = legacy default stream)
 * Asynchronous: a tripped guard is reported by gz_stream_check().  Exception: one
 * stream of at least 2^15 deviates (the reference's engine.fill_gaussians call
 * shape, no checksum/psum, guard >= 8192) is decoded by the whole GPU
 * (csrc/gz_single.cuh) and synchronises `cuda_stream` once or twice inside the
 * call; gz_set_kernel_policy(1) keeps the plain warp-per-stream schedule.
 */
int gz_fill_gaussians(int alg, int src, int table_slot, int64_t n_streams, int64_t n_per, int64_t ld,
                      const uint64_t* state_in, uint64_t* state_out,
                      const double* spare_in, const uint8_t* has_spare_in,
                      double* spare_out, uint8_t* has_spare_out,
                      double* out, uint64_t* checksum_out, double* psum_out,
                      int64_t guard, void* cuda_stream);

/*
 * Same contract with HOST buffers (the reference-facing call: numpy arrays in
 * and out).  Copies state in, generates, copies deviates and state out, in a
 * chunked pipeline on internal CUDA streams; synchronous; returns the guard
 * status like gz_stream_check().  checksum_out (host, optional) as above.
 */
int gz_fill_gaussians_host(int alg, int src, int table_slot, int64_t n_streams, int64_t n_per,
                           const uint64_t* state_in, uint64_t* state_out,
                           const double* spare_in, const uint8_t* has_spare_in,
                           double* spare_out, uint8_t* has_spare_out,
                           double* out, uint64_t* checksum_out, int64_t guard);

/* Raw 64-bit draws: row s = engine.fill_u64(source_s, row) (engine.py:224-232). */
int gz_fill_u64(int src, int64_t n_streams, int64_t n_per, int64_t ld, const uint64_t* state_in,
                uint64_t* state_out, uint64_t* out, void* cuda_stream);

/*
 * Device-side seeding of `count` streams with ids first_id .. first_id+count-1
 * (scheme GZ_SEED_*); writes the state layout of the scheme's source.
 */
int gz_seed_streams(int scheme, uint64_t master, int64_t first_id, int64_t count, uint64_t* state_out,
                    void* cuda_stream);

/*
 * out[j] = a + b * next_f64_unit() for the first n draws of ONE stream
 * (sources.py:45-47; two roundings), e.g. the config-5 population init
 * x = -5 + 10*u.  state: that stream's state (device, layout of `src`); it is
 * advanced by n draws.
 */
int gz_fill_unit_affine(int src, uint64_t* state, int64_t n, double a, double b, double* out,
                        void* cuda_stream);

/*
 * Fused Gaussian mutation (config 5): for each individual i (a SplitMix64
 * stream), `generations` times, for each gene j in order:
 *   x[i][j] = x[i][j] + sigma[i] * z        (samplers.py:195-200 gaussian_affine,
 *                                             two roundings)
 * with z the next original-ziggurat deviate of stream i (tables in
 * table_slot).  x has row stride ld.  The deviates never touch memory.
 */
int gz_mutate(int table_slot, int64_t n_ind, int64_t n_genes, int64_t ld, const uint64_t* state_in,
              uint64_t* state_out, double* x, const double* sigma, int generations, int64_t guard,
              void* cuda_stream);

/*
 * Deterministic reduction of per-row power sums (gz_fill_gaussians psum_out)
 * to out5 = {n, mean, M2, M3, M4} (central sums; device pointer).  The
 * reduction order depends only on n_rows, so results are bit-reproducible.
 * Feeds the moments of stats.py:232-259 (mean, M2/(n-1), ...).
 */
int gz_moments_reduce(const double* psum, int64_t n_rows, int64_t values_per_row, double* out5,
                      void* cuda_stream);

/*
 * out5 = {n, mean, M2, M3, M4} of a raw f64 buffer x[n] (device pointers), by
 * fixed-order block power sums: the moments of stats.py:232-259 for the
 * `verify` command (cli.py:160-175) over deviates already in HBM.
 */
int gz_moments_buffer(const double* x, int64_t n, double* out5, void* cuda_stream);

/*
 * Layer occupancy of one ziggurat stream (samplers.py:89-93 / 138-142
 * sample_with_occupancy, used by cli.py:185-192): n_calls sequential calls,
 * counts[i] (device u64[n_layers]) = attempts that selected layer i, out
 * (device f64[n_calls], may be NULL) = the deviates, state advanced
 * (state_in/state_out device, 1 or 2 words).  Single-threaded on the device;
 * meant for <= 1e6 calls.  Guard trips are reported by gz_stream_check.
 */
int gz_zig_occupancy(int alg, int src, int table_slot, const uint64_t* state_in, uint64_t* state_out,
                     int64_t n_calls, double* out, uint64_t* counts, int64_t guard, void* cuda_stream);

/*
 * Self-check of the wedge pre-filters' error budget for a table slot: over n
 * random wedge candidates, out3 (device f64[3]) = {max |y_f/y - 1|,
 * max |e_f/e - 1| of the float exp2 filter, max |__expf/e - 1| of the warp
 * kernels' filter}, e = the bit-exact glibc exp.  Both filters fall back to the
 * exact test within 2^-15 of the accept boundary, so each maximum must stay
 * well below 2^-16.  Test infrastructure; not on the generation path.
 */
int gz_wedge_filter_error(int table_slot, int64_t n, uint64_t seed, double* out3, void* cuda_stream);

/*
 * Self-check of the branch-free correctly rounded divide and square root used by
 * the polar drains, against div.rn / sqrt.rn, over n samples of the polar
 * operand domain (s = v1^2 + v2^2 in (0, 1) incl. tiny s; a = -2 log s):
 * counts2 (device u64[2]) = {quotient mismatches, sqrt mismatches}; both must
 * be 0.  Test infrastructure; not on the generation path.
 */
int gz_polar_ops_selftest(int64_t n, uint64_t seed, uint64_t* counts2, void* cuda_stream);

/*
 * One tail_sample(src, r) call (samplers.py:40-57): a deviate beyond r > 0 from the
 * stream at `state` (device, 1 or 2 words, advanced in place) into *out (device).
 * Guard trips are reported by gz_stream_check.
 */
int gz_tail_sample(int src, uint64_t* state, double r, int64_t guard, double* out, void* cuda_stream);

/*
 * Deviates from a scripted source (sources.py ScriptedSource, the reference's test
 * double): the sampler loop of samplers.py run by one device thread over the
 * words[n_words] (device) from *cursor (device, advanced past the consumed
 * words).  n deviates into out (device); polar spares as in gz_fill_gaussians
 * (single values, device).  Reading past the last word reports GZ_ERR_EXHAUSTED
 * through gz_stream_check.  For tests and per-call replay, not throughput.
 */
int gz_fill_scripted(int alg, int table_slot, const uint64_t* words, int64_t n_words, int64_t* cursor, int64_t n,
                     double* out, const double* spare_in, const uint8_t* has_spare_in, double* spare_out,
                     uint8_t* has_spare_out, int64_t guard, void* cuda_stream);

/* gz_tail_sample over scripted words (words/cursor as in gz_fill_scripted). */
int gz_tail_scripted(const uint64_t* words, int64_t n_words, int64_t* cursor, double r, int64_t guard, double* out,
                     void* cuda_stream);

/* xor-fold of u64[n] (device) into *out (device): the global checksum. */
int gz_xor_reduce(const uint64_t* in, int64_t n, uint64_t* out, void* cuda_stream);

/*
 * Synchronise `cuda_stream` and report any rejection-guard trip or CUDA error
 * raised by work enqueued before (then clears it).
 */
int gz_stream_check(void* cuda_stream);

/*
 * On-device verification statistics (device pointers):
 *   gz_hist_edges   counts[k] = #{x : number of edges <= x == k}, k = 0..n_edges
 *                   (numpy.searchsorted(edges, x, side="right"); edges sorted;
 *                   stats.py:276-315 chi_square_gof binning); n_edges < 4096
 *   gz_ks_stat      d_out = {D+, D-} of the sample against 0.5*erfc(-x/sqrt 2)
 *                   (stats.py:262-273); n < 2^31
 *   gz_lowbits_hist counts[c] = #{x : (x & (2^k - 1)) == c}, 1 <= k <= 8
 *                   (stats.py:334-353 low_bits_chi_square)
 */
int gz_hist_edges(const double* x, int64_t n, const double* edges, int n_edges, uint64_t* counts, void* cuda_stream);
int gz_ks_stat(const double* x, int64_t n, double* d_out, void* cuda_stream);
int gz_lowbits_hist(const uint64_t* x, int64_t n, int k_bits, uint64_t* counts, void* cuda_stream);

/* Pinned host memory helpers (for gz_fill_gaussians_host at full PCIe speed). */
int gz_host_alloc(void** ptr, int64_t bytes);
int gz_host_free(void* ptr);

/*
 * Host (CPU) table builder: build_ziggurat_tables (tables.py:107-131) in C++,
 * bit-identical to the reference.  Arrays: x[n+1], ktab[n], wtab[n], ytab[n+1].
 * GZ_ERR_INVALID for a bad layer count, GZ_ERR_GUARD for TableConstructionError.
 */
int gz_build_tables(int n, double* r, double* v, double* x, uint64_t* ktab, double* wtab, double* ytab);

/* Device evaluation of the restated exp (fn = 0) / log (fn = 1) over in[n] -> out[n]
 * (device pointers), for bit-for-bit sweeps against the host libm. */
int gz_libm_eval_device(int fn, const double* in, double* out, int64_t n, void* cuda_stream);

/* Host restatements of glibc exp/log used by the kernels (for CPU sweep tests). */
double gz_libm_exp(double x);
double gz_libm_log(double x);

#ifdef __cplusplus
}
#endif
#endif /* GZ_B200_H */
