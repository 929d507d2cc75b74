/*
 * ttcross.h -- C-ABI of the B200-native dimension-parallel TT-cross quadrature.
 *
 * Method: Dolgov & Savostyanov, "Parallel cross interpolation for high-precision
 * calculation of high-dimensional integrals", arXiv:1903.11554.  The calls
 * follow the paper's problem statement (§4.1): a function on a
 * tensor-product grid (nodes), quadrature weights, a rank cap and a tolerance.  The cross is
 * the dimension-parallel greedy algorithm of Alg. 6 (lines 624-641) with the pivot search of
 * Alg. 2 (lines 231-253); the integral is the §4.1 product of 2d-1 matrices (lines 689-693).
 * The exact semantics (readings R1-R9) are in DESIGN.md §2.
 *
 * Conventions
 *   - modes m = 0..d-1, interfaces k = 0..d-2 (interface k separates modes <= k | > k);
 *   - pivot s of interface k is stored as a full d-tuple of node indices
 *     PIV[k][s][0..d-1] = (I_{<=k}[s], I_{>k}[s])  (eq. (3)) and its
 *     parents PAR[k][s] = (alpha, beta): the slot of its left part in I_{<=k-1} and of its
 *     right part in I_{>k+1} (nestedness, eq. (4));
 *   - pivot sets only grow (Alg. 6 line 4): slots never move once written;
 *   - all functions return TTC_OK (0) or an error code; tt_last_error() returns a
 *     thread-local message.  Any CUDA error is reported, never silently recovered; there
 *     is no CPU fallback.
 *   - all device work is issued on the stream given to tt_cross_init (NULL = legacy
 *     default stream); functions that return host data synchronise that stream.
 */
#ifndef TTCROSS_H
#define TTCROSS_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define TTC_OK            0
#define TTC_ERR_ARG       1  /* invalid argument / unsupported size                       */
#define TTC_ERR_CUDA      2  /* a CUDA runtime call or kernel failed                      */
#define TTC_ERR_SINGULAR  3  /* an intersection matrix A(I_{<=k}, I_{>k}) is singular     */
#define TTC_ERR_STATE     4  /* call order violated (e.g. commit without a local sweep)   */

/* t-form (BASELINE.json configs): nodes are u = e^t, integral prefactor 4/d!              */
#define TTC_FAMILY_C 0  /* C_d : f = 1/(sum_j (u_j + 1/u_j))^2                 (eq. (9))  */
#define TTC_FAMILY_D 1  /* D_d : f = prod_{i<j} ((u_i-u_j)/(u_i+u_j))^2 / (...)^2 (eq. (10)) */
/* x-form (eq. (9)-(11), lines 843-851): the d-1 variables x_2..x_d in (0,1) are the
 * modes (cfg.d = d-1), nodes are x (e.g. Gauss-Legendre), integral prefactor 2              */
#define TTC_FAMILY_CX 2 /* C_d = 2 int B_d                                                    */
#define TTC_FAMILY_DX 3 /* D_d = 2 int A_d B_d                                                */
#define TTC_FAMILY_EX 4 /* E_d = 2 int A_d                                                    */

#define TTC_MEM_HOST   0
#define TTC_MEM_DEVICE 1

#define TTC_MAX_RANK    64    /* rank cap limit                     */
#define TTC_MAX_SAMPLES 1024  /* random samples per Alg. 2 step      */

typedef struct ttc_ctx ttc_ctx;

typedef struct ttc_config {
  int32_t  family;     /* TTC_FAMILY_C, _D (t-form) or TTC_FAMILY_CX, _DX, _EX (x-form)     */
  int32_t  d;          /* number of modes of the tensor, 2 <= d <= 2000                   */
  int32_t  n;          /* nodes per mode, 2 <= n <= 4096 (same for every mode)             */
  int32_t  rank_cap;   /* 1 <= rank_cap <= TTC_MAX_RANK                                    */
  int32_t  n_samples;  /* |L| of Alg. 2 line 1 (random superblock entries), 1..1024        */
  int32_t  rook_iters; /* column+row rounds of the rook search (Alg. 2 lines 2-5), 0..64   */
  double   tol;        /* add a pivot only if |E(i*,j*)| > tol * max|A| at the pivots, [0,1) */
  uint64_t seed;       /* counter-based RNG seed of the first pivot and the samples        */
  int32_t  rank;       /* this process' index among `world` (superblocks are partitioned)  */
  int32_t  world;      /* number of processes (GPUs) sharing the problem, >= 1             */
  int32_t  fold_weights; /* 1: cross on B = w x ... x w * f and contract with unit weights
                          (§4.1); x-form families only; 0: off   */
} ttc_config;

typedef struct ttc_stats {
  int64_t evals;           /* tensor entries evaluated since the last reset (all kernels)  */
  int64_t launches;        /* kernels launched since the last reset                        */
  int32_t sweeps;          /* Alg. 6 sweeps committed since the last reset                 */
  int32_t pad;
  double  ms_fiber;        /* device time: quadrature fibers (k_frozen_*, k_fiber)          */
  double  ms_cross;        /* device time: k_sweep (tables, u/v extension, Alg. 2 search)   */
  double  ms_quad;         /* device time: quadrature contraction kernels                  */
  double  ms_other;        /* device time: init kernels                                    */
  int64_t fiber_entries;   /* entries written by k_fiber (quadrature fibers)               */
  int64_t sb_entries;      /* superblock entries evaluated by k_sweep                      */
  int64_t sb_updates;      /* multiply-subtract terms u_t(x) v_t(y) of those kernels        */
  int64_t rook_steps;      /* column+row rounds of the rook searches                        */
  int64_t ext_entries;     /* ... of which by the u/v extension phase (batched fibers)      */
  int64_t ext_updates;     /* multiply-subtract terms of the extension phase                */
  int64_t ring_steps;      /* (CTA, rook step) pairs that streamed the u/v factors from HBM
                              through the shared-memory ring (the non-cached launch shape)  */
} ttc_stats;

/*
 * tt_cross_init -- create a context, upload the grid, precompute the per-node tables and draw
 * the seed-fixed rank-1 start (R5; 64 entry evaluations, redrawn by every reset /
 * solve -- not counted in the per-solve statistics, which tt_cross_reset zeroes).
 *   out      : receives the context (owned by the caller; free with tt_cross_destroy)
 *   cfg      : problem configuration (copied)
 *   nodes_u  : d*n doubles, row-major [mode][node], > 0: u-nodes (u = e^t, R1) for
 *              the t-form families, x-nodes in (0,1) for the x-form families
 *   weights  : d*n doubles, quadrature weights [mode][node]
 *   mem_kind : TTC_MEM_HOST (pageable/pinned host arrays, copied H2D on `stream`) or
 *              TTC_MEM_DEVICE (device arrays, copied D2D).  The copies are asynchronous:
 *              the caller keeps nodes_u / weights alive and unmodified until the stream
 *              has completed them (any synchronising call of this library does that).
 *   stream   : cudaStream_t to issue all work on (may be NULL)
 * Errors: TTC_ERR_ARG for out-of-range sizes or non-positive host nodes, TTC_ERR_CUDA.
 */
int tt_cross_init(ttc_ctx** out, const ttc_config* cfg, const double* nodes_u,
                  const double* weights, int32_t mem_kind, void* stream);

/*
 * tt_cross_load_grid -- replace the grid of an existing context (same d and n) and reset.
 * nodes_u / weights / mem_kind as in tt_cross_init; host arrays should be pinned for an
 * asynchronous copy.  This is the per-problem input upload of the end-to-end path.
 * Errors: TTC_ERR_ARG (non-positive host node), TTC_ERR_STATE (uncommitted sweep).
 */
int tt_cross_load_grid(ttc_ctx* ctx, const double* nodes_u, const double* weights, int32_t mem_kind);

/* tt_cross_reset -- draw the rank-1 start of the loaded grid again (k_init_pivot: first argmax
 * |A| over the seeded samples) and reset every interface to it (device kernels, asynchronous),
 * zero the statistics.  Lets a benchmark time repeated whole solves from the same seed. */
int tt_cross_reset(ttc_ctx* ctx);

/*
 * tt_cross_sweep -- n_sweeps dimension-parallel sweeps (Alg. 6): every superblock
 * adds at most one pivot found by Alg. 2 from the index sets of the previous sweep.
 * world == 1 only (multi-process callers use tt_cross_sweep_local + exchange + commit).
 * When every superblock's thread-block cluster fits on the device at once (see
 * tt_cross_get_launch_shape), the n sweeps run as ONE persistent launch in which superblock k
 * starts sweep s as soon as superblocks k-1 and k+1 have published sweep s-1 (the
 * neighbour-only exchange of Alg. 6 lines 6-8, through release/acquire flags); otherwise one
 * launch per sweep.  Results are identical either way.  A neighbour wait longer than ~2 s
 * (clusters not co-resident, e.g. under MPS or beside concurrent kernels) abandons the launch
 * and is reported as TTC_ERR_CUDA by the next synchronising call (tt_integrate*,
 * tt_cross_get_state, tt_cross_get_stats); the cross is then incomplete.
 * Fully asynchronous on the context stream.
 */
int tt_cross_sweep(ttc_ctx* ctx, int32_t n_sweeps);

/*
 * tt_cross_sweep_local -- one sweep over the superblocks owned by cfg.rank; the updated
 * records go to the "next" record buffer.  After the caller has all-gathered that buffer
 * (tt_cross_exchange_buffer) it calls tt_cross_commit.  For world == 1 no exchange is needed.
 */
int tt_cross_sweep_local(ttc_ctx* ctx);
int tt_cross_commit(ttc_ctx* ctx);

/*
 * tt_cross_exchange_buffer -- device pointer of the exchange buffer of one sweep.  A record is
 * (1 + rank_cap*d + 2*rank_cap) int32: [r_k, PIV[k][0..cap)[0..d), PAR[k][0..cap)[0..2)].
 * Interfaces are partitioned in balanced contiguous blocks (Alg. 6 line 1): with
 * q = (d-1) / world, m = (d-1) % world, rank p owns [kb_p, kb_{p+1}), kb_p = p*q + min(p, m).
 * world > 1: world slots of chunk = ceil((d-1)/world) records; tt_cross_sweep_local writes
 * this rank's records of [kb_p, kb_{p+1}) to the start of slot p; an in-place all-gather of
 * the slots (*bytes_per_rank = chunk*record bytes) followed by tt_cross_commit completes the
 * sweep (Alg. 6 lines 6-8).  The buffer stays at the same address for the life of the context.
 * world == 1: the "next" records of all d-1 interfaces (no exchange needed); commit swaps the
 * two record buffers, so re-query the pointer after every commit.
 */
int tt_cross_exchange_buffer(ttc_ctx* ctx, void** dev_ptr, int64_t* bytes_total,
                             int64_t* bytes_per_rank);

/*
 * Cross-GPU wavefront (world > 1; Alg. 6 lines 6-8, lines 604-608: after a sweep a
 * process sends its new pivots to its neighbouring processes only).  Instead of one launch and
 * one all-gather per sweep (tt_cross_sweep_local / exchange / commit), every rank runs its
 * superblocks' sweeps as ONE persistent launch, as tt_cross_sweep does on one GPU: a rank's
 * first and last superblock publish their new pivot record, rank and done flag also into the
 * neighbour rank's copies through CUDA IPC peer memory (NVLink), the flag with a system-scope
 * release, and wait on the neighbour rank's flag with a system-scope acquire.  The pivots are
 * those of tt_cross_sweep on one GPU, bit for bit.
 *
 * tt_cross_peer_handles -- writes TTC_PEER_HANDLE_BYTES bytes to `out` (host): the CUDA IPC
 *   handles of this context's record buffer, rank ring and done flags, for the neighbour ranks
 *   (exchange them with any host collective).  world > 1, else TTC_ERR_STATE.
 * tt_cross_peer_open -- maps the left (rank-1) and right (rank+1) neighbours' handles (as written
 *   by their tt_cross_peer_handles; host pointers, read during the call).  `left` must be NULL
 *   exactly when rank == 0, `right` exactly when rank == world-1 (TTC_ERR_ARG).  Needs a t-form
 *   family (TTC_FAMILY_C / D) with every owned superblock's cluster resident at once
 *   (tt_cross_get_launch_shape bit 2), else TTC_ERR_STATE.  Synchronises the context stream.  Mappings are closed by tt_cross_destroy.
 * tt_cross_sweep_peer -- n_sweeps >= 1 sweeps of the owned superblocks (one persistent launch),
 *   then this rank's records to its slot of the exchange buffer; the caller all-gathers the
 *   exchange buffer (tt_cross_exchange_buffer) and calls tt_cross_commit, which advances the
 *   sweep count by n_sweeps.  All ranks must call it with the same n_sweeps, and no rank may
 *   launch it before every rank's previous reset / commit has completed on its device (the
 *   neighbours write into this rank's buffers): put a device-side barrier (e.g. a one-element
 *   NCCL all-reduce) after tt_cross_reset and after tt_cross_commit.  TTC_ERR_STATE after a
 *   tt_cross_sweep_local since the last reset (its neighbour flags are not published).  A
 *   neighbour wait longer than ~2 s abandons the launch (reported as by tt_cross_sweep).
 *   Asynchronous on the context stream.
 *
 * Loopback test of the same code path on one GPU (world == 1, persistent launch):
 * tt_cross_set_loopback -- boundary b in [1, d-2] splits the interfaces as if [0, b) and
 *   [b, d-1) were on two ranks: superblocks b-1 and b exchange flag and rank through a mirror
 *   buffer (system-scope release / acquire) and publish their records into the mirror's record
 *   copy; b = 0 turns it off.  Resets the context to the rank-1 start (tt_cross_reset).
 * tt_cross_get_loopback -- the mirror after the last sweep (synchronising): the record copy
 *   (the layout of tt_cross_exchange_buffer's world == 1 records, d-1 records), the rank ring
 *   [d-1][2] (rank of interface k after sweep s at [k][s & 1]) and the done flags [d-1].
 */
#define TTC_PEER_HANDLE_BYTES 192
int tt_cross_peer_handles(ttc_ctx* ctx, void* out, int64_t capacity);
int tt_cross_peer_open(ttc_ctx* ctx, const void* left, const void* right);
int tt_cross_sweep_peer(ttc_ctx* ctx, int32_t n_sweeps);
int tt_cross_set_loopback(ttc_ctx* ctx, int32_t boundary);
int tt_cross_get_loopback(ttc_ctx* ctx, int32_t* rec_out, int32_t* ring_out, int32_t* done_out);

/*
 * tt_solve_launch -- enqueue one whole solve on the context stream, asynchronously: reset to
 * the rank-1 start, n_sweeps sweeps (as tt_cross_sweep) and the quadrature (as
 * tt_integrate_launch).  use_graph != 0 captures this sequence once as a CUDA graph
 * (re-captured when n_sweeps changes) and replays it; the result is bit-identical to the
 * eager sequence.  world == 1 only.  Read the result with tt_integrate_read.
 */
int tt_solve_launch(ttc_ctx* ctx, int32_t n_sweeps, int32_t use_graph);

/*
 * tt_integrate -- the TT quadrature of the current cross (§4.1):
 *   I = (4/d!) W_0 M_0^{-1} W_1 M_1^{-1} ... W_{d-1},  W_m = sum_a w_{m,a} A(I_{<=m-1}, a, I_{>m}),
 *   M_k = A(I_{<=k}, I_{>k}).
 * Synchronises the stream.  value may be +-0/inf when outside the fp64 range (C_200);
 * log10_abs and sign are always valid (sign 0 for an exactly zero integral).
 * world == 1 only (multi-process: tt_integrate_local / tt_integrate_finish).
 * The contraction runs in double-double: the result is the §4.1 product for the given fp64
 * entries to ~1e-30 * cond (R9).
 * Errors: TTC_ERR_SINGULAR if some M_k has a zero pivot in LU with partial pivoting.
 */
int tt_integrate(ttc_ctx* ctx, double* value, double* log10_abs, int32_t* sign);

/*
 * tt_integrate_launch / tt_integrate_read -- tt_integrate split in two: _launch enqueues
 * the quadrature kernels and the device->host copy of the 20-byte result into pinned memory
 * (no synchronisation); _read synchronises the stream and decodes value / log10|value| /
 * sign exactly as tt_integrate.  world == 1 for _launch.
 */
int tt_integrate_launch(ttc_ctx* ctx);
int tt_integrate_read(ttc_ctx* ctx, double* value, double* log10_abs, int32_t* sign);

/*
 * Multi-process quadrature: tt_integrate_local computes, for the owned interfaces
 * [kb, ke), the partial product Q_p = prod_{k in [kb,ke)} M_k^{-1} W_{k+1} (rank 0 also
 * prepends W_0) into a device record of (3 + 2*rank_cap*rank_cap) doubles
 * [rows, cols, log2scale, Q_hi (row-major, stride rank_cap), Q_lo] (double-double);
 * tt_integrate_partials_buffer returns the world records buffer to all-gather in place;
 * tt_integrate_finish multiplies the records in rank order and returns the result.
 */
int tt_integrate_local(ttc_ctx* ctx);
int tt_integrate_partials_buffer(ttc_ctx* ctx, void** dev_ptr, int64_t* bytes_total,
                                 int64_t* bytes_per_rank);
int tt_integrate_finish(ttc_ctx* ctx, double* value, double* log10_abs, int32_t* sign);

/*
 * State inspection (synchronise the stream).
 *   tt_cross_get_state : ranks_out[d-1]; piv_out[(d-1)*rank_cap*d] (slots >= r_k are -1);
 *                        par_out[(d-1)*rank_cap*2] (may be NULL)
 *   tt_cross_get_fiber : fiber A(I_{<=m-1}, i_m, I_{>m}) of mode m of the current cross,
 *                        evaluated on demand by the quadrature's own fiber kernel
 *                        (k_fiber_wsum storing the entries it contracts; it also refreshes
 *                        W_m, see tt_cross_get_wsum),
 *                        out[rx*ry*n] as [alpha][beta][a]; capacity in doubles; out NULL:
 *                        only rx, ry.  TTC_ERR_STATE while a local sweep is uncommitted.
 *   tt_cross_get_stats : counters and (if enabled) device times.
 */
int tt_cross_get_state(ttc_ctx* ctx, int32_t* ranks_out, int32_t* piv_out, int32_t* par_out);
int tt_cross_get_fiber(ttc_ctx* ctx, int32_t mode, double* out, int64_t capacity,
                       int32_t* rx, int32_t* ry);
int tt_cross_get_stats(ttc_ctx* ctx, ttc_stats* out);

/*
 * tt_cross_get_wsum -- the weighted fiber sums W_m[alpha][beta] = sum_a w_{m,a}
 * A(I_{<=m-1}[alpha], a, I_{>m}[beta]) (§4.1) of mode m as the last
 * tt_integrate / tt_integrate_local / tt_cross_get_fiber of this context computed them, in
 * double-double: hi_out[rx*ry], lo_out[rx*ry] row-major [alpha][beta] (value = hi + lo).
 * capacity in doubles per array; hi_out NULL: only rx, ry.  Synchronises the stream.
 * Only modes this rank contracts are defined (world > 1: modes kb+1..ke, and 0 on rank 0).
 * Errors: TTC_ERR_ARG (mode out of range, buffer too small), TTC_ERR_STATE (pending sweep).
 */
int tt_cross_get_wsum(ttc_ctx* ctx, int32_t mode, double* hi_out, double* lo_out, int64_t capacity,
                      int32_t* rx, int32_t* ry);

/* tt_cross_get_kernel_time -- per-kernel launch count and accumulated device time (ms,
 * timing enabled) since the last reset, for kernel id kid in [0, 13): 0 k_prep_nodes,
 * 1 k_init_pivot, 2 k_init_records, 3 k_sweep, 4 k_frozen_sides, 5 k_frozen_q,
 * 6 k_frozen_lr, 7 k_fiber, 8 k_wsum, 9 k_intersection, 10 k_solve, 11 k_chain, 12 k_finish.
 * *name is a static string.  Errors: TTC_ERR_ARG for kid out of range. */
int tt_cross_get_kernel_time(ttc_ctx* ctx, int32_t kid, const char** name, int64_t* launches, double* ms);

/* tt_cross_get_launch_shape -- the k_sweep launch chosen at init: CTAs per superblock cluster,
 * threads per CTA, flags in *cached (bit 0: the rook search keeps its rows/columns in shared
 * memory; bit 1: tt_cross_sweep runs the persistent wavefront launch; bit 2: the cross-GPU
 * wavefront is available -- a t-form family with every owned superblock's cluster resident at
 * once, tt_cross_peer_open's condition), and the dynamic shared
 * memory per CTA (bytes).  Any pointer may be NULL. */
int tt_cross_get_launch_shape(ttc_ctx* ctx, int32_t* cluster, int32_t* threads, int32_t* cached,
                              int64_t* smem_bytes);

/* tt_cross_get_phase_times -- with timing enabled, k_sweep's first CTA of one owned
 * superblock (the first, or the one environment variable TTC_PHASE_JOB names when the context
 * is created) accumulates its phases (globaltimer): us_out[0..6] = microseconds spent in
 * [neighbour wait of the persistent kernel, tables, u/v extension, samples, rook search, final
 * column/row + append, exit barrier], us_out[7] = sweeps measured, us_out[8..11] = [column
 * evaluation, column argmax (CTA + cluster), row evaluation, row argmax] summed over the search
 * steps, us_out[12..13] = [raw entries, recurrence] of the extension's row tiles (written when
 * count >= 14); with count >= 14 + 16*256 also a per-sweep log: us_out[14 + 16*s + p] = slot p
 * (0..13 as above) for sweep s < 256 alone, except slot 7 = the sweep's rook rounds.  count >= 12.
 * Reset by tt_cross_set_timing(1).  Diagnostics: only a library compiled with
 * -DTTC_PHASE_CLOCKS=1 keeps the clocks (tools/probe_phases.py builds one); the default build
 * returns TTC_ERR_STATE. */
int tt_cross_get_phase_times(ttc_ctx* ctx, double* us_out, int32_t count);

/* tt_cross_set_timing -- 1: bracket every kernel launch with CUDA events on the context
 * stream and accumulate per-kernel device time; 0: off (default).  Ignored while a CUDA
 * graph is captured (tt_solve_launch with use_graph). */
int tt_cross_set_timing(ttc_ctx* ctx, int32_t enable);

/* tt_cross_destroy -- free all device and host memory of the context (NULL is a no-op). */
void tt_cross_destroy(ttc_ctx* ctx);

/* Thread-local description of the last error (never NULL). */
const char* tt_last_error(void);

/* tt_selftest_division -- diagnostics for the division the u/v extension uses with a
 * divisor known in advance (u_t(x_t)): q_pre[i] = the hoisted-reciprocal quotient,
 * q_ieee[i] = __ddiv_rn(a[i], b[i]); the two must agree bit for bit.
 * a, b, q_pre, q_ieee: DEVICE pointers to n doubles (caller-owned); synchronises the device.
 * TTC_ERR_ARG on n < 0 or a NULL pointer, TTC_ERR_CUDA on a launch failure. */
int tt_selftest_division(const double* a, const double* b, double* q_pre, double* q_ieee, int64_t n);

/* Library build identifier (compile arch, version). */
const char* tt_build_info(void);

#ifdef __cplusplus
}
#endif
#endif /* TTCROSS_H */
