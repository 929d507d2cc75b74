/*
 * ttcross.h -- C-ABI of the B200-native dimension-parallel TT-cross quadrature.
 *
 * Method: Dolgov & Savostyanov, "Parallel cross interpolation for high-precision
 * calculation of high-dimensional integrals", arXiv:1903.11554.  The calls
 * follow the paper's problem statement (§4.1): a function on a
 * tensor-product grid (nodes), quadrature weights, a rank cap and a tolerance.  The exact
 * semantics (readings R1-R8) are in DESIGN.md §2.
 *
 * Conventions
 *   - modes m = 0..d-1, interfaces i = 0..d-2 (interface i separates modes <= i | > i);
 *   - every pivot of interface i is stored as a full d-tuple of node indices
 *     PIV[i][s][0..d-1] = (I_{<=i}[s], I_{>i}[s])  (eq. (3));
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
#define TTC_ERR_SINGULAR  3  /* an intersection matrix A(I_{<=i}, I_{>i}) is singular     */
#define TTC_ERR_STATE     4  /* call order violated (e.g. commit without half-sweep)      */

#define TTC_FAMILY_C 0  /* C_d : f = 1/(sum_j (u_j + 1/u_j))^2                 (eq. (9))  */
#define TTC_FAMILY_D 1  /* D_d : f = prod_{i<j} ((u_i-u_j)/(u_i+u_j))^2 / (...)^2 (eq. (10)) */

#define TTC_DIR_LR 0    /* left-to-right half-sweep: updates I_{<=i} (Alg. 3 direction) */
#define TTC_DIR_RL 1    /* right-to-left half-sweep: updates I_{>i}                      */

#define TTC_MEM_HOST   0
#define TTC_MEM_DEVICE 1

#define TTC_MAX_RANK   64   /* rank cap limit                        */
#define TTC_MAX_ENRICH 16   /* random superblock columns per interface */

typedef struct ttc_ctx ttc_ctx;

typedef struct ttc_config {
  int32_t  family;     /* TTC_FAMILY_C or TTC_FAMILY_D                                   */
  int32_t  d;          /* number of modes, 2 <= d <= 2000                                */
  int32_t  n;          /* nodes per mode, 2 <= n <= 4096 (same for every mode)            */
  int32_t  rank_cap;   /* 1 <= rank_cap <= TTC_MAX_RANK                                   */
  int32_t  n_enrich;   /* p, random extra columns per interface and half-sweep, 0..16     */
  int32_t  max_swaps;  /* maxvol swap cap per interface and half-sweep; 0 -> 2*rank_cap   */
  double   tol;        /* cross truncation: stop when |pivot| <= tol * max|fiber|, 0<=tol<1 */
  double   delta;      /* maxvol: swap while max|B| > 1 + delta (Alg. 1), delta >= 0      */
  uint64_t seed;       /* counter-based RNG seed for initial pivots and enrichment        */
  int32_t  rank;       /* this process' index among `world` (interfaces are partitioned)  */
  int32_t  world;      /* number of processes (GPUs) sharing the problem, >= 1            */
} ttc_config;

typedef struct ttc_stats {
  int64_t evals;           /* tensor entries evaluated by this process (fibers + M_i)      */
  int64_t launches;        /* kernels launched by this process since the last reset        */
  int32_t sweeps;          /* full sweeps done since init/reset                            */
  int32_t half_sweeps;     /* half-sweeps done since init/reset                            */
  double  ms_fiber;        /* device time of fiber evaluation kernels (timing enabled)     */
  double  ms_cross;        /* device time of the cross/maxvol kernel                       */
  double  ms_quad;         /* device time of the quadrature kernels                        */
  double  ms_other;        /* device time of the remaining kernels                         */
  int64_t fiber_launches;  /* k_fiber launches since the last reset                        */
  int64_t cross_launches;  /* k_cross launches since the last reset                        */
  int64_t fiber_entries;   /* entries written by k_fiber (device counter)                  */
  int64_t cross_updates;   /* matrix elements updated by k_cross: sum over jobs of
                              nrows*ncols*rank + nrows*rank*swaps (algorithmic)            */
  int64_t cross_steps;     /* pivot + swap steps of k_cross, summed over jobs              */
  int64_t cross_elems;     /* fiber-matrix elements loaded by k_cross (nrows*ncols per job) */
} ttc_stats;

/*
 * tt_cross_init -- create a context, upload the grid, draw the seed-fixed nested initial
 * pivots (R5) and precompute the per-node tables.
 *   out      : receives the context (owned by the caller; free with tt_cross_destroy)
 *   cfg      : problem configuration (copied)
 *   nodes_u  : d*n doubles, row-major [mode][node], u-nodes (u = e^t, R1), > 0
 *   weights  : d*n doubles, quadrature weights [mode][node]
 *   mem_kind : TTC_MEM_HOST (pageable/pinned host arrays, copied H2D on `stream`) or
 *              TTC_MEM_DEVICE (device arrays, copied D2D)
 *   stream   : cudaStream_t to issue all work on (may be NULL)
 * Errors: TTC_ERR_ARG for out-of-range sizes or non-positive nodes, TTC_ERR_CUDA.
 */
int tt_cross_init(ttc_ctx** out, const ttc_config* cfg, const double* nodes_u,
                  const double* weights, int32_t mem_kind, void* stream);

/* tt_cross_reset -- restore the initial pivots (device copy, no host work) and zero the
 * statistics.  Lets a benchmark time repeated solves from the same seed. */
int tt_cross_reset(ttc_ctx* ctx);

/*
 * tt_cross_load_grid -- replace the grid of an existing context (same d and n) and restore
 * the initial pivots (tt_cross_reset).  nodes_u / weights / mem_kind as in tt_cross_init;
 * host arrays should be pinned for an asynchronous copy.  This is the per-problem input
 * upload of the end-to-end path (§4.1: a new function on the tensor grid).
 * Errors: TTC_ERR_ARG (non-positive host node), TTC_ERR_STATE (pending half-sweep).
 */
int tt_cross_load_grid(ttc_ctx* ctx, const double* nodes_u, const double* weights, int32_t mem_kind);

/*
 * tt_solve_launch -- enqueue one whole solve on the context stream, asynchronously:
 * reset to the initial pivots, n_sweeps full sweeps (as tt_cross_sweep) and the quadrature
 * (as tt_integrate_launch).  use_graph != 0 captures this sequence once as a CUDA graph
 * (re-captured when n_sweeps changes) and replays it; the result is bit-identical to the
 * eager sequence.  world == 1 only.  Read the result with tt_integrate_read.
 */
int tt_solve_launch(ttc_ctx* ctx, int32_t n_sweeps, int32_t use_graph);

/*
 * tt_integrate_launch / tt_integrate_read -- tt_integrate split in two: _launch enqueues
 * the quadrature kernels and the device->host copy of the 16-byte result into pinned memory
 * (no synchronisation); _read synchronises the stream and decodes value / log10|value| /
 * sign exactly as tt_integrate.  world == 1 for _launch.  _read returns TTC_ERR_SINGULAR
 * like tt_integrate.
 */
int tt_integrate_launch(ttc_ctx* ctx);
int tt_integrate_read(ttc_ctx* ctx, double* value, double* log10_abs, int32_t* sign);

/*
 * tt_cross_sweep -- n_sweeps full sweeps (L->R half-sweep then R->L half-sweep), each
 * half-sweep dimension-parallel over all interfaces (Alg. 6 + §3.4).  Only for
 * world == 1 (multi-process callers use tt_cross_half_sweep + exchange + commit).
 * Fully asynchronous on the context stream.
 */
int tt_cross_sweep(ttc_ctx* ctx, int32_t n_sweeps);

/*
 * tt_cross_half_sweep -- one half-sweep over the interfaces owned by cfg.rank; results go
 * to the "next" pivot buffer.  After the caller has all-gathered that buffer (see
 * tt_cross_exchange_buffer) it calls tt_cross_commit.  For world == 1 the commit is a
 * no-op exchange.  direction: TTC_DIR_LR or TTC_DIR_RL.
 */
int tt_cross_half_sweep(ttc_ctx* ctx, int32_t direction);
int tt_cross_commit(ttc_ctx* ctx);

/*
 * tt_cross_exchange_buffer -- device pointer of the "next" pivot record buffer:
 * world*chunk records of (1 + rank_cap*d) int32 (record i = [r_i, PIV[i][0][0..d-1], ...]),
 * where chunk = ceil((d-1)/world) interfaces are owned by each rank, rank p owning records
 * [p*chunk, (p+1)*chunk).  *bytes_per_rank = chunk*(1+rank_cap*d)*4.  An in-place
 * all-gather of this buffer completes a half-sweep.
 */
int tt_cross_exchange_buffer(ttc_ctx* ctx, void** dev_ptr, int64_t* bytes_total,
                             int64_t* bytes_per_rank);

/*
 * tt_integrate -- the TT quadrature of the current cross (§4.1):
 *   I = (4/d!) W_0 M_0^{-1} W_1 M_1^{-1} ... W_{d-1},  W_m = sum_a w_{m,a} A(I_{<=m-1}, a, I_{>m}),
 *   M_i = A(I_{<=i}, I_{>i}).
 * Synchronises the stream.  value may be +-0/inf when outside the fp64 range (C_200);
 * log10_abs and sign are always valid (sign 0 for an exactly zero integral).
 * world == 1 only (multi-process: tt_integrate_local / tt_integrate_finish).
 * Errors: TTC_ERR_SINGULAR if some M_i has a zero pivot in LU with partial pivoting.
 */
int tt_integrate(ttc_ctx* ctx, double* value, double* log10_abs, int32_t* sign);

/*
 * Multi-process quadrature: tt_integrate_local computes, for the owned interfaces
 * [kb, ke), the partial product Q_p = prod_{i in [kb,ke)} M_i^{-1} W_{i+1} (rank 0 also
 * prepends W_0) into a device record of (3 + 2*rank_cap*rank_cap) doubles
 * [rows, cols, log2scale, Q_hi (row-major, stride rank_cap), Q_lo] (double-double);
 * tt_integrate_partials_buffer returns the world records buffer to all-gather in place;
 * tt_integrate_finish multiplies the records in rank order.
 * The contraction is carried out in double-double, so the result is the §4.1 product for
 * the given fp64 fiber entries to ~1e-30 * cond (R9).
 */
int tt_integrate_local(ttc_ctx* ctx);
int tt_integrate_partials_buffer(ttc_ctx* ctx, void** dev_ptr, int64_t* bytes_total,
                                 int64_t* bytes_per_rank);
int tt_integrate_finish(ttc_ctx* ctx, double* value, double* log10_abs, int32_t* sign);

/*
 * State inspection (synchronise the stream).
 *   tt_cross_get_state : ranks_out[d-1]; piv_out[(d-1)*rank_cap*d] (slots >= r_i are -1)
 *   tt_cross_get_fiber : fiber of mode m from the last tt_integrate / fiber pass,
 *                        out[rx*ry*n] as [alpha][beta][a]; capacity in doubles.
 *   tt_cross_get_stats : counters and (if enabled) device times.
 */
int tt_cross_get_state(ttc_ctx* ctx, int32_t* ranks_out, int32_t* piv_out);
int tt_cross_get_fiber(ttc_ctx* ctx, int32_t mode, double* out, int64_t capacity,
                       int32_t* rx, int32_t* ry);
int tt_cross_get_stats(ttc_ctx* ctx, ttc_stats* out);

/* tt_cross_get_kernel_time -- per-kernel launch count and accumulated device time (ms,
 * timing enabled) for kernel id kid in [0, 13): 0 k_prep_nodes, 1 k_enrich,
 * 2 k_frozen_sides, 3 k_frozen_q, 4 k_frozen_lr, 5 k_fiber, 6 k_cross, 7 k_commit, 8 k_wsum,
 * 9 k_intersection, 10 k_solve, 11 k_chain, 12 k_finish.  *name is a static string.
 * Errors: TTC_ERR_ARG for kid out of range. */
int tt_cross_get_kernel_time(ttc_ctx* ctx, int32_t kid, const char** name, int64_t* launches, double* ms);

/* tt_cross_set_timing -- 1: bracket every kernel launch with CUDA events on the context
 * stream and accumulate per-class device time (ttc_stats.ms_*); 0: off (default). */
int tt_cross_set_timing(ttc_ctx* ctx, int32_t enable);

/* tt_cross_destroy -- free all device and host memory of the context (NULL is a no-op). */
void tt_cross_destroy(ttc_ctx* ctx);

/* Thread-local description of the last error (never NULL). */
const char* tt_last_error(void);

/* Library build identifier (compile arch, version). */
const char* tt_build_info(void);

#ifdef __cplusplus
}
#endif
#endif /* TTCROSS_H */
