// ttc_greedy.cuh -- the dimension-parallel greedy cross (Alg. 6 with Alg. 2).
//
// One sweep updates every owned interface k from the index sets of the previous sweep
// (§3.4 relaxation).  Interface k works on its superblock
//   A_k(x, y) = A(I_{<=k-1}[alpha], a, b, I_{>k+1}[beta]),  x = alpha*n + a,  y = beta*n + b
// (Alg. 5), an (r_{k-1} n) x (n r_{k+1}) matrix, and keeps its cross in the
// incomplete-LU form A~(x, y) = sum_t u_t(x) v_t(y) (oracle/cross.py).
//
//   k_init_pivot / k_init_records : the rank-1 start (first argmax |A| over seeded samples)
//   k_sweep                       : one thread-block cluster per superblock, three phases
//                                   separated by cluster barriers:
//     1. factor tables of the superblock entries for the rows / columns that are new this
//        sweep (the frozen left/right pivot coordinates, staged once per sweep);
//     2. u_s(x) / v_s(y) of the existing pivots on the new rows / columns -- the batched
//        fiber evaluation of the sweep;
//     3. Alg. 2: random samples (line 1), rook search (lines 2-5), append the new pivot
//        (Alg. 6 line 4) to the next record buffer.
//
// Arithmetic is bit-identical to the oracle (R3, R4): entries are exactly rounded
// functions of the coordinate multiset (any factorisation gives the same bits), every sum
// over t runs t = 0, 1, ... with __dmul_rn / __dsub_rn (no FMA), argmax = first maximiser.
#pragma once
#include <cooperative_groups.h>
#include "ttc_common.cuh"

namespace cg = cooperative_groups;

namespace ttc {

#define N_INIT 64
#ifndef TTC_PHASE_CLOCKS
// per-phase device clocks of one superblock (tt_cross_get_phase_times): a diagnostics build
// only (tools/probe_phases.py builds build/libttcross_clocks.so) -- the clock code's live
// registers cost the sweep kernel spills even when the clocks are off (D_20 14.52 vs 14.21 ms,
// C_200 4.81 vs 4.61, profiles/r02t_phase_clocks.log)
#define TTC_PHASE_CLOCKS 0
#endif
#define N_INIT_WARPS 32
#define INIT_UQ 128   // coordinates per sample staged in shared memory by init_entry_warp
#define TTC_MAX_SAMPLES 1024

// ---------------------------------------------------------------------------------------
// direct O(d^2) entry of a full tuple given coordinate by coordinate (init only)
// ---------------------------------------------------------------------------------------
__device__ __forceinline__ int init_coord(const DevCtx& c, int q, int j) {
  return (int)(splitmix64(c.seed, draw_ctr(0, c.d, 0, q * c.d + j)) % (uint64_t)c.n);
}

__device__ double init_entry(const DevCtx& c, int q) {
  const int d = c.d, n = c.n;
  if (c.family >= 2) return x_entry_dyn(c.family, c.u, c.wf, d, n, [&](int j) { return init_coord(c, q, j); });
  ESum s = esum_zero();
  for (int j = 0; j < d; ++j) {
    const int t = init_coord(c, q, j);
    esum_add(s, c.chi[j * n + t], c.clo[j * n + t]);
  }
  const double S = esum_round(s);
  const double SS = __dmul_rn(S, S);
  if (c.family == 0) return __drcp_rn(SS);
  DDE p = dde_one();
  for (int i = 0; i < d; ++i) {
    const double ui = c.u[i * n + init_coord(c, q, i)];
    for (int j = i + 1; j < d; ++j) dde_mul_d(p, rho_ool(ui, c.u[j * n + init_coord(c, q, j)]));
  }
  return dde_div(p, SS);
}

// init_entry by one warp (t-form families): the lanes split the coordinates (exact integer
// sums) and the d(d-1)/2 rho pairs (partial double-double products, rho on its branch-free
// fast path), then a shuffle tree -- the product is rounded once, so the grouping gives the
// entry of init_entry (R3); lane 0's value is returned on every lane.  (A thread per
// sample ran its 190 IEEE-division pairs of D_20 one after another: ~110 us per solve.)
__device__ double init_entry_warp(const DevCtx& c, int q) {
  const int lane = threadIdx.x & 31;
  const int d = c.d, n = c.n;
  if (c.family >= 2) {
    const double v = lane == 0 ? init_entry(c, q) : 0.0;
    return __shfl_sync(0xffffffffu, v, 0);
  }
  ESum s = esum_zero();
  for (int j = lane; j < d; j += 32) {
    const int t = init_coord(c, q, j);
    esum_add(s, c.chi[j * n + t], c.clo[j * n + t]);
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    s.h += __shfl_xor_sync(0xffffffffu, s.h, o);
    s.l += __shfl_xor_sync(0xffffffffu, s.l, o);
  }
  const double S = esum_round(s);
  const double SS = __dmul_rn(S, S);
  if (c.family == 0) return __drcp_rn(SS);
  DDE p = dde_one();
  // the sample's node values, gathered once per warp (one round of loads instead of a
  // dependent pair of loads per rho pair)
  __shared__ double s_uq[N_INIT_WARPS][INIT_UQ];
  double* uq = s_uq[threadIdx.x >> 5];
  const bool staged = d <= INIT_UQ;
  if (staged)
    for (int j = lane; j < d; j += 32) uq[j] = c.u[j * n + init_coord(c, q, j)];
  __syncwarp();
  for (int e = lane; e < d * d; e += 32) {
    const int i = e / d, j = e - i * d;
    if (j <= i) continue;
    const double ui = staged ? uq[i] : c.u[i * n + init_coord(c, q, i)];
    const double uj = staged ? uq[j] : c.u[j * n + init_coord(c, q, j)];
    bool ok;
    double rr = rho_fast(ui, uj, ok);
    if (!ok) rr = rho_ool(ui, uj);
    dde_mul_d(p, rr);
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    DDE y;
    y.hi = __shfl_xor_sync(0xffffffffu, p.hi, o);
    y.lo = __shfl_xor_sync(0xffffffffu, p.lo, o);
    y.e = __shfl_xor_sync(0xffffffffu, p.e, o);
    y.pad = 0;
    dde_mul(p, y);
  }
  const double v = lane == 0 ? dde_div(p, SS) : 0.0;
  __syncwarp();   // (uq is rewritten by this warp's next sample)
  return __shfl_sync(0xffffffffu, v, 0);
}

// one block of N_INIT_WARPS warps: t0 = first argmax |A| over the N_INIT seeded samples (a warp
// per sample) -> t0buf[d], A(t0) -> p0val.  Part of loading a grid (tt_cross_init /
// tt_cross_load_grid) and of every tt_cross_reset.
__global__ void __launch_bounds__(N_INIT_WARPS * 32) k_init_pivot(DevCtx c, int* t0buf) {
  __shared__ double sv[N_INIT], sgn[N_INIT];
  __shared__ int best;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int q = warp; q < N_INIT; q += N_INIT_WARPS) {
    const double v = init_entry_warp(c, q);
    if (lane == 0) {
      sgn[q] = v;
      sv[q] = fabs(v);
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    int b = 0;
    for (int t = 1; t < N_INIT; ++t)
      if (sv[t] > sv[b]) b = t;
    best = b;
    *c.p0val = sgn[b];  // A(t0): u_0(x_0) of every superblock at the first sweep
  }
  __syncthreads();
  for (int j = threadIdx.x; j < c.d; j += blockDim.x) t0buf[j] = init_coord(c, best, j);
}

// rank-1 records (t0, parents (0, 0)) for every interface + fresh superblock state
__global__ void k_init_records(DevCtx c, const int* t0buf, int nrec, int n_owned) {
  const int i = blockIdx.x;
  const int d = c.d, cap = c.cap;
  if (i < nrec) {
    int* R = c.rec_cur + (long long)i * c.RS;
    for (int t = threadIdx.x; t < c.RS; t += blockDim.x) {
      int v = -1;
      if (t == 0) v = (i < d - 1) ? 1 : 0;
      else if (t <= d) v = (i < d - 1) ? t0buf[t - 1] : -1;
      else if (t == 1 + cap * d || t == 2 + cap * d) v = 0;  // parents of slot 0
      R[t] = v;
    }
  }
  if (i < d - 1 && threadIdx.x == 0) {
    c.rank_ring[2 * i] = 1;
    c.rank_ring[2 * i + 1] = 1;
    c.done[i] = 0;
    if (c.loopback) {   // the loopback test's mirror of a neighbour rank's copies
      c.rring[2 * i] = 1;
      c.rring[2 * i + 1] = 1;
      c.rdone[i] = 0;
    }
  }
  if (c.loopback && i < nrec)
    for (int t = threadIdx.x; t < c.RS; t += blockDim.x) c.prec[0][(long long)i * c.RS + t] = c.rec_cur[(long long)i * c.RS + t];
  if (i < n_owned && threadIdx.x == 0) {
    c.sbstate[i * 4 + 0] = 0;
    c.sbstate[i * 4 + 1] = 0;
    c.sbstate[i * 4 + 2] = 0;
    c.sbstate[i * 4 + 3] = 0;
    c.praw_max[i] = -1.0;
  }
  if (i == 0 && threadIdx.x == 0) c.flags[1] = 0;
}

// Balanced superblock partition (Alg. 6 line 1): rank p owns the interfaces
// [kb_p, ke_p), the first (d-1) mod world ranks one more than the others.
__host__ __device__ __forceinline__ int part_begin(int nif, int world, int p) {
  const int base = nif / world, rem = nif % world;
  return p * base + (p < rem ? p : rem);
}

// multi-process commit: rank p's slot of the all-gathered exchange buffer (its records of
// interfaces [kb_p, ke_p), slot stride `chunk` records) -> the current records; one block per rank
__global__ void k_unpack_records(const int* xbuf, int* rec_cur, int nif, int world, int chunk, int RS) {
  const int p = blockIdx.x;
  const int kb = part_begin(nif, world, p), ke = part_begin(nif, world, p + 1);
  const int* src = xbuf + (long long)p * chunk * RS;
  int* dst = rec_cur + (long long)kb * RS;
  for (long long t = threadIdx.x; t < (long long)(ke - kb) * RS; t += blockDim.x) dst[t] = src[t];
}

// CX[alpha][beta] by one warp: lanes split the k * (d-k-2) cross pairs (i < k, j > k+1), each
// lane a partial double-double product, then the shuffle tree -- the product is rounded once
// later, so any grouping gives the same entries (R3).  (A thread per entry ran the
// whole chain alone: D_20's middle superblocks have ~80 pairs per entry, ~24k cycles.)
__device__ void sb_cx_table_warp(const DevCtx& c, int job, int al, int be) {
  const int k = c.kb + job, d = c.d, n = c.n;
  const int lane = threadIdx.x & 31;
  DDE p = dde_one();
  int act = 0;   // lanes holding a factor (the tree's levels beyond combine identities: skipped)
  if (k > 0 && k < d - 2) {
    const int* TX = rec_piv(c.rec_cur, c.RS, k - 1) + (long long)al * d;
    const int* TY = rec_piv(c.rec_cur, c.RS, k + 1) + (long long)be * d;
    const int nj = d - k - 2, np = k * nj;
    act = min(32, np);
    for (int q = lane; q < np; q += 32) {
      const int i = q / nj, j = k + 2 + (q - i * nj);
      const double xi = c.u[i * n + TX[i]], yj = c.u[j * n + TY[j]];
      bool ok;
      double rr = rho_fast(xi, yj, ok);   // (the IEEE division's bits; its slow path out of line)
      if (!ok) rr = rho_ool(xi, yj);
      dde_mul_d(p, rr);
    }
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    if (o >= act) continue;
    DDE y;
    y.hi = __shfl_xor_sync(0xffffffffu, p.hi, o);
    y.lo = __shfl_xor_sync(0xffffffffu, p.lo, o);
    y.e = __shfl_xor_sync(0xffffffffu, p.e, o);
    y.pad = 0;
    dde_mul(p, y);
  }
  if (lane == 0) c.CX[((long long)job * c.cap + al) * c.cap + be] = p;
}

// this warp's share of the sweep's new CX pairs (new alpha x all beta, then old alpha x new
// beta): warps 1.. of every CTA of the cluster, global warp index gw of nwg (warp 0 of each CTA
// is busy with the frozen-tuple scalars of the side tables meanwhile)
__device__ void sb_cx_share(const DevCtx& c, int job, int rows_done, int cols_done, int rl, int rr, int gw,
                            int nwg) {
  const int na = (rl - rows_done) * rr, nb = rows_done * (rr - cols_done);
  for (int e = gw; e < na + nb; e += nwg) {   // (warp-uniform)
    int al, be;
    if (e < na) { al = rows_done + e / rr; be = e % rr; }
    else { const int f = e - na; al = f / (rr - cols_done); be = cols_done + f % (rr - cols_done); }
    sb_cx_table_warp(c, job, al, be);
  }
}

// ---------------------------------------------------------------------------------------
// superblock factor tables (eq. (9)-(10) integrands split over the frozen parts)
// ---------------------------------------------------------------------------------------
// One launch, block 128.  blockIdx.z < 2*jobs: side tables, z = job*2 + side, x = node chunk,
// y = slot (alpha or beta):
//   side 0 (alpha >= rows_done): SA = S_L + c_k[a], PA = P_LL * prod_{i<k} rho(u_k[a], X_i),
//                                QL1 = prod_{i<k} rho(u_{k+1}[b], X_i)
//   side 1 (beta >= cols_done):  SB = c_{k+1}[b] + S_R, PB = P_RR * prod_{j>k+1} rho(u_{k+1}[b], Y_j),
//                                QR0 = prod_{j>k+1} rho(u_k[a], Y_j)
// blockIdx.z >= 2*jobs (family D): CX[alpha][beta] = prod_{i<k} prod_{j>k+1} rho(X_alpha,i, Y_beta,j)
// for the new (alpha, beta) pairs, z = 2*jobs + job, y = alpha, x*128 + tid = beta.
__device__ __noinline__ void sb_side_tables(const DevCtx& c, int job, int side, int slot, int a0, int astride, int rl,
                               int rr, int cx_rows_done, int cx_cols_done, int cx_gw, int cx_nwg) {
  const int k = c.kb + job, d = c.d, n = c.n;
  __shared__ ESum sS;
  __shared__ DDE sP;
  __shared__ double sX[64];   // node values of the frozen tuple's first 64 coordinates
  const int* T;
  int lo, hi;  // coordinate range of the frozen tuple
  // (the callers pass only the slots that are new this sweep)
  if (side == 0) {
    if (slot >= rl) return;
    T = k > 0 ? rec_piv(c.rec_cur, c.RS, k - 1) + (long long)slot * d : nullptr;
    lo = 0;
    hi = k;
  } else {
    if (slot >= rr) return;
    T = k < d - 2 ? rec_piv(c.rec_cur, c.RS, k + 1) + (long long)slot * d : nullptr;
    lo = k + 2;
    hi = d;
  }
  if (!T) hi = lo;
  if (threadIdx.x < 32) {
    // the frozen tuple's S (exact limbs) and P (double-double) by warp 0: lanes split the
    // coordinates and the pair rows, then a shuffle reduction -- any order gives the same
    // rounded entries (R3)
    const int lane = threadIdx.x;
    ESum s = esum_zero();
    DDE p = dde_one();
    for (int q = lo + lane; q < hi; q += 32) {
      esum_add(s, c.chi[q * n + T[q]], c.clo[q * n + T[q]]);
      if (q - lo < 64) sX[q - lo] = c.u[q * n + T[q]];
    }
    if (c.family == 1)
      for (int a = lo + lane; a < hi; a += 32) {
        const double ua = c.u[a * n + T[a]];
        for (int b = a + 1; b < hi; ++b) {
          const double ub = c.u[b * n + T[b]];
          bool ok;
          double rr = rho_fast(ua, ub, ok);
          if (!ok) rr = rho_ool(ua, ub);
          dde_mul_d(p, rr);
        }
      }
    // butterfly levels with offset >= the lanes holding data only combine identities (exact
    // no-ops: +0, *1): skipped
    const int act = min(32, hi - lo);
#pragma unroll
    for (int o = 16; o; o >>= 1) {
      if (o >= act) continue;
      s.h += __shfl_xor_sync(0xffffffffu, s.h, o);
      s.l += __shfl_xor_sync(0xffffffffu, s.l, o);
      DDE y;
      y.hi = __shfl_xor_sync(0xffffffffu, p.hi, o);
      y.lo = __shfl_xor_sync(0xffffffffu, p.lo, o);
      y.e = __shfl_xor_sync(0xffffffffu, p.e, o);
      y.pad = 0;
      dde_mul(p, y);
    }
    if (lane == 0) {
      sS = s;
      sP = p;
    }
  } else if (cx_nwg > 0) {   // family D, first new slot: the CX pairs overlap warp 0's scalars
    sb_cx_share(c, job, cx_rows_done, cx_cols_done, rl, rr, cx_gw, cx_nwg);
  }
  __syncthreads();
  const long long o = ((long long)job * c.cap + slot) * n;
  const int mode_own = side == 0 ? k : k + 1;    // mode summed into SA / SB
  const int mode_oth = side == 0 ? k + 1 : k;    // mode of QL1 / QR0
  for (int a = a0 + threadIdx.x; a < n; a += astride) {
    ESum s = sS;
    esum_add(s, c.chi[mode_own * n + a], c.clo[mode_own * n + a]);
    if (side == 0) c.SA[o + a] = s;
    else c.SB[o + a] = s;
    if (c.family == 1) {
      const double uo = c.u[mode_own * n + a], ux = c.u[mode_oth * n + a];
      DDE p = sP, q = dde_one();
      bool ok = true;
#pragma unroll 2
      for (int t = lo; t < hi; ++t) {   // (branch-free rho: the two chains and consecutive t overlap)
        const double x = t - lo < 64 ? sX[t - lo] : c.u[t * n + T[t]];
        bool o1, o2;
        dde_mul_d(p, rho_fast(uo, x, o1));
        dde_mul_d(q, rho_fast(ux, x, o2));
        ok = ok && o1 && o2;
      }
      if (!ok) {   // (a division off its fast path: the chains again with the IEEE division)
        p = sP;
        q = dde_one();
        for (int t = lo; t < hi; ++t) {
          const double x = t - lo < 64 ? sX[t - lo] : c.u[t * n + T[t]];
          dde_mul_d(p, rho(uo, x));
          dde_mul_d(q, rho(ux, x));
        }
      }
      if (side == 0) { c.PA[o + a] = p; c.QL1[o + a] = q; }
      else { c.PB[o + a] = p; c.QR0[o + a] = q; }
    }
  }
}

// A_k(alpha, a; beta, b) from the tables (single rounding, R3)
template <int FAMILY>
__device__ __forceinline__ double sb_entry(const DevCtx& c, int job, int k, int al, int a, int be, int b) {
  const int n = c.n;
  if (FAMILY >= 2) {  // x-form: direct evaluation of the full coordinate tuple
    const int d = c.d;
    const int* TL = k > 0 ? rec_piv(c.rec_cur, c.RS, k - 1) + (long long)al * d : nullptr;
    const int* TR = k < d - 2 ? rec_piv(c.rec_cur, c.RS, k + 1) + (long long)be * d : nullptr;
    return x_entry_at<FAMILY>(c.u, c.wf, d, n,
                              [&](int j) { return j < k ? TL[j] : (j == k ? a : (j == k + 1 ? b : TR[j])); });
  }
  const long long oa = ((long long)job * c.cap + al) * n;
  const long long ob = ((long long)job * c.cap + be) * n;
  ESum s = c.SA[oa + a];
  esum_add(s, c.SB[ob + b]);
  const double S = esum_round(s);
  const double SS = __dmul_rn(S, S);
  if (FAMILY == 0) return __drcp_rn(SS);
  DDE p = c.PA[oa + a];
  dde_mul(p, c.PB[ob + b]);
  dde_mul(p, c.CX[((long long)job * c.cap + al) * c.cap + be]);
  dde_mul(p, c.QL1[oa + b]);
  dde_mul(p, c.QR0[ob + a]);
  dde_mul_d(p, rho(c.u[k * n + a], c.u[(k + 1) * n + b]));
  return dde_div(p, SS);
}

// sb_entry with the divisions on their branch-free fast paths (ok: the bits of sb_entry; !ok:
// the caller recomputes with sb_entry, out of its hot loop)
template <int FAMILY>
__device__ __forceinline__ double sb_entry_fast(const DevCtx& c, int job, int k, int al, int a, int be, int b,
                                                bool& ok) {
  if (FAMILY >= 2) {
    ok = true;
    return sb_entry<FAMILY>(c, job, k, al, a, be, b);
  }
  const int n = c.n;
  const long long oa = ((long long)job * c.cap + al) * n;
  const long long ob = ((long long)job * c.cap + be) * n;
  ESum s = c.SA[oa + a];
  esum_add(s, c.SB[ob + b]);
  const double S = esum_round(s);
  const double SS = __dmul_rn(S, S);
  if (FAMILY == 0) return div_pre_fast(1.0, SS, rcp_refined(SS), ok);   // = __drcp_rn(SS) when ok
  DDE p = c.PA[oa + a];
  dde_mul(p, c.PB[ob + b]);
  dde_mul(p, c.CX[((long long)job * c.cap + al) * c.cap + be]);
  dde_mul(p, c.QL1[oa + b]);
  dde_mul(p, c.QR0[ob + a]);
  bool o1, o2;
  dde_mul_d(p, rho_fast(c.u[k * n + a], c.u[(k + 1) * n + b], o1));
  const double v = dde_div_fast(p, SS, o2);
  ok = o1 && o2;
  return v;
}

// pivot positions of interface k: xs = alpha_s*n + a_s, ys = beta_s*n + b_s
__device__ __forceinline__ void pivot_pos(const DevCtx& c, int k, int s, int& x, int& y) {
  const int* T = rec_piv(c.rec_cur, c.RS, k) + (long long)s * c.d;
  const int* P = rec_par(c.rec_cur, c.RS, c.cap, c.d, k) + 2 * s;
  x = P[0] * c.n + T[k];
  y = P[1] * c.n + T[k + 1];
}

// ---------------------------------------------------------------------------------------
// phase 2: u/v of the existing pivots on the rows / columns that are new this sweep, in tiles
// of c.ext_tile rows: (1) all raw entries A(x, y_s) (A(x_s, y)) of the tile at once, one per
// thread, into shared memory -- the batched fiber evaluation; (2) a thread per row runs the
// triangular recurrence column-oriented:
//   for t = 0..r-1: u_t final; acc_s -= u_t * V[t][y_s]  (s > t)
// -- per s the same operations in the same order as the oracle's row-oriented
// u_s = A(x, y_s) - sum_{t<s} u_t(x) v_t(y_s) (t ascending), hence the same bits.
// Columns: v_t = acc_t / u_t(x_t) final; acc_s -= U[t][x_s] * v_t.
// Rows [x_lo, x_hi) of this CTA; coef = [t][s] (stride cap), tile = [s][TS], TS <= c.ext_tile + 1.
// ---------------------------------------------------------------------------------------
// rows per tile: c.ext_tile (host: as many as fit in EXT_SMEM_DOUBLES next to the coefficients)
#define EXT_SMEM_DOUBLES 8192
#ifndef EXT_REG
#define EXT_REG 1    // 1: phase 2 of the t-form families in registers (extend_side_reg)
#endif
#ifndef EXT_ILP
#define EXT_ILP 4   // raw entries per thread per iteration of the extension
#endif

template <int FAMILY>
__device__ __noinline__ void extend_side(const DevCtx& c, int sweep, int job, int k, int side, int r, int x_lo, int x_hi,
                            const int* p_al, const int* p_a, const double* pdiag, const double* prcp,
                            double* coef, double* tile,
                            unsigned long long& ent, unsigned long long& upd) {
  const int n = c.n, cap = c.cap;
  const int sbn = (int)c.sbn;
  double* U = c.U + (long long)job * cap * sbn;
  double* V = c.V + (long long)job * cap * sbn;
  if (x_lo >= x_hi) return;
  for (int e = threadIdx.x; e < r * r; e += blockDim.x) {
    const int t = e / r, s = e - t * r;
    double v = 0.0;
    if (t < s) {
      const int q = p_al[s] * n + p_a[s];
      v = side == 0 ? V[t * sbn + q] : U[t * sbn + q];
    }
    coef[t * cap + s] = v;
  }
  // rows per tile, tile stride and lanes per row of the recurrence (host: extend_tile_shape)
  const int tile_rows = c.ext_tile;
  double* dst = side == 0 ? U : V;
  const bool timer = TTC_PHASE_CLOCKS && c.phase_ns && job == c.phase_job && threadIdx.x == 0 && cg::this_cluster().block_rank() == 0;
  unsigned long long tm = timer ? gtimer() : 0;
  auto clock_to = [&](int ph) {
    if (timer) {
      const unsigned long long t = gtimer();
      ph_add(c.phase_ns, sweep, ph, t - tm);
      tm = t;
    }
  };
  int nrow;
  for (int x0 = x_lo; x0 < x_hi; x0 += nrow) {
    // tile shape: nrow rows, L recurrence lanes per row (as many as the rows leave threads
    // for, <= 8), stride TS <= tile_rows + 1.  L adjacent lanes work on L different s of one
    // row: TS = 8 (L = 4) or 4 (L = 8) mod 16 doubles spreads a warp's 32 accesses evenly over
    // the banks (L <= 2: any stride does); a full tile shrinks to such a stride when needed.
    nrow = min(tile_rows, x_hi - x0);
    int L = 1;
    while (L < 8 && 2 * L * nrow <= (int)blockDim.x) L *= 2;
    int TS = nrow + 1;
    if (L >= 4) {
      const int res = L == 4 ? 8 : 4;
      TS = ((nrow + 15 - res) & ~15) + res;   // smallest >= nrow with TS = res mod 16
      if (TS > tile_rows + 1) {
        TS = ((tile_rows + 1 - res) & ~15) + res;   // largest <= capacity
        if (TS >= 16) nrow = TS;
        else TS = nrow + 1;
      }
    }
    // (1) raw entries of the tile, one per thread, EXT_ILP per iteration: the independent
    // latency chains (table loads, double-double products, division) overlap
    {
      const int ne = nrow * r, B = blockDim.x;
      int e = threadIdx.x;
#pragma unroll 1
      for (; e + (EXT_ILP - 1) * B < ne; e += EXT_ILP * B) {
        double v[EXT_ILP];
        int at[EXT_ILP];
        bool ok[EXT_ILP];
#pragma unroll
        for (int u = 0; u < EXT_ILP; ++u) {   // (branch-free: the EXT_ILP chains interleave)
          const int eu = e + u * B;
          const int s = eu / nrow, j = eu - s * nrow;
          const int x = x0 + j;
          const int al = x / n, a = x - al * n;
          v[u] = side == 0 ? sb_entry_fast<FAMILY>(c, job, k, al, a, p_al[s], p_a[s], ok[u])
                           : sb_entry_fast<FAMILY>(c, job, k, p_al[s], p_a[s], al, a, ok[u]);
          at[u] = s * TS + j;
        }
#pragma unroll
        for (int u = 0; u < EXT_ILP; ++u) {
          if (!ok[u]) {
            const int eu = e + u * B;
            const int s = eu / nrow, j = eu - s * nrow;
            const int x = x0 + j;
            const int al = x / n, a = x - al * n;
            v[u] = side == 0 ? sb_entry<FAMILY>(c, job, k, al, a, p_al[s], p_a[s])
                             : sb_entry<FAMILY>(c, job, k, p_al[s], p_a[s], al, a);
          }
          tile[at[u]] = v[u];
        }
      }
#pragma unroll 1
      for (; e < ne; e += B) {
        const int s = e / nrow, j = e - s * nrow;
        const int x = x0 + j;
        const int al = x / n, a = x - al * n;
        tile[s * TS + j] = side == 0 ? sb_entry<FAMILY>(c, job, k, al, a, p_al[s], p_a[s])
                                     : sb_entry<FAMILY>(c, job, k, p_al[s], p_a[s], al, a);
      }
    }
    __syncthreads();
    clock_to(PH_EXT_RAW);
    // (2) the recurrence, L adjacent lanes per row (L = 1, 2, 4, 8: as many as the tile's rows
    // leave threads for), column-oriented (t outer, s > t inner), lane l updating s = l mod L:
    // for every s the same subtractions in the same t order as the oracle's row-oriented sum.
    // Columns divide by u_t(x_t) on the fly (every lane computes the same v_t bits); the final
    // v_t = tile / u_t(x_t) is formed again in the store below.  (A warp per row with lanes
    // over s measured slower at r = 16 and at r = 64.)
    {
      const int ln = threadIdx.x & (L - 1), lane = threadIdx.x & 31;
      const unsigned gmask = (L == 32 ? 0xffffffffu : ((1u << L) - 1u)) << (lane & ~(L - 1));
#pragma unroll 1
      for (int j = threadIdx.x / L; j < nrow; j += blockDim.x / L) {
#pragma unroll 1
        for (int t = 0; t < r; ++t) {
          if (L > 1) __syncwarp(gmask);   // tile[t][j] final (updated at step t-1 by lane t mod L)
          double f = tile[t * TS + j];
          if (side == 1) {   // v_t (= __ddiv_rn bits)
            bool ok;
            const double q = div_pre_fast(f, pdiag[t], prcp[t], ok);
            f = ok ? q : div_pre(f, pdiag[t], prcp[t]);
          }
          const int q0 = t + 1 + ((ln - (t + 1)) & (L - 1));
          const double* cf = coef + t * cap;
          int q = q0;
          // four independent read-modify-writes per iteration (distinct q: the loads of one
          // group do not depend on its stores, so they are issued together)
#pragma unroll 1
          for (; q + 3 * L < r; q += 4 * L) {
            double* p0 = tile + q * TS + j;
            const double a0 = p0[0], a1 = p0[L * TS], a2 = p0[2 * L * TS], a3 = p0[3 * L * TS];
            const double c0 = cf[q], c1 = cf[q + L], c2 = cf[q + 2 * L], c3 = cf[q + 3 * L];
            p0[0] = __dsub_rn(a0, __dmul_rn(f, c0));
            p0[L * TS] = __dsub_rn(a1, __dmul_rn(f, c1));
            p0[2 * L * TS] = __dsub_rn(a2, __dmul_rn(f, c2));
            p0[3 * L * TS] = __dsub_rn(a3, __dmul_rn(f, c3));
          }
          for (; q < r; q += L) tile[q * TS + j] = __dsub_rn(tile[q * TS + j], __dmul_rn(f, cf[q]));
        }
        if (L > 1) __syncwarp(gmask);
      }
    }
    __syncthreads();
    clock_to(PH_EXT_REC);
    for (int e = threadIdx.x; e < r * nrow; e += blockDim.x) {
      const int s = e / nrow, j = e - s * nrow;
      const double f = tile[s * TS + j];
      dst[s * sbn + x0 + j] = side == 1 ? div_pre(f, pdiag[s], prcp[s]) : f;
    }
    __syncthreads();
  }
  ent += (unsigned long long)(x_hi - x_lo) * r;
  upd += (unsigned long long)(x_hi - x_lo) * r * (r - 1) / 2;
}

// Phase 2, register-resident variant (t-form families, the default): the tile variant above
// runs its recurrence through shared memory -- a load and a store per multiply-subtract, the
// SM's shared-memory bandwidth is its roof (D_20: ~690 cycles per t step, half of a late
// sweep's extension) -- and evaluates each raw entry from seven table loads.  Here a row x is
// held by L adjacent lanes, lane l keeping acc[i] = the value of s = L*i + l (EXR_NS slots, so
// L = 1, 2, 4 covers r <= 16, 32, 64), in registers from the raw entry to the final store:
//   (1) raw entries straight into the slots.  The factors that depend only on the pivot s
//       (rows: SB, PB * CX * QL1 and u_{k+1}[b_s] of column y_s; columns: SA, PA * CX * QR0
//       and u_k[a_s] of row x_s) are formed once per call in shared memory (ExtFix), so an
//       entry is P_own * F_s * Q_s[node] * rho(u_own, u_s) / (S_own + S_s)^2 -- three
//       double-double products instead of five; the product is rounded once, so the grouping
//       gives the same entries (R3);
//   (2) the triangular recurrence column-oriented (t ascending): the owner lane of t (lane
//       t mod L of the row group, slot t / L) holds the final acc_t, the group reads it with a
//       shuffle (columns: v_t = acc_t / u_t(x_t)), every lane subtracts f * coef[t][s] from its
//       slots s > t -- per s the same operations in the same t order as the oracle's
//       u_s = A(x, y_s) - sum_{t<s} u_t(x) v_t(y_s), hence the same bits;
//   (3) the final values (columns: acc_s / u_s(x_s)) straight to U / V.
// coef[t][s] is kept as coefL[t][l][i] (s = L*i + l), so a lane's slots are contiguous.
#define EXR_NS 16
#ifndef TTC_EXT_PREFETCH
#define TTC_EXT_PREFETCH 0   // phase 2 raw entries: the next group's Q gathers prefetched into L1 (D_20 14.52 -> 14.70 ms: off)
#endif
__device__ __forceinline__ void prefetch_l1(const void* p) { asm volatile("prefetch.global.L1 [%0];" ::"l"(p)); }
#ifndef TTC_EXT_ALL
#define TTC_EXT_ALL 1   // phase 2, streaming shapes: every CTA extends a share of the rows, then of the columns
#endif
#ifndef TTC_EXT_INLINE
#define TTC_EXT_INLINE __noinline__   // (A/B: __forceinline__ puts phase 2 in the kernel's register allocation)
#endif
struct ExtFix {
  DDE F;      // rows: PB[be_s][b_s] * CX[al][be_s] * QL1[al][b_s]; columns: PA[al_s][a_s] * CX[al_s][be] * QR0[be][a_s]
  ESum S;     // rows: SB[be_s][b_s]; columns: SA[al_s][a_s]
  double u;   // rows: u_{k+1}[b_s]; columns: u_k[a_s]
  int q;      // rows: offset of QR0[be_s][.]; columns: offset of QL1[al_s][.]
  int pad;
};
// coefficient row stride (doubles): the L lanes of a row group read L different rows of
// coefL at once; 18 puts them on disjoint banks (16 = 128 bytes put all on the same ones --
// a 4-way conflict on every read, ncu: short-scoreboard stalls on the update line) and keeps
// the rows 16-byte aligned for paired reads
#define EXR_CS 18
// lanes per row: the fewest that give every pivot a slot (L * EXR_NS >= r)
__host__ __device__ __forceinline__ int ext_reg_lanes(int r) { return r <= EXR_NS ? 1 : (r <= 2 * EXR_NS ? 2 : 4); }
template <int FAMILY>
__device__ __noinline__ double sb_entry_ool(const DevCtx& c, int job, int k, int al, int a, int be, int b) {
  return sb_entry<FAMILY>(c, job, k, al, a, be, b);
}

// raw entries of slots [i0, i0 + 4) of this lane (s = L*i + l) into v; slow bit u: entry u
// left the division's fast path
template <int FAMILY>
__device__ __forceinline__ void ext_raw4(double (&v)[4], int i0, int L, int l, int r, const ExtFix* fix,
                                         const ESum& so, const DDE& po, double uo, const DDE* Qg, int z,
                                         unsigned& slow) {
  DDE q[4];
#pragma unroll
  for (int u = 0; u < 4; ++u) {
    const int s = min(L * (i0 + u) + l, r - 1);
    if (FAMILY == 1) q[u] = Qg[fix[s].q + z];
  }
#pragma unroll
  for (int u = 0; u < 4; ++u) {
    const int s = min(L * (i0 + u) + l, r - 1);
    const ExtFix& f = fix[s];
    ESum sm = so;
    esum_add(sm, f.S);
    const double Sd = esum_round(sm);
    const double SS = __dmul_rn(Sd, Sd);
    bool ok;
    if (FAMILY == 0) {
      v[u] = div_pre_fast(1.0, SS, rcp_refined(SS), ok);
    } else {
      DDE p = po;
      dde_mul(p, f.F);
      dde_mul(p, q[u]);
      bool o1, o2;
      dde_mul_d(p, rho_fast(uo, f.u, o1));
      v[u] = dde_div_fast(p, SS, o2);
      ok = o1 && o2;
    }
    slow |= (ok ? 0u : 1u) << u;
  }
}

// the column recurrence's divisors u_t(x_t) and their refined reciprocals: file-scope shared
// arrays (constant addresses: ext_rec reads them without a pointer that the register
// allocator of the sweep kernel would spill to local memory)
__shared__ double s_pdiag[TTC_MAX_RANK_DEV], s_prcp[TTC_MAX_RANK_DEV];

// phase-2 recurrence of one row group (see extend_side_reg): lane l of the L lanes holds
// acc[i] = slot s = L*i + l; for t = 0..r-1 the owner lane's acc_t (columns: / u_t(x_t)) is
// broadcast and every slot s > t subtracts f * coef[t][s] -- per s the oracle's operations in
// its t order.
template <int L>
__device__ __forceinline__ void ext_rec(double (&acc)[EXR_NS], int r, int l, int gbase, int side, const double* pdiag,
                                        const double* prcp, const double* coefL) {
  constexpr int LG = L == 1 ? 0 : (L == 2 ? 1 : 2);
#pragma unroll
  for (int ph = 0; ph < EXR_NS / 4; ++ph) {
    const int tb = 4 * L * ph;   // (a constant: the phase loop is unrolled)
    if (tb >= r) break;          // (warp-uniform)
#pragma unroll 1
    for (int t = tb; t < tb + 4 * L; ++t) {   // (constant trip count: no bound to spill)
      if (t >= r) continue;                    // (warp-uniform)
      const int it = t >> LG, lt = t & (L - 1);
      double own = acc[4 * ph];
#pragma unroll
      for (int u = 1; u < 4; ++u)
        if (it == 4 * ph + u) own = acc[4 * ph + u];
      const double2* cf = reinterpret_cast<const double2*>(coefL + (t * L + l) * EXR_CS);
      // the phase's own four coefficients and the divisor, loaded before the broadcast
      const double2 c0 = cf[2 * ph], c1 = cf[2 * ph + 1];
      const double pd = s_pdiag[t], pr = s_prcp[t];
      double f = __shfl_sync(0xffffffffu, own, gbase + lt);
      if (side == 1) {   // v_t = acc_t / u_t(x_t) (= __ddiv_rn bits)
        bool ok;
        const double q = div_pre_fast(f, pd, pr, ok);
        f = ok ? q : div_pre(f, pd, pr);
      }
      const int thr = (t - l) >> LG;   // slots i <= thr hold s <= t (arithmetic shift: -1 for t < l)
      // the phase's own four slots: s > t depends on the lane
      if (4 * ph > thr) acc[4 * ph] = __dsub_rn(acc[4 * ph], __dmul_rn(f, c0.x));
      if (4 * ph + 1 > thr) acc[4 * ph + 1] = __dsub_rn(acc[4 * ph + 1], __dmul_rn(f, c0.y));
      if (4 * ph + 2 > thr) acc[4 * ph + 2] = __dsub_rn(acc[4 * ph + 2], __dmul_rn(f, c1.x));
      if (4 * ph + 3 > thr) acc[4 * ph + 3] = __dsub_rn(acc[4 * ph + 3], __dmul_rn(f, c1.y));
      // later slots: s >= L*(4*ph + 4) > t on every lane (no predicate), in groups of four
      // whose coefficient loads the compiler is free to hoist (no stores in between)
#pragma unroll
      for (int i = 4 * ph + 4; i < EXR_NS; i += 4) {
        if (L * i >= r) break;   // (warp-uniform: no lane has a slot s < r from here on)
        const double2 a0 = cf[i >> 1], a1 = cf[(i >> 1) + 1];
        acc[i] = __dsub_rn(acc[i], __dmul_rn(f, a0.x));
        acc[i + 1] = __dsub_rn(acc[i + 1], __dmul_rn(f, a0.y));
        acc[i + 2] = __dsub_rn(acc[i + 2], __dmul_rn(f, a1.x));
        acc[i + 3] = __dsub_rn(acc[i + 3], __dmul_rn(f, a1.y));
      }
    }
  }
}

template <int FAMILY>
__device__ TTC_EXT_INLINE void extend_side_reg(const DevCtx& c, int sweep, int job, int k, int side, int r, int x_lo,
                                             int x_hi, const int* p_al, const int* p_a, const double* pdiag,
                                             const double* prcp, double* dyn, long long smem_doubles,
                                             unsigned long long& ent, unsigned long long& upd) {
  static_assert(FAMILY <= 1, "t-form families only");
  const int n = c.n, cap = c.cap;
  const int sbn = (int)c.sbn;
  const int jo = job * cap * n, jcx = job * cap * cap;
  double* U = c.U + (long long)job * cap * sbn;
  double* V = c.V + (long long)job * cap * sbn;
  if (x_lo >= x_hi || r == 0) return;
  const int T = blockDim.x, tid = threadIdx.x, lane = tid & 31;
  const int L = ext_reg_lanes(r);
  const int l = tid & (L - 1), P = T / L;   // slot lane, rows per pass
  (void)smem_doubles;   // (cap * 4 * EXR_CS + 8 * cap <= extend_smem_doubles(cap) for cap <= 64)
  double* coefL = dyn;                                                  // [cap][L][EXR_CS]
  ExtFix* fix = reinterpret_cast<ExtFix*>(dyn + (long long)cap * L * EXR_CS);   // [cap]
  {
    // coefL[t][ls][i] = coef[t][L*i + ls] (i < EXR_NS; the padding is never read): eight
    // independent loads per thread per iteration
    const int ne = r * L * EXR_CS;
    const double* F = side == 0 ? V : U;
#pragma unroll 1
    for (int e0 = tid; e0 < ne; e0 += 8 * T) {
      double v[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int e = e0 + u * T;
        const int t = e / (L * EXR_CS), ls = (e / EXR_CS) % L, i = e % EXR_CS;
        const int s = L * i + ls;
        v[u] = 0.0;
        if (e < ne && i < EXR_NS && t < s && s < r) v[u] = F[t * sbn + p_al[s] * n + p_a[s]];
      }
#pragma unroll
      for (int u = 0; u < 8; ++u)
        if (e0 + u * T < ne) coefL[e0 + u * T] = v[u];
    }
  }
  double* dst = side == 0 ? U : V;
  const bool timer = TTC_PHASE_CLOCKS && c.phase_ns && job == c.phase_job && tid == 0 && cg::this_cluster().block_rank() == 0;
  unsigned long long tm = timer ? gtimer() : 0;
  auto clock_to = [&](int ph) {
    if (timer) {
      const unsigned long long t = gtimer();
      ph_add(c.phase_ns, sweep, ph, t - tm);
      tm = t;
    }
  };
  // own-side tables and node values: rows SA / PA / u_k, columns SB / PB / u_{k+1}
  const ESum* Sown = side == 0 ? c.SA + jo : c.SB + jo;
  const DDE* Pown = side == 0 ? c.PA + jo : c.PB + jo;
  const DDE* Qg = side == 0 ? c.QR0 : c.QL1;
  const double* uown = c.u + (long long)(side == 0 ? k : k + 1) * n;
  int fslot = -1;   // the slot (rows: alpha, columns: beta) the ExtFix entries were formed for
  const int gbase = lane & ~(L - 1);
#pragma unroll 1
  for (int x0 = x_lo; x0 < x_hi;) {
    const int sl0 = x0 / n;
    const int x1 = min(min(x_hi, x0 + P), (sl0 + 1) * n);   // (a pass stays inside one slot)
    if (sl0 != fslot) {
      __syncthreads();   // (previous users of fix / coefL done)
      if (tid < r) {
        ExtFix f;
        const int ps = p_al[tid], pn = p_a[tid];
        if (side == 0) {   // pivot column y_s = (be, b) = (ps, pn), row slot al = sl0
          f.S = c.SB[jo + ps * n + pn];
          f.u = c.u[(long long)(k + 1) * n + pn];
          f.q = jo + ps * n;
          if (FAMILY == 1) {
            DDE F = c.PB[jo + ps * n + pn];
            const DDE F1 = c.CX[jcx + sl0 * cap + ps], F2 = c.QL1[jo + sl0 * n + pn];
            dde_mul(F, F1);
            dde_mul(F, F2);
            f.F = F;
          }
        } else {           // pivot row x_s = (al, a) = (ps, pn), column slot be = sl0
          f.S = c.SA[jo + ps * n + pn];
          f.u = c.u[(long long)k * n + pn];
          f.q = jo + ps * n;
          if (FAMILY == 1) {
            DDE F = c.PA[jo + ps * n + pn];
            const DDE F1 = c.CX[jcx + ps * cap + sl0], F2 = c.QR0[jo + sl0 * n + pn];
            dde_mul(F, F1);
            dde_mul(F, F2);
            f.F = F;
          }
        }
        f.pad = 0;
        fix[tid] = f;
      }
      fslot = sl0;
      __syncthreads();
    }
    const int nrow = x1 - x0;
    const int j = tid / L;
    const bool valid = j < nrow;
    if ((tid & ~31) / L >= nrow) {   // a warp with no row in this pass (the last, partial one) idles
      x0 = x1;
      continue;
    }
    const int x = x0 + (valid ? j : nrow - 1);   // (a lane past the pass repeats the last row)
    const int z = x - sl0 * n;                   // node of the row within its slot
    // (1) raw entries, four slots per iteration (their table gathers issued together: a
    // dependent global load waits a loaded-L2 round trip), placed into the slots by selects
    double acc[EXR_NS];
#pragma unroll
    for (int i = 0; i < EXR_NS; ++i) acc[i] = 0.0;
    {
      const ESum so = Sown[x];
      DDE po;
      if (FAMILY == 1) po = Pown[x];
      else po = dde_one();
      const double uo = uown[z];
      if (TTC_EXT_PREFETCH && FAMILY == 1)   // the first group's Q factors into L1
#pragma unroll
        for (int u = 0; u < 4; ++u) prefetch_l1(&Qg[fix[min(L * u + l, r - 1)].q + z]);
#pragma unroll 1
      for (int g = 0; g < EXR_NS / 4 && 4 * L * g < r; ++g) {   // (warp-uniform)
        double v[4];
        unsigned slow = 0;
        // the next group's Q gathers go out now (L1 prefetch: no registers), so its loads hit L1
        // instead of waiting a loaded-L2 round trip after this group's arithmetic
        if (TTC_EXT_PREFETCH && FAMILY == 1 && 4 * L * (g + 1) < r)
#pragma unroll
          for (int u = 0; u < 4; ++u) prefetch_l1(&Qg[fix[min(L * (4 * (g + 1) + u) + l, r - 1)].q + z]);
        ext_raw4<FAMILY>(v, 4 * g, L, l, r, fix, so, po, uo, Qg, z, slow);
        if (slow) {   // (rare: a division off its fast path -- the entry the plain way, out of line)
#pragma unroll 1
          for (int u = 0; u < 4; ++u)
            if ((slow >> u) & 1u) {
              const int s = min(L * (4 * g + u) + l, r - 1);
              const int al = side == 0 ? sl0 : p_al[s], a = side == 0 ? z : p_a[s];
              const int be = side == 0 ? p_al[s] : sl0, b = side == 0 ? p_a[s] : z;
              const double w = sb_entry_ool<FAMILY>(c, job, k, al, a, be, b);
              if (u == 0) v[0] = w;
              else if (u == 1) v[1] = w;
              else if (u == 2) v[2] = w;
              else v[3] = w;
            }
        }
#pragma unroll
        for (int i = 0; i < EXR_NS; ++i)
          if ((i >> 2) == g) acc[i] = v[i & 3];
      }
    }
    clock_to(PH_EXT_RAW);
    // (2) the recurrence: t in four phases of 4 * L (a runtime loop each, its slot updates
    // unrolled over the slots a phase can still reach, predicated on s > t; f = acc_t read
    // from the phase's four candidate slots by selects): small, spill-free code.  L is a
    // template constant here (ext_rec<L>): the slot predicate is one compare with an
    // immediate, and a phase's coefficient pairs are all read before the first update (the
    // runtime-L form re-used one register quad per pair: eight dependent shared-memory round
    // trips per t, ~800 cycles per t on D_20)
    if (L == 1) ext_rec<1>(acc, r, l, gbase, side, pdiag, prcp, coefL);
    else if (L == 2) ext_rec<2>(acc, r, l, gbase, side, pdiag, prcp, coefL);
    else ext_rec<4>(acc, r, l, gbase, side, pdiag, prcp, coefL);
    clock_to(PH_EXT_REC);
    // (3) final values
    if (valid) {
#pragma unroll
      for (int i = 0; i < EXR_NS; ++i) {
        const int s = L * i + l;
        if (s < r) dst[(long long)s * sbn + x] = side == 1 ? div_pre(acc[i], pdiag[s], prcp[s]) : acc[i];
      }
    }
    x0 = x1;
  }
  __syncthreads();
  ent += (unsigned long long)(x_hi - x_lo) * r;
  upd += (unsigned long long)(x_hi - x_lo) * r * (r - 1) / 2;
}

// phase-2 tile rows and dynamic shared memory: coef [cap][cap] + tile [cap][rows + 1]
__host__ __device__ __forceinline__ int extend_tile_rows(int cap) {
  const long long rows = (EXT_SMEM_DOUBLES - (long long)cap * cap) / cap - 1;
  return (int)(rows < 32 ? 32 : (rows > 256 ? 256 : rows));
}
__host__ __device__ __forceinline__ long long extend_smem_doubles(int cap) {
  return (long long)cap * cap + (long long)cap * (extend_tile_rows(cap) + 1);
}

// ---------------------------------------------------------------------------------------
// k_sweep phase 3 (Alg. 2): helpers
// ---------------------------------------------------------------------------------------
#define GREEDY_MAX_THREADS 512
#define TMA_PMAX 16   // stages of the TMA ring (at most)
#define TMA_NBAR 128  // TMA ring barriers: warps x stages
#define STAGE_N 1024  // n up to which the n-indexed factor of a step is staged in shared memory

#ifndef TTC_PREFETCH
#define TTC_PREFETCH 0   // rook steps: prefetch the next row block's tables into L1 (A/B)
#endif
struct Cand {
  double val;
  long long idx;
};

__device__ __forceinline__ bool cand_better(double v, long long f, double bv, long long bf) {
  return v > bv || (v == bv && f < bf);
}

// warp argmax of (v, f) with cand_better's order (largest v, then smallest f) on every lane.
// Candidates are |E| >= 0 with an index < 2^31, or (-1, LLONG_MAX) for none; the bit pattern
// of a non-negative double orders like its value, so three warp reductions (max of the high
// words, max of the low words among those, min of the indices among the maxima: REDUX)
// replace the five-round shuffle tree (tools/microbench.cu: warp_argmax probes).  NaN is
// never chosen, as with cand_better.
__device__ __forceinline__ void warp_argmax(double& v, long long& f) {
  const bool has = v >= 0.0;
  const unsigned hi = has ? (unsigned)__double2hiint(v) : 0u;
  const unsigned lo = has ? (unsigned)__double2loint(v) : 0u;
  const unsigned mh = __reduce_max_sync(0xffffffffu, hi);
  const unsigned ml = __reduce_max_sync(0xffffffffu, hi == mh ? lo : 0u);
  const unsigned mf = __reduce_min_sync(0xffffffffu, (has && hi == mh && lo == ml) ? (unsigned)f : 0xffffffffu);
  if (mf == 0xffffffffu) {
    v = -1.0;
    f = LLONG_MAX;
  } else {
    v = __hiloint2double((int)mh, (int)ml);
    f = (long long)mf;
  }
}
// the five-round shuffle tree (kept for the microbenchmark comparison)
__device__ __forceinline__ void warp_argmax_shfl(double& v, long long& f) {
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    const double ov = __shfl_xor_sync(0xffffffffu, v, o);
    const long long of = __shfl_xor_sync(0xffffffffu, f, o);
    if (cand_better(ov, of, v, f)) { v = ov; f = of; }
  }
}

struct GreedySmem {
  Cand xc[2][16];                    // cluster exchange: candidate of CTA j in xc[step & 1][j]
  unsigned long long xbar[2];        // mbarriers of the two exchange buffers
  Cand red[GREEDY_MAX_THREADS / 32];
  Cand best;                         // CTA argmax / cluster winner
  int xs[TTC_MAX_RANK_DEV];          // pivot rows
  int ys[TTC_MAX_RANK_DEV];          // pivot columns
  alignas(16) double vec[TTC_MAX_RANK_DEV];   // V[t][y*] (column step) or U[t][x*] (row step) (paired reads)
  // factors of the fixed column (row) of a step
  DDE f_slot[TTC_MAX_RANK_DEV];      // column step: CX[alpha][beta]*QL1[alpha][b]; row step: CX*QR0
  // (f_node -- column step: QR0[beta][a]; row step: QL1[alpha][b] -- lives in the dynamic
  // shared memory at c.fnode_off, sized for n: the static footprint stays small, so the
  // rook-step ring can take the rest of the SM's shared memory)
  ESum fs;                           // SB[beta][b] (column step) or SA[alpha][a] (row step)
  DDE fp;                            // PB[beta][b] or PA[alpha][a]
  double pv;                         // E(x*, y*) of the final pivot (owner CTA of column y*)
  double pa;                         // A(x*, y*) (CACHED: owner CTA of row x*)
  unsigned long long rfull[TMA_NBAR];   // TMA ring: stage landed (1 arrival + the box bytes), [warp][P]
};

// asynchronous global -> shared copies (LDGSTS): the whole cache fill is one round trip
__device__ __forceinline__ void cp_async8(void* smem, const void* gmem) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(sa), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait_group() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

// Per-thread staging ring of the non-cached rook steps.  A column step needs, for each of the
// thread's rows x, the r factors F[t][x] = U[t][x] (a row step: V[t][y]) -- an HBM stream of
// r*8 bytes per row (D_20: 2 MB per CTA per step).  Loading them with plain loads leaves one
// unrolled batch (8 loads) in flight per thread and the step latency-bound; here each thread
// streams its own factors through shared memory with cp.async in RING_P stages of `tb` terms,
// RING_P - 1 stages ahead of the chain, so ~ (RING_P - 1) * tb loads per thread are in flight.
// A thread reads back only what it copied itself: no block barrier, only cp.async.wait_group.
// Layout: buf[stage][i][T] (conflict-free per warp).  Stage s = (row j, term block b), row-major.
#define RING_P 4
#define RING_MIN_ROWS 4   // rows per thread from which a step streams through the ring
// L2 evict_first hint on the factor stream (TMA ring only).  For cp.async with
// .L2::cache_hint, ptxas 12.9 (sm_100a) emits LDGSTS whose cache-policy operand names uniform
// registers the policy was never written to (SASS in profiles/r02_illegal_instruction.txt): a
// garbage descriptor, "illegal instruction" in some builds -- the DotRing therefore streams
// without a hint.  UTMALDG takes the policy registers correctly.
#ifndef TTC_TMA
#define TTC_TMA 1   // the rook steps stream through the TMA ring (0: the per-thread cp.async DotRing)
#endif
#ifndef TTC_EVICT_FIRST
#define TTC_EVICT_FIRST 1
#endif
// L2 policy of the stream: the u/v factors of all superblocks exceed the
// 126 MB L2 many times over (D_20 640 MB, C_200 840 MB), so no factor line survives in L2
// until the superblock's next step anyway.  EVICT_FIRST loads them evict_first, so the stream
// stops displacing the tables and records the steps reuse: C_200 -8%, D_20 -1%
// (profiles/r01n_l2_policy.log); t-form families.  (Keeping a fraction of the lines with
// evict_last measured slower for every fraction tried, 0.15-0.5.)
__device__ __forceinline__ void cp_async8_ef(void* smem, const void* gmem, unsigned long long pol) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.ca.shared.global.L2::cache_hint [%0], [%1], 8, %2;" ::"r"(sa), "l"(gmem), "l"(pol) : "memory");
}
template <bool EVICT_FIRST>
struct DotRing {
  double* buf;
  const double* F;
  unsigned long long pol;   // L2 cache policy of the factor stream (EVICT_FIRST)
  int T, tid, tb, nb, sbn, r;
  int z0, total;          // first row of the thread, stages in all
  int is, irow, iblk;     // next stage to issue
  int cs;                 // next stage to consume
  __device__ __forceinline__ void init(double* b, const double* f, int T_, int tid_, int tb_, int sbn_, int r_, int zb,
                                       int ze) {
    buf = b; F = f; T = T_; tid = tid_; tb = tb_; sbn = sbn_; r = r_;
    nb = (r + tb - 1) / tb;
    z0 = zb + tid;
    const int rows = z0 < ze ? (ze - z0 + T - 1) / T : 0;
    total = rows * nb;
    is = irow = iblk = cs = 0;
#pragma unroll 1
    for (int q = 0; q < RING_P - 1; ++q) issue();
  }
  __device__ __forceinline__ void issue() {
    if (is < total) {
      double* dst = buf + (is & (RING_P - 1)) * tb * T + tid;
      const int t0 = iblk * tb, tn = min(tb, r - t0);
      const double* src = F + t0 * sbn + z0 + irow * T;
      // (loops left to the compiler's unrolling: measured faster than unroll 1 on D_20)
      if (EVICT_FIRST) {
        // the policy is created right before its copies: LDGSTS takes it from a uniform
        // register, and a policy created once in init() and carried across the out-of-line
        // calls of the step reached the copies as garbage in some builds (SASS
        // `LDGSTS desc[UR]` -> "illegal instruction", found with cuda-gdb)
        asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
        for (int i = 0; i < tn; ++i) cp_async8_ef(dst + i * T, src + i * sbn, pol);
      }
      else
        for (int i = 0; i < tn; ++i) cp_async8(dst + i * T, src + i * sbn);
      if (++iblk == nb) { iblk = 0; ++irow; }
    }
    ++is;
    cp_async_commit();   // (empty groups keep the wait count uniform)
  }
  // e -= F[t][row] * vec[t], t = 0 .. r-1 in order, for the thread's next row
  __device__ __forceinline__ double dot_sub(double e, const double* vec) {
#pragma unroll 1
    for (int b = 0; b < nb; ++b) {
      issue();
      cp_async_wait_group<RING_P - 1>();
      const double* src = buf + (cs & (RING_P - 1)) * tb * T + tid;
      const int t0 = b * tb, tn = min(tb, r - t0);
      for (int i = 0; i < tn; ++i) e = __dsub_rn(e, __dmul_rn(src[i * T], vec[t0 + i]));
      ++cs;
    }
    return e;
  }
};

// TMA ring of the non-cached rook steps (c.tma), one ring per warp: a warp's u/v factor
// stream F[t][x] (its 32 rows x of each row block, t = 0..r-1) is cut into stages of tb terms,
// each one 2-D box {32, tb} of F's tensor map (dims {sbn, jobs * cap}: x fastest, one row per
// (job, t)), landing as [tb][32] in the warp's part of the shared-memory ring.  Lane 0 issues
// stage q + P - 1 (cp.async.bulk.tensor, complete_tx on the warp's rfull[slot], L2 evict_first
// for the t-form families) when the warp starts consuming stage q -- the slot of stage q - 1,
// which every lane finished reading before the __syncwarp that ends it; every lane waits on
// rfull and reads back its own row's terms.  Warps never wait for each other (the cp.async
// DotRing's property, without its 8-byte copy per thread and term).  The ring position
// (slot, phase) is the same in every thread and persists across steps and sweeps (RingPos).
#ifndef TTC_RING_PREFETCH
#define TTC_RING_PREFETCH 0   // bit 0: the first column step's first stage during the samples; bit 1: a row step's after its column step (both measured slower: C_200 5.09 -> 5.39 ms, profiles/r02k_prefetch.log)
#endif
#ifndef TTC_FENCE_ALL
#define TTC_FENCE_ALL 1       // the post-extension proxy fence covers shared memory too
#endif
struct RingPos {
  int slot;
  unsigned phase;
  int pre;   // 1: the next step's first stage is already in flight (TmaRing::prefetch)
};

__device__ __forceinline__ unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_wait(const unsigned long long* b, unsigned parity) {
  const unsigned a = smem_u32(b);
  unsigned ok = 0;
  while (!ok)
    asm volatile(
        "{\n .reg .pred q;\n"
        " mbarrier.try_wait.parity.shared::cta.b64 q, [%1], %2;\n"
        " selp.u32 %0, 1, 0, q;\n}"
        : "=r"(ok) : "r"(a), "r"(parity) : "memory");
}

__device__ __forceinline__ void tma_ring_init(GreedySmem* S) {
  if (threadIdx.x == 0) {
    for (int q = 0; q < TMA_NBAR; ++q)
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&S->rfull[q])) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  // (ordered before any use by the kernel's first cluster barrier)
}

template <bool EVICT_FIRST>
struct TmaRing {
  double* wbuf;               // this warp's P stages of [tb][32]
  const void* tmap;
  unsigned long long* full;   // this warp's P barriers
  // (two stages of 16 terms per warp: compile-time constants -- the best measured shape, and
  // fewer live registers in the consumer loop; the host sets ring_tb = 16, ring_p = 2)
  static constexpr int tb = 16, P = 2;
  int lane, nb, r, ybase, x0, T;
  int total, is;              // stages of this step, issued (lane 0)
  float keep;                 // L2 evict_last fraction of the stream (c.l2_keep)
  int ijb, ib;                // row block and term block of the next stage to issue (no division per stage)
  RingPos pos, ipos;          // consumption / issue position
  __device__ __forceinline__ void setup(double* buf, const void* tmap_, GreedySmem* S, int T_, int tid, int tb_, int P_,
                                        int r_, int ybase_, int xb, int xe, RingPos p, float keep_) {
    const int warp = tid >> 5;
    keep = keep_;
    lane = tid & 31;
    tmap = tmap_; T = T_; r = r_; ybase = ybase_;
    (void)tb_;
    (void)P_;
    wbuf = buf + (long long)warp * P * tb * 32;
    full = &S->rfull[warp * P];
    x0 = xb + warp * 32;
    nb = (r + tb - 1) / tb;
    total = xe > xb ? ((xe - xb + T - 1) / T) * nb : 0;
    pos = p;
    pos.pre = 0;
    ipos = pos;
    is = 0;
    ijb = 0;
    ib = 0;
  }
  __device__ __forceinline__ void start(double* buf, const void* tmap_, GreedySmem* S, int T_, int tid, int tb_,
                                        int P_, int r_, int ybase_, int xb, int xe, RingPos p, float keep_) {
    setup(buf, tmap_, S, T_, tid, tb_, P_, r_, ybase_, xb, xe, p, keep_);
    if (p.pre && total > 0) {   // stage 0 was issued by prefetch() into slot p.slot
      is = 1;
      if (++ib == nb) { ib = 0; ++ijb; }
      if (++ipos.slot == P) { ipos.slot = 0; ipos.phase ^= 1u; }
    }
    if (lane == 0)
      for (int q = is; q < P - 1 && is < total; ++q) issue();
  }
  // the first stage of a step that is certain to follow (the ring is empty: every stage of the
  // previous step consumed), issued while the current step's argmax -- or the samples phase --
  // still runs: the data of a column step (U of the CTA's rows) does not depend on the column y,
  // nor a row step's (V of its columns) on the row x.  Every thread marks p.pre.
  __device__ __forceinline__ void prefetch(double* buf, const void* tmap_, GreedySmem* S, int T_, int tid, int tb_,
                                           int P_, int r_, int ybase_, int xb, int xe, RingPos& p, float keep_) {
    setup(buf, tmap_, S, T_, tid, tb_, P_, r_, ybase_, xb, xe, p, keep_);
    if (total <= 0) return;
    if (lane == 0) issue();
    p.pre = 1;
  }
  __device__ __forceinline__ void issue() {   // lane 0: stage `is` into slot ipos
    const unsigned fa = smem_u32(&full[ipos.slot]);
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(fa), "r"(tb * 256) : "memory");
    const unsigned dst = smem_u32(wbuf + ipos.slot * tb * 32);
    const int x = x0 + ijb * T, y = ybase + ib * tb;
    if (EVICT_FIRST) {
      unsigned long long pol;
      if (keep > 0.f)   // a fraction of the lines evict_last: they survive until the next step
        asm volatile("createpolicy.fractional.L2::evict_last.L2::evict_first.b64 %0, %1;" : "=l"(pol) : "f"(keep));
      else
        asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
      asm volatile(
          "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes.L2::cache_hint"
          " [%0], [%1, {%2, %3}], [%4], %5;" ::"r"(dst), "l"(tmap), "r"(x), "r"(y), "r"(fa), "l"(pol)
          : "memory");
    } else {
      asm volatile(
          "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
          " [%0], [%1, {%2, %3}], [%4];" ::"r"(dst), "l"(tmap), "r"(x), "r"(y), "r"(fa)
          : "memory");
    }
    ++is;
    if (++ib == nb) { ib = 0; ++ijb; }
    if (++ipos.slot == P) { ipos.slot = 0; ipos.phase ^= 1u; }
  }
  // e -= F[t][row] * vec[t], t = 0 .. r-1 in order, for this thread's row of the next row
  // block (every lane of the warp calls this for every row block)
  __device__ __forceinline__ double dot_sub(double e, const double* vec) {
#pragma unroll 1
    for (int b = 0; b < nb; ++b) {
      if (lane == 0 && is < total) issue();
      mbar_wait(&full[pos.slot], pos.phase);
      const double* src = wbuf + pos.slot * tb * 32 + lane;
      const int t0 = b * tb, tn = min(tb, r - t0);
      if (tn == 16) {   // (a full stage of the usual shape: unrolled, vec read in pairs)
        const double2* v2 = reinterpret_cast<const double2*>(vec + t0);
#pragma unroll
        for (int i = 0; i < 16; i += 2) {
          const double2 vv = v2[i >> 1];
          e = __dsub_rn(e, __dmul_rn(src[i * 32], vv.x));
          e = __dsub_rn(e, __dmul_rn(src[(i + 1) * 32], vv.y));
        }
      } else {   // (the last stage of a rank that is not a multiple of 16: unrolled, guarded)
#pragma unroll
        for (int i = 0; i < 15; ++i)
          if (i < tn) e = __dsub_rn(e, __dmul_rn(src[i * 32], vec[t0 + i]));
      }
      __syncwarp();   // (the slot is refilled two issues later, by lane 0 of this warp)
      if (++pos.slot == P) { pos.slot = 0; pos.phase ^= 1u; }
    }
    return e;
  }
};

// dynamic shared memory of the CACHED variant (phase 3): own rows' U[t][x], SA, PA and own
// columns' V[t][y], SB, PB stay on chip for the whole rook search, plus the E / raw values of
// the last steps.  Phase 2 uses the same buffer first.
__host__ __device__ __forceinline__ long long greedy_cache_doubles(long long rpcap, int cap) {
  // U[cap-1] Ecol Acol SA(2) PA(3) | V[cap-1] Erow SB(2) PB(3)
  return rpcap * ((cap - 1) + 1 + 1 + 2 + 3 + (cap - 1) + 1 + 2 + 3);
}

#ifndef TTC_STEP_INLINE
#define TTC_STEP_INLINE __forceinline__   // (__noinline__: StepCtx goes to local memory, D_20 14.7 -> 17.1 ms)
#endif
// everything a rook step needs (one per CTA, built once per launch)
struct StepCtx {
  const DevCtx* c;
  GreedySmem* S;
  int job, k, n, cap, r, rl, rr, tid, T;
  int xb, xe, yb, ye, sbn, rpcap, jo, jcx;  // intra-superblock indices: < 2^31 (n <= 4096, cap <= 64)
  double *U, *V, *Araw, *Uc, *Ecol, *Acol, *Vc, *Erow;
  ESum* SAc;
  DDE* PAc;
  ESum* SBc;
  DDE* PBc;
  const double *uk, *uk1;
  bool stage_n;
  unsigned long long rowmask, colmask;  // bit j: this thread's j-th row / column is a pivot's
  bool timer;                           // phase clock owner (tt_cross_get_phase_times)
  double* ring;                         // non-cached: DotRing / TmaRing buffer (dyn)
  int ring_tb;                          // terms per ring stage
  int ring_p;                           // TMA ring stages
  bool tma;                             // stream through the TMA ring (else the cp.async DotRing)
  RingPos* rpos;                        // TMA ring position (persists across steps and sweeps)
  DDE* f_node;                          // staged node factors (dynamic shared memory, stage_n)
};

// column step E(:, y) on this CTA's rows -> U[r][:] (or the row cache), raw values; returns
// the thread's (|E|, row) candidate.  The factors that depend on the fixed column are staged
// once per step: S.fs = SB[beta][b], S.fp = PB[beta][b], f_slot[alpha] = CX[alpha][beta] *
// QL1[alpha][b], f_node[a] = QR0[beta][a].
template <int FAMILY, bool CACHED>
__device__ TTC_STEP_INLINE void column_eval(const StepCtx& X, int y, double& bv_out, long long& bf_out) {
  const DevCtx& c = *X.c;
  GreedySmem& S = *X.S;
  const int n = X.n, cap = X.cap, r = X.r, tid = X.tid, T = X.T;
  const int sbn = X.sbn, jo = X.jo, jcx = X.jcx, xb = X.xb, xe = X.xe, rpcap = X.rpcap;
  const int be = y / n, b = y - (y / n) * n;
  TRACE(10);
  if (tid < r) S.vec[tid] = X.V[tid * sbn + y];
  if (tid == 0 && FAMILY < 2) {
    S.fs = c.SB[jo + be * n + b];
    if (FAMILY == 1) S.fp = c.PB[jo + be * n + b];
  }
  if (FAMILY == 1) {
    for (int al = tid; al < X.rl; al += T) {
      DDE f = c.CX[jcx + al * cap + be];
      dde_mul(f, c.QL1[jo + al * n + b]);
      S.f_slot[al] = f;
    }
    if (X.stage_n)
      for (int a = tid; a < n; a += T) X.f_node[a] = c.QR0[jo + be * n + a];
  }
  const double ub = X.uk1[b];
  __syncthreads();
  TRACE(11);
  double bv = -1.0;
  long long bf = LLONG_MAX;
  const bool stream = !CACHED && xe - xb >= c.ring_min * T;
#if TTC_TMA
  // (one ring kind per build: both live at once cost ~1 KB of spills per thread)
  constexpr bool use_ring = false;
  const bool use_tma = stream && X.tma;   // (else plain loads)
  TmaRing<TTC_EVICT_FIRST && FAMILY <= 1> ring;
  if (use_tma) ring.start(X.ring, c.tmapU, &S, T, tid, X.ring_tb, X.ring_p, r, X.job * cap, xb, xe, *X.rpos, c.l2_keep);
#else
  constexpr bool use_tma = false;
  const bool use_ring = stream;
  DotRing<false> ring;   // (no cache hint: see TTC_EVICT_FIRST)
  if (use_ring) ring.init(X.ring, X.U, T, tid, X.ring_tb, sbn, r, xb, xe);
#endif
#if TTC_TMA
  // (the TMA ring's barriers count every warp: all threads run every row block, a thread
  // past the last row computes a clamped duplicate and stores nothing)
  const int nblk = xe > xb ? (xe - xb + T - 1) / T : 0;
  #pragma unroll 1
  for (int jrow = 0; jrow < nblk; ++jrow) {
    const bool valid = xb + jrow * T + tid < xe;
    const int x = valid ? xb + jrow * T + tid : xe - 1;
#else
  int jrow = 0;
  #pragma unroll 1
  for (int x = xb + tid; x < xe; x += T, ++jrow) {
    constexpr bool valid = true;
#endif
    if (TTC_PREFETCH && !CACHED && FAMILY < 2 && valid && x + T < xe) {   // the next row block's tables
      prefetch_l1(&c.SA[jo + x + T]);
      if (FAMILY == 1) prefetch_l1(&c.PA[jo + x + T]);
    }
    const int al = x / n, a = x - al * n;
    const double ua = X.uk[a];
    double raw;
    if (FAMILY >= 2) {
      raw = sb_entry<FAMILY>(c, X.job, X.k, al, a, be, b);
    } else if (FAMILY == 0) {
      ESum s = CACHED ? X.SAc[x - xb] : c.SA[jo + x];
      esum_add(s, S.fs);
      const double Sd = esum_round(s);
      const double SS = __dmul_rn(Sd, Sd);
      bool ok;
      raw = div_pre_fast(1.0, SS, rcp_refined(SS), ok);
      if (!ok) raw = __drcp_rn(SS);
    } else {
      ESum s = CACHED ? X.SAc[x - xb] : c.SA[jo + x];
      esum_add(s, S.fs);
      const double Sd = esum_round(s);
      const double SS = __dmul_rn(Sd, Sd);
      DDE p = CACHED ? X.PAc[x - xb] : c.PA[jo + x];
      dde_mul(p, S.fp);
      dde_mul(p, S.f_slot[al]);
      dde_mul(p, X.stage_n ? X.f_node[a] : c.QR0[jo + be * n + a]);
      bool o1, o2;
      DDE pr = p;
      dde_mul_d(pr, rho_fast(ua, ub, o1));
      raw = dde_div_fast(pr, SS, o2);
      if (!(o1 && o2)) {
        dde_mul_d(p, rho(ua, ub));
        raw = dde_div(p, SS);
      }
    }
    double e = raw;
    if (CACHED)
      for (int t = 0; t < r; ++t) e = __dsub_rn(e, __dmul_rn(X.Uc[t * rpcap + (x - xb)], S.vec[t]));
    else if (use_tma || use_ring)
      e = ring.dot_sub(e, S.vec);
    else
      for (int t = 0; t < r; ++t) e = __dsub_rn(e, __dmul_rn(X.U[t * sbn + x], S.vec[t]));
    if (!valid) continue;
    bool piv = jrow < 64 && ((X.rowmask >> jrow) & 1ULL);   // a pivot row (E is exactly 0 there)
    if (jrow >= 64)
      for (int t = 0; t < r; ++t) piv |= (S.xs[t] == x);
    if (piv) e = 0.0;
    if (CACHED) {
      X.Acol[x - xb] = raw;
      X.Ecol[x - xb] = e;
    } else {
      X.Araw[x] = raw;
      X.U[r * sbn + x] = e;
    }
    if (cand_better(fabs(e), x, bv, bf)) { bv = fabs(e); bf = x; }
  }
#if TTC_TMA
  if (use_tma) *X.rpos = ring.pos;
#endif
  bv_out = bv;
  bf_out = bf;
}

// row step E(x, :) on this CTA's columns -> V[r][:] (or the column cache); staged:
// S.fs = SA[alpha][a], S.fp = PA[alpha][a], f_slot[beta] = CX[alpha][beta] * QR0[beta][a],
// f_node[b] = QL1[alpha][b]
template <int FAMILY, bool CACHED>
__device__ TTC_STEP_INLINE void row_eval(const StepCtx& X, int x, double& bv_out, long long& bf_out) {
  const DevCtx& c = *X.c;
  GreedySmem& S = *X.S;
  const int n = X.n, cap = X.cap, r = X.r, tid = X.tid, T = X.T;
  const int sbn = X.sbn, jo = X.jo, jcx = X.jcx, yb = X.yb, ye = X.ye, rpcap = X.rpcap;
  const int al = x / n, a = x - (x / n) * n;
  TRACE(20);
  if (tid < r) S.vec[tid] = X.U[tid * sbn + x];
  if (tid == 0 && FAMILY < 2) {
    S.fs = c.SA[jo + x];
    if (FAMILY == 1) S.fp = c.PA[jo + x];
  }
  if (FAMILY == 1) {
    for (int be = tid; be < X.rr; be += T) {
      DDE f = c.CX[jcx + al * cap + be];
      dde_mul(f, c.QR0[jo + be * n + a]);
      S.f_slot[be] = f;
    }
    if (X.stage_n)
      for (int b = tid; b < n; b += T) X.f_node[b] = c.QL1[jo + al * n + b];
  }
  const double ua = X.uk[a];
  __syncthreads();
  TRACE(21);
  double bv = -1.0;
  long long bf = LLONG_MAX;
  const bool stream = !CACHED && ye - yb >= c.ring_min * T;
#if TTC_TMA
  // (one ring kind per build: both live at once cost ~1 KB of spills per thread)
  constexpr bool use_ring = false;
  const bool use_tma = stream && X.tma;   // (else plain loads)
  TmaRing<TTC_EVICT_FIRST && FAMILY <= 1> ring;
  if (use_tma) ring.start(X.ring, c.tmapV, &S, T, tid, X.ring_tb, X.ring_p, r, X.job * cap, yb, ye, *X.rpos, c.l2_keep);
#else
  constexpr bool use_tma = false;
  const bool use_ring = stream;
  DotRing<false> ring;   // (no cache hint: see TTC_EVICT_FIRST)
  if (use_ring) ring.init(X.ring, X.V, T, tid, X.ring_tb, sbn, r, yb, ye);
#endif
#if TTC_TMA
  const int nblk = ye > yb ? (ye - yb + T - 1) / T : 0;
  #pragma unroll 1
  for (int jcol = 0; jcol < nblk; ++jcol) {
    const bool valid = yb + jcol * T + tid < ye;
    const int y = valid ? yb + jcol * T + tid : ye - 1;
#else
  int jcol = 0;
  #pragma unroll 1
  for (int y = yb + tid; y < ye; y += T, ++jcol) {
    constexpr bool valid = true;
#endif
    if (TTC_PREFETCH && !CACHED && FAMILY < 2 && valid && y + T < ye) {   // the next column block's tables
      prefetch_l1(&c.SB[jo + y + T]);
      if (FAMILY == 1) prefetch_l1(&c.PB[jo + y + T]);
    }
    const int be = y / n, b = y - be * n;
    const double ub = X.uk1[b];
    double e;
    if (FAMILY >= 2) {
      e = sb_entry<FAMILY>(c, X.job, X.k, al, a, be, b);
    } else if (FAMILY == 0) {
      ESum s = CACHED ? X.SBc[y - yb] : c.SB[jo + y];
      esum_add(s, S.fs);
      const double Sd = esum_round(s);
      const double SS = __dmul_rn(Sd, Sd);
      bool ok;
      e = div_pre_fast(1.0, SS, rcp_refined(SS), ok);
      if (!ok) e = __drcp_rn(SS);
    } else {
      ESum s = CACHED ? X.SBc[y - yb] : c.SB[jo + y];
      esum_add(s, S.fs);
      const double Sd = esum_round(s);
      const double SS = __dmul_rn(Sd, Sd);
      DDE p = CACHED ? X.PBc[y - yb] : c.PB[jo + y];
      dde_mul(p, S.fp);
      dde_mul(p, S.f_slot[be]);
      dde_mul(p, X.stage_n ? X.f_node[b] : c.QL1[jo + al * n + b]);
      bool o1, o2;
      DDE pr = p;
      dde_mul_d(pr, rho_fast(ua, ub, o1));
      e = dde_div_fast(pr, SS, o2);
      if (!(o1 && o2)) {
        dde_mul_d(p, rho(ua, ub));
        e = dde_div(p, SS);
      }
    }
    if (CACHED)
      for (int t = 0; t < r; ++t) e = __dsub_rn(e, __dmul_rn(S.vec[t], X.Vc[t * rpcap + (y - yb)]));
    else if (use_tma || use_ring)
      e = ring.dot_sub(e, S.vec);   // (S.vec[t] * V[t][y]: the product commutes bitwise)
    else
      for (int t = 0; t < r; ++t) e = __dsub_rn(e, __dmul_rn(S.vec[t], X.V[t * sbn + y]));
    if (!valid) continue;
    bool piv = jcol < 64 && ((X.colmask >> jcol) & 1ULL);   // a pivot column
    if (jcol >= 64)
      for (int t = 0; t < r; ++t) piv |= (S.ys[t] == y);
    if (piv) e = 0.0;
    if (CACHED) X.Erow[y - yb] = e;
    else X.V[r * sbn + y] = e;
    if (cand_better(fabs(e), y, bv, bf)) { bv = fabs(e); bf = y; }
  }
#if TTC_TMA
  if (use_tma) *X.rpos = ring.pos;
#endif
  bv_out = bv;
  bf_out = bf;
}

// cluster exchange of the per-CTA candidates without a cluster barrier: CTA j writes its
// candidate into slot j of every CTA's xc[p] with st.async, which completes bytes on the
// receiver's mbarrier xbar[p]; each CTA waits on its own barrier (expecting 16*G bytes) and
// reduces the G slots in cluster-rank order.  p = step & 1 double-buffers the slots: a CTA can
// send step s+2 only after every CTA has sent step s+1, i.e. finished reading step s.
__device__ __forceinline__ void xbar_init(GreedySmem* S) {
  if (threadIdx.x == 0) {
    for (int p = 0; p < 2; ++p) {
      const unsigned a = (unsigned)__cvta_generic_to_shared(&S->xbar[p]);
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(a) : "memory");
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  // (the caller's cluster barrier orders the init before any remote complete_tx)
}

__device__ __forceinline__ unsigned cluster_addr(const void* p, int cta) {
  unsigned r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"((unsigned)__cvta_generic_to_shared(p)), "r"(cta));
  return r;
}

// CTA argmax + cluster argmax of (v, f) -> S->best, out of line (one copy of the shuffle
// trees for all steps: the sweep kernel is instruction-cache bound).  xstep counts the
// cluster exchanges of this launch (identical on every CTA of the cluster).
__device__ __noinline__ void argmax_step(GreedySmem* S, double v, long long f, int G, int xstep) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  warp_argmax(v, f);
  if (lane == 0) S->red[warp] = {v, f};
  __syncthreads();
  TRACE(31);
  if (warp == 0) {
    const int nw = blockDim.x >> 5;
    double bv = lane < nw ? S->red[lane].val : -1.0;
    long long bf = lane < nw ? S->red[lane].idx : LLONG_MAX;
    TRACE(35);
    warp_argmax(bv, bf);
    TRACE(36);
    if (G == 1) {
      if (lane == 0) S->best = {bv, bf};
    } else {
      const int p = xstep & 1;
      const unsigned bar = (unsigned)__cvta_generic_to_shared(&S->xbar[p]);
      if (lane == 0)
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(16 * G) : "memory");
      TRACE(37);
      if (lane < G) {
        const int me = (int)cg::this_cluster().block_rank();
        const unsigned ra = cluster_addr(&S->xc[p][me], lane), rb = cluster_addr(&S->xbar[p], lane);
        asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v2.b64 [%0], {%1, %2}, [%3];" ::"r"(ra),
                     "l"(__double_as_longlong(bv)), "l"(bf), "r"(rb)
                     : "memory");
      }
      TRACE(32);
      const unsigned par = (unsigned)(xstep >> 1) & 1u;
      unsigned ok = 0;
      while (!ok)
        asm volatile(
            "{\n .reg .pred q;\n"
            " mbarrier.try_wait.parity.shared::cta.b64 q, [%1], %2;\n"
            " selp.u32 %0, 1, 0, q;\n}"
            : "=r"(ok) : "r"(bar), "r"(par) : "memory");
      TRACE(33);
      bv = -1.0;
      bf = LLONG_MAX;
      if (lane < G) {
        bv = S->xc[p][lane].val;
        bf = S->xc[p][lane].idx;
      }
      warp_argmax(bv, bf);
      if (lane == 0) S->best = {bv, bf};
    }
  }
  __syncthreads();
  TRACE(34);
}

// One Alg. 6 sweep of superblock `job` (all CTAs of its cluster): phases 1-3 with the ranks
// r (own), rl / rr (neighbours, at the end of the previous sweep) given by the caller; the
// new pivot (if any) is written to the record Rn (slot r and rank); returns the new rank.
// release / acquire flags of the persistent sweep loop (global memory, gpu scope)
__device__ __forceinline__ int ld_acquire(const int* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release(int* p, int v) {
  asm volatile("st.release.gpu.global.s32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
// system scope: a flag written by (or for) a kernel on another GPU through NVLink peer memory
__device__ __forceinline__ int ld_acquire_sys(const int* p) {
  int v;
  asm volatile("ld.acquire.sys.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_sys(int* p, int v) {
  asm volatile("st.release.sys.global.s32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// Cross-GPU wavefront (DevCtx prec/pring/pdone): superblock k's new record (slot r: tuple and
// parents; the rank word), its rank after the sweep and its done flag, written into the copies
// of the neighbour rank `side` -- plain stores over NVLink, then the flag with a system-scope
// release, which orders them before it for the peer's system-scope acquire (Alg. 6
// lines 6-8: the new pivots go to the neighbouring processes only).  Rn: this rank's record
// of k, already complete (same thread).
__device__ __noinline__ void peer_publish(const DevCtx& c, int side, int k, int sweep, int r, bool add, const int* Rn) {
  int* R = c.prec[side] + (long long)k * c.RS;
  if (add) {
    const int d = c.d;
    for (int q = 0; q < d; ++q) R[1 + (long long)r * d + q] = Rn[1 + (long long)r * d + q];
    R[1 + (long long)c.cap * d + 2 * r] = Rn[1 + (long long)c.cap * d + 2 * r];
    R[2 + (long long)c.cap * d + 2 * r] = Rn[2 + (long long)c.cap * d + 2 * r];
    R[0] = r + 1;
  }
  c.pring[side][k * 2 + (sweep & 1)] = add ? r + 1 : r;
  st_release_sys(&c.pdone[side][k], sweep + 1);
}

template <int FAMILY, bool CACHED, bool PEER = false>
__device__ __forceinline__ int sweep_body(const DevCtx& c, const DevCtx& cs, GreedySmem& S, double* dyn, int sweep, int job, int r,
                                          int rl, int rr, int* Rn, int& xstep, RingPos& rpos, bool end_sync,
                                          int rows_done, int cols_done, bool xy_known, bool release) {
  cg::cluster_group cl = cg::this_cluster();
  const int G = c.G;
  const int cr = (int)cl.block_rank();
  const int k = c.kb + job, d = c.d, n = c.n, cap = c.cap;
  const int tid = threadIdx.x, T = blockDim.x;
  // intra-superblock indices are int: n <= 4096, cap <= 64 (tt_cross_init)
  const int R = rl * n, C = rr * n;
  // rows / columns of this CTA (contiguous blocks); the cached variant's shared-memory
  // stride is the capacity block rpcap >= rpc, cpc
  // (TMA ring: even block sizes, so every CTA's first row starts a 16-byte aligned TMA box --
  // an odd start raised "illegal instruction", tools/tma_probe.cu)
  const int rpc = c.tma ? (((R + G - 1) / G + 1) & ~1) : (R + G - 1) / G;
  const int cpc = c.tma ? (((C + G - 1) / G + 1) & ~1) : (C + G - 1) / G;
  const int rpcap = (int)((c.sbn + G - 1) / G);
  const int xb = cr * rpc, xe = min(R, xb + rpc);
  const int yb = cr * cpc, ye = min(C, yb + cpc);
  const int sbn = (int)c.sbn;
  double* U = c.U + (long long)job * cap * sbn;
  double* V = c.V + (long long)job * cap * sbn;
  double* Araw = c.Araw + (long long)job * sbn;
  const int jo = job * cap * n;   // table offset of this job
  const int jcx = job * cap * cap;
  const double* uk = c.u + (long long)k * n;
  const double* uk1 = c.u + (long long)(k + 1) * n;
  // cached layout (rpcap rows / columns per CTA)
  double* Uc = dyn;                                  // [t][rpcap]
  double* Ecol = Uc + (long long)(cap - 1) * rpcap;  // [rpcap]
  double* Acol = Ecol + rpcap;                       // [rpcap]
  ESum* SAc = reinterpret_cast<ESum*>(Acol + rpcap);  // [rpcap]
  DDE* PAc = reinterpret_cast<DDE*>(SAc + rpcap);     // [rpcap]
  double* Vc = reinterpret_cast<double*>(PAc + rpcap);  // [t][rpcap]
  double* Erow = Vc + (long long)(cap - 1) * rpcap;  // [rpcap]
  ESum* SBc = reinterpret_cast<ESum*>(Erow + rpcap);  // [rpcap]
  DDE* PBc = reinterpret_cast<DDE*>(SBc + rpcap);     // [rpcap]

  const bool timer = TTC_PHASE_CLOCKS && c.phase_ns && job == c.phase_job && cr == 0 && tid == 0;
  unsigned long long t_last = timer ? gtimer() : 0;
  auto phase = [&](int ph) {
    if (timer) {
      const unsigned long long t = gtimer();
      ph_add(c.phase_ns, sweep, ph, t - t_last);
      t_last = t;
    }
  };
  if (!xy_known && tid < r) {   // (the persistent loop keeps them in S.xs / S.ys: appended below)
    int px, py;
    pivot_pos(c, k, tid, px, py);
    S.xs[tid] = px;
    S.ys[tid] = py;
  }
  // Alg. 2 line 1 sample positions of this sweep, drawn now (they depend only on the sweep,
  // k and the superblock shape) by the warps after warp 0, which starts the tables; kept in
  // the f_node region until the samples phase (the rook steps restage it afterwards)
  DDE* f_node = reinterpret_cast<DDE*>(dyn + c.fnode_off);
  int* smp = reinterpret_cast<int*>(f_node);
  {
    const uint64_t tag = 1ULL + (uint64_t)sweep;
    for (int q = tid >= 32 ? tid - 32 : tid + T - 32; q < c.ns; q += T) {
      smp[2 * q] = (int)(splitmix64(c.seed, draw_ctr(tag, d, k, 2 * q)) % (uint64_t)R);
      smp[2 * q + 1] = (int)(splitmix64(c.seed, draw_ctr(tag, d, k, 2 * q + 1)) % (uint64_t)C);
    }
  }
  const bool first = rows_done == 0 && cols_done == 0;
  __syncthreads();
  TRACE(1);
  unsigned long long ext_ent = 0, ext_upd = 0;

  // ---- phase 1: factor tables of the new left slots [rows_done, rl) and right slots
  // [cols_done, rr); every CTA of the cluster takes a strided share of the nodes a
  if (FAMILY < 2) {
    // with G >= 2 the first half of the cluster builds the left tables, the second half the
    // right ones; each CTA takes a strided share of the nodes a
    const int gl = G >= 2 ? G / 2 : 1;
    const bool do_l = G == 1 || cr < gl, do_r = G == 1 || cr >= gl;
    const int il = G == 1 ? 0 : cr, ir = G == 1 ? 0 : cr - gl;
    // family D: the CX pairs of the new slots go to warps 1.. of every CTA, during the first
    // side-table call (or on their own when this CTA has no new slot)
    const int nwc = (T >> 5) - 1;
    const int cx_gw = cr * nwc + (tid >> 5) - 1, cx_nwg = FAMILY == 1 ? G * nwc : 0;
    bool cx_pending = FAMILY == 1;
    if (do_l)
      for (int slot = rows_done; slot < rl; ++slot) {
        sb_side_tables(cs, job, 0, slot, il * T, gl * T, rl, rr, rows_done, cols_done, cx_gw, cx_pending ? cx_nwg : 0);
        cx_pending = false;
        __syncthreads();
      }
    if (do_r)
      for (int slot = cols_done; slot < rr; ++slot) {
        sb_side_tables(cs, job, 1, slot, ir * T, (G >= 2 ? G - gl : 1) * T, rl, rr, rows_done, cols_done, cx_gw,
                       cx_pending ? cx_nwg : 0);
        cx_pending = false;
        __syncthreads();
      }
    if (cx_pending && tid >= 32) sb_cx_share(cs, job, rows_done, cols_done, rl, rr, cx_gw, cx_nwg);
  }
  TRACE(2);
  cl.sync();  // tables visible to the whole cluster
  TRACE(3);
  phase(PH_TABLES);

  // ---- phase 2: u / v of the existing pivots on the new rows and columns
  // (per-sweep log slots 14 / 15: this phase's own time in the first row CTA / the first column
  // CTA of the logged superblock, before the cluster barrier)
  const bool ext_clock = TTC_PHASE_CLOCKS && c.phase_ns && job == c.phase_job && tid == 0 && (cr == 0 || cr == (G >= 2 ? G / 2 : 0));
  const unsigned long long t_ext0 = ext_clock ? gtimer() : 0;
  {
    __shared__ int p_al[TTC_MAX_RANK_DEV], p_a[TTC_MAX_RANK_DEV];
    double* pdiag = s_pdiag;
    double* prcp = s_prcp;
    double* coef = dyn;
    double* tile = dyn + (long long)cap * cap;
    const long long ext_dyn = extend_smem_doubles(cap);   // (dynamic shared memory is at least this)
    const int nr_new = (rl - rows_done) * n, nc_new = (rr - cols_done) * n;
    // with G >= 2 the first half of the cluster extends the rows, the second half the columns
    // (independent: the column recurrence reads u only at old pivot rows, or A(t0) at the
    // first sweep), so the two latency chains overlap
    // streaming shapes: every CTA extends a share of the rows, then of the columns (D_20:
    // 14.80 -> 14.65 ms -- the slower column half no longer sets the pace alone); the cached
    // shapes of the small problems keep the halves (D_5: 0.76 vs 0.82 ms)
    constexpr bool ext_all = TTC_EXT_ALL && !CACHED && FAMILY == 1;   // (family C: its tile variant on few rows per CTA -- C_10 1.63 -> 1.73 ms -- keeps the halves)
    const int gr = ext_all ? G : (G >= 2 ? G / 2 : 1), gc = ext_all ? G : (G >= 2 ? G - gr : 1);
    const bool do_rows = ext_all || G == 1 || cr < gr, do_cols = ext_all || G == 1 || cr >= gr;
    const int rr_i = ext_all ? cr : (G == 1 ? 0 : cr), cc_i = ext_all ? cr : (G == 1 ? 0 : cr - gr);
    const int rchunk = (nr_new + gr - 1) / gr, cchunk = (nc_new + gc - 1) / gc;
    // the register variant when a CTA's rows fill its threads at the lanes per row the rank
    // needs (D_20 from rank 17); else the tile variant spreads the few rows' entries over all
    // threads (D_5: ~33 rows per CTA -- the register variant measured 0.93 vs 0.77 ms there)
    const bool ext_reg = EXT_REG && FAMILY == 1 && min(rchunk, cchunk) * ext_reg_lanes(r) >= (ext_all ? T / 2 : T);
    if (do_rows) {   // rows: fixed index = pivot columns y_s
      if (tid < r) {
        p_al[tid] = S.ys[tid] / n;
        p_a[tid] = S.ys[tid] - (S.ys[tid] / n) * n;
      }
      __syncthreads();
      const int lo = rows_done * n + rr_i * rchunk;
      if (ext_reg)
        extend_side_reg<1>(cs, sweep, job, k, 0, r, lo, min(lo + rchunk, rl * n), p_al, p_a,
                                                  pdiag, prcp, dyn, ext_dyn, ext_ent, ext_upd);
      else
        extend_side<FAMILY>(cs, sweep, job, k, 0, r, lo, min(lo + rchunk, rl * n), p_al, p_a, pdiag, prcp, coef, tile,
                            ext_ent, ext_upd);
      __syncthreads();
    }
    if (do_cols) {   // columns: fixed index = pivot rows x_s, divisors u_s(x_s) (A(t0) at first)
      if (tid < r) {
        p_al[tid] = S.xs[tid] / n;
        p_a[tid] = S.xs[tid] - (S.xs[tid] / n) * n;
        pdiag[tid] = first ? *c.p0val : U[tid * sbn + S.xs[tid]];
        prcp[tid] = rcp_refined(pdiag[tid]);
      }
      __syncthreads();
      const int lo = cols_done * n + cc_i * cchunk;
      if (ext_reg)
        extend_side_reg<1>(cs, sweep, job, k, 1, r, lo, min(lo + cchunk, rr * n), p_al, p_a,
                                                  pdiag, prcp, dyn, ext_dyn, ext_ent, ext_upd);
      else
        extend_side<FAMILY>(cs, sweep, job, k, 1, r, lo, min(lo + cchunk, rr * n), p_al, p_a, pdiag, prcp, coef, tile,
                            ext_ent, ext_upd);
    }
  }
  TRACE(4);
  // (the rook steps read U / V through the TMA engine -- the async proxy: order this thread's
  // generic-proxy stores before the barrier that publishes them)
  // (and the extension's shared-memory scratch, which the TMA ring overwrites next)
  if (c.tma) {
    if (TTC_FENCE_ALL) asm volatile("fence.proxy.async;" ::: "memory");
    else asm volatile("fence.proxy.async.global;" ::: "memory");
  }
  if (ext_clock && sweep < TTC_LOG_SWEEPS) c.phase_ns[TTC_NPHASES + sweep * TTC_LOG_W + 14 + (cr != 0)] += gtimer() - t_ext0;
  cl.sync();  // u / v of the new rows and columns visible to the whole cluster
  TRACE(5);
  phase(PH_EXTEND);

  bool active = r < cap;
  const double p0 = U[S.xs[0]];  // u_0(x_0) = A(x_0, y_0)
  if (p0 == 0.0) active = false;  // singular first pivot: leave the interface (R8)
  double scale = c.praw_max[job];
  if (scale < 0.0) scale = fabs(p0);
  unsigned long long evals = 0, upd = 0, ring_steps = 0;
  int steps = 0;
  int xst = 0, yst = 0;
  bool added = false;
  double raw_star = 0.0;
  // the new pivot record (Alg. 6 line 4), the superblock state and -- persistent loop -- the
  // rank ring and the release of done[k] for the neighbours, by thread 0 of CTA 0
  auto publish = [&](bool add, double raw) {
    if (cr != 0 || tid != 0) return;
    if (add) {
      const int al = xst / n, a = xst - al * n, be = yst / n, b = yst - be * n;
      const int* TL = k > 0 ? rec_piv(c.rec_cur, c.RS, k - 1) + (long long)al * d : nullptr;
      const int* TR = k < d - 2 ? rec_piv(c.rec_cur, c.RS, k + 1) + (long long)be * d : nullptr;
      int* tup = Rn + 1 + (long long)r * d;
      for (int q = 0; q < k; ++q) tup[q] = TL[q];
      tup[k] = a;
      tup[k + 1] = b;
      for (int q = k + 2; q < d; ++q) tup[q] = TR[q];
      int* par = Rn + 1 + (long long)cap * d + 2 * r;
      par[0] = al;
      par[1] = be;
      Rn[0] = r + 1;
      scale = fmax(scale, fabs(raw));
    }
    c.praw_max[job] = scale;
    c.sbstate[job * 4 + 0] = rl;
    c.sbstate[job * 4 + 1] = rr;
    if (release) {
      c.rank_ring[k * 2 + (sweep & 1)] = add ? r + 1 : r;
      st_release(&c.done[k], sweep + 1);  // the record writes above happen-before this release
      // boundary superblocks of a rank: the same to the neighbour rank's copies
      if (PEER && c.pdone[0] && k == c.pb_lo) peer_publish(cs, 0, k, sweep, r, add, Rn);   // (cs: the shared copy -- a
      if (PEER && c.pdone[1] && k + 1 == c.pb_hi) peer_publish(cs, 1, k, sweep, r, add, Rn);   // reference to c would copy it to local memory)
    }
  };
  const bool stage_n = n <= STAGE_N;

  if (active) {
    if (CACHED) {
#pragma unroll 1
      for (int t = 0; t < r; ++t)
#pragma unroll 1
        for (int j = tid; j < rpcap; j += T) {
          if (xb + j < xe) cp_async8(&Uc[t * rpcap + j], &U[t * sbn + xb + j]);
          if (yb + j < ye) cp_async8(&Vc[t * rpcap + j], &V[t * sbn + yb + j]);
        }
#pragma unroll 1
      for (int j = tid; j < rpcap; j += T) {
        if (xb + j < xe) {
          const double* sa = reinterpret_cast<const double*>(&c.SA[jo + xb + j]);
          double* da = reinterpret_cast<double*>(&SAc[j]);
          cp_async8(da, sa);
          cp_async8(da + 1, sa + 1);
          if (FAMILY == 1) {
            const double* pa = reinterpret_cast<const double*>(&c.PA[jo + xb + j]);
            double* dp = reinterpret_cast<double*>(&PAc[j]);
            cp_async8(dp, pa);
            cp_async8(dp + 1, pa + 1);
            cp_async8(dp + 2, pa + 2);
          }
        }
        if (yb + j < ye) {
          const double* sb = reinterpret_cast<const double*>(&c.SB[jo + yb + j]);
          double* db = reinterpret_cast<double*>(&SBc[j]);
          cp_async8(db, sb);
          cp_async8(db + 1, sb + 1);
          if (FAMILY == 1) {
            const double* pb = reinterpret_cast<const double*>(&c.PB[jo + yb + j]);
            double* dp = reinterpret_cast<double*>(&PBc[j]);
            cp_async8(dp, pb);
            cp_async8(dp + 1, pb + 1);
            cp_async8(dp + 2, pb + 2);
          }
        }
      }
      cp_async_wait_all();
      TRACE(6);
      // visibility of the cache to the other threads: the __syncthreads of the first step
    }
    // the first column step's first ring stage, in flight during the samples phase (U of this
    // CTA's rows: independent of the sampled column)
    if ((TTC_RING_PREFETCH & 1) && !CACHED && c.tma && xe - xb >= c.ring_min * T) {
      TmaRing<TTC_EVICT_FIRST && FAMILY <= 1> pf;
      pf.prefetch(dyn, c.tmapU, &S, T, tid, c.ring_tb, c.ring_p, r, job * cap, xb, xe, rpos, c.l2_keep);
    }
    // ---- Alg. 2 line 1: n_samples random entries, largest |E| (every CTA, identically).
    // A warp per four samples: the lanes load the u/v factors of all four at once (t = lane,
    // lane + 32) and form the products u_t(x) v_t(y); lanes 0-3 evaluate the raw entries;
    // then the four E = A - sum_t u_t v_t run their t-ascending subtraction chains side by
    // side through shuffles -- the oracle's operations in its order.  (A thread per sample
    // waited for its 2r scattered factor loads in dependent batches: ~16 us per late D_20
    // sweep.)
    {
      double bv = -1.0;
      long long bf = LLONG_MAX;
      const int lane = tid & 31, nw = T >> 5;
#pragma unroll 1
      for (int q0 = (tid >> 5) * 4; q0 < c.ns; q0 += nw * 4) {   // (warp-uniform)
        double pa[4], pb[4];
        bool msk[4];
#pragma unroll
        for (int m = 0; m < 4; ++m) {
          const int q = min(q0 + m, c.ns - 1);
          const int sx = smp[2 * q], sy = smp[2 * q + 1];
          const int t1 = lane + 32;
          pa[m] = lane < r ? __dmul_rn(U[lane * sbn + sx], V[lane * sbn + sy]) : 0.0;
          pb[m] = t1 < r ? __dmul_rn(U[t1 * sbn + sx], V[t1 * sbn + sy]) : 0.0;
          msk[m] = (lane < r && (S.xs[lane] == sx || S.ys[lane] == sy)) || (t1 < r && (S.xs[t1] == sx || S.ys[t1] == sy));
        }
        double raw;
        {
          const int q = min(q0 + (lane & 3), c.ns - 1);
          const int sx = smp[2 * q], sy = smp[2 * q + 1];
          const int al = sx / n, a = sx - al * n;
          const int be = sy / n, b = sy - be * n;
          raw = sb_entry<FAMILY>(c, job, k, al, a, be, b);
        }
        double e[4];
#pragma unroll
        for (int m = 0; m < 4; ++m) e[m] = __shfl_sync(0xffffffffu, raw, m);
#pragma unroll 4
        for (int t = 0; t < r; ++t)
#pragma unroll
          for (int m = 0; m < 4; ++m) e[m] = __dsub_rn(e[m], __shfl_sync(0xffffffffu, t < 32 ? pa[m] : pb[m], t & 31));
#pragma unroll
        for (int m = 0; m < 4; ++m) {
          if (__any_sync(0xffffffffu, msk[m])) e[m] = 0.0;   // a pivot row or column: E is exactly 0
          if (q0 + m < c.ns && cand_better(fabs(e[m]), q0 + m, bv, bf)) { bv = fabs(e[m]); bf = q0 + m; }
        }
      }
      TRACE(7);
      argmax_step(&S, bv, bf, 1, 0);   // CTA-local: every CTA drew the same samples
      const int q = (int)S.best.idx;
      xst = smp[2 * q];
      yst = smp[2 * q + 1];
      // smp aliases f_node, which the first column step (family D, staged) overwrites
      // before its own barrier: every thread must have read the winner first
      if (FAMILY == 1 && stage_n) __syncthreads();
      if (cr == 0 && tid == 0) {
        evals += c.ns;
        upd += (unsigned long long)c.ns * r;
      }
      phase(PH_SAMPLES);
    }
    // column step E(:, y) on this CTA's rows; returns the cluster argmax row when `search`.
    // The factors that depend on the fixed column are staged once per step:
    //   S.fs = SB[beta][b], S.fp = PB[beta][b], f_slot[alpha] = CX[alpha][beta]*QL1[alpha][b],
    //   f_node[a] = QR0[beta][a]
    // pivot rows / columns among this thread's first 64 rows / columns (a search beyond)
    unsigned long long rowmask = 0, colmask = 0;
#pragma unroll 1
    for (int t = 0; t < r; ++t) {   // (32-bit: a superblock side has < 2^31 rows)
      const int jx = S.xs[t] - (int)xb, jy = S.ys[t] - (int)yb;
      if (jx >= 0 && jx < (int)(xe - xb)) {
        const int q = jx / T;
        if (jx - q * T == tid && q < 64) rowmask |= 1ULL << q;
      }
      if (jy >= 0 && jy < (int)(ye - yb)) {
        const int q = jy / T;
        if (jy - q * T == tid && q < 64) colmask |= 1ULL << q;
      }
    }
    StepCtx X{&cs, &S, job, k, n, cap, r, rl, rr, tid, T, xb, xe, yb, ye, sbn, rpcap, jo, jcx,
              U, V, Araw, Uc, Ecol, Acol, Vc, Erow, SAc, PAc, SBc, PBc, uk, uk1, stage_n, rowmask, colmask,
              timer, dyn, c.ring_tb, c.ring_p, c.tma != 0, &rpos, f_node};
    auto column = [&](int y, bool search) -> int {
      double bv;
      long long bf;
      const unsigned long long t0 = timer ? gtimer() : 0;
      column_eval<FAMILY, CACHED>(X, y, bv, bf);
      const unsigned long long t1 = timer ? gtimer() : 0;
      if (tid == 0) {
        evals += (unsigned long long)max(0, xe - xb);
        upd += (unsigned long long)max(0, xe - xb) * r;
        ring_steps += !CACHED && xe - xb >= c.ring_min * T;   // (column_eval's stream)
      }
      if (!search) {
        __syncthreads();
        return -1;
      }
      // a search column step is always followed by a row step: its first ring stage (V of this
      // CTA's columns) goes out before the argmax
      if ((TTC_RING_PREFETCH & 2) && !CACHED && c.tma && ye - yb >= c.ring_min * T) {
        TmaRing<TTC_EVICT_FIRST && FAMILY <= 1> pf;
        pf.prefetch(dyn, c.tmapV, &S, T, tid, c.ring_tb, c.ring_p, r, job * cap, yb, ye, rpos, c.l2_keep);
      }
      argmax_step(&S, bv, bf, G, xstep);
      if (timer) {
        ph_add(c.phase_ns, sweep, PH_COL_EVAL, t1 - t0);
        ph_add(c.phase_ns, sweep, PH_COL_ARGMAX, gtimer() - t1);
      }
      ++xstep;
      return (int)S.best.idx;
    };
    auto row = [&](int x, bool search) -> int {
      double bv;
      long long bf;
      const unsigned long long t0 = timer ? gtimer() : 0;
      row_eval<FAMILY, CACHED>(X, x, bv, bf);
      const unsigned long long t1 = timer ? gtimer() : 0;
      if (tid == 0) {
        evals += (unsigned long long)max(0, ye - yb);
        upd += (unsigned long long)max(0, ye - yb) * r;
        ring_steps += !CACHED && ye - yb >= c.ring_min * T;   // (row_eval's stream)
      }
      if (!search) {
        __syncthreads();
        return -1;
      }
      argmax_step(&S, bv, bf, G, xstep);
      if (timer) {
        ph_add(c.phase_ns, sweep, PH_ROW_EVAL, t1 - t0);
        ph_add(c.phase_ns, sweep, PH_ROW_ARGMAX, gtimer() - t1);
      }
      ++xstep;
      return (int)S.best.idx;
    };
    // ---- Alg. 2 lines 2-5: rook search
    // one call site per step kind (the kernel is instruction-cache bound): the loop runs
    // the rook rounds, then at most one extra column and one extra row for the final pivot
    int c_at = -1, g_at = -1;
    int it = 0;
    bool done = c.rook == 0;
    int stage = 0;  // 0: column, 1: row
    while (true) {
      if (stage == 0) {
        const bool search = !done;
        if (!search && c_at == yst) { stage = 1; continue; }
        const int xn = column(yst, search);
        c_at = yst;
        if (search) xst = xn;
        stage = 1;
      } else {
        const bool search = !done;
        if (!search && g_at == xst) break;
        const int yn = row(xst, search);
        g_at = xst;
        if (!search) break;
        steps += 1;
        const bool conv = (yn == yst);
        yst = yn;
        ++it;
        if (conv || it >= c.rook) {
          done = true;
          phase(PH_ROOK);
        }
        stage = 0;
      }
    }
    // the pivot value E(x*, y*) from the shared memory of the CTA owning column y* (cached:
    // also A(x*, y*) from the owner of row x*), read through DSMEM after the barrier
    const int own = (int)(yst / cpc);
    if (cr == own && tid == 0) S.pv = CACHED ? Erow[yst - yb] : V[r * sbn + yst];
    if (CACHED && cr == (int)(xst / rpc) && tid == 0) S.pa = Acol[xst - xb];
    TRACE(8);
    if (G > 1) cl.sync();  // S.pv, S.pa (non-cached: U[r][:], V[r][:], Araw) visible cluster-wide
    else __syncthreads();
    TRACE(9);
    const double pv = G > 1 ? cl.map_shared_rank(&S.pv, own)[0] : S.pv;
    raw_star = CACHED ? (G > 1 ? cl.map_shared_rank(&S.pa, (int)(xst / rpc))[0] : S.pa) : Araw[xst];
    added = fabs(pv) > c.tol * scale;
    // publish first (the neighbours wait for it), then the copy-out / rescale of v_r
    publish(added, raw_star);
    if (CACHED) {   // the final column / row leave the chip once
      for (int x = xb + tid; x < xe; x += T) {
        U[r * sbn + x] = Ecol[x - xb];
        Araw[x] = Acol[x - xb];
      }
#pragma unroll 1
      for (int y = yb + tid; y < ye; y += T) V[r * sbn + y] = added ? __ddiv_rn(Erow[y - yb], pv) : Erow[y - yb];
    } else if (added) {
#pragma unroll 1
      for (int y = yb + tid; y < ye; y += T) V[r * sbn + y] = __ddiv_rn(V[r * sbn + y], pv);
    }
  } else {
    publish(false, 0.0);
  }

  if (c.tma) asm volatile("fence.proxy.async.global;" ::: "memory");   // (U[r], V[r] for the next sweep's TMA reads)
  phase(PH_FINAL);
  if (added && tid == 0) {   // the new pivot's position, for the next sweep of a persistent loop
    S.xs[r] = xst;
    S.ys[r] = yst;
  }
  if (c.counters && tid == 0) {
    evals += ext_ent;
    upd += ext_upd;
    if (evals) {
      atomicAdd(&c.counters[CNT_EVALS], evals);
      atomicAdd(&c.counters[CNT_SB_ENTRIES], evals);
    }
    if (upd) atomicAdd(&c.counters[CNT_SB_UPDATES], upd);
    if (ext_ent) atomicAdd(&c.counters[CNT_EXT_ENTRIES], ext_ent);
    if (ext_upd) atomicAdd(&c.counters[CNT_EXT_UPDATES], ext_upd);
    if (cr == 0 && steps) atomicAdd(&c.counters[CNT_ROOK_STEPS], (unsigned long long)steps);
    if (timer && sweep < TTC_LOG_SWEEPS) c.phase_ns[TTC_NPHASES + sweep * TTC_LOG_W + PH_LAUNCHES] += (unsigned long long)steps;
    if (ring_steps) atomicAdd(&c.counters[CNT_RING_STEPS], ring_steps);
  }
  TRACE(40);
  // no CTA may leave while another can still read its shared memory; inside the persistent
  // loop the next sweep's start barrier does this (nothing a CTA writes to its shared memory
  // before that barrier is read remotely: the exchange slots alternate by step parity, S.pv
  // is rewritten only in the next sweep's final phase)
  if (G > 1 && end_sync) cl.sync();
  TRACE(41);
  phase(PH_END);
  if (timer) atomicAdd(&c.phase_ns[PH_LAUNCHES], 1ULL);
  return added ? r + 1 : r;
}

// neighbour ranks published at the end of each sweep (a ring of two: a neighbour can be at
// most one sweep ahead) and the sweeps each superblock has completed

// single sweep (any world size): ranks from the current records, the updated record goes to
// rec_next (the multi-process exchange buffer)
template <int FAMILY, bool CACHED, int THREADS>
__global__ void __launch_bounds__(THREADS, 512 / THREADS) k_sweep(DevCtx c, int sweep) {
  __shared__ GreedySmem S;
  __shared__ DevCtx s_ctx;   // (see k_sweeps)
  extern __shared__ __align__(1024) double dyn[];
  cg::cluster_group cl = cg::this_cluster();
  if (threadIdx.x == 0) s_ctx = c;
  const int job = blockIdx.x / c.G, k = c.kb + job, d = c.d;
  const int r = rec_rank(c.rec_cur, c.RS, k);
  const int rl = k > 0 ? rec_rank(c.rec_cur, c.RS, k - 1) : 1;
  const int rr = k < d - 2 ? rec_rank(c.rec_cur, c.RS, k + 1) : 1;
  int* Rn = c.rec_next + (long long)k * c.RS;
  const int* Rc = c.rec_cur + (long long)k * c.RS;
  TRACE_INIT();
  xbar_init(&S);
  tma_ring_init(&S);
  if (cl.block_rank() == 0)
    for (int t = threadIdx.x; t < c.RS; t += blockDim.x) Rn[t] = Rc[t];
  cl.sync();  // record copy and exchange barriers ready
  int xstep = 0;
  RingPos rpos{0, 0u, 0};
  const int rn = sweep_body<FAMILY, CACHED>(c, s_ctx, S, dyn, sweep, job, r, rl, rr, Rn, xstep, rpos, true,
                                            c.sbstate[job * 4 + 0], c.sbstate[job * 4 + 1], false, false);
  if (cl.block_rank() == 0 && threadIdx.x == 0) {
    c.rank_ring[k * 2 + (sweep & 1)] = rn;
    c.done[k] = sweep + 1;
  }
  TRACE_FLUSH();
}

// Sweeps [s0, s0 + nsweeps) in one launch (world == 1, all clusters resident): superblock k
// starts sweep s as soon as its neighbours k-1 and k+1 have finished sweep s-1 -- the
// neighbour-only pivot exchange of PAPER.md Alg. 6 lines 6-8, through release/acquire flags
// in global memory instead of a grid-wide barrier.  Records are appended in place (slots
// below a published rank never change).  A wait longer than ~2 s sets flags[1] and abandons
// the launch (reported as an error), so a scheduling failure cannot hang the device.
// PEER: the cross-GPU wavefront variant (boundary superblocks exchange through peer memory,
// DevCtx prec/pring/pdone); a separate instantiation, so the one-GPU kernel carries none of its
// code (its branches cost the one-GPU kernel ~0.8% on D_20: 14.33 vs 14.22 ms, profiles/r02w_*)
template <int FAMILY, bool CACHED, int THREADS, bool PEER = false>
__global__ void __launch_bounds__(THREADS, 512 / THREADS) k_sweeps(DevCtx c, int s0, int nsweeps) {
  __shared__ GreedySmem S;
  __shared__ int s_abort[2];   // by sweep parity: one cluster barrier per sweep start
  // The parameters as seen by the out-of-line helpers (tables, extension, rook-step context):
  // a reference to the kernel parameter itself would make the compiler copy it to local
  // memory and every helper read its fields with LDL -- L1 misses (shared memory leaves L1
  // ~50 KB) that wait a loaded-L2 round trip while the other superblocks stream.  (Ordered
  // before use by the first sweep's cluster barrier.)
  __shared__ DevCtx s_ctx;
  extern __shared__ __align__(1024) double dyn[];
  cg::cluster_group cl = cg::this_cluster();
  if (threadIdx.x == 0) s_ctx = c;
  const int job = blockIdx.x / c.G, k = c.kb + job, d = c.d;
  int* Rk = c.rec_cur + (long long)k * c.RS;
  int r = c.rank_ring[k * 2 + ((s0 - 1) & 1)];
  int rdone = c.sbstate[job * 4 + 0], cdone = c.sbstate[job * 4 + 1];
  int xstep = 0;
  RingPos rpos{0, 0u, 0};
  TRACE_INIT();
  xbar_init(&S);  // ordered before remote use by the cluster barriers of the first sweep
  tma_ring_init(&S);
  for (int s = s0; s < s0 + nsweeps; ++s) {
    TRACE_FLUSH();
    TRACE(49);
    // every CTA acquires the neighbours' flags itself: the acquire also makes this SM's L1
    // drop lines of neighbour data (records, rank ring) cached in an earlier sweep, which a
    // cluster barrier after a single CTA's acquire does not guarantee
    if (threadIdx.x == 0) {
      int abort = 0;
      const long long t0 = clock64();
      const unsigned long long w0 = (TTC_PHASE_CLOCKS && c.phase_ns) ? gtimer() : 0;
      // a neighbour on another rank (cross-GPU wavefront): its flag, written by the peer with a
      // system-scope release, is acquired at system scope from rdone
      const bool lrem = PEER && c.pdone[0] && k == c.pb_lo, rrem = PEER && c.pdone[1] && k + 1 == c.pb_hi;
      if (k > 0)
        while ((lrem ? ld_acquire_sys(&c.rdone[k - 1]) : ld_acquire(&c.done[k - 1])) < s &&
               !(abort = (clock64() - t0 > (1LL << 32)) || c.flags[1])) {
        }
      if (!abort && k < d - 2)
        while ((rrem ? ld_acquire_sys(&c.rdone[k + 1]) : ld_acquire(&c.done[k + 1])) < s &&
               !(abort = (clock64() - t0 > (1LL << 32)) || c.flags[1])) {
        }
      if (abort) atomicOr(&c.flags[1], 1);
      s_abort[s & 1] = abort;
      if (TTC_PHASE_CLOCKS && c.phase_ns && job == c.phase_job && cl.block_rank() == 0) {
        ph_add(c.phase_ns, s, PH_START, gtimer() - w0);
      }
    }
    TRACE(50);
    cl.sync();
    // every warp reads the cluster's abort flags (lane i: CTA i) -- no second barrier: slot
    // s & 1 is rewritten two sweeps later, after this sweep's barriers
    {
      const int lane = threadIdx.x & 31;
      const int mine = lane < (int)cl.num_blocks() ? cl.map_shared_rank(&s_abort[s & 1], lane)[0] : 0;
      TRACE(51);
      if (__any_sync(0xffffffffu, mine)) {   // (the same on every CTA of the cluster)
        cl.sync();   // no CTA exits while another may still read its flags
        break;
      }
    }
    const bool lrem = PEER && c.pdone[0] && k == c.pb_lo, rrem = PEER && c.pdone[1] && k + 1 == c.pb_hi;
    const int rl = k > 0 ? (lrem ? c.rring : c.rank_ring)[(k - 1) * 2 + ((s - 1) & 1)] : 1;
    const int rr = k < d - 2 ? (rrem ? c.rring : c.rank_ring)[(k + 1) * 2 + ((s - 1) & 1)] : 1;
    // (sweep_body publishes rank_ring[k] and releases done[k] as soon as the pivot is known)
    r = sweep_body<FAMILY, CACHED, PEER>(c, s_ctx, S, dyn, s, job, r, rl, rr, Rk, xstep, rpos, s + 1 == s0 + nsweeps, rdone, cdone,
                                   s > s0, true);
    rdone = rl;   // (= the sbstate the sweep wrote)
    cdone = rr;
  }
  TRACE_FLUSH();
}

}  // namespace ttc
