// ttc_greedy.cuh -- the dimension-parallel greedy cross (Alg. 6 with Alg. 2).
//
// One sweep updates every owned interface k from the index sets of the previous sweep
// (§3.4 relaxation).  Interface k works on its superblock
//   A_k(x, y) = A(I_{<=k-1}[alpha], a, b, I_{>k+1}[beta]),  x = alpha*n + a,  y = beta*n + b
// (Alg. 5), an (r_{k-1} n) x (n r_{k+1}) matrix, and keeps its cross in the
// incomplete-LU form A~(x, y) = sum_t u_t(x) v_t(y) (oracle/cross.py).
//
//   k_init_pivot / k_init_records : the rank-1 start (first argmax |A| over seeded samples)
//   k_sb_sides / k_sb_cx          : factor tables of the superblock entries for the rows /
//                                   columns that are new this sweep (the frozen left/right
//                                   pivot coordinates, staged once per sweep)
//   k_sb_extend_rows / _cols      : u_s(x) / v_s(y) of the existing pivots on the new rows /
//                                   columns -- the batched fiber evaluation of the sweep
//   k_greedy                      : one thread-block cluster per superblock: random samples
//                                   (Alg. 2 line 1), rook search (lines 2-5), append the new
//                                   pivot (Alg. 6 line 4) to the next record buffer.
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
#define GREEDY_THREADS 512
#define TTC_MAX_SAMPLES 1024

// ---------------------------------------------------------------------------------------
// direct O(d^2) entry of a full tuple given coordinate by coordinate (init only)
// ---------------------------------------------------------------------------------------
__device__ __forceinline__ int init_coord(const DevCtx& c, int q, int j) {
  return (int)(splitmix64(c.seed, draw_ctr(0, c.d, 0, q * c.d + j)) % (uint64_t)c.n);
}

__device__ double init_entry(const DevCtx& c, int q) {
  const int d = c.d, n = c.n;
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
    for (int j = i + 1; j < d; ++j) dde_mul_d(p, rho(ui, c.u[j * n + init_coord(c, q, j)]));
  }
  return __ddiv_rn(dde_round(p), SS);
}

// one block of N_INIT threads: t0 = first argmax |A| over the seeded samples -> t0buf[d]
__global__ void __launch_bounds__(N_INIT) k_init_pivot(DevCtx c, int* t0buf) {
  __shared__ double sv[N_INIT];
  __shared__ int best;
  const int q = threadIdx.x;
  sv[q] = fabs(init_entry(c, q));
  __syncthreads();
  if (q == 0) {
    int b = 0;
    for (int t = 1; t < N_INIT; ++t)
      if (sv[t] > sv[b]) b = t;
    best = b;
    if (c.counters) atomicAdd(&c.counters[CNT_EVALS], (unsigned long long)N_INIT);
  }
  __syncthreads();
  for (int j = q; j < c.d; j += blockDim.x) t0buf[j] = init_coord(c, best, j);
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
  if (i < n_owned && threadIdx.x == 0) {
    c.sbstate[i * 4 + 0] = 0;
    c.sbstate[i * 4 + 1] = 0;
    c.sbstate[i * 4 + 2] = 0;
    c.sbstate[i * 4 + 3] = 0;
    c.praw_max[i] = -1.0;
  }
}

// ---------------------------------------------------------------------------------------
// superblock factor tables (eq. (9)-(10) integrands split over the frozen parts)
// ---------------------------------------------------------------------------------------
// grid: x = node chunk, y = slot (alpha or beta), z = job*2 + side; block 128.
// side 0 (alpha >= rows_done): SA = S_L + c_k[a], PA = P_LL * prod_{i<k} rho(u_k[a], X_i),
//                              QL1 = prod_{i<k} rho(u_{k+1}[b], X_i)
// side 1 (beta >= cols_done):  SB = c_{k+1}[b] + S_R, PB = P_RR * prod_{j>k+1} rho(u_{k+1}[b], Y_j),
//                              QR0 = prod_{j>k+1} rho(u_k[a], Y_j)
__global__ void __launch_bounds__(128) k_sb_sides(DevCtx c) {
  const int job = blockIdx.z >> 1, side = blockIdx.z & 1, slot = blockIdx.y;
  const int k = c.kb + job, d = c.d, n = c.n;
  const int* st = c.sbstate + job * 4;
  __shared__ ESum sS;
  __shared__ DDE sP;
  const int* T;
  int lo, hi;  // coordinate range of the frozen tuple
  if (side == 0) {
    const int rl = k > 0 ? rec_rank(c.rec_cur, c.RS, k - 1) : 1;
    if (slot < st[0] || slot >= rl) return;
    T = k > 0 ? rec_piv(c.rec_cur, c.RS, k - 1) + (long long)slot * d : nullptr;
    lo = 0;
    hi = k;
  } else {
    const int rr = k < d - 2 ? rec_rank(c.rec_cur, c.RS, k + 1) : 1;
    if (slot < st[1] || slot >= rr) return;
    T = k < d - 2 ? rec_piv(c.rec_cur, c.RS, k + 1) + (long long)slot * d : nullptr;
    lo = k + 2;
    hi = d;
  }
  if (!T) hi = lo;
  if (threadIdx.x == 0) {
    ESum s = esum_zero();
    DDE p = dde_one();
    for (int q = lo; q < hi; ++q) esum_add(s, c.chi[q * n + T[q]], c.clo[q * n + T[q]]);
    if (c.family == 1)
      for (int a = lo; a < hi; ++a) {
        const double ua = c.u[a * n + T[a]];
        for (int b = a + 1; b < hi; ++b) dde_mul_d(p, rho(ua, c.u[b * n + T[b]]));
      }
    sS = s;
    sP = p;
  }
  __syncthreads();
  const long long o = ((long long)job * c.cap + slot) * n;
  const int mode_own = side == 0 ? k : k + 1;    // mode summed into SA / SB
  const int mode_oth = side == 0 ? k + 1 : k;    // mode of QL1 / QR0
  for (int a = blockIdx.x * blockDim.x + threadIdx.x; a < n; a += gridDim.x * blockDim.x) {
    ESum s = sS;
    esum_add(s, c.chi[mode_own * n + a], c.clo[mode_own * n + a]);
    if (side == 0) c.SA[o + a] = s;
    else c.SB[o + a] = s;
    if (c.family == 1) {
      const double uo = c.u[mode_own * n + a], ux = c.u[mode_oth * n + a];
      DDE p = sP, q = dde_one();
      for (int t = lo; t < hi; ++t) {
        const double x = c.u[t * n + T[t]];
        dde_mul_d(p, rho(uo, x));
        dde_mul_d(q, rho(ux, x));
      }
      if (side == 0) { c.PA[o + a] = p; c.QL1[o + a] = q; }
      else { c.PB[o + a] = p; c.QR0[o + a] = q; }
    }
  }
}

// CX[alpha][beta] = prod_{i<k} prod_{j>k+1} rho(X_alpha,i, Y_beta,j) for the new pairs;
// grid: x = beta chunk (64), y = alpha, z = job
__global__ void __launch_bounds__(64) k_sb_cx(DevCtx c) {
  const int job = blockIdx.z, al = blockIdx.y;
  const int be = blockIdx.x * blockDim.x + threadIdx.x;
  const int k = c.kb + job, d = c.d, n = c.n;
  const int* st = c.sbstate + job * 4;
  const int rl = k > 0 ? rec_rank(c.rec_cur, c.RS, k - 1) : 1;
  const int rr = k < d - 2 ? rec_rank(c.rec_cur, c.RS, k + 1) : 1;
  if (al >= rl || be >= rr || (al < st[0] && be < st[1])) return;
  DDE p = dde_one();
  if (k > 0 && k < d - 2) {
    const int* TX = rec_piv(c.rec_cur, c.RS, k - 1) + (long long)al * d;
    const int* TY = rec_piv(c.rec_cur, c.RS, k + 1) + (long long)be * d;
    for (int i = 0; i < k; ++i) {
      const double ui = c.u[i * n + TX[i]];
      for (int j = k + 2; j < d; ++j) dde_mul_d(p, rho(ui, c.u[j * n + TY[j]]));
    }
  }
  c.CX[((long long)job * c.cap + al) * c.cap + be] = p;
}

// A_k(alpha, a; beta, b) from the tables (single rounding, R3)
template <int FAMILY>
__device__ __forceinline__ double sb_entry(const DevCtx& c, int job, int k, int al, int a, int be, int b) {
  const int n = c.n;
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
  return __ddiv_rn(dde_round(p), SS);
}

// pivot positions of interface k: xs = alpha_s*n + a_s, ys = beta_s*n + b_s
__device__ __forceinline__ void pivot_pos(const DevCtx& c, int k, int s, int& x, int& y) {
  const int* T = rec_piv(c.rec_cur, c.RS, k) + (long long)s * c.d;
  const int* P = rec_par(c.rec_cur, c.RS, c.cap, c.d, k) + 2 * s;
  x = P[0] * c.n + T[k];
  y = P[1] * c.n + T[k + 1];
}

// ---------------------------------------------------------------------------------------
// u_s(x) on the new rows:  u_s(x) = A(x, y_s) - sum_{t<s} u_t(x) v_t(y_s)
// grid: x = row chunk (256), y = job
// ---------------------------------------------------------------------------------------
template <int FAMILY>
__global__ void __launch_bounds__(256) k_sb_extend_rows(DevCtx c) {
  const int job = blockIdx.y, k = c.kb + job, n = c.n;
  __shared__ int syb[TTC_MAX_RANK_DEV], sbb[TTC_MAX_RANK_DEV];
  const int r = rec_rank(c.rec_cur, c.RS, k);
  const int rl = k > 0 ? rec_rank(c.rec_cur, c.RS, k - 1) : 1;
  const long long x0 = (long long)c.sbstate[job * 4 + 0] * n;
  const long long x = x0 + blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (x0 + blockIdx.x * (long long)blockDim.x >= (long long)rl * n) return;
  if (threadIdx.x < r) {
    int px, py;
    pivot_pos(c, k, threadIdx.x, px, py);
    syb[threadIdx.x] = py / n;
    sbb[threadIdx.x] = py - (py / n) * n;
  }
  __syncthreads();
  if (x >= (long long)rl * n) return;
  const int al = (int)(x / n), a = (int)(x - (long long)al * n);
  const long long sbn = c.sbn;
  const double* V = c.V + (long long)job * c.cap * sbn;
  double* U = c.U + (long long)job * c.cap * sbn;
  for (int s = 0; s < r; ++s) {
    const long long ys = (long long)syb[s] * n + sbb[s];
    double acc = sb_entry<FAMILY>(c, job, k, al, a, syb[s], sbb[s]);
    for (int t = 0; t < s; ++t) acc = __dsub_rn(acc, __dmul_rn(U[t * sbn + x], V[t * sbn + ys]));
    U[s * sbn + x] = acc;
  }
  if (c.counters) {
    // one atomic per warp
    const unsigned mask = __activemask();
    const int cnt = __popc(mask);
    if ((threadIdx.x & 31) == __ffs(mask) - 1) {
      atomicAdd(&c.counters[CNT_EVALS], (unsigned long long)cnt * r);
      atomicAdd(&c.counters[CNT_SB_ENTRIES], (unsigned long long)cnt * r);
      atomicAdd(&c.counters[CNT_EXT_ENTRIES], (unsigned long long)cnt * r);
      atomicAdd(&c.counters[CNT_SB_UPDATES], (unsigned long long)cnt * r * (r - 1) / 2);
      atomicAdd(&c.counters[CNT_EXT_UPDATES], (unsigned long long)cnt * r * (r - 1) / 2);
    }
  }
}

// v_s(y) on the new columns:  v_s(y) = (A(x_s, y) - sum_{t<s} u_t(x_s) v_t(y)) / u_s(x_s)
template <int FAMILY>
__global__ void __launch_bounds__(256) k_sb_extend_cols(DevCtx c) {
  const int job = blockIdx.y, k = c.kb + job, d = c.d, n = c.n;
  __shared__ int sal[TTC_MAX_RANK_DEV], sa[TTC_MAX_RANK_DEV];
  __shared__ long long sx[TTC_MAX_RANK_DEV];
  const int r = rec_rank(c.rec_cur, c.RS, k);
  const int rr = k < d - 2 ? rec_rank(c.rec_cur, c.RS, k + 1) : 1;
  const long long y0 = (long long)c.sbstate[job * 4 + 1] * n;
  const long long y = y0 + blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (y0 + blockIdx.x * (long long)blockDim.x >= (long long)rr * n) return;
  if (threadIdx.x < r) {
    int px, py;
    pivot_pos(c, k, threadIdx.x, px, py);
    sal[threadIdx.x] = px / n;
    sa[threadIdx.x] = px - (px / n) * n;
    sx[threadIdx.x] = px;
  }
  __syncthreads();
  if (y >= (long long)rr * n) return;
  const int be = (int)(y / n), b = (int)(y - (long long)be * n);
  const long long sbn = c.sbn;
  const double* U = c.U + (long long)job * c.cap * sbn;
  double* V = c.V + (long long)job * c.cap * sbn;
  for (int s = 0; s < r; ++s) {
    double acc = sb_entry<FAMILY>(c, job, k, sal[s], sa[s], be, b);
    for (int t = 0; t < s; ++t) acc = __dsub_rn(acc, __dmul_rn(U[t * sbn + sx[s]], V[t * sbn + y]));
    V[s * sbn + y] = __ddiv_rn(acc, U[s * sbn + sx[s]]);
  }
  if (c.counters) {
    const unsigned mask = __activemask();
    const int cnt = __popc(mask);
    if ((threadIdx.x & 31) == __ffs(mask) - 1) {
      atomicAdd(&c.counters[CNT_EVALS], (unsigned long long)cnt * r);
      atomicAdd(&c.counters[CNT_SB_ENTRIES], (unsigned long long)cnt * r);
      atomicAdd(&c.counters[CNT_EXT_ENTRIES], (unsigned long long)cnt * r);
      atomicAdd(&c.counters[CNT_SB_UPDATES], (unsigned long long)cnt * r * (r - 1) / 2);
      atomicAdd(&c.counters[CNT_EXT_UPDATES], (unsigned long long)cnt * r * (r - 1) / 2);
    }
  }
}

// ---------------------------------------------------------------------------------------
// k_greedy: one cluster of G CTAs per superblock
// ---------------------------------------------------------------------------------------
struct Cand {
  double val;
  long long idx;
};

__device__ __forceinline__ bool cand_better(double v, long long f, double bv, long long bf) {
  return v > bv || (v == bv && f < bf);
}

__device__ __forceinline__ void warp_argmax(double& v, long long& f) {
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    const double ov = __shfl_xor_sync(0xffffffffu, v, o);
    const long long of = __shfl_xor_sync(0xffffffffu, f, o);
    if (cand_better(ov, of, v, f)) { v = ov; f = of; }
  }
}

struct GreedySmem {
  Cand cand[2];                      // published CTA candidate (double-buffered per step)
  Cand red[GREEDY_THREADS / 32];
  Cand best;                         // CTA argmax / cluster winner
  int xs[TTC_MAX_RANK_DEV];          // pivot rows
  int ys[TTC_MAX_RANK_DEV];          // pivot columns
  double vec[TTC_MAX_RANK_DEV];      // V[t][y*] (column step) or U[t][x*] (row step)
};

// CTA-wide argmax of (v, f) -> S.best (all threads call)
__device__ __forceinline__ void cta_argmax(GreedySmem& S, double v, long long f) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  warp_argmax(v, f);
  if (lane == 0) S.red[warp] = {v, f};
  __syncthreads();
  if (warp == 0) {
    const int nw = blockDim.x >> 5;
    double bv = lane < nw ? S.red[lane].val : -1.0;
    long long bf = lane < nw ? S.red[lane].idx : LLONG_MAX;
    warp_argmax(bv, bf);
    if (lane == 0) S.best = {bv, bf};
  }
  __syncthreads();
}

// cluster-wide argmax: every CTA publishes S.best in cand[ph]; after the barrier every CTA
// reduces all G candidates (DSMEM) in cluster-rank order -> S.best
__device__ __forceinline__ void cluster_argmax(GreedySmem& S, cg::cluster_group& cl, int G, int& ph) {
  if (threadIdx.x == 0) S.cand[ph] = S.best;
  cl.sync();
  if (threadIdx.x < 32) {
    const int lane = threadIdx.x;
    double bv = -1.0;
    long long bf = LLONG_MAX;
    if (lane < G) {
      const GreedySmem* R = cl.map_shared_rank(&S, lane);
      bv = R->cand[ph].val;
      bf = R->cand[ph].idx;
    }
    warp_argmax(bv, bf);
    if (lane == 0) S.best = {bv, bf};
  }
  ph ^= 1;
  __syncthreads();
}

template <int FAMILY>
__global__ void __launch_bounds__(GREEDY_THREADS, 1) k_greedy(DevCtx c, int sweep) {
  cg::cluster_group cl = cg::this_cluster();
  const int G = c.G;
  const int cr = (int)cl.block_rank();
  const int job = blockIdx.x / G;
  const int k = c.kb + job, d = c.d, n = c.n, cap = c.cap;
  const int tid = threadIdx.x, T = blockDim.x;
  __shared__ GreedySmem S;

  const int r = rec_rank(c.rec_cur, c.RS, k);
  const int rl = k > 0 ? rec_rank(c.rec_cur, c.RS, k - 1) : 1;
  const int rr = k < d - 2 ? rec_rank(c.rec_cur, c.RS, k + 1) : 1;
  const long long R = (long long)rl * n, C = (long long)rr * n;
  const long long rpc = (R + G - 1) / G, cpc = (C + G - 1) / G;
  const long long xb = cr * rpc, xe = min(R, xb + rpc);
  const long long yb = cr * cpc, ye = min(C, yb + cpc);
  const long long sbn = c.sbn;
  double* U = c.U + (long long)job * cap * sbn;
  double* V = c.V + (long long)job * cap * sbn;
  double* Araw = c.Araw + (long long)job * sbn;
  int* Rn = c.rec_next + (long long)k * c.RS;
  const int* Rc = c.rec_cur + (long long)k * c.RS;

  if (cr == 0)
    for (int t = tid; t < c.RS; t += T) Rn[t] = Rc[t];
  if (tid < r) {
    int px, py;
    pivot_pos(c, k, tid, px, py);
    S.xs[tid] = px;
    S.ys[tid] = py;
  }
  __syncthreads();

  bool active = r < cap;
  const double p0 = U[S.xs[0]];  // u_0(x_0) = A(x_0, y_0)
  if (p0 == 0.0) active = false;  // singular first pivot: leave the interface (R8)
  double scale = c.praw_max[job];
  if (scale < 0.0) scale = fabs(p0);
  unsigned long long evals = 0, steps = 0, upd = 0;
  int ph = 0;
  int xst = 0, yst = 0;
  bool added = false;
  double raw_star = 0.0;

  if (active) {
    // ---- Alg. 2 line 1: n_samples random entries, largest |E| (every CTA, identically)
    {
      const uint64_t tag = 1ULL + (uint64_t)sweep;
      double bv = -1.0;
      long long bf = LLONG_MAX;
      for (int q = tid; q < c.ns; q += T) {
        const long long sx = (long long)(splitmix64(c.seed, draw_ctr(tag, d, k, 2 * q)) % (uint64_t)R);
        const long long sy = (long long)(splitmix64(c.seed, draw_ctr(tag, d, k, 2 * q + 1)) % (uint64_t)C);
        const int al = (int)(sx / n), a = (int)(sx - (long long)al * n);
        const int be = (int)(sy / n), b = (int)(sy - (long long)be * n);
        double e = sb_entry<FAMILY>(c, job, k, al, a, be, b);
        for (int t = 0; t < r; ++t) e = __dsub_rn(e, __dmul_rn(U[t * sbn + sx], V[t * sbn + sy]));
        bool masked = false;
        for (int t = 0; t < r; ++t) masked |= (S.xs[t] == sx) | (S.ys[t] == sy);
        if (masked) e = 0.0;
        if (cand_better(fabs(e), q, bv, bf)) { bv = fabs(e); bf = q; }
      }
      cta_argmax(S, bv, bf);
      const int q = (int)S.best.idx;
      xst = (int)(splitmix64(c.seed, draw_ctr(tag, d, k, 2 * q)) % (uint64_t)R);
      yst = (int)(splitmix64(c.seed, draw_ctr(tag, d, k, 2 * q + 1)) % (uint64_t)C);
      if (cr == 0 && tid == 0) {
        evals += c.ns;
        upd += (unsigned long long)c.ns * r;
      }
    }
    // column step E(:, y) -> U[r][:], Araw; returns the cluster argmax row when `search`
    auto column = [&](int y, bool search) -> int {
      if (tid < r) S.vec[tid] = V[tid * sbn + y];
      __syncthreads();
      const int be = y / n, b = y - (y / n) * n;
      double bv = -1.0;
      long long bf = LLONG_MAX;
      for (long long x = xb + tid; x < xe; x += T) {
        const int al = (int)(x / n), a = (int)(x - (long long)al * n);
        const double raw = sb_entry<FAMILY>(c, job, k, al, a, be, b);
        double e = raw;
        for (int t = 0; t < r; ++t) e = __dsub_rn(e, __dmul_rn(U[t * sbn + x], S.vec[t]));
        for (int t = 0; t < r; ++t)
          if (S.xs[t] == x) e = 0.0;
        Araw[x] = raw;
        U[r * sbn + x] = e;
        if (cand_better(fabs(e), x, bv, bf)) { bv = fabs(e); bf = x; }
      }
      if (tid == 0) {
        evals += (unsigned long long)max(0LL, xe - xb);
        upd += (unsigned long long)max(0LL, xe - xb) * r;
      }
      int win = -1;
      if (search) {
        cta_argmax(S, bv, bf);
        cluster_argmax(S, cl, G, ph);
        win = (int)S.best.idx;
      } else {
        __syncthreads();
      }
      return win;
    };
    auto row = [&](int x, bool search) -> int {
      if (tid < r) S.vec[tid] = U[tid * sbn + x];
      __syncthreads();
      const int al = x / n, a = x - (x / n) * n;
      double bv = -1.0;
      long long bf = LLONG_MAX;
      for (long long y = yb + tid; y < ye; y += T) {
        const int be = (int)(y / n), b = (int)(y - (long long)be * n);
        double e = sb_entry<FAMILY>(c, job, k, al, a, be, b);
        for (int t = 0; t < r; ++t) e = __dsub_rn(e, __dmul_rn(S.vec[t], V[t * sbn + y]));
        for (int t = 0; t < r; ++t)
          if (S.ys[t] == y) e = 0.0;
        V[r * sbn + y] = e;
        if (cand_better(fabs(e), y, bv, bf)) { bv = fabs(e); bf = y; }
      }
      if (tid == 0) {
        evals += (unsigned long long)max(0LL, ye - yb);
        upd += (unsigned long long)max(0LL, ye - yb) * r;
      }
      int win = -1;
      if (search) {
        cta_argmax(S, bv, bf);
        cluster_argmax(S, cl, G, ph);
        win = (int)S.best.idx;
      } else {
        __syncthreads();
      }
      return win;
    };
    // ---- Alg. 2 lines 2-5: rook search
    int c_at = -1, g_at = -1;
    for (int it = 0; it < c.rook; ++it) {
      const int xn = column(yst, true);
      c_at = yst;
      const int yn = row(xn, true);
      g_at = xn;
      steps += 1;
      const bool conv = (yn == yst);
      xst = xn;
      yst = yn;
      if (conv) break;
    }
    if (c_at != yst) column(yst, false);
    if (g_at != xst) row(xst, false);
    cl.sync();  // U[r][:], V[r][:], Araw visible to the whole cluster
    const double pv = V[r * sbn + yst];
    raw_star = Araw[xst];
    if (fabs(pv) > c.tol * scale) {
      added = true;
      for (long long y = yb + tid; y < ye; y += T) V[r * sbn + y] = __ddiv_rn(V[r * sbn + y], pv);
    }
  }

  if (cr == 0 && tid == 0) {
    if (added) {
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
      scale = fmax(scale, fabs(raw_star));
    }
    c.praw_max[job] = scale;
    c.sbstate[job * 4 + 0] = rl;
    c.sbstate[job * 4 + 1] = rr;
  }
  if (c.counters) {
    // per-thread tallies reduced by one atomic per thread with nonzero work
    if (evals) {
      atomicAdd(&c.counters[CNT_EVALS], evals);
      atomicAdd(&c.counters[CNT_SB_ENTRIES], evals);
    }
    if (upd) atomicAdd(&c.counters[CNT_SB_UPDATES], upd);
    if (cr == 0 && tid == 0 && steps) atomicAdd(&c.counters[CNT_ROOK_STEPS], steps);
  }
  cl.sync();  // no CTA may exit while another can still read its shared memory
}

}  // namespace ttc
