// ttc_cross.cuh -- batched rank-revealing cross + maxvol on the fiber matrices.
//
// One thread-block cluster of G CTAs per interface.  The (nrows x ncols) fiber matrix
// (rows (outer, a) -> outer*n + a) is distributed by row blocks over the
// cluster's shared memory (global memory when it does not fit), each thread owning a
// strided set of rows.  Every step is: fused rank-1 update + local |max| (first index wins
// ties), warp-shuffle and CTA reductions, one cluster barrier, and a DSMEM read of the
// winning candidate and its row.  B = F(:,J) F(I,J)^{-1} lives in the columns that the
// complete pivoting has retired, so the storage is exactly nrows x ncols.
//
// Arithmetic follows oracle/cross.py::rrcross / ::maxvol operation by operation
// (__dmul_rn/__dsub_rn/__ddiv_rn, no FMA), so pivots agree bit for bit (R4):
//   cross : b = R[:,c]/piv ; B -= b (x) B[i,:] ; R -= R[:,c] (x) (R[i,:]/piv) ; R[i,:] = 0
//   maxvol: g = (B[i,:] - e_j)/B[i,j] ; B -= B[:,j] (x) g            (Alg. 1)
#pragma once
#include <cooperative_groups.h>
#include "ttc_common.cuh"

namespace cg = cooperative_groups;

namespace ttc {

#define CROSS_THREADS 512

struct Cand {
  double val;
  long long flat;
};

__device__ __forceinline__ bool cand_better(double v, long long f, double bv, long long bf) {
  return v > bv || (v == bv && f < bf);
}

__device__ __forceinline__ void warp_argmax(double& v, long long& f) {
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    double ov = __shfl_xor_sync(0xffffffffu, v, o);
    long long of = __shfl_xor_sync(0xffffffffu, f, o);
    if (cand_better(ov, of, v, f)) { v = ov; f = of; }
  }
}

struct CrossSmem {
  Cand cand[2];
  Cand red[CROSS_THREADS / 32];
  Cand cta_best;
  Cand win;
  int win_cta;
  int live[TTC_MAX_COLS];
  int col_of_slot[TTC_MAX_RANK_DEV];
  long long row_of_slot[TTC_MAX_RANK_DEV];
  double stage[2][TTC_MAX_COLS];
  double prow[TTC_MAX_COLS];
  double gco[TTC_MAX_COLS];
};

// CTA-wide argmax of (v, f); result in S.cta_best (all threads must call)
__device__ __forceinline__ void cta_argmax(CrossSmem& S, double v, long long f) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  warp_argmax(v, f);
  if (lane == 0) S.red[warp] = {v, f};
  __syncthreads();
  if (warp == 0) {
    const int nw = blockDim.x >> 5;
    double bv = lane < nw ? S.red[lane].val : -1.0;
    long long bf = lane < nw ? S.red[lane].flat : LLONG_MAX;
    warp_argmax(bv, bf);
    if (lane == 0) S.cta_best = {bv, bf};
  }
  __syncthreads();
}

// cluster-wide winner among the published candidates cand[ph] of every CTA
__device__ __forceinline__ void cluster_winner(CrossSmem& S, cg::cluster_group& cl, int G, int ph) {
  const int lane = threadIdx.x & 31;
  if (threadIdx.x < 32) {
    double bv = -1.0;
    long long bf = LLONG_MAX;
    int bc = 0;
    if (lane < G) {
      CrossSmem* R = cl.map_shared_rank(&S, lane);
      bv = R->cand[ph].val;
      bf = R->cand[ph].flat;
      bc = lane;
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) {
      double ov = __shfl_xor_sync(0xffffffffu, bv, o);
      long long of = __shfl_xor_sync(0xffffffffu, bf, o);
      int oc = __shfl_xor_sync(0xffffffffu, bc, o);
      if (cand_better(ov, of, bv, bf)) { bv = ov; bf = of; bc = oc; }
    }
    if (lane == 0) {
      S.win = {bv, bf};
      S.win_cta = bc;
    }
  }
  __syncthreads();
}

template <bool SMEM>
__global__ void __launch_bounds__(CROSS_THREADS, 1) k_cross(DevCtx c, int kind, int G, int rpc) {
  cg::cluster_group cl = cg::this_cluster();
  const int cr = (int)cl.block_rank();
  const int job = blockIdx.x / G;
  extern __shared__ __align__(16) unsigned char smraw[];
  CrossSmem& S = *reinterpret_cast<CrossSmem*>(smraw);
  double* st = reinterpret_cast<double*>(smraw + ((sizeof(CrossSmem) + 127) / 128) * 128);

  Job jb = make_job(c, kind, job);
  const int n = c.n;
  const int rx = jb.rx, ry = jb.ry;
  const bool lr = (kind == JOB_LR);
  const long long nrows = (long long)(lr ? rx : ry) * n;
  const int ncols = lr ? ry : rx;
  double* F = c.fib + (long long)job * c.fib_stride;
  const long long row0 = (long long)cr * rpc;
  const int nloc = (int)max(0LL, min(nrows - row0, (long long)rpc));
  const int T = blockDim.x, tid = threadIdx.x;

  auto gaddr = [&](long long grow, int col) -> long long {
    long long outer = grow / n;
    long long a = grow - outer * n;
    return lr ? ((outer * ry + col) * n + a) : (((long long)col * ry + outer) * n + a);
  };
  auto E = [&](int x, int col) -> double& {
    if (SMEM) return st[(long long)col * rpc + x];
    return F[gaddr(row0 + x, col)];
  };

  if (SMEM) {
    for (int col = 0; col < ncols; ++col)
      for (int x = tid; x < nloc; x += T) st[(long long)col * rpc + x] = F[gaddr(row0 + x, col)];
  }
  if (tid < TTC_MAX_COLS) S.live[tid] = tid < ncols ? 1 : 0;
  __syncthreads();

  // ---------------- rank-revealing cross by complete pivoting ----------------
  double bv = -1.0;
  long long bf = LLONG_MAX;
  for (int x = tid; x < nloc; x += T)
    for (int col = 0; col < ncols; ++col) {
      double v = fabs(E(x, col));
      long long f = (row0 + x) * ncols + col;
      if (cand_better(v, f, bv, bf)) { bv = v; bf = f; }
    }

  const int smax = (int)min((long long)c.cap, min(nrows, (long long)ncols));
  // Published candidate/stage buffers alternate with every cluster step (ph = step & 1):
  // a CTA can only overwrite buffer ph again after the next cluster barrier, which every
  // reader of step `step` reaches only after it finished reading.
  int ph = 0;
  int s = 0;
  double scale = 0.0;
  for (; s < smax; ++s) {
    cta_argmax(S, bv, bf);
    if (S.cta_best.val >= 0.0) {
      const int xb = (int)(S.cta_best.flat / ncols - row0);
      if (tid < ncols) S.stage[ph][tid] = E(xb, tid);
    }
    if (tid == 0) S.cand[ph] = S.cta_best;
    cl.sync();
    cluster_winner(S, cl, G, ph);
    const int rph = ph;
    ph ^= 1;
    const double pv = S.win.val;
    if (s == 0) scale = pv;
    if (!(pv > c.tol * scale)) break;
    const long long p = S.win.flat / ncols;
    const int colc = (int)(S.win.flat - p * ncols);
    if (tid < ncols) {
      CrossSmem* R = cl.map_shared_rank(&S, S.win_cta);
      S.prow[tid] = R->stage[rph][tid];
    }
    __syncthreads();
    const double piv = S.prow[colc];
    if (tid < ncols) S.gco[tid] = (S.live[tid] && tid != colc) ? __ddiv_rn(S.prow[tid], piv) : 0.0;
    __syncthreads();
    bv = -1.0;
    bf = LLONG_MAX;
    for (int x = tid; x < nloc; x += T) {
      const long long grow = row0 + x;
      const double rxc = E(x, colc);
      const double b = __ddiv_rn(rxc, piv);
      for (int l = 0; l < s; ++l) {
        const int cl_ = S.col_of_slot[l];
        E(x, cl_) = __dsub_rn(E(x, cl_), __dmul_rn(b, S.prow[cl_]));
      }
      E(x, colc) = b;
      for (int y = 0; y < ncols; ++y) {
        if (!S.live[y] || y == colc) continue;
        const double v = (grow == p) ? 0.0 : __dsub_rn(E(x, y), __dmul_rn(rxc, S.gco[y]));
        E(x, y) = v;
        const double av = fabs(v);
        const long long f = grow * ncols + y;
        if (cand_better(av, f, bv, bf)) { bv = av; bf = f; }
      }
    }
    __syncthreads();
    if (tid == 0) {
      S.live[colc] = 0;
      S.col_of_slot[s] = colc;
      S.row_of_slot[s] = p;
    }
    __syncthreads();
  }
  const int r = s;

  // ---------------- maxvol swaps (Alg. 1) ----------------
  int nsw = 0;
  if (r > 0 && c.max_swaps > 0) {
    bv = -1.0;
    bf = LLONG_MAX;
    for (int x = tid; x < nloc; x += T)
      for (int l = 0; l < r; ++l) {
        const double v = fabs(E(x, S.col_of_slot[l]));
        const long long f = (row0 + x) * r + l;
        if (cand_better(v, f, bv, bf)) { bv = v; bf = f; }
      }
    while (true) {
      cta_argmax(S, bv, bf);
      if (S.cta_best.val >= 0.0) {
        const int xb = (int)(S.cta_best.flat / r - row0);
        if (tid < r) S.stage[ph][tid] = E(xb, S.col_of_slot[tid]);
      }
      if (tid == 0) S.cand[ph] = S.cta_best;
      cl.sync();
      cluster_winner(S, cl, G, ph);
      const int rph = ph;
      ph ^= 1;
      if (!(S.win.val > 1.0 + c.delta)) break;
      const long long iw = S.win.flat / r;
      const int jw = (int)(S.win.flat - iw * r);
      if (tid < r) {
        CrossSmem* R = cl.map_shared_rank(&S, S.win_cta);
        S.prow[tid] = R->stage[rph][tid];
      }
      __syncthreads();
      const double piv = S.prow[jw];
      if (tid < r) {
        const double e = (tid == jw) ? __dsub_rn(S.prow[tid], 1.0) : S.prow[tid];
        S.gco[tid] = __ddiv_rn(e, piv);
      }
      __syncthreads();
      bv = -1.0;
      bf = LLONG_MAX;
      const int cj = S.col_of_slot[jw];
      for (int x = tid; x < nloc; x += T) {
        const long long grow = row0 + x;
        const double bxj = E(x, cj);
        for (int l = 0; l < r; ++l) {
          const int cc = S.col_of_slot[l];
          const double v = __dsub_rn(E(x, cc), __dmul_rn(bxj, S.gco[l]));
          E(x, cc) = v;
          const double av = fabs(v);
          const long long f = grow * r + l;
          if (cand_better(av, f, bv, bf)) { bv = av; bf = f; }
        }
      }
      __syncthreads();
      if (tid == 0) S.row_of_slot[jw] = iw;
      ++nsw;
      __syncthreads();
      if (nsw >= c.max_swaps) break;
    }
  }

  if (cr == 0 && tid < c.cap) {
    if (tid == 0) {
      c.sel_rank[job] = r;
      c.sel_nsw[job] = nsw;
      if (c.counters) {
        atomicAdd(&c.counters[CNT_CROSS_UPDATES],
                  (unsigned long long)(nrows * ncols * r + nrows * (long long)r * nsw));
        atomicAdd(&c.counters[CNT_CROSS_STEPS], (unsigned long long)(r + nsw));
        atomicAdd(&c.counters[CNT_CROSS_ELEMS], (unsigned long long)(nrows * ncols));
      }
    }
    if (tid < r) {
      c.sel_row[(long long)job * c.cap + tid] = (int)S.row_of_slot[tid];
      c.sel_col[(long long)job * c.cap + tid] = S.col_of_slot[tid];
    }
  }
  cl.sync();  // no CTA may leave while others can still read its shared memory
}

}  // namespace ttc
