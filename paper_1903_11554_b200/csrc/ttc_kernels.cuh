// ttc_kernels.cuh -- node tables, fiber evaluation and quadrature kernels.
//
// Fiber of mode m for a job: F[alpha][beta][a] = A(X[alpha][0:m], a, Y[beta][m+1:d])
// (eq. (3) factors A(I_{<=k-1}, i_k, I_{>k}), lines 312-320).  The entry is
// factorised over the frozen coordinates (DESIGN.md §5 "fiber kernel"):
//   S = S_L[alpha] + S_R[beta] + c_m[a]                               (exact int64 limbs)
//   P = Pf[alpha][beta] * Q_L[alpha][a] * Q_R[beta][a]                (double-double)
//   Pf = P_LL[alpha] * P_RR[beta] * prod_{i<m<j} rho(X_i, Y_j),
//   Q_L = prod_{j<m} rho(u_m[a], X_j),  Q_R = prod_{j>m} rho(u_m[a], Y_j).
// Because S and P are rounded once from exactly (resp. to 2^-100) accumulated values, the
// result equals the oracle's plain O(d^2)-per-entry evaluation bit for bit.
#pragma once
#include "ttc_common.cuh"
#include "ttc_greedy.cuh"   // cooperative_groups, cp.async helpers

namespace ttc {

// ---------------------------------------------------------------------------------------
// per-node tables: c = fl(u + fl(1/u)) split into (floor(c), frac(c)*2^52)
// ---------------------------------------------------------------------------------------
__global__ void k_prep_nodes(const double* __restrict__ u, long long* chi, long long* clo, int total) {
  int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= total) return;
  double x = u[t];
  double c = __dadd_rn(x, __ddiv_rn(1.0, x));
  double h = floor(c);
  chi[t] = __double2ll_rn(h);
  clo[t] = __double2ll_rn(__dmul_rn(__dsub_rn(c, h), 0x1p52));
}

// ---------------------------------------------------------------------------------------
// frozen parts, per (job, side, tuple): S_L / P_LL (side 0), S_R / P_RR (side 1)
// grid: x = tuple (<= ncols_max), y = side, z = job
// ---------------------------------------------------------------------------------------
__global__ void k_frozen_sides(DevCtx c, int kind, int jbase) {
  const int j = jbase + blockIdx.z, side = blockIdx.y;
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  Job jb = make_job(c, kind, j);
  const int d = c.d, n = c.n, m = jb.m;
  const long long so = (long long)j * c.cap + t;
  if (side == 0 && t == 0 && c.counters) {
    atomicAdd(&c.counters[CNT_EVALS], (unsigned long long)jb.rx * jb.ry * n);
    atomicAdd(&c.counters[CNT_FIBER_ENTRIES], (unsigned long long)jb.rx * jb.ry * n);
  }
  if (side == 0) {
    if (t >= jb.rx) return;
    ESum s = esum_zero();
    DDE p = dde_one();
    if (jb.X) {
      const int* T = jb.X + (long long)t * d;
      for (int q = 0; q < m; ++q) esum_add(s, c.chi[q * n + T[q]], c.clo[q * n + T[q]]);
      if (c.family == 1)
        for (int a = 0; a < m; ++a) {
          double ua = c.u[a * n + T[a]];
          for (int b = a + 1; b < m; ++b) dde_mul_d(p, rho(ua, c.u[b * n + T[b]]));
        }
    }
    c.sl[so] = s;
    c.pll[so] = p;
  } else {
    if (t >= jb.ry) return;
    ESum s = esum_zero();
    DDE p = dde_one();
    if (jb.Y) {
      const int* T = jb.Y + (long long)t * d;
      for (int q = m + 1; q < d; ++q) esum_add(s, c.chi[q * n + T[q]], c.clo[q * n + T[q]]);
      if (c.family == 1)
        for (int a = m + 1; a < d; ++a) {
          double ua = c.u[a * n + T[a]];
          for (int b = a + 1; b < d; ++b) dde_mul_d(p, rho(ua, c.u[b * n + T[b]]));
        }
    }
    c.sr[so] = s;
    c.prr[so] = p;
  }
}

// Q_L[alpha][a] (side 0) and Q_R[beta][a] (side 1); grid: x = node a, y = tuple, z = job*2+side
__global__ void k_frozen_q(DevCtx c, int kind, int jbase) {
  const int j = jbase + (blockIdx.z >> 1), side = blockIdx.z & 1;
  const int tup = blockIdx.y;
  const int a = blockIdx.x * blockDim.x + threadIdx.x;
  const int d = c.d, n = c.n;
  if (a >= n) return;
  Job jb = make_job(c, kind, j);
  const int m = jb.m;
  const double um = c.u[m * n + a];
  DDE p = dde_one();
  const long long o = ((long long)j * c.cap + tup) * n + a;
  if (side == 0) {
    if (tup >= jb.rx) return;
    if (jb.X) {
      const int* T = jb.X + (long long)tup * d;
      for (int q = 0; q < m; ++q) dde_mul_d(p, rho(um, c.u[q * n + T[q]]));
    }
    c.ql[o] = p;
  } else {
    if (tup >= jb.ry) return;
    if (jb.Y) {
      const int* T = jb.Y + (long long)tup * d;
      for (int q = m + 1; q < d; ++q) dde_mul_d(p, rho(um, c.u[q * n + T[q]]));
    }
    c.qr[o] = p;
  }
}

// Pf[alpha][beta] = P_LL * P_RR * prod_{i<m<j} rho(X_i, Y_j); grid: x = beta, y = alpha, z = job
__global__ void k_frozen_lr(DevCtx c, int kind, int jbase) {
  const int j = jbase + blockIdx.z, al = blockIdx.y;
  const int be = blockIdx.x * blockDim.x + threadIdx.x;
  Job jb = make_job(c, kind, j);
  if (al >= jb.rx || be >= jb.ry) return;
  const int d = c.d, n = c.n, m = jb.m;
  const long long base = (long long)j * c.cap;
  DDE p = c.pll[base + al];
  dde_mul(p, c.prr[base + be]);
  if (jb.X && jb.Y) {
    const int* TX = jb.X + (long long)al * d;
    const int* TY = jb.Y + (long long)be * d;
    for (int a = 0; a < m; ++a) {
      double ua = c.u[a * n + TX[a]];
      for (int b = m + 1; b < d; ++b) dde_mul_d(p, rho(ua, c.u[b * n + TY[b]]));
    }
  }
  c.pf[(base + al) * c.cap + be] = p;
}

__global__ void k_fill(double* p, double v, long long count) {
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < count; t += (long long)gridDim.x * blockDim.x)
    p[t] = v;
}

__device__ __forceinline__ void dd_mul_raw(double& h, double& l, double yh, double yl) {
  const double p = __dmul_rn(h, yh);
  const double err = fma(h, yh, -p);
  const double t = fma(h, yl, fma(l, yh, err));
  const double s = __dadd_rn(p, t);
  l = __dsub_rn(t, __dsub_rn(s, p));
  h = s;
}


// Fused quadrature fibers + weighted sums (t-form families), the product path of
// tt_integrate: W_m[alpha][beta] = sum_a w_{m,a} A(X_alpha, a, Y_beta) with the entries
// evaluated on the fly, nothing written per entry.
// A CTA owns a tile of FW_TA x FW_TB fibers (thread = fiber) and one of NS node ranges; the
// NS CTAs of a tile write their partial sums to global memory and the last one to arrive
// combines them in node-range order.  The CTA stages its node range (<= FW_CH
// nodes: every configuration's range fits in one chunk, so one barrier pair per CTA instead of
// one per 33-node chunk) in shared memory with cp.async: the Q_L rows of the tile's alphas, Q_R
// rows of its betas (hi / lo / e planes, odd row stride FW_CH + 1 so the 16 rows a warp reads
// at one node fall in distinct banks) and c_m, w_m of its nodes -- every factor is fetched once
// per tile instead of once per entry.  The fiber's frozen factors (S_L + S_R, Pf) stay in
// registers.
#define FW_TA 16
#define FW_TB 16
#define FW_CH 72   // max nodes per chunk (row stride 73 doubles: 16 rows in distinct banks)
#define FW_RS (FW_CH + 1)
#define FW_NSMAX 8   // node ranges per tile (at most)
#ifndef FW_MINB
#define FW_MINB 4    // resident CTAs per SM the register budget is sized for
#endif

struct FwBuf {
  double qlh[FW_TA][FW_RS], qll[FW_TA][FW_RS];
  double qrh[FW_TB][FW_RS], qrl[FW_TB][FW_RS];
  int qle[FW_TA][FW_RS], qre[FW_TB][FW_RS];
  long long chi[FW_CH], clo[FW_CH];
  double w[FW_CH];
};
__host__ __device__ constexpr int fw_smem_bytes() { return (int)sizeof(FwBuf); }

__device__ __forceinline__ void cp_async4(void* smem, const void* gmem) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(sa), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async8g(void* smem, const void* gmem) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(sa), "l"(gmem) : "memory");
}

// EMIT = true (tt_cross_get_fiber): the same kernel also stores every entry it contracts,
// F[alpha][beta][a] -> c.fib, so the fiber entries checked against the oracle are the product
// path's own (the stores are uncoalesced; diagnostics only).
template <int FAMILY, bool EMIT>
__global__ void __launch_bounds__(FW_TA * FW_TB, FW_MINB) k_fiber_wsum(DevCtx c, int kind, int jbase, int tiles_b) {
  extern __shared__ __align__(16) unsigned char fw_dyn[];
  FwBuf* buf = reinterpret_cast<FwBuf*>(fw_dyn);
  const int j = jbase + blockIdx.z;
  Job jb = make_job(c, kind, j);   // (entries counted by k_frozen_sides)
  const int A0 = (blockIdx.x / tiles_b) * FW_TA, B0 = (blockIdx.x % tiles_b) * FW_TB;
  if (A0 >= jb.rx || B0 >= jb.ry) return;   // (uniform over the tile's NS CTAs)
  const int tid = threadIdx.x;
  const int ra = tid / FW_TB, rb = tid % FW_TB;
  const int al = A0 + ra, be = B0 + rb;
  const bool live = al < jb.rx && be < jb.ry;
  const int n = c.n, m = jb.m;
  const int NS = gridDim.y, ns = blockIdx.y;
  const int len = (n + NS - 1) / NS;
  const int a_lo = min(n, ns * len), a_hi = min(n, a_lo + len);
  const int na = min(FW_TA, jb.rx - A0), nb = min(FW_TB, jb.ry - B0);
  const long long base = (long long)j * c.cap;
  const long long* gchi = c.chi + (long long)m * n;
  const long long* gclo = c.clo + (long long)m * n;
  const double* gw = c.w + (long long)m * n;
  const DDE* gql = FAMILY == 1 ? c.ql + (base + A0) * n : nullptr;
  const DDE* gqr = FAMILY == 1 ? c.qr + (base + B0) * n : nullptr;
  // stage chunk [a0, a0 + cn) into buffer b
  auto stage = [&](int b, int a0, int cn) {
    FwBuf& B = buf[b];
    if (tid < cn) {
      cp_async8g(&B.chi[tid], gchi + a0 + tid);
      cp_async8g(&B.clo[tid], gclo + a0 + tid);
      cp_async8g(&B.w[tid], gw + a0 + tid);
    }
    if (FAMILY == 1) {
      // (row, node) pairs of the tile's rows, node fastest (coalesced along each row)
      for (int e = tid; e < (na + nb) * cn; e += FW_TA * FW_TB) {
        const int row = e / cn, a = e - row * cn;
        const bool left = row < na;
        const int rr = left ? row : row - na;
        const double* src = reinterpret_cast<const double*>((left ? gql : gqr) + (long long)rr * n + a0 + a);
        if (left) {
          cp_async8g(&B.qlh[rr][a], src);
          cp_async8g(&B.qll[rr][a], src + 1);
          cp_async4(&B.qle[rr][a], src + 2);
        } else {
          cp_async8g(&B.qrh[rr][a], src);
          cp_async8g(&B.qrl[rr][a], src + 1);
          cp_async4(&B.qre[rr][a], src + 2);
        }
      }
    }
    cp_async_commit();
  };
  ESum s0 = esum_zero();
  DDE p0 = dde_one();
  if (live) {
    s0 = c.sl[base + al];
    esum_add(s0, c.sr[base + be]);
    if (FAMILY == 1) p0 = c.pf[(base + al) * c.cap + be];
  }
  double hi = 0.0, lo = 0.0;
  double* F = EMIT ? c.fib + (long long)j * c.fib_stride + ((long long)al * jb.ry + be) * n : nullptr;
  // balanced chunks of <= FW_CH nodes (one for every configuration's node range)
  const int nchunk = (a_hi - a_lo + FW_CH - 1) / FW_CH;
  const int csz = nchunk > 0 ? (a_hi - a_lo + nchunk - 1) / nchunk : 0;
  for (int ci = 0; ci < nchunk; ++ci) {
    const int a0 = a_lo + ci * csz, cn = min(csz, a_hi - a0);
    if (ci > 0) __syncthreads();   // (the previous chunk is read by every thread before restaging)
    stage(0, a0, cn);
    cp_async_wait_group<0>();
    __syncthreads();
    const FwBuf& B = buf[0];
    if (live) {
      // groups of FW_ILP nodes: the entries of a group on their branch-free fast paths side by
      // side (their dependent chains interleave), an entry off the fast path redone the plain
      // way after the group, then the weighted terms accumulated in node order
      // (family C: 4 -- 74 vs 84 us on C_200; family D: 2 -- its longer entry fills the issue
      // slots already, 4 measured 3% slower on D_20)
      constexpr int FW_ILP = FAMILY == 0 ? 4 : 2;
#pragma unroll 1
      for (int g0 = 0; g0 < cn; g0 += FW_ILP) {
        double v[FW_ILP];
        unsigned slow = 0;
#pragma unroll
        for (int u = 0; u < FW_ILP; ++u) {
          const int a = min(g0 + u, cn - 1);
          ESum s = s0;
          esum_add(s, B.chi[a], B.clo[a]);
          const double S = esum_round(s);
          const double SS = __dmul_rn(S, S);
          bool ok;
          if (FAMILY == 0) {
            v[u] = div_pre_fast(1.0, SS, rcp_refined(SS), ok);
          } else {
            double ph = p0.hi, pl = p0.lo;
            dd_mul_raw(ph, pl, B.qlh[ra][a], B.qll[ra][a]);
            dd_mul_raw(ph, pl, B.qrh[rb][a], B.qrl[rb][a]);
            v[u] = dde_div_fast(DDE{ph, pl, p0.e + B.qle[ra][a] + B.qre[rb][a], 0}, SS, ok);
          }
          slow |= (ok ? 0u : 1u) << u;
        }
        if (slow) {   // (rare: the IEEE division, out of the group's chains)
#pragma unroll 1
          for (int u = 0; u < FW_ILP; ++u) {
            if (!((slow >> u) & 1u)) continue;
            const int a = min(g0 + u, cn - 1);
            ESum s = s0;
            esum_add(s, B.chi[a], B.clo[a]);
            const double S = esum_round(s);
            const double SS = __dmul_rn(S, S);
            double w;
            if (FAMILY == 0) {
              w = __drcp_rn(SS);
            } else {
              double ph = p0.hi, pl = p0.lo;
              dd_mul_raw(ph, pl, B.qlh[ra][a], B.qll[ra][a]);
              dd_mul_raw(ph, pl, B.qrh[rb][a], B.qrl[rb][a]);
              w = dde_div(DDE{ph, pl, p0.e + B.qle[ra][a] + B.qre[rb][a], 0}, SS);
            }
#pragma unroll
            for (int q = 0; q < FW_ILP; ++q)
              if (q == u) v[q] = w;
          }
        }
#pragma unroll
        for (int u = 0; u < FW_ILP; ++u) {
          if (g0 + u >= cn) break;
          const int a = g0 + u;
          if (EMIT) F[a0 + a] = v[u];
          const double wa = B.w[a];
          const double pr = __dmul_rn(wa, v[u]);
          const double pe = fma(wa, v[u], -pr);
          const double s1 = __dadd_rn(hi, pr);
          const double bb = __dsub_rn(s1, hi);
          const double er = __dadd_rn(__dsub_rn(hi, __dsub_rn(s1, bb)), __dsub_rn(pr, bb));
          const double l1 = __dadd_rn(lo, __dadd_rn(er, pe));
          hi = __dadd_rn(s1, l1);
          lo = __dsub_rn(l1, __dsub_rn(hi, s1));
        }
      }
    }
  }
  const long long wi = ((long long)j * c.cap + al) * c.cap + be;
  if (NS == 1) {
    if (live) c.W[wi] = DD{hi, lo};
    return;
  }
  // the NS node-range partials go to global memory; the last CTA of the tile to arrive (a
  // counter per tile) sums them in node-range order -- no CTA waits for the others (a cluster
  // reduction kept every CTA of the tile resident until the slowest one finished)
  if (live) c.wpart[wi * FW_NSMAX + ns] = DD{hi, lo};
  __threadfence();
  __syncthreads();
  __shared__ int s_last;
  if (tid == 0) {
    int* cnt = &c.wcnt[(long long)j * gridDim.x + blockIdx.x];
    const int old = atomicAdd(cnt, 1);
    s_last = old == NS - 1;
    if (s_last) *cnt = 0;   // (every CTA of the tile has arrived: ready for the next launch)
  }
  __syncthreads();
  if (s_last && live) {
    __threadfence();
    const double2 v0 = __ldcg(reinterpret_cast<const double2*>(&c.wpart[wi * FW_NSMAX]));   // (L2: written by other SMs)
    DD acc = DD{v0.x, v0.y};
    for (int q = 1; q < NS; ++q) {
      const double2 v = __ldcg(reinterpret_cast<const double2*>(&c.wpart[wi * FW_NSMAX + q]));
      acc = dd_add(acc, DD{v.x, v.y});
    }
    c.W[wi] = acc;
  }
}

// quadrature fibers of the x-form families: direct evaluation of every entry (the x-form
// integrand is not a function of per-mode node values, so the frozen-part factorisation
// of the t-form does not apply); grid x = flat (beta*n + a) chunks, y = alpha, z = job
template <int FAM>
__global__ void __launch_bounds__(256) k_fiber_x(DevCtx c, int kind, int jbase) {
  const int j = jbase + blockIdx.z, al = blockIdx.y;
  Job jb = make_job(c, kind, j);
  if (al >= jb.rx) return;
  const int n = c.n, m = jb.m, d = c.d;
  const int total = jb.ry * n;
  if (al == 0 && blockIdx.x == 0 && threadIdx.x == 0 && c.counters) {
    atomicAdd(&c.counters[CNT_EVALS], (unsigned long long)jb.rx * jb.ry * n);
    atomicAdd(&c.counters[CNT_FIBER_ENTRIES], (unsigned long long)jb.rx * jb.ry * n);
  }
  const int* TX = jb.X ? jb.X + (long long)al * d : nullptr;
  double* F = c.fib + (long long)j * c.fib_stride + (long long)al * jb.ry * n;
  for (int f = blockIdx.x * blockDim.x + threadIdx.x; f < total; f += gridDim.x * blockDim.x) {
    const int be = f / n;
    const int a = f - be * n;
    const int* TY = jb.Y ? jb.Y + (long long)be * d : nullptr;
    F[f] = x_entry_at<FAM>(c.u, c.wf, d, n, [&](int q) { return q < m ? TX[q] : (q == m ? a : TY[q]); });
  }
}

// ---------------------------------------------------------------------------------------
// quadrature (§4.1)
// ---------------------------------------------------------------------------------------
// intersection matrices M_i[s][t] = A(left(PIV[i][s]), right(PIV[i][t])), direct O(d^2)
__global__ void k_intersection(DevCtx c, int ibase) {
  const int i = ibase + blockIdx.z;
  const int s = blockIdx.y;
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  const int d = c.d, n = c.n;
  const int r = rec_rank(c.rec_cur, c.RS, i);
  if (s == 0 && t == 0 && c.counters) atomicAdd(&c.counters[CNT_EVALS], (unsigned long long)r * r);
  if (s >= r || t >= r) return;
  const int* Ps = rec_piv(c.rec_cur, c.RS, i) + (long long)s * d;
  const int* Pt = rec_piv(c.rec_cur, c.RS, i) + (long long)t * d;
  if (c.family >= 2) {
    c.M[((long long)i * c.cap + s) * c.cap + t] =
        x_entry_dyn(c.family, c.u, c.wf, d, n, [&](int q) { return q <= i ? Ps[q] : Pt[q]; });
    return;
  }
  ESum S = esum_zero();
  for (int q = 0; q < d; ++q) {
    int node = q <= i ? Ps[q] : Pt[q];
    esum_add(S, c.chi[q * n + node], c.clo[q * n + node]);
  }
  const double Sd = esum_round(S);
  const double SS = __dmul_rn(Sd, Sd);
  double v;
  if (c.family == 0) {
    v = __drcp_rn(SS);
  } else {
    DDE p = dde_one();
    for (int a = 0; a < d; ++a) {
      double ua = c.u[a * n + (a <= i ? Ps[a] : Pt[a])];
      for (int b = a + 1; b < d; ++b) dde_mul_d(p, rho(ua, c.u[b * n + (b <= i ? Ps[b] : Pt[b])]));
    }
    v = dde_div(p, SS);
  }
  c.M[((long long)i * c.cap + s) * c.cap + t] = v;
}

// W_m[alpha][beta] = sum_a w_{m,a} F_m[alpha][beta][a] in double-double; one warp per entry
__global__ void k_wsum(DevCtx c, int mode_base) {
  const int m = mode_base + blockIdx.z;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int al = blockIdx.y;
  const int be = blockIdx.x * (blockDim.x >> 5) + warp;
  Job jb = make_job(c, JOB_INT, m);
  if (al >= jb.rx || be >= jb.ry) return;
  const int n = c.n;
  const double* F = c.fib + (long long)m * c.fib_stride + ((long long)al * jb.ry + be) * n;
  const double* w = c.w + (long long)m * n;
  DD acc = dd_make(0.0);
  for (int a = lane; a < n; a += 32) {
    double p = w[a] * F[a];
    acc = dd_add(acc, DD{p, fma(w[a], F[a], -p)});
  }
  for (int o = 16; o; o >>= 1) {
    DD other{__shfl_xor_sync(0xffffffffu, acc.hi, o), __shfl_xor_sync(0xffffffffu, acc.lo, o)};
    acc = dd_add(acc, other);
  }
  if (lane == 0) c.W[((long long)m * c.cap + al) * c.cap + be] = acc;
}

// H_i = M_i^{-1} W_{i+1}: LU with partial pivoting in double-double on [M_i | W_{i+1}] in
// shared memory, one CTA per owned interface.  Rows are permuted through an index array (no
// row swaps).  Elimination step k: warp 0 picks the pivot (first maximiser of |A[row][k].hi|
// over the remaining rows in their current order) -- barrier -- every thread forms the pivot
// reciprocal itself (one IEEE division + a double-double Newton step: the same bits on every
// thread) and updates its share of the trailing block of [A | B] with l = A[row][k] * 1/akk --
// barrier.  Back substitution, one barrier per step: X[k] = B[k] / U[k][k] goes straight to
// H, and B[q] -= U[q][k] X[k] (q < k) recomputes X[k] locally.  (Double-double throughout:
// the contraction is compared with the exact value at 1e-12, R9.)  grid: x = owned
// interface, y = a share of the right-hand-side columns (each CTA eliminates A itself and
// carries only its columns of B: the elimination is r^3/3, the right-hand sides r^2 nc).
__device__ __forceinline__ DD dd_recip(DD y) {
  const double q1 = 1.0 / y.hi;
  const DD e = dd_sub(dd_make(1.0), dd_mul_d(y, q1));   // 1 - y q1, tiny
  return dd_add(dd_make(q1), dd_mul_d(e, q1));
}

__global__ void __launch_bounds__(512) k_solve(DevCtx c) {
  const int i = blockIdx.x + c.kb;
  const int cap = c.cap, d = c.d;
  extern __shared__ DD smd[];
  DD* A = smd;                 // [cap][cap]
  DD* Bm = smd + cap * cap;    // [cap][cap]
  __shared__ DD dinv[TTC_MAX_RANK_DEV], lmul[TTC_MAX_RANK_DEV];
  __shared__ int perm[TTC_MAX_RANK_DEV];
  const int r = rec_rank(c.rec_cur, c.RS, i);
  const int nc_all = (i + 1 < d - 1) ? rec_rank(c.rec_cur, c.RS, i + 1) : 1;
  const int cps = (nc_all + gridDim.y - 1) / gridDim.y, c0 = blockIdx.y * cps;
  const int nc = min(nc_all - c0, cps);   // this CTA's columns [c0, c0 + nc)
  if (nc <= 0) return;
  for (int t = threadIdx.x; t < r * r; t += blockDim.x) {
    const int a = t / r, b = t % r;
    A[a * cap + b] = dd_make(c.M[((long long)i * cap + a) * cap + b]);
  }
  for (int t = threadIdx.x; t < r * nc; t += blockDim.x) {
    const int a = t / nc, b = t % nc;
    Bm[a * cap + b] = c.W[((long long)(i + 1) * cap + a) * cap + c0 + b];
  }
  for (int t = threadIdx.x; t < r; t += blockDim.x) perm[t] = t;
  __syncthreads();
  for (int k = 0; k < r; ++k) {
    if (threadIdx.x < 32) {
      // partial pivoting: first row of the largest |hi| (a warp argmax by REDUX: the bit
      // pattern of a non-negative double orders like its value; rows with no candidate: none)
      double bv = -1.0;
      int bq = k;
      for (int q = k + threadIdx.x; q < r; q += 32) {
        const double v = fabs(A[perm[q] * cap + k].hi);
        if (v > bv) { bv = v; bq = q; }
      }
      {
        const bool has = bv >= 0.0;
        const unsigned hi = has ? (unsigned)__double2hiint(bv) : 0u, lo = has ? (unsigned)__double2loint(bv) : 0u;
        const unsigned mh = __reduce_max_sync(0xffffffffu, hi);
        const unsigned ml = __reduce_max_sync(0xffffffffu, hi == mh ? lo : 0u);
        const unsigned mq = __reduce_min_sync(0xffffffffu, (has && hi == mh && lo == ml) ? (unsigned)bq : 0xffffffffu);
        bv = mq == 0xffffffffu ? -1.0 : __hiloint2double((int)mh, (int)ml);
        bq = mq == 0xffffffffu ? k : (int)mq;
      }
      if (threadIdx.x == 0) {
        const int t = perm[k];
        perm[k] = perm[bq];
        perm[bq] = t;
        if (!(bv > 0.0) && blockIdx.y == 0) atomicOr(&c.flags[0], 1);
      }
    }
    __syncthreads();
    const int pk = perm[k];
    const DD inv = dd_recip(A[pk * cap + k]);
    if (threadIdx.x == 0) dinv[k] = inv;
    const int nr = r - k - 1, width = nr + nc;
    // the step's multipliers once per row (not once per updated element)
    for (int q = threadIdx.x; q < nr; q += blockDim.x) lmul[q] = dd_mul(A[perm[k + 1 + q] * cap + k], inv);
    __syncthreads();
    // a thread keeps one column and steps over the rows (no integer division per element: the
    // 512 threads as qs row lanes x width columns, the last partial row lane idle); the pivot
    // row's entry of the column is loaded once
    if (nr > 0) {
      const int qs = blockDim.x / width, colx = threadIdx.x % width, q0 = threadIdx.x / width;
      if (q0 < qs) {
        const bool inA = colx < nr;
        DD* base = inA ? A + k + 1 + colx : Bm + (colx - nr);
        const DD pv = base[pk * cap];
#pragma unroll 2
        for (int q = q0; q < nr; q += qs) {
          DD* e = base + perm[k + 1 + q] * cap;
          *e = dd_sub(*e, dd_mul(lmul[q], pv));
        }
      }
    }
    __syncthreads();
  }
  DD* H = c.H + (long long)i * cap * cap;
  for (int k = r - 1; k >= 0; --k) {
    const int pk = perm[k];
    const DD dk = dinv[k];
    // a thread keeps one column, rows q0, q0 + qs, ... (q == k: write X[k]; q < k: update row q)
    {
      const int qs = blockDim.x / nc, col = threadIdx.x % nc, q0 = threadIdx.x / nc;
      if (q0 < qs) {
        const DD xk = dd_mul(Bm[pk * cap + col], dk);
        for (int q = q0; q <= k; q += qs) {
          if (q == k) {
            H[(long long)k * cap + c0 + col] = xk;
          } else {
            const int pq = perm[q];
            Bm[pq * cap + col] = dd_sub(Bm[pq * cap + col], dd_mul(A[pq * cap + k], xk));
          }
        }
      }
    }
    __syncthreads();
  }
}

// record layout (doubles): [rows, cols, log2scale, V_hi[cap*cap], V_lo[cap*cap]]
__host__ __device__ __forceinline__ long long chain_record_size(int cap) { return 3 + 2LL * cap * cap; }

__device__ double block_absmax(double v, double* red) {
  red[threadIdx.x] = v;
  __syncthreads();
  for (int s2 = blockDim.x / 2; s2; s2 >>= 1) {
    if (threadIdx.x < s2) red[threadIdx.x] = fmax(red[threadIdx.x], red[threadIdx.x + s2]);
    __syncthreads();
  }
  double m = red[0];
  __syncthreads();
  return m;
}

// ---------------------------------------------------------------------------------------
// tree-reduced chain: the rank's partial product W_0 H_kb ... H_{ke-1} (rank 0) or
// H_kb ... H_{ke-1} (others) as a balanced binary tree of double-double matrix products,
// ceil(log2(items)) launches instead of d sequential vector-matrix steps.  Each item carries
// its dimensions and a power-of-two scale (exact), renormalised after every product so that
// d = 200 neither overflows nor underflows.  The §4.1 product is associative; the tree only
// changes the double-double rounding (R9).
// item layout: DD [cap][cap] (row-major, stride cap) + int dims [3] = rows, cols, log2scale
// ---------------------------------------------------------------------------------------
__global__ void __launch_bounds__(256) k_chain_init(DevCtx c, int i_begin, int i_end, int with_head, DD* dst,
                                                      int* ddim) {
  const int cap = c.cap, d = c.d;
  const int item = blockIdx.x;  // 0..count-1
  int i;
  int rows, cols;
  const DD* src;
  long long src_stride = cap;
  if (with_head && item == 0) {
    rows = 1;
    cols = (d > 1) ? rec_rank(c.rec_cur, c.RS, 0) : 1;
    src = c.W;  // W_0, row 0
  } else {
    i = i_begin + item - (with_head ? 1 : 0);
    rows = rec_rank(c.rec_cur, c.RS, i);
    cols = (i + 1 < d - 1) ? rec_rank(c.rec_cur, c.RS, i + 1) : 1;
    src = c.H + (long long)i * cap * cap;
  }
  DD* D = dst + (long long)item * cap * cap;
  for (int t = threadIdx.x; t < rows * cols; t += blockDim.x) {
    const int a = t / cols, b = t % cols;
    D[a * cap + b] = src[a * src_stride + b];
  }
  if (threadIdx.x == 0) {
    ddim[item * 3 + 0] = rows;
    ddim[item * 3 + 1] = cols;
    ddim[item * 3 + 2] = 0;
  }
}

// dst[j] = src[2j] * src[2j+1] (or src[2j] if it has no partner); when `final` (one output
// item), also write the chain record [rows, cols, log2scale, hi, lo]
__global__ void __launch_bounds__(256) k_chain_level(int cap, const DD* src, const int* sdim, int count, DD* dst,
                                                       int* ddim, double* rec, int final) {
  __shared__ double red[256];
  const int j = blockIdx.x, ia = 2 * j, ib = 2 * j + 1;
  const DD* A = src + (long long)ia * cap * cap;
  DD* C = dst + (long long)j * cap * cap;
  const int p = sdim[ia * 3 + 0], q = sdim[ia * 3 + 1];
  int s_, ex = 0;
  long long lg = sdim[ia * 3 + 2];
  if (ib >= count) {
    s_ = q;
    for (int t = threadIdx.x; t < p * q; t += blockDim.x) C[(t / q) * cap + t % q] = A[(t / q) * cap + t % q];
  } else {
    const DD* B = src + (long long)ib * cap * cap;
    s_ = sdim[ib * 3 + 1];
    lg += sdim[ib * 3 + 2];
    double mx = 0.0;
    for (int t = threadIdx.x; t < p * s_; t += blockDim.x) {
      const int a = t / s_, col = t % s_;
      DD acc = dd_make(0.0);
      for (int k = 0; k < q; ++k) acc = dd_add(acc, dd_mul(A[a * cap + k], B[k * cap + col]));
      C[a * cap + col] = acc;
      mx = fmax(mx, fabs(acc.hi));
    }
    mx = block_absmax(mx, red);
    if (mx > 0.0 && isfinite(mx)) frexp(mx, &ex);
    __syncthreads();
    for (int t = threadIdx.x; t < p * s_; t += blockDim.x) {
      const int a = t / s_, col = t % s_;
      C[a * cap + col] = dd_ldexp(C[a * cap + col], -ex);
    }
    lg += ex;
  }
  if (threadIdx.x == 0) {
    ddim[j * 3 + 0] = p;
    ddim[j * 3 + 1] = s_;
    ddim[j * 3 + 2] = (int)lg;
  }
  if (final) {
    __syncthreads();
    if (threadIdx.x == 0) { rec[0] = p; rec[1] = s_; rec[2] = (double)lg; }
    for (int t = threadIdx.x; t < p * s_; t += blockDim.x) {
      const int a = t / s_, col = t % s_;
      rec[3 + a * cap + col] = C[a * cap + col].hi;
      rec[3 + (long long)cap * cap + a * cap + col] = C[a * cap + col].lo;
    }
  }
}

// Rank 0's partial product as a vector chain: v = W_0 H_kb H_kb+1 ... H_{ke-1}, one
// vector-matrix product per interface in one CTA (r^2 double-double terms per step instead of
// the tree's r^3 per product).  Column col of a step is summed by 4 adjacent lanes (terms
// k = sub mod 4, then an xor combine); after every step v is rescaled by the exact power of
// two 2^-e of its largest entry (e accumulated in log2scale) so long chains neither overflow
// nor underflow.  Writes the chain record [1, cols, log2scale, hi[cols], lo[cols]].
#define CHAIN_VEC_MAX 64   // interfaces up to which rank 0 uses the vector chain
__global__ void __launch_bounds__(256) k_chain_vec(DevCtx c, int i_begin, int i_end, double* rec) {
  const int cap = c.cap, d = c.d;
  __shared__ DD v[2][TTC_MAX_RANK_DEV];
  __shared__ double wmax[2][8];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int col = tid >> 2, sub = tid & 3;
  int len = d > 1 ? rec_rank(c.rec_cur, c.RS, 0) : 1;
  for (int t = tid; t < len; t += blockDim.x) v[0][t] = c.W[t];   // W_0, row 0
  long long lg = 0;
  int cur = 0, ex = 0;
  // this lane's terms of the next step's H column, prefetched a step ahead (cap <= 64)
  constexpr int KPL = TTC_MAX_RANK_DEV / 4;
  DD hn[KPL];
  auto fetch = [&](int i) {
    const int rows = i == i_begin ? len : rec_rank(c.rec_cur, c.RS, i);
    const int cols = (i + 1 < d - 1) ? rec_rank(c.rec_cur, c.RS, i + 1) : 1;
    const DD* H = c.H + (long long)i * cap * cap;
#pragma unroll
    for (int q = 0; q < KPL; ++q) {
      const int k = sub + 4 * q;
      hn[q] = (col < cols && k < rows) ? H[(long long)k * cap + col] : dd_make(0.0);
    }
  };
  if (i_begin < i_end) fetch(i_begin);
  __syncthreads();
  for (int i = i_begin; i < i_end; ++i) {
    const int rows = len;
    const int cols = (i + 1 < d - 1) ? rec_rank(c.rec_cur, c.RS, i + 1) : 1;
    DD hc[KPL];
#pragma unroll
    for (int q = 0; q < KPL; ++q) hc[q] = hn[q];
    if (i + 1 < i_end) fetch(i + 1);
    // v * 2^-ex by two exact power-of-two factors (|ex| <= 1074)
    const double sc1 = ldexp(1.0, -(ex / 2)), sc2 = ldexp(1.0, -(ex - ex / 2));
    DD acc = dd_make(0.0);
#pragma unroll
    for (int q = 0; q < KPL; ++q) {
      const int k = sub + 4 * q;
      if (k < rows) {
        const DD vk = v[cur][k];
        acc = dd_add(acc, dd_mul(DD{vk.hi * sc1 * sc2, vk.lo * sc1 * sc2}, hc[q]));
      }
    }
    acc = dd_add(acc, DD{__shfl_xor_sync(0xffffffffu, acc.hi, 1), __shfl_xor_sync(0xffffffffu, acc.lo, 1)});
    acc = dd_add(acc, DD{__shfl_xor_sync(0xffffffffu, acc.hi, 2), __shfl_xor_sync(0xffffffffu, acc.lo, 2)});
    double mx = (col < cols) ? fabs(acc.hi) : 0.0;
#pragma unroll
    for (int o = 16; o; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    const int p = (i - i_begin) & 1;
    if (lane == 0) wmax[p][warp] = mx;
    if (sub == 0 && col < cols) v[cur ^ 1][col] = acc;
    __syncthreads();
    mx = 0.0;
    for (int q = 0; q < (int)(blockDim.x >> 5); ++q) mx = fmax(mx, wmax[p][q]);
    ex = 0;
    if (mx > 0.0 && isfinite(mx)) frexp(mx, &ex);
    lg += ex;
    cur ^= 1;
    len = cols;
  }
  if (tid == 0) { rec[0] = 1; rec[1] = len; rec[2] = (double)lg; }
  const long long LO = (long long)cap * cap;
  for (int t = tid; t < len; t += blockDim.x) {
    const DD x = dd_ldexp(v[cur][t], -ex);
    rec[3 + t] = x.hi;
    rec[3 + LO + t] = x.lo;
  }
}

// Multiply the world records in rank order: out = [core_hi, log2scale, core_lo]; one CTA.
__global__ void __launch_bounds__(256) k_finish(const double* recs, int world, int cap, double* out) {
  __shared__ DD v[TTC_MAX_RANK_DEV], v2[TTC_MAX_RANK_DEV];
  __shared__ double red[256];
  __shared__ long long lg2;
  __shared__ int len;
  const long long RSZ = chain_record_size(cap);
  const long long LO = (long long)cap * cap;
  if (threadIdx.x == 0) {
    lg2 = (long long)recs[2];
    len = (int)recs[1];
  }
  __syncthreads();
  for (int t = threadIdx.x; t < len; t += blockDim.x) v[t] = DD{recs[3 + t], recs[3 + LO + t]};
  __syncthreads();
  for (int p = 1; p < world; ++p) {
    const double* R = recs + p * RSZ;
    const int rows = (int)R[0], cols = (int)R[1];
    if (rows == 0) continue;
    double mx = 0.0;
    for (int col = threadIdx.x; col < cols; col += blockDim.x) {
      DD acc = dd_make(0.0);
      for (int k = 0; k < rows; ++k)
        acc = dd_add(acc, dd_mul(v[k], DD{R[3 + k * cap + col], R[3 + LO + k * cap + col]}));
      v2[col] = acc;
      mx = fmax(mx, fabs(acc.hi));
    }
    mx = block_absmax(mx, red);
    int ex = 0;
    if (mx > 0.0 && isfinite(mx)) frexp(mx, &ex);
    for (int col = threadIdx.x; col < cols; col += blockDim.x) v[col] = dd_ldexp(v2[col], -ex);
    if (threadIdx.x == 0) { lg2 += ex + (long long)R[2]; len = cols; }
    __syncthreads();
  }
  if (threadIdx.x == 0) { out[0] = v[0].hi + v[0].lo; out[1] = (double)lg2; }
}

}  // namespace ttc
