// ttc_api.cu -- host side of libttcross: context, memory, launch sequences, C-ABI
// (include/ttcross.h).  One translation unit; compiled for sm_100a only.
#include <cuda.h>          // CUtensorMap and its enums (types only: the driver entry point is
#include <cudaTypedefs.h>  // fetched at run time, libcuda is not linked)
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/ttcross.h"
#include "ttc_common.cuh"
#include "ttc_greedy.cuh"
#include "ttc_kernels.cuh"

using namespace ttc;

namespace {

thread_local std::string g_err = "no error";

int fail(int code, const std::string& msg) {
  g_err = msg;
  return code;
}

#define CK(call)                                                                         \
  do {                                                                                   \
    cudaError_t e_ = (call);                                                             \
    if (e_ != cudaSuccess)                                                               \
      return fail(TTC_ERR_CUDA, std::string(#call) + ": " + cudaGetErrorString(e_));     \
  } while (0)

enum KClass { KC_FIBER = 0, KC_CROSS = 1, KC_QUAD = 2, KC_OTHER = 3 };

// per-kernel identifiers for tt_cross_get_kernel_time (class = accounting bucket of ttc_stats)
enum KId {
  K_PREP = 0, K_INIT_PIVOT, K_INIT_RECORDS, K_SWEEP, K_FROZEN_SIDES, K_FROZEN_Q, K_FROZEN_LR, K_FIBER,
  K_WSUM, K_INTERSECTION, K_SOLVE, K_CHAIN, K_FINISH, K_COUNT
};
const char* const kKernelName[K_COUNT] = {
    "k_prep_nodes", "k_init_pivot", "k_init_records", "k_sweep", "k_frozen_sides", "k_frozen_q",
    "k_frozen_lr", "k_fiber", "k_wsum", "k_intersection", "k_solve", "k_chain", "k_finish"};
const int kKernelClass[K_COUNT] = {KC_OTHER, KC_OTHER, KC_OTHER, KC_CROSS, KC_FIBER, KC_FIBER, KC_FIBER,
                                   KC_FIBER, KC_QUAD,  KC_QUAD,  KC_QUAD,  KC_QUAD,  KC_QUAD};

const char* const kWaveTimeout =
    "k_sweeps: a superblock waited > 2 s for a neighbour (clusters not co-resident); the sweeps are incomplete";

struct EvRec {
  cudaEvent_t a, b;
  int kid;
};

}  // namespace

struct ttc_ctx {
  ttc_config cfg{};
  cudaStream_t stream = nullptr;
  cudaStream_t ls = nullptr;          // launch stream: `stream`, or the capture stream while a graph is built
  cudaStream_t cap_stream = nullptr;  // private stream used to capture the solve graph
  // quadrature branches that do not depend on each other (k_intersection, k_frozen_q) run on
  // two side streams forked from / joined to ls by events -- concurrent branches of the graph
  cudaStream_t side[2] = {nullptr, nullptr};
  cudaEvent_t ev_fork[2] = {nullptr, nullptr}, ev_join[2] = {nullptr, nullptr};
  cudaGraph_t graph = nullptr;
  cudaGraphExec_t graph_exec = nullptr;
  int graph_sweeps = -1;
  long long graph_launches = 0;
  DevCtx dc{};
  int chunk = 0, kb = 0, ke = 0, n_owned = 0, slots = 0, nrec = 0;
  int* xbuf = nullptr;  // world > 1: exchange buffer [world][chunk][RS] (rank p's records in slot p)
  int sweeps = 0;
  int pending = 0;  // a local sweep waits for commit
  int* t0buf = nullptr;
  unsigned long long* phase_buf = nullptr;  // k_sweep phase timer (enabled with timing)
  int sms = 148;               // multiprocessors of the device
  bool greedy_cached = false;  // k_sweep keeps its rows' u / columns' v in shared memory
  size_t greedy_smem = 0;      // dynamic shared memory of k_sweep
  int greedy_threads = 256;    // CTA size of k_sweep (256: two CTAs per SM, 512: one)
  int fw_ns = 0;               // k_fiber_wsum node ranges per tile override (TTC_FW_NS; 0 = host rule)
  const void* greedy_fn = nullptr;   // k_sweep variant (one sweep)
  const void* sweeps_fn = nullptr;   // k_sweeps variant (persistent, world == 1)
  const void* sweeps_peer_fn = nullptr;   // its cross-GPU wavefront instantiation (t-form families), or null
  bool peer_resident = false;        // sweeps_peer_fn's clusters all resident at once
  bool persistent = false;           // k_sweeps usable (all clusters resident)
  bool resident_all = false;         // every owned superblock's cluster resident at once (any world)
  // cross-GPU wavefront (tt_cross_peer_open / tt_cross_sweep_peer)
  void* peer_maps[2][3] = {{nullptr, nullptr, nullptr}, {nullptr, nullptr, nullptr}};   // opened IPC mappings
  bool peer_consistent = true;       // rank_ring / done of every interface current (no tt_cross_sweep_local since reset)
  int* lb_rec = nullptr;             // loopback mirror (tt_cross_set_loopback)
  int* lb_ring = nullptr;
  int* lb_done = nullptr;
  // buffers
  std::vector<void*> allocs;
  long long rec_ints = 0;
  double* partials = nullptr;  // [world][3 + 2*cap*cap] (see k_chain_level)
  DD *chainA = nullptr, *chainB = nullptr;  // tree-chain ping-pong items [d][cap][cap]
  int *chainAd = nullptr, *chainBd = nullptr;  // their dims [d][3]
  double* out_dev = nullptr;   // [4]
  double* out_host = nullptr;  // pinned [8]
  // accounting
  long long launches = 0;
  bool timing = false;
  std::vector<EvRec> evs;
  std::vector<cudaEvent_t> ev_pool;
  double ms[4] = {0, 0, 0, 0};
  double kms[K_COUNT] = {};
  long long klaunch[K_COUNT] = {};
};

namespace {

template <typename T>
int dalloc(ttc_ctx* c, T** p, size_t count) {
  void* q = nullptr;
  size_t bytes = std::max<size_t>(count * sizeof(T), 16);
  cudaError_t e = cudaMalloc(&q, bytes);
  if (e != cudaSuccess)
    return fail(TTC_ERR_CUDA, std::string("cudaMalloc(") + std::to_string(bytes) + "): " + cudaGetErrorString(e));
  c->allocs.push_back(q);
  *p = static_cast<T*>(q);
  return TTC_OK;
}

cudaEvent_t get_event(ttc_ctx* c) {
  if (!c->ev_pool.empty()) {
    cudaEvent_t e = c->ev_pool.back();
    c->ev_pool.pop_back();
    return e;
  }
  cudaEvent_t e;
  cudaEventCreate(&e);
  return e;
}

// bracket a launch with events when timing is enabled
struct Timed {
  ttc_ctx* c;
  int kid;
  cudaStream_t s;
  cudaEvent_t a = nullptr;
  Timed(ttc_ctx* c_, int kid_, cudaStream_t s_ = nullptr) : c(c_), kid(kid_), s(s_ ? s_ : c_->ls) {
    c->launches++;
    c->klaunch[kid]++;
    if (c->timing) {
      a = get_event(c);
      cudaEventRecord(a, s);
    }
  }
  ~Timed() {
    if (c->timing) {
      cudaEvent_t b = get_event(c);
      cudaEventRecord(b, s);
      c->evs.push_back({a, b, kid});
    }
  }
};

// side stream i joins the work already issued on ls (fork) / ls waits for side stream i (join)
int side_fork(ttc_ctx* c, int i) {
  if (!c->side[i]) {
    if (cudaStreamCreateWithFlags(&c->side[i], cudaStreamNonBlocking) != cudaSuccess ||
        cudaEventCreateWithFlags(&c->ev_fork[i], cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&c->ev_join[i], cudaEventDisableTiming) != cudaSuccess)
      return fail(TTC_ERR_CUDA, "side stream / event creation failed");
  }
  if (cudaEventRecord(c->ev_fork[i], c->ls) != cudaSuccess || cudaStreamWaitEvent(c->side[i], c->ev_fork[i], 0) != cudaSuccess)
    return fail(TTC_ERR_CUDA, "side stream fork failed");
  return TTC_OK;
}
int side_join(ttc_ctx* c, int i) {
  if (cudaEventRecord(c->ev_join[i], c->side[i]) != cudaSuccess || cudaStreamWaitEvent(c->ls, c->ev_join[i], 0) != cudaSuccess)
    return fail(TTC_ERR_CUDA, "side stream join failed");
  return TTC_OK;
}

int check_launch(const char* what) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return fail(TTC_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
  return TTC_OK;
}

// ------------------------------------------------------------------ launch sequences
// quadrature fibers: frozen parts + entries for modes [jbase, jbase+njobs).  t-form
// families: k_fiber_wsum contracts the entries with the weights into W directly, nothing
// stored per entry (the product path of tt_integrate); emit (tt_cross_get_fiber): the same
// kernel also writes every entry to dc.fib.  x-form: k_fiber_x writes dc.fib and the caller
// runs k_wsum.
int launch_fibers(ttc_ctx* c, int kind, int jbase, int njobs, bool emit = false, bool count = true) {
  DevCtx dc = c->dc;
  if (!count) dc.counters = nullptr;   // (tt_cross_get_fiber: not part of the method's work)
  const int n = dc.n, tup = dc.cap;
  if (dc.family >= 2) {
    const int gx = std::min(4096, (tup * n + 255) / 256);
    {
      Timed t(c, K_FIBER);
      if (dc.family == 2) k_fiber_x<2><<<dim3(gx, tup, njobs), 256, 0, c->ls>>>(dc, kind, jbase);
      else if (dc.family == 3) k_fiber_x<3><<<dim3(gx, tup, njobs), 256, 0, c->ls>>>(dc, kind, jbase);
      else k_fiber_x<4><<<dim3(gx, tup, njobs), 256, 0, c->ls>>>(dc, kind, jbase);
    }
    return check_launch("k_fiber_x");
  }
  {
    Timed t(c, K_FROZEN_SIDES);
    k_frozen_sides<<<dim3((tup + 63) / 64, 2, njobs), 64, 0, c->ls>>>(dc, kind, jbase);
  }
  if (int e = check_launch("k_frozen_sides")) return e;
  if (dc.family == TTC_FAMILY_D) {
    // k_frozen_q needs only the records: a concurrent branch (side stream 1), joined before
    // the fiber kernel; k_frozen_lr follows k_frozen_sides on ls
    if (int e = side_fork(c, 1)) return e;
    {
      Timed t(c, K_FROZEN_Q, c->side[1]);
      k_frozen_q<<<dim3((n + 127) / 128, tup, 2 * njobs), 128, 0, c->side[1]>>>(dc, kind, jbase);
    }
    if (int e = check_launch("k_frozen_q")) return e;
    {
      Timed t(c, K_FROZEN_LR);
      k_frozen_lr<<<dim3((tup + 63) / 64, tup, njobs), 64, 0, c->ls>>>(dc, kind, jbase);
    }
    if (int e = check_launch("k_frozen_lr")) return e;
    if (int e = side_join(c, 1)) return e;
  }
  {
    Timed t(c, K_FIBER);
    // tiles of FW_TA x FW_TB fibers (the grid covers rank = cap; tiles beyond the actual
    // ranks exit at once) x NS node ranges, NS doubled up to 8 while
    // the grid has fewer than 4 waves of 4 CTAs per SM and the ranges keep >= 32 nodes
    const int ta = (tup + FW_TA - 1) / FW_TA, tb = (tup + FW_TB - 1) / FW_TB;
    const long long tiles = (long long)ta * tb * njobs;
    int ns = 1;
    while (ns < 8 && tiles * ns < 16LL * c->sms && n / (2 * ns) >= 32) ns *= 2;
    if (c->fw_ns > 0) ns = c->fw_ns;   // (experiments: TTC_FW_NS)
    cudaLaunchConfig_t lc = {};
    lc.gridDim = dim3(ta * tb, ns, njobs);
    lc.blockDim = dim3(FW_TA * FW_TB);
    lc.dynamicSmemBytes = fw_smem_bytes();
    lc.stream = c->ls;
    lc.numAttrs = 0;   // (the NS CTAs of a tile are independent: last-arrival reduction)
    cudaError_t e;
    if (dc.family == TTC_FAMILY_C)
      e = emit ? cudaLaunchKernelEx(&lc, k_fiber_wsum<0, true>, dc, kind, jbase, tb)
               : cudaLaunchKernelEx(&lc, k_fiber_wsum<0, false>, dc, kind, jbase, tb);
    else
      e = emit ? cudaLaunchKernelEx(&lc, k_fiber_wsum<1, true>, dc, kind, jbase, tb)
               : cudaLaunchKernelEx(&lc, k_fiber_wsum<1, false>, dc, kind, jbase, tb);
    if (e != cudaSuccess) return fail(TTC_ERR_CUDA, std::string("k_fiber_wsum launch: ") + cudaGetErrorString(e));
  }
  return check_launch("k_fiber_wsum");
}

// one Alg. 6 sweep over the owned superblocks -> rec_next
int do_sweep_local(ttc_ctx* c) {
  if (c->n_owned > 0) {
    DevCtx& dc = c->dc;
    const int nj = c->n_owned;
    cudaLaunchConfig_t lc = {};
    lc.gridDim = dim3(nj * dc.G);
    lc.blockDim = dim3(c->greedy_threads);
    lc.dynamicSmemBytes = 0;
    lc.stream = c->ls;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = dc.G;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    lc.attrs = at;
    lc.numAttrs = 1;
    cudaError_t e;
    {
      Timed t(c, K_SWEEP);
      lc.dynamicSmemBytes = c->greedy_smem;
      e = cudaLaunchKernelEx(&lc, (void (*)(DevCtx, int))c->greedy_fn, dc, c->sweeps);
    }
    if (e != cudaSuccess) return fail(TTC_ERR_CUDA, std::string("k_sweep launch: ") + cudaGetErrorString(e));
    if (int e2 = check_launch("k_sweep")) return e2;
  }
  c->peer_consistent = false;   // (the neighbour ranks' flags and ranks are not published here)
  if (c->cfg.world > 1 && c->n_owned > 0)   // own records -> own slot of the exchange buffer
    CK(cudaMemcpyAsync(c->xbuf + (long long)c->cfg.rank * c->chunk * c->dc.RS, c->dc.rec_next + (long long)c->kb * c->dc.RS,
                       sizeof(int32_t) * c->n_owned * c->dc.RS, cudaMemcpyDeviceToDevice, c->ls));
  c->pending = 1;
  return TTC_OK;
}

// n sweeps [c->sweeps, c->sweeps + n) of the owned superblocks in one persistent launch
// (k_sweeps); c->sweeps is advanced by the caller
int launch_sweeps(ttc_ctx* c, int n) {
  DevCtx& dc = c->dc;
  cudaLaunchConfig_t lc = {};
  lc.gridDim = dim3(c->n_owned * dc.G);
  lc.blockDim = dim3(c->greedy_threads);
  lc.dynamicSmemBytes = c->greedy_smem;
  lc.stream = c->ls;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = dc.G;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  lc.attrs = at;
  lc.numAttrs = 1;
  cudaError_t e;
  {
    Timed t(c, K_SWEEP);
    const bool peer = dc.pdone[0] || dc.pdone[1];   // (tt_cross_peer_open / tt_cross_set_loopback)
    e = cudaLaunchKernelEx(&lc, (void (*)(DevCtx, int, int))(peer ? c->sweeps_peer_fn : c->sweeps_fn), dc, c->sweeps, n);
  }
  if (e != cudaSuccess) return fail(TTC_ERR_CUDA, std::string("k_sweeps launch: ") + cudaGetErrorString(e));
  return check_launch("k_sweeps");
}

// n sweeps in one persistent launch (world == 1)
int do_sweeps_persistent(ttc_ctx* c, int n) {
  if (n <= 0) return TTC_OK;
  if (int e = launch_sweeps(c, n)) return e;
  c->sweeps += n;
  return TTC_OK;
}

// n sweeps of this rank's superblocks in one persistent launch, the boundary superblocks
// exchanging their records with the neighbour ranks' kernels through peer memory (world > 1),
// then this rank's records -> its slot of the exchange buffer; tt_cross_commit after the
// caller's all-gather completes the n sweeps
int do_sweeps_peer(ttc_ctx* c, int n) {
  if (n > 0 && c->n_owned > 0)
    if (int e = launch_sweeps(c, n)) return e;
  if (c->n_owned > 0)
    CK(cudaMemcpyAsync(c->xbuf + (long long)c->cfg.rank * c->chunk * c->dc.RS, c->dc.rec_cur + (long long)c->kb * c->dc.RS,
                       sizeof(int32_t) * c->n_owned * c->dc.RS, cudaMemcpyDeviceToDevice, c->ls));
  c->pending = n;
  return TTC_OK;
}

int do_commit(ttc_ctx* c) {
  if (!c->pending) return fail(TTC_ERR_STATE, "tt_cross_commit without a pending local sweep");
  if (c->cfg.world == 1) {
    std::swap(c->dc.rec_cur, c->dc.rec_next);
  } else {
    // every rank's slot of the all-gathered exchange buffer -> the current records
    k_unpack_records<<<c->cfg.world, 256, 0, c->ls>>>(c->xbuf, c->dc.rec_cur, c->dc.d - 1, c->cfg.world, c->chunk,
                                                      c->dc.RS);
    if (int e = check_launch("k_unpack_records")) return e;
  }
  c->sweeps += c->pending;   // (1 after tt_cross_sweep_local, n after tt_cross_sweep_peer)
  c->pending = 0;
  return TTC_OK;
}

int do_integrate_local(ttc_ctx* c) {
  DevCtx dc = c->dc;
  const int cap = dc.cap;
  const int rank = c->cfg.rank;
  // modes whose fibers are needed: i+1 for the owned interfaces i, and mode 0 on rank 0
  int m_lo = c->kb + 1, m_hi = c->ke;  // inclusive range
  if (rank == 0) m_lo = 0;
  const int nm = (c->n_owned > 0) ? (m_hi - m_lo + 1) : (rank == 0 ? 1 : 0);
  // the intersection matrices need only the records: a concurrent branch (side stream 0)
  // alongside the fibers, joined before k_solve
  if (c->n_owned > 0) {
    if (int e = side_fork(c, 0)) return e;
    {
      Timed t(c, K_INTERSECTION, c->side[0]);
      k_intersection<<<dim3((cap + 63) / 64, cap, c->n_owned), 64, 0, c->side[0]>>>(dc, c->kb);
    }
    if (int e = check_launch("k_intersection")) return e;
  }
  if (nm > 0) {
    if (int e = launch_fibers(c, JOB_INT, m_lo, nm)) return e;
    if (dc.family >= TTC_FAMILY_CX) {
      {
        Timed t(c, K_WSUM);
        k_wsum<<<dim3((cap + 7) / 8, cap, nm), 256, 0, c->ls>>>(dc, m_lo);
      }
      if (int e = check_launch("k_wsum")) return e;
    }
  }
  CK(cudaMemsetAsync(dc.flags, 0, sizeof(int), c->ls));  // flags[1] (sweep timeout) stays
  if (c->n_owned > 0) {
    if (int e = side_join(c, 0)) return e;
    {
      Timed t(c, K_SOLVE);
      // split the right-hand sides over CTAs while the interfaces leave SMs idle (each CTA
      // repeats the LU of M_k): up to 8 x 512 threads at cap 64 (D_20 0.20 -> 0.16 ms), 4 x 256
      // at cap 32 (more CTAs or threads measured slower on the smaller matrices)
      const int split = cap >= 64 ? std::max(1, std::min(8, c->sms / std::max(1, c->n_owned)))
                                  : ((cap >= 32 && 4 * c->n_owned <= c->sms) ? 4 : 1);
      k_solve<<<dim3(c->n_owned, split), cap >= 64 ? 512 : 256, 2 * cap * cap * sizeof(DD), c->ls>>>(dc);
    }
    if (int e = check_launch("k_solve")) return e;
  }
  double* rec = c->partials + (long long)rank * chain_record_size(cap);
  const int with_head = rank == 0 ? 1 : 0;
  const int items = c->n_owned + with_head;
  if (items == 0) {  // a rank without superblocks contributes an empty record
    CK(cudaMemsetAsync(rec, 0, 3 * sizeof(double), c->ls));
    return TTC_OK;
  }
  if (with_head && c->n_owned <= CHAIN_VEC_MAX) {   // rank 0: a vector chain (see k_chain_vec)
    {
      Timed t(c, K_CHAIN);
      k_chain_vec<<<1, 256, 0, c->ls>>>(dc, c->kb, c->kb + c->n_owned, rec);
    }
    return check_launch("k_chain_vec");
  }
  {
    Timed t(c, K_CHAIN);
    k_chain_init<<<items, 256, 0, c->ls>>>(dc, c->kb, c->ke, with_head, c->chainA, c->chainAd);
  }
  if (int e = check_launch("k_chain_init")) return e;
  DD* src = c->chainA;
  int* sd = c->chainAd;
  DD* dst = c->chainB;
  int* dd_ = c->chainBd;
  int count = items;
  if (count == 1) {  // a single item: one level that only copies and emits the record
    Timed t(c, K_CHAIN);
    k_chain_level<<<1, 256, 0, c->ls>>>(cap, src, sd, 1, dst, dd_, rec, 1);
    return check_launch("k_chain_level");
  }
  while (count > 1) {
    const int out = (count + 1) / 2;
    {
      Timed t(c, K_CHAIN);
      k_chain_level<<<out, 256, 0, c->ls>>>(cap, src, sd, count, dst, dd_, rec, out == 1 ? 1 : 0);
    }
    if (int e = check_launch("k_chain_level")) return e;
    std::swap(src, dst);
    std::swap(sd, dd_);
    count = out;
  }
  return TTC_OK;
}

// enqueue k_finish and the D2H copy of the result into pinned host memory (no sync)
int do_integrate_finish_launch(ttc_ctx* c) {
  const int cap = c->dc.cap;
  {
    Timed t(c, K_FINISH);
    k_finish<<<1, 256, 0, c->ls>>>(c->partials, c->cfg.world, cap, c->out_dev);
  }
  if (int e = check_launch("k_finish")) return e;
  CK(cudaMemcpyAsync(c->out_host, c->out_dev, 2 * sizeof(double), cudaMemcpyDeviceToHost, c->ls));
  CK(cudaMemcpyAsync(c->out_host + 2, c->dc.flags, 2 * sizeof(int), cudaMemcpyDeviceToHost, c->ls));
  return TTC_OK;
}

// wait for the enqueued result and decode it (value outside the fp64 range -> +-0/inf)
int do_integrate_read(ttc_ctx* c, double* value, double* log10_abs, int32_t* sign) {
  const int d = c->dc.d;
  CK(cudaStreamSynchronize(c->stream));
  int flag = 0, flag2[2] = {0, 0};
  std::memcpy(flag2, c->out_host + 2, 2 * sizeof(int));
  flag = flag2[0];
  if (flag2[1]) return fail(TTC_ERR_CUDA, kWaveTimeout);
  if (flag) return fail(TTC_ERR_SINGULAR, "an intersection matrix A(I_{<=k}, I_{>k}) is singular");
  const double core = c->out_host[0];
  const double lg2 = c->out_host[1];
  int sg = core > 0 ? 1 : (core < 0 ? -1 : 0);
  double l10, val;
  if (core == 0.0 || !std::isfinite(core)) {
    l10 = core == 0.0 ? -INFINITY : NAN;
    val = core;
  } else {
    const bool xform = c->dc.family >= 2;  // PAPER.md eq. (9)-(11): prefactor 2
    const double lnpre = xform ? std::log(2.0) : std::log(4.0) - std::lgamma((double)d + 1.0);
    const double ln_abs = std::log(std::fabs(core)) + lg2 * std::log(2.0) + lnpre;
    l10 = ln_abs / std::log(10.0);
    if (ln_abs > -700.0 && ln_abs < 700.0) {
      if (lg2 > -1000 && lg2 < 1000 && (xform || d <= 170)) {
        double pre = xform ? 2.0 : 4.0;
        if (!xform)
          for (int k = 2; k <= d; ++k) pre /= (double)k;
        val = std::ldexp(core, (int)lg2) * pre;
      } else {
        val = sg * std::exp(ln_abs);
      }
    } else {
      val = sg * (ln_abs > 0 ? INFINITY : 0.0);
    }
  }
  if (value) *value = val;
  if (log10_abs) *log10_abs = l10;
  if (sign) *sign = sg;
  return TTC_OK;
}

int resolve_timing(ttc_ctx* c) {
  if (c->evs.empty()) return TTC_OK;
  CK(cudaStreamSynchronize(c->stream));
  for (auto& r : c->evs) {
    float ms = 0.f;
    cudaEventElapsedTime(&ms, r.a, r.b);
    c->ms[kKernelClass[r.kid]] += ms;
    c->kms[r.kid] += ms;
    c->ev_pool.push_back(r.a);
    c->ev_pool.push_back(r.b);
  }
  c->evs.clear();
  return TTC_OK;
}

// device part of a reset (async, capturable): rank-1 start (the seeded first pivot, DESIGN.md
// R5 -- part of every timed solve), superblock state, counters
int reset_device(ttc_ctx* c) {
  CK(cudaMemsetAsync(c->dc.counters, 0, TTC_NCOUNTERS * sizeof(unsigned long long), c->ls));
  {
    Timed t(c, K_INIT_PIVOT);
    k_init_pivot<<<1, N_INIT_WARPS * 32, 0, c->ls>>>(c->dc, c->t0buf);
  }
  if (int e = check_launch("k_init_pivot")) return e;
  {
    Timed t(c, K_INIT_RECORDS);
    k_init_records<<<std::max(std::max(c->nrec, c->n_owned), c->dc.d - 1), 128, 0, c->ls>>>(c->dc, c->t0buf, c->nrec,
                                                                                      c->n_owned);
  }
  return check_launch("k_init_records");
}

int reset_host(ttc_ctx* c) {
  c->sweeps = 0;
  c->pending = 0;
  c->peer_consistent = true;
  c->launches = 0;
  if (int e = resolve_timing(c)) return e;
  for (double& m : c->ms) m = 0.0;
  for (int k = 0; k < K_COUNT; ++k) { c->kms[k] = 0.0; c->klaunch[k] = 0; }
  return TTC_OK;
}

int do_reset(ttc_ctx* c) {
  if (int e = reset_host(c)) return e;
  return reset_device(c);
}

// n_sweeps sweeps + the quadrature, enqueued on c->ls (world == 1)
int enqueue_solve(ttc_ctx* c, int n_sweeps) {
  if (c->persistent) {
    if (int e = do_sweeps_persistent(c, n_sweeps)) return e;
  } else {
    for (int s = 0; s < n_sweeps; ++s) {
      if (int e = do_sweep_local(c)) return e;
      if (int e = do_commit(c)) return e;
    }
  }
  if (int e = do_integrate_local(c)) return e;
  return do_integrate_finish_launch(c);
}

// Capture reset + n_sweeps sweeps + quadrature as one CUDA graph.  Every launch shape
// depends only on (d, n, cap); ranks are read on the device, so the graph is valid for any
// grid loaded into this context.
int capture_solve(ttc_ctx* c, int n_sweeps) {
  if (c->graph_exec) { cudaGraphExecDestroy(c->graph_exec); c->graph_exec = nullptr; }
  if (c->graph) { cudaGraphDestroy(c->graph); c->graph = nullptr; }
  if (!c->cap_stream) CK(cudaStreamCreateWithFlags(&c->cap_stream, cudaStreamNonBlocking));
  if (int e = reset_host(c)) return e;
  const bool timing = c->timing;
  c->timing = false;
  c->ls = c->cap_stream;
  int rc = TTC_OK;
  cudaError_t ce = cudaStreamBeginCapture(c->cap_stream, cudaStreamCaptureModeThreadLocal);
  if (ce != cudaSuccess) rc = fail(TTC_ERR_CUDA, std::string("cudaStreamBeginCapture: ") + cudaGetErrorString(ce));
  if (!rc) rc = reset_device(c);
  if (!rc) rc = enqueue_solve(c, n_sweeps);
  cudaGraph_t g = nullptr;
  ce = cudaStreamEndCapture(c->cap_stream, &g);
  c->ls = c->stream;
  c->timing = timing;
  if (rc) { if (g) cudaGraphDestroy(g); return rc; }
  if (ce != cudaSuccess) return fail(TTC_ERR_CUDA, std::string("cudaStreamEndCapture: ") + cudaGetErrorString(ce));
  c->graph = g;
  CK(cudaGraphInstantiate(&c->graph_exec, g, 0));
  c->graph_sweeps = n_sweeps;
  c->graph_launches = c->launches;
  return reset_host(c);
}

}  // namespace

// ====================================================================================
// C-ABI
// ====================================================================================
extern "C" {

const char* tt_last_error(void) { return g_err.c_str(); }

#ifdef TTC_TRACE
// trace build only (tools/trace_steps.py): copy out and clear the step trace
int ttc_trace_read(unsigned long long* events, int* counts) {
  if (cudaMemcpyFromSymbol(events, ttc::g_trace, sizeof(ttc::g_trace)) != cudaSuccess) return TTC_ERR_CUDA;
  if (cudaMemcpyFromSymbol(counts, ttc::g_trace_n, sizeof(ttc::g_trace_n)) != cudaSuccess) return TTC_ERR_CUDA;
  static int zero[TTC_TRACE_SLOTS];
  if (cudaMemcpyToSymbol(ttc::g_trace_n, zero, sizeof(zero)) != cudaSuccess) return TTC_ERR_CUDA;
  return TTC_OK;
}
#endif

// diagnostics: q_pre[i] = div_pre_fast (when its test passes) else div_pre, both with
// rcp_refined(b[i]); q_ieee[i] = __ddiv_rn(a[i], b[i])
namespace ttc {
__global__ void k_selftest_division(const double* a, const double* b, double* qp, double* qi, long long n) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    const double r2 = rcp_refined(b[i]);
    bool ok;
    const double q = div_pre_fast(a[i], b[i], r2, ok);   // (the extension's branch-free path)
    qp[i] = ok ? q : div_pre(a[i], b[i], r2);
    qi[i] = __ddiv_rn(a[i], b[i]);
  }
}
}  // namespace ttc

int tt_selftest_division(const double* a, const double* b, double* q_pre, double* q_ieee, int64_t n) {
  if (n < 0 || (n > 0 && (!a || !b || !q_pre || !q_ieee))) return fail(TTC_ERR_ARG, "tt_selftest_division: bad arguments");
  if (n == 0) return TTC_OK;
  ttc::k_selftest_division<<<(unsigned)std::min<long long>(4096, (n + 255) / 256), 256>>>(a, b, q_pre, q_ieee, n);
  if (int e = check_launch("k_selftest_division")) return e;
  if (cudaDeviceSynchronize() != cudaSuccess) return fail(TTC_ERR_CUDA, "tt_selftest_division: sync");
  return TTC_OK;
}

const char* tt_build_info(void) {
  return "libttcross 0.2 (sm_100a, fp64, -fmad=false, dimension-parallel greedy cross, cluster rook search)";
}

int tt_cross_init(ttc_ctx** out, const ttc_config* cfg, const double* nodes_u, const double* weights,
                  int32_t mem_kind, void* stream) {
  if (!out || !cfg || !nodes_u || !weights) return fail(TTC_ERR_ARG, "null argument");
  *out = nullptr;
  const ttc_config& k = *cfg;
  if (k.family < TTC_FAMILY_C || k.family > TTC_FAMILY_EX)
    return fail(TTC_ERR_ARG, "family must be 0 (C), 1 (D), 2 (Cx), 3 (Dx) or 4 (Ex)");
  if (k.d < 2 || k.d > 2000) return fail(TTC_ERR_ARG, "d must be in [2, 2000]");
  if (k.n < 2 || k.n > 4096) return fail(TTC_ERR_ARG, "n must be in [2, 4096]");
  if (k.rank_cap < 1 || k.rank_cap > TTC_MAX_RANK) return fail(TTC_ERR_ARG, "rank_cap must be in [1, 64]");
  if (k.n_samples < 1 || k.n_samples > TTC_MAX_SAMPLES) return fail(TTC_ERR_ARG, "n_samples must be in [1, 1024]");
  if (k.rook_iters < 0 || k.rook_iters > 64) return fail(TTC_ERR_ARG, "rook_iters must be in [0, 64]");
  if (!(k.tol >= 0.0 && k.tol < 1.0)) return fail(TTC_ERR_ARG, "tol must be in [0, 1)");
  if (k.world < 1 || k.rank < 0 || k.rank >= k.world) return fail(TTC_ERR_ARG, "need 0 <= rank < world");
  if (k.fold_weights != 0 && k.fold_weights != 1) return fail(TTC_ERR_ARG, "fold_weights must be 0 or 1");
  if (k.fold_weights && k.family < TTC_FAMILY_CX)
    return fail(TTC_ERR_ARG, "weight folding is supported for the x-form families (uniform trapezoid weights)");
  if (mem_kind != TTC_MEM_HOST && mem_kind != TTC_MEM_DEVICE) return fail(TTC_ERR_ARG, "mem_kind");
  if (mem_kind == TTC_MEM_HOST) {
    for (long long t = 0; t < (long long)k.d * k.n; ++t)
      if (!(nodes_u[t] > 0.0) || !std::isfinite(nodes_u[t])) return fail(TTC_ERR_ARG, "u-nodes must be finite and > 0");
  }

  ttc_ctx* c = new ttc_ctx();
  c->cfg = k;
  c->stream = static_cast<cudaStream_t>(stream);
  c->ls = c->stream;
  const int d = k.d, n = k.n, cap = k.rank_cap;
  DevCtx& dc = c->dc;
  dc.family = k.family;
  dc.d = d;
  dc.n = n;
  dc.cap = cap;
  dc.ns = k.n_samples;
  dc.rook = k.rook_iters;
  dc.tol = k.tol;
  dc.seed = k.seed;
  dc.world = k.world;
  dc.rank = k.rank;
  // balanced partition (part_begin): D_20 on 8 ranks owns 3,3,3,2,2,2,2,2 superblocks
  c->chunk = (d - 1 + k.world - 1) / k.world;   // the largest share: exchange slot size
  dc.chunk = c->chunk;
  c->kb = part_begin(d - 1, k.world, k.rank);
  c->ke = part_begin(d - 1, k.world, k.rank + 1);
  c->n_owned = c->ke - c->kb;
  dc.kb = c->kb;
  dc.ke = c->ke;
  dc.RS = 1 + cap * d + 2 * cap;
  // row / column capacity of a superblock, padded to an even count: the u/v factor rows
  // (stride sbn doubles) then start 16-byte aligned, as the TMA tensor maps need
  dc.sbn = ((long long)cap * n + 1) & ~1LL;
  dc.G = 1;  // cluster size of k_sweep, chosen below once the device is known
  c->slots = d;
  c->nrec = d - 1;   // record i = interface i
  c->rec_ints = (long long)c->nrec * dc.RS;
  dc.fib_stride = (long long)cap * cap * n;
  const int nj = std::max(1, c->n_owned);

  auto bail = [&](int e) {
    tt_cross_destroy(c);
    return e;
  };
  int e = 0;
  double *u = nullptr, *w = nullptr, *wf = nullptr;
  long long *chi = nullptr, *clo = nullptr;
  if ((e = dalloc(c, &u, (size_t)d * n)) || (e = dalloc(c, &w, (size_t)d * n)) ||
      (k.fold_weights && (e = dalloc(c, &wf, (size_t)d * n))) ||
      (e = dalloc(c, &chi, (size_t)d * n)) || (e = dalloc(c, &clo, (size_t)d * n)))
    return bail(e);
  dc.u = u;
  dc.w = w;
  dc.wf = wf;
  dc.chi = chi;
  dc.clo = clo;
  const size_t tab = (size_t)nj * cap * n;
  if ((e = dalloc(c, &dc.rec_cur, (size_t)c->rec_ints)) || (e = dalloc(c, &dc.rec_next, (size_t)c->rec_ints)) ||
      (e = dalloc(c, &c->t0buf, (size_t)d)) ||
      (k.world > 1 && (e = dalloc(c, &c->xbuf, (size_t)k.world * c->chunk * dc.RS))) ||
      (e = dalloc(c, &dc.SA, tab)) || (e = dalloc(c, &dc.SB, tab)) ||
      (e = dalloc(c, &dc.U, (size_t)nj * cap * dc.sbn)) || (e = dalloc(c, &dc.V, (size_t)nj * cap * dc.sbn)) ||
      (e = dalloc(c, &dc.Araw, (size_t)nj * dc.sbn)) || (e = dalloc(c, &dc.praw_max, (size_t)nj)) ||
      (e = dalloc(c, &dc.p0val, 1)) ||
      (e = dalloc(c, &dc.sbstate, (size_t)nj * 4)) ||
      (e = dalloc(c, &dc.fib, (size_t)c->slots * dc.fib_stride)) ||
      (e = dalloc(c, &dc.sl, (size_t)c->slots * cap)) || (e = dalloc(c, &dc.sr, (size_t)c->slots * cap)) ||
      (e = dalloc(c, &dc.pll, (size_t)c->slots * cap)) || (e = dalloc(c, &dc.prr, (size_t)c->slots * cap)) ||
      (e = dalloc(c, &dc.pf, (size_t)c->slots * cap * cap)) ||
      (e = dalloc(c, &dc.W, (size_t)d * cap * cap)) || (e = dalloc(c, &dc.M, (size_t)d * cap * cap)) ||
      (e = dalloc(c, &dc.wpart, (size_t)d * cap * cap * FW_NSMAX)) ||
      (e = dalloc(c, &dc.wcnt, (size_t)d * ((cap + FW_TA - 1) / FW_TA) * ((cap + FW_TB - 1) / FW_TB))) ||
      (e = dalloc(c, &dc.H, (size_t)d * cap * cap)) || (e = dalloc(c, &dc.flags, 4)) ||
      (e = dalloc(c, &dc.rank_ring, (size_t)2 * d)) || (e = dalloc(c, &dc.done, (size_t)d)) ||
      (e = dalloc(c, &dc.counters, TTC_NCOUNTERS)) || (e = dalloc(c, &c->phase_buf, TTC_PHASE_WORDS)) ||
      (e = dalloc(c, &c->partials, (size_t)k.world * chain_record_size(cap))) || (e = dalloc(c, &c->out_dev, 4)) ||
      (e = dalloc(c, &c->chainA, (size_t)(nj + 1) * cap * cap)) || (e = dalloc(c, &c->chainB, (size_t)(nj + 1) * cap * cap)) ||
      (e = dalloc(c, &c->chainAd, (size_t)(nj + 1) * 3)) || (e = dalloc(c, &c->chainBd, (size_t)(nj + 1) * 3)))
    return bail(e);
  dc.rdone = dc.done;        // (a remote neighbour's flag and rank land in this rank's own copies)
  dc.rring = dc.rank_ring;
  if (cudaMemset(dc.wcnt, 0, sizeof(int) * d * ((cap + FW_TA - 1) / FW_TA) * ((cap + FW_TB - 1) / FW_TB)) != cudaSuccess)
    return bail(fail(TTC_ERR_CUDA, "cudaMemset(wcnt) failed"));
  if (k.family == TTC_FAMILY_D) {
    if ((e = dalloc(c, &dc.ql, (size_t)c->slots * cap * n)) || (e = dalloc(c, &dc.qr, (size_t)c->slots * cap * n)) ||
        (e = dalloc(c, &dc.PA, tab)) || (e = dalloc(c, &dc.PB, tab)) || (e = dalloc(c, &dc.QL1, tab)) ||
        (e = dalloc(c, &dc.QR0, tab)) || (e = dalloc(c, &dc.CX, (size_t)nj * cap * cap)))
      return bail(e);
  }
  {
    cudaError_t ce = cudaMallocHost(&c->out_host, 8 * sizeof(double));
    if (ce != cudaSuccess) return bail(fail(TTC_ERR_CUDA, std::string("cudaMallocHost: ") + cudaGetErrorString(ce)));
  }
  {
    cudaError_t ce = cudaSuccess;
    int optin = 0, dev0 = 0;
    cudaGetDevice(&dev0);
    cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev0);
    // smem < 0: everything the device allows a block beside the kernel's static shared memory
    auto allow = [&](const void* f, int smem) {
      if (ce == cudaSuccess) ce = cudaFuncSetAttribute(f, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
      if (smem < 0 && ce == cudaSuccess) {
        cudaFuncAttributes fa = {};
        ce = cudaFuncGetAttributes(&fa, f);
        smem = optin - (int)fa.sharedSizeBytes;
      }
      if (ce == cudaSuccess) ce = cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    };
    allow((const void*)k_sweeps<0, false, 256>, -1);
    allow((const void*)k_sweeps<1, false, 256>, -1);
    allow((const void*)k_sweeps<0, true, 256>, -1);
    allow((const void*)k_sweeps<1, true, 256>, -1);
    allow((const void*)k_sweeps<0, false, 512>, -1);
    allow((const void*)k_sweeps<1, false, 512>, -1);
    allow((const void*)k_sweeps<0, true, 512>, -1);
    allow((const void*)k_sweeps<1, true, 512>, -1);
    for (const void* f : {(const void*)k_sweeps<0, false, 256, true>, (const void*)k_sweeps<1, false, 256, true>,
                          (const void*)k_sweeps<0, true, 256, true>, (const void*)k_sweeps<1, true, 256, true>,
                          (const void*)k_sweeps<0, false, 512, true>, (const void*)k_sweeps<1, false, 512, true>,
                          (const void*)k_sweeps<0, true, 512, true>, (const void*)k_sweeps<1, true, 512, true>})
      allow(f, -1);   // (the cross-GPU wavefront instantiations)
    for (const void* f : {(const void*)k_sweep<2, false, 256>, (const void*)k_sweep<2, false, 512>,
                          (const void*)k_sweep<3, false, 256>, (const void*)k_sweep<3, false, 512>,
                          (const void*)k_sweep<4, false, 256>, (const void*)k_sweep<4, false, 512>,
                          (const void*)k_sweeps<2, false, 256>, (const void*)k_sweeps<2, false, 512>,
                          (const void*)k_sweeps<3, false, 256>, (const void*)k_sweeps<3, false, 512>,
                          (const void*)k_sweeps<4, false, 256>, (const void*)k_sweeps<4, false, 512>})
      allow(f, -1);
    allow((const void*)k_sweep<0, false, 256>, -1);
    allow((const void*)k_sweep<1, false, 256>, -1);
    allow((const void*)k_sweep<0, true, 256>, -1);
    allow((const void*)k_sweep<1, true, 256>, -1);
    allow((const void*)k_sweep<0, false, 512>, -1);
    allow((const void*)k_sweep<1, false, 512>, -1);
    allow((const void*)k_sweep<0, true, 512>, -1);
    allow((const void*)k_sweep<1, true, 512>, -1);
    allow((const void*)k_fiber_wsum<0, false>, fw_smem_bytes());
    allow((const void*)k_fiber_wsum<1, false>, fw_smem_bytes());
    allow((const void*)k_fiber_wsum<0, true>, fw_smem_bytes());
    allow((const void*)k_fiber_wsum<1, true>, fw_smem_bytes());
    const int quad_smem = 2 * cap * cap * (int)sizeof(DD);
    if (ce == cudaSuccess) ce = cudaFuncSetAttribute(k_solve, cudaFuncAttributeMaxDynamicSharedMemorySize, quad_smem);
    if (ce != cudaSuccess) return bail(fail(TTC_ERR_CUDA, std::string("cudaFuncSetAttribute: ") + cudaGetErrorString(ce)));
  }
  {
    // k_sweep shape: G CTAs (a power of two <= 16, at least 128 superblock rows each) per
    // owned superblock, all resident at once.  512-thread CTAs (one per SM) when that gives
    // at least as many threads per superblock as 256-thread CTAs (two per SM); the CACHED
    // variant when the CTA's rows/columns fit in shared memory.
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    c->sms = sms;
    const long long by_rows = std::max<long long>(1, (dc.sbn + 127) / 128);
    auto pick_g = [&](long long slots) -> int {
      if (slots < nj) return 0;
      int G = 16;
      while (G > 1 && (G * (long long)nj > slots || G > by_rows)) G >>= 1;
      return G;
    };
    // 256-thread CTAs measured faster than 512 at equal cluster size (profiles/r01d_probe_*)
    int T = 256;
    int G = std::max(1, pick_g(2LL * sms));
    // tuning overrides (benchmarks / experiments): TTC_GREEDY_T in {256, 512}, TTC_GREEDY_G
    if (const char* e = std::getenv("TTC_GREEDY_T")) {
      const int t = std::atoi(e);
      if (t == 256 || t == 512) { T = t; G = std::max(1, pick_g(t == 512 ? sms : 2LL * sms)); }
    }
    if (const char* e = std::getenv("TTC_FW_NS")) {
      const int v = std::atoi(e);
      if (v == 1 || v == 2 || v == 4 || v == 8) c->fw_ns = v;
    }
    if (const char* e = std::getenv("TTC_PHASE_JOB")) {   // profiling: superblock of the phase clocks
      const int j = std::atoi(e);
      dc.phase_job = (j >= 0 && j < nj) ? j : 0;
    }
    if (const char* e = std::getenv("TTC_GREEDY_G")) {   // (experiments: any cluster size 1..16)
      const int g = std::atoi(e);
      if (g >= 1 && g <= 16) G = g;
    }
    auto cache_for = [&](int g) -> size_t {
      const long long rpcap = (dc.sbn + g - 1) / g;
      return (size_t)greedy_cache_doubles(rpcap, cap) * sizeof(double);
    };
    const size_t ext_bytes = (size_t)extend_smem_doubles(cap) * sizeof(double);
    const size_t smem_lim = 180 * 1024;
    // after the ring / cache / extension part: the staged node factors f_node (family D, n <=
    // STAGE_N) or the Alg. 2 sample positions, whichever is larger
    const size_t fnode_bytes =
        ((std::max<size_t>(k.family == TTC_FAMILY_D && n <= STAGE_N ? (size_t)n * sizeof(DDE) : 0,
                           (size_t)2 * dc.ns * sizeof(int)) + 15) / 16) * 16;
    // (TTC_RING_KB: experiments, the ring part of a non-cached shape in KB)
    const size_t ring_env = std::getenv("TTC_RING_KB") ? (size_t)std::atoi(std::getenv("TTC_RING_KB")) * 1024 : 0;
    size_t ring = ring_env ? ring_env : (size_t)RING_P * 4 * T * sizeof(double);
    auto base_for = [&](int g, bool cached) -> size_t { return std::max(ext_bytes, cached ? cache_for(g) : ring); };
    auto smem_for = [&](int g, bool cached) -> size_t { return base_for(g, cached) + fnode_bytes; };
    // T = threads per CTA; kernels are compiled for 256 (two CTAs per SM) and 512 (one)
    auto fn_for = [&](bool cached) -> const void* {
      const bool big = T > 256;
      switch (k.family) {
        case TTC_FAMILY_C:
          return big ? (cached ? (const void*)k_sweep<0, true, 512> : (const void*)k_sweep<0, false, 512>)
                     : (cached ? (const void*)k_sweep<0, true, 256> : (const void*)k_sweep<0, false, 256>);
        case TTC_FAMILY_D:
          return big ? (cached ? (const void*)k_sweep<1, true, 512> : (const void*)k_sweep<1, false, 512>)
                     : (cached ? (const void*)k_sweep<1, true, 256> : (const void*)k_sweep<1, false, 256>);
        case TTC_FAMILY_CX: return big ? (const void*)k_sweep<2, false, 512> : (const void*)k_sweep<2, false, 256>;
        case TTC_FAMILY_DX: return big ? (const void*)k_sweep<3, false, 512> : (const void*)k_sweep<3, false, 256>;
        default: return big ? (const void*)k_sweep<4, false, 512> : (const void*)k_sweep<4, false, 256>;
      }
    };
    auto sweeps_for = [&](bool cached) -> const void* {
      const bool big = T > 256;
      switch (k.family) {
        case TTC_FAMILY_C:
          return big ? (cached ? (const void*)k_sweeps<0, true, 512> : (const void*)k_sweeps<0, false, 512>)
                     : (cached ? (const void*)k_sweeps<0, true, 256> : (const void*)k_sweeps<0, false, 256>);
        case TTC_FAMILY_D:
          return big ? (cached ? (const void*)k_sweeps<1, true, 512> : (const void*)k_sweeps<1, false, 512>)
                     : (cached ? (const void*)k_sweeps<1, true, 256> : (const void*)k_sweeps<1, false, 256>);
        case TTC_FAMILY_CX: return big ? (const void*)k_sweeps<2, false, 512> : (const void*)k_sweeps<2, false, 256>;
        case TTC_FAMILY_DX: return big ? (const void*)k_sweeps<3, false, 512> : (const void*)k_sweeps<3, false, 256>;
        default: return big ? (const void*)k_sweeps<4, false, 512> : (const void*)k_sweeps<4, false, 256>;
      }
    };
    auto sweeps_peer_for = [&](bool cached) -> const void* {
      const bool big = T > 256;
      switch (k.family) {
        case TTC_FAMILY_C:
          return big ? (cached ? (const void*)k_sweeps<0, true, 512, true> : (const void*)k_sweeps<0, false, 512, true>)
                     : (cached ? (const void*)k_sweeps<0, true, 256, true> : (const void*)k_sweeps<0, false, 256, true>);
        case TTC_FAMILY_D:
          return big ? (cached ? (const void*)k_sweeps<1, true, 512, true> : (const void*)k_sweeps<1, false, 512, true>)
                     : (cached ? (const void*)k_sweeps<1, true, 256, true> : (const void*)k_sweeps<1, false, 256, true>);
        default: return nullptr;   // (x-form families: the per-sweep exchange only)
      }
    };
    // resident clusters for (G, cached)
    auto resident_of = [&](const void* fn, int g, bool cached) -> int {
      cudaLaunchConfig_t lc = {};
      lc.gridDim = dim3(g);
      lc.blockDim = dim3(T);
      lc.dynamicSmemBytes = smem_for(g, cached);
      cudaLaunchAttribute at[1];
      at[0].id = cudaLaunchAttributeClusterDimension;
      at[0].val.clusterDim.x = g;
      at[0].val.clusterDim.y = 1;
      at[0].val.clusterDim.z = 1;
      lc.attrs = at;
      lc.numAttrs = 1;
      int nclus = 0;
      if (cudaOccupancyMaxActiveClusters(&nclus, fn, &lc) != cudaSuccess) {
        cudaGetLastError();
        return 0;
      }
      return nclus;
    };
    auto resident = [&](int g, bool cached) -> int { return resident_of(fn_for(cached), g, cached); };
    // prefer: all nj clusters resident; cached rows when they fit; then the largest G
    bool cached = false;
    for (;; G >>= 1) {
      const bool can_cache = cache_for(G) <= smem_lim && k.family < TTC_FAMILY_CX;
      if (can_cache && resident(G, true) >= std::min(nj, 1 << 30)) { cached = true; break; }
      if (resident(G, false) >= nj) { cached = false; break; }
      if (G == 1) { cached = false; break; }
    }
    dc.G = G;
    // the block size covers a CTA's rows/columns at full rank in one pass when that takes at
    // most 512 threads (the 512-thread variant is launched with fewer threads then)
    {
      const long long per = (dc.sbn + G - 1) / G;
      const int want = (int)std::min<long long>(512, ((per + 31) / 32) * 32);
      if (!std::getenv("TTC_GREEDY_T") && want > T) {
        const int Tsave = T;
        T = want;
        if (resident(G, cached) < nj) T = Tsave;
      }
    }
    // Streaming shapes (the rook steps read U / V from HBM through the TMA ring): a step of a
    // CTA is bound by the bytes its ring keeps in flight (~ the ring: 64 KB at ~1.8 us per
    // round trip = 36 GB/s per CTA, D_20), so the shape maximises the ring capacity of all
    // resident CTAs -- (threads, CTAs per SM, cluster size) with every cluster resident and
    // each CTA's ring as large as the SM's shared memory allows (whole 16-term stages per
    // warp).  D_20: 19 clusters of 6 x 512 threads (one CTA per SM, 192 KB rings) instead of
    // 8 x 256 (two per SM, 64 KB): 18.5 -> ~15 ms (profiles/r02c_*).
    const bool shape_env = std::getenv("TTC_GREEDY_T") || std::getenv("TTC_GREEDY_G");
    if (!cached && TTC_TMA && !shape_env) {
      int smem_sm = 0, optin = 0;
      const long long ring_sm = std::getenv("TTC_RING_SM_KB") ? std::atoll(std::getenv("TTC_RING_SM_KB")) * 1024 : 128 * 1024;
      cudaDeviceGetAttribute(&smem_sm, cudaDevAttrMaxSharedMemoryPerMultiprocessor, dev);
      cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
      double best = -1.0;
      int bT = T, bG = G;
      const size_t ring0 = ring;
      size_t bring = ring;
      const int Tsave = T;
      for (int t : {512, 256})
        for (int cps : {1, 2}) {
          if (t * cps > 512) continue;
          T = t;
          cudaFuncAttributes fa = {};
          if (cudaFuncGetAttributes(&fa, sweeps_for(false)) != cudaSuccess) { cudaGetLastError(); continue; }
          const long long avail = std::min<long long>(smem_sm / cps - 1024, optin) - (long long)fa.sharedSizeBytes -
                                  (long long)fnode_bytes;
          const long long unit = (long long)t * 16 * (long long)sizeof(double);   // a 16-term stage per warp
          // (at most ring_sm per SM: the rest of the 256 KB L1 / shared memory stays L1 for the
          // tables and factor rows the steps read through it -- 192 KB rings measured slower)
          const long long cap_b = std::min<long long>(avail, ring_sm / cps);
          const size_t rg = ring_env ? ring_env : (size_t)std::max(0LL, cap_b / unit * unit);
          if (rg < (size_t)2 * unit || rg < ext_bytes || (long long)rg > avail) continue;
          ring = rg;
          for (int g = std::min<long long>(16, by_rows); g >= 1; --g) {
            if (resident(g, false) < nj || resident_of(sweeps_for(false), g, false) < nj) continue;
            const double score = (double)nj * g * rg + 1e-3 * (double)nj * g * t;   // ring, then threads
            if (score > best) { best = score; bT = t; bG = g; bring = rg; }
            break;   // (the largest resident g for this (t, cps))
          }
        }
      T = Tsave;
      ring = ring0;
      if (best > 0) { T = bT; G = bG; ring = bring; dc.G = G; }
    }
    c->greedy_threads = T;
    c->greedy_cached = cached;
    c->greedy_smem = smem_for(G, cached);
    dc.fnode_off = (int)(base_for(G, cached) / sizeof(double));
    const size_t ring_part = base_for(G, cached);
    dc.ring_tb = (int)std::min<size_t>(8, ring_part / (sizeof(double) * RING_P * T));
    // TMA ring: 16 terms per stage when two stages per warp fit (D_20: 20.8 ms vs 24.0 with 8
    // terms x 4 stages, C_200 5.39 vs 6.01; profiles/r02_ring_shape.log)
    if (TTC_TMA && !cached && ring_part >= 2 * 16 * (size_t)T * sizeof(double)) dc.ring_tb = 16;
    if (const char* e = std::getenv("TTC_RING_TB")) {   // (experiments: terms per ring stage)
      const int v = std::atoi(e);
      if (v >= 1 && v <= 64 && (size_t)v * 2 * T * sizeof(double) <= ring_part) dc.ring_tb = v;
    }
    // TMA ring (non-cached shape): stages of T rows x ring_tb terms in the ring part of the
    // dynamic shared memory, as many as fit (<= TMA_PMAX)
    dc.ring_tb = std::max(1, dc.ring_tb);   // (cached shapes: the ring is not used)
    dc.ring_p = (int)std::min<size_t>(std::min(TMA_PMAX, TMA_NBAR / std::max(1, T / 32)),
                                      ring_part / (sizeof(double) * (size_t)T * dc.ring_tb));
    dc.tma = TTC_TMA && !cached && dc.ring_p >= 2 && dc.ring_tb == 16;
    if (dc.tma) dc.ring_p = 2;   // (TmaRing: two 16-term stages per warp, compile-time)
    // rows per thread from which a step streams through the ring (the DotRing needs a few rows
    // per thread to fill its stages; the TMA ring streams any row count)
    dc.ring_min = dc.tma ? 1 : RING_MIN_ROWS;
    dc.l2_keep = 0.f;
    if (const char* e = std::getenv("TTC_L2_KEEP")) {   // (experiments)
      const float v = (float)std::atof(e);
      if (v >= 0.f && v <= 1.f) dc.l2_keep = v;
    }
    if (const char* e = std::getenv("TTC_RING_MIN")) {   // (experiments)
      const int v = std::atoi(e);
      if (v >= 1 && v <= 64) dc.ring_min = v;
    }
    dc.ext_tile = extend_tile_rows(cap);
    c->greedy_fn = fn_for(c->greedy_cached);
    {
      c->sweeps_fn = sweeps_for(cached);
      // the wavefront needs every cluster resident at once
      // (queried for the persistent kernel itself: its register / shared-memory footprint
      // differs from the single-sweep kernel's)
      c->resident_all = resident_of(c->sweeps_fn, G, cached) >= nj && resident(G, cached) >= nj &&
                        !std::getenv("TTC_NO_PERSISTENT");
      c->persistent = k.world == 1 && c->resident_all;
      c->sweeps_peer_fn = sweeps_peer_for(cached);
      c->peer_resident = c->sweeps_peer_fn && resident_of(c->sweeps_peer_fn, G, cached) >= nj && c->resident_all;
    }
  }
  if (dc.tma) {
    // 2-D tensor maps of U and V: dims {sbn (x, fastest), jobs * cap (t of job j at j*cap + t)},
    // boxes of {32, ring_tb} doubles: a warp's rows (see TmaRing)
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess || !fn)
      return bail(fail(TTC_ERR_CUDA, "cuTensorMapEncodeTiled: driver entry point not found"));
    auto encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
    CUtensorMap maps[2];
    const cuuint32_t bw = 32;   // a warp's rows (TmaRing: one ring per warp)
    const cuuint64_t dims[2] = {(cuuint64_t)dc.sbn, (cuuint64_t)nj * cap};
    const cuuint64_t strides[1] = {(cuuint64_t)dc.sbn * sizeof(double)};
    const cuuint32_t box[2] = {bw, (cuuint32_t)dc.ring_tb};
    const cuuint32_t estr[2] = {1, 1};
    double* bases[2] = {dc.U, dc.V};
    for (int i = 0; i < 2; ++i) {
      const CUresult cr = encode(&maps[i], CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, bases[i], dims, strides, box, estr,
                                 CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                                 CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
      if (cr != CUDA_SUCCESS)
        return bail(fail(TTC_ERR_CUDA, "cuTensorMapEncodeTiled failed (code " + std::to_string((int)cr) + ")"));
    }
    unsigned char* dmaps = nullptr;
    if ((e = dalloc(c, &dmaps, sizeof(maps)))) return bail(e);
    if (cudaMemcpy(dmaps, maps, sizeof(maps), cudaMemcpyHostToDevice) != cudaSuccess)
      return bail(fail(TTC_ERR_CUDA, "tensor map upload failed"));
    dc.tmapU = dmaps;
    dc.tmapV = dmaps + sizeof(CUtensorMap);
  }
  int rc = tt_cross_load_grid(c, nodes_u, weights, mem_kind);
  if (rc) return bail(rc);
  *out = c;
  return TTC_OK;
}

int tt_cross_load_grid(ttc_ctx* c, const double* nodes_u, const double* weights, int32_t mem_kind) {
  if (!c || !nodes_u || !weights) return fail(TTC_ERR_ARG, "null argument");
  if (mem_kind != TTC_MEM_HOST && mem_kind != TTC_MEM_DEVICE) return fail(TTC_ERR_ARG, "mem_kind");
  const int d = c->dc.d, n = c->dc.n;
  if (mem_kind == TTC_MEM_HOST)
    for (long long t = 0; t < (long long)d * n; ++t)
      if (!(nodes_u[t] > 0.0) || !std::isfinite(nodes_u[t])) return fail(TTC_ERR_ARG, "u-nodes must be finite and > 0");
  if (c->pending) return fail(TTC_ERR_STATE, "uncommitted local sweep");
  const cudaMemcpyKind kind = mem_kind == TTC_MEM_HOST ? cudaMemcpyHostToDevice : cudaMemcpyDeviceToDevice;
  CK(cudaMemcpyAsync(const_cast<double*>(c->dc.u), nodes_u, sizeof(double) * d * n, kind, c->stream));
  if (c->dc.wf) {  // folded: the entries carry the weights, the contraction sums with ones
    CK(cudaMemcpyAsync(const_cast<double*>(c->dc.wf), weights, sizeof(double) * d * n, kind, c->stream));
    k_fill<<<(d * n + 255) / 256, 256, 0, c->stream>>>(const_cast<double*>(c->dc.w), 1.0, (long long)d * n);
    if (int e = check_launch("k_fill")) return e;
  } else {
    CK(cudaMemcpyAsync(const_cast<double*>(c->dc.w), weights, sizeof(double) * d * n, kind, c->stream));
  }
  {
    Timed t(c, K_PREP);
    k_prep_nodes<<<(d * n + 255) / 256, 256, 0, c->stream>>>(c->dc.u, const_cast<long long*>(c->dc.chi),
                                                             const_cast<long long*>(c->dc.clo), d * n);
  }
  if (int e = check_launch("k_prep_nodes")) return e;
  return tt_cross_reset(c);
}

int tt_cross_reset(ttc_ctx* c) {
  if (!c) return fail(TTC_ERR_ARG, "null context");
  return do_reset(c);
}

int tt_cross_sweep_local(ttc_ctx* c) {
  if (!c) return fail(TTC_ERR_ARG, "null context");
  if (c->pending) return fail(TTC_ERR_STATE, "previous local sweep not committed");
  return do_sweep_local(c);
}

int tt_cross_commit(ttc_ctx* c) {
  if (!c) return fail(TTC_ERR_ARG, "null context");
  return do_commit(c);
}

int tt_cross_sweep(ttc_ctx* c, int32_t n_sweeps) {
  if (!c) return fail(TTC_ERR_ARG, "null context");
  if (c->cfg.world != 1) return fail(TTC_ERR_STATE, "tt_cross_sweep needs world == 1");
  if (n_sweeps < 0) return fail(TTC_ERR_ARG, "n_sweeps < 0");
  if (c->pending) return fail(TTC_ERR_STATE, "uncommitted local sweep");
  if (c->persistent) return do_sweeps_persistent(c, n_sweeps);
  for (int s = 0; s < n_sweeps; ++s) {
    if (int e = do_sweep_local(c)) return e;
    if (int e = do_commit(c)) return e;
  }
  return TTC_OK;
}

int tt_cross_exchange_buffer(ttc_ctx* c, void** dev_ptr, int64_t* bytes_total, int64_t* bytes_per_rank) {
  if (!c) return fail(TTC_ERR_ARG, "null context");
  if (c->cfg.world == 1) {
    if (dev_ptr) *dev_ptr = c->dc.rec_next;
    if (bytes_total) *bytes_total = c->rec_ints * (int64_t)sizeof(int32_t);
    if (bytes_per_rank) *bytes_per_rank = c->rec_ints * (int64_t)sizeof(int32_t);
    return TTC_OK;
  }
  if (dev_ptr) *dev_ptr = c->xbuf;
  if (bytes_total) *bytes_total = (int64_t)c->cfg.world * c->chunk * c->dc.RS * (int64_t)sizeof(int32_t);
  if (bytes_per_rank) *bytes_per_rank = (int64_t)c->chunk * c->dc.RS * (int64_t)sizeof(int32_t);
  return TTC_OK;
}

int tt_solve_launch(ttc_ctx* c, int32_t n_sweeps, int32_t use_graph) {
  if (!c) return fail(TTC_ERR_ARG, "null context");
  if (c->cfg.world != 1) return fail(TTC_ERR_STATE, "tt_solve_launch needs world == 1");
  if (n_sweeps < 0) return fail(TTC_ERR_ARG, "n_sweeps < 0");
  if (c->pending) return fail(TTC_ERR_STATE, "uncommitted local sweep");
  if (!use_graph) {
    if (int e = do_reset(c)) return e;
    return enqueue_solve(c, n_sweeps);
  }
  if (!c->graph_exec || c->graph_sweeps != n_sweeps) {
    if (int e = capture_solve(c, n_sweeps)) return e;
  }
  if (int e = reset_host(c)) return e;
  CK(cudaGraphLaunch(c->graph_exec, c->stream));
  c->launches = c->graph_launches;
  c->sweeps = n_sweeps;
  return TTC_OK;
}

int tt_integrate(ttc_ctx* c, double* value, double* log10_abs, int32_t* sign) {
  if (!c) return fail(TTC_ERR_ARG, "null context");
  if (c->cfg.world != 1) return fail(TTC_ERR_STATE, "tt_integrate needs world == 1");
  if (c->pending) return fail(TTC_ERR_STATE, "uncommitted local sweep");
  if (int e = do_integrate_local(c)) return e;
  if (int e = do_integrate_finish_launch(c)) return e;
  return do_integrate_read(c, value, log10_abs, sign);
}

int tt_integrate_launch(ttc_ctx* c) {
  if (!c) return fail(TTC_ERR_ARG, "null context");
  if (c->cfg.world != 1) return fail(TTC_ERR_STATE, "tt_integrate_launch needs world == 1");
  if (c->pending) return fail(TTC_ERR_STATE, "uncommitted local sweep");
  if (int e = do_integrate_local(c)) return e;
  return do_integrate_finish_launch(c);
}

int tt_integrate_read(ttc_ctx* c, double* value, double* log10_abs, int32_t* sign) {
  if (!c) return fail(TTC_ERR_ARG, "null context");
  return do_integrate_read(c, value, log10_abs, sign);
}

int tt_integrate_local(ttc_ctx* c) {
  if (!c) return fail(TTC_ERR_ARG, "null context");
  if (c->pending) return fail(TTC_ERR_STATE, "uncommitted local sweep");
  return do_integrate_local(c);
}

int tt_integrate_partials_buffer(ttc_ctx* c, void** dev_ptr, int64_t* bytes_total, int64_t* bytes_per_rank) {
  if (!c) return fail(TTC_ERR_ARG, "null context");
  const int64_t rsz = chain_record_size(c->dc.cap) * (int64_t)sizeof(double);
  if (dev_ptr) *dev_ptr = c->partials;
  if (bytes_total) *bytes_total = rsz * c->cfg.world;
  if (bytes_per_rank) *bytes_per_rank = rsz;
  return TTC_OK;
}

int tt_integrate_finish(ttc_ctx* c, double* value, double* log10_abs, int32_t* sign) {
  if (!c) return fail(TTC_ERR_ARG, "null context");
  if (int e = do_integrate_finish_launch(c)) return e;
  return do_integrate_read(c, value, log10_abs, sign);
}

int tt_cross_get_state(ttc_ctx* c, int32_t* ranks_out, int32_t* piv_out, int32_t* par_out) {
  if (!c) return fail(TTC_ERR_ARG, "null context");
  const int d = c->dc.d, cap = c->dc.cap, RS = c->dc.RS;
  std::vector<int32_t> rec(c->rec_ints);
  int32_t flags[2] = {0, 0};
  CK(cudaMemcpyAsync(rec.data(), c->dc.rec_cur, sizeof(int32_t) * c->rec_ints, cudaMemcpyDeviceToHost, c->stream));
  CK(cudaMemcpyAsync(flags, c->dc.flags, sizeof(flags), cudaMemcpyDeviceToHost, c->stream));
  CK(cudaStreamSynchronize(c->stream));
  if (flags[1]) return fail(TTC_ERR_CUDA, kWaveTimeout);
  for (int i = 0; i < d - 1; ++i) {
    const int32_t* R = rec.data() + (long long)i * RS;
    if (ranks_out) ranks_out[i] = R[0];
    if (piv_out)
      for (long long t = 0; t < (long long)cap * d; ++t)
        piv_out[(long long)i * cap * d + t] = (t / d) < R[0] ? R[1 + t] : -1;
    if (par_out)
      for (long long t = 0; t < 2LL * cap; ++t)
        par_out[(long long)i * cap * 2 + t] = (t / 2) < R[0] ? R[1 + (long long)cap * d + t] : -1;
  }
  return TTC_OK;
}

int tt_cross_get_fiber(ttc_ctx* c, int32_t mode, double* out, int64_t capacity, int32_t* rx, int32_t* ry) {
  if (!c) return fail(TTC_ERR_ARG, "null context");
  const int d = c->dc.d, n = c->dc.n, RS = c->dc.RS;
  if (mode < 0 || mode >= d) return fail(TTC_ERR_ARG, "mode out of range");
  int32_t a = 1, b = 1;
  if (mode > 0) CK(cudaMemcpyAsync(&a, c->dc.rec_cur + (long long)(mode - 1) * RS, sizeof(int32_t), cudaMemcpyDeviceToHost, c->stream));
  if (mode < d - 1) CK(cudaMemcpyAsync(&b, c->dc.rec_cur + (long long)mode * RS, sizeof(int32_t), cudaMemcpyDeviceToHost, c->stream));
  CK(cudaStreamSynchronize(c->stream));
  if (rx) *rx = a;
  if (ry) *ry = b;
  const long long cnt = (long long)a * b * n;
  if (out) {
    if (capacity < cnt) return fail(TTC_ERR_ARG, "fiber buffer too small");
    if (c->pending) return fail(TTC_ERR_STATE, "uncommitted local sweep");
    // evaluated on demand from the current index sets (the quadrature pass contracts the
    // t-form fibers without storing them)
    if (int e = launch_fibers(c, JOB_INT, mode, 1, true, false)) return e;
    if (c->dc.family >= TTC_FAMILY_CX) {   // (x-form: W from the stored entries, as tt_integrate)
      Timed t(c, K_WSUM);
      k_wsum<<<dim3((c->dc.cap + 7) / 8, c->dc.cap, 1), 256, 0, c->ls>>>(c->dc, mode);
    }
    if (int e = check_launch("k_wsum")) return e;
    CK(cudaMemcpyAsync(out, c->dc.fib + (long long)mode * c->dc.fib_stride, sizeof(double) * cnt, cudaMemcpyDeviceToHost, c->stream));
    CK(cudaStreamSynchronize(c->stream));
  }
  return TTC_OK;
}

int tt_cross_get_wsum(ttc_ctx* c, int32_t mode, double* hi_out, double* lo_out, int64_t capacity, int32_t* rx,
                      int32_t* ry) {
  if (!c) return fail(TTC_ERR_ARG, "null context");
  const int d = c->dc.d, cap = c->dc.cap, RS = c->dc.RS;
  if (mode < 0 || mode >= d) return fail(TTC_ERR_ARG, "mode out of range");
  if (c->pending) return fail(TTC_ERR_STATE, "uncommitted local sweep");
  int32_t a = 1, b = 1;
  if (mode > 0) CK(cudaMemcpyAsync(&a, c->dc.rec_cur + (long long)(mode - 1) * RS, sizeof(int32_t), cudaMemcpyDeviceToHost, c->stream));
  if (mode < d - 1) CK(cudaMemcpyAsync(&b, c->dc.rec_cur + (long long)mode * RS, sizeof(int32_t), cudaMemcpyDeviceToHost, c->stream));
  CK(cudaStreamSynchronize(c->stream));
  if (rx) *rx = a;
  if (ry) *ry = b;
  if (!hi_out) return TTC_OK;
  if (!lo_out) return fail(TTC_ERR_ARG, "lo_out is NULL");
  if (capacity < (int64_t)a * b) return fail(TTC_ERR_ARG, "wsum buffer too small");
  std::vector<DD> W((size_t)cap * cap);
  CK(cudaMemcpyAsync(W.data(), c->dc.W + (long long)mode * cap * cap, sizeof(DD) * cap * cap, cudaMemcpyDeviceToHost,
                     c->stream));
  CK(cudaStreamSynchronize(c->stream));
  for (int i = 0; i < a; ++i)
    for (int j = 0; j < b; ++j) {
      hi_out[(long long)i * b + j] = W[(size_t)i * cap + j].hi;
      lo_out[(long long)i * b + j] = W[(size_t)i * cap + j].lo;
    }
  return TTC_OK;
}

int tt_cross_get_stats(ttc_ctx* c, ttc_stats* out) {
  if (!c || !out) return fail(TTC_ERR_ARG, "null argument");
  unsigned long long cnt[TTC_NCOUNTERS] = {};
  int32_t flags[2] = {0, 0};
  CK(cudaMemcpyAsync(cnt, c->dc.counters, sizeof(cnt), cudaMemcpyDeviceToHost, c->stream));
  CK(cudaMemcpyAsync(flags, c->dc.flags, sizeof(flags), cudaMemcpyDeviceToHost, c->stream));
  CK(cudaStreamSynchronize(c->stream));
  if (flags[1]) return fail(TTC_ERR_CUDA, kWaveTimeout);
  if (int e = resolve_timing(c)) return e;
  std::memset(out, 0, sizeof(*out));
  out->evals = (int64_t)cnt[CNT_EVALS];
  out->launches = c->launches;
  out->sweeps = c->sweeps;
  out->ms_fiber = c->ms[KC_FIBER];
  out->ms_cross = c->ms[KC_CROSS];
  out->ms_quad = c->ms[KC_QUAD];
  out->ms_other = c->ms[KC_OTHER];
  out->fiber_entries = (int64_t)cnt[CNT_FIBER_ENTRIES];
  out->sb_entries = (int64_t)cnt[CNT_SB_ENTRIES];
  out->sb_updates = (int64_t)cnt[CNT_SB_UPDATES];
  out->rook_steps = (int64_t)cnt[CNT_ROOK_STEPS];
  out->ext_entries = (int64_t)cnt[CNT_EXT_ENTRIES];
  out->ext_updates = (int64_t)cnt[CNT_EXT_UPDATES];
  out->ring_steps = (int64_t)cnt[CNT_RING_STEPS];
  return TTC_OK;
}

int tt_cross_get_kernel_time(ttc_ctx* c, int32_t kid, const char** name, int64_t* launches, double* ms) {
  if (!c) return fail(TTC_ERR_ARG, "null context");
  if (kid < 0 || kid >= K_COUNT) return fail(TTC_ERR_ARG, "kernel id out of range");
  if (int e = resolve_timing(c)) return e;
  if (name) *name = kKernelName[kid];
  if (launches) *launches = c->klaunch[kid];
  if (ms) *ms = c->kms[kid];
  return TTC_OK;
}

int tt_cross_get_launch_shape(ttc_ctx* c, int32_t* cluster, int32_t* threads, int32_t* cached,
                              int64_t* smem_bytes) {
  if (!c) return fail(TTC_ERR_ARG, "null context");
  if (cluster) *cluster = c->dc.G;
  if (threads) *threads = c->greedy_threads;
  if (cached) *cached = (c->greedy_cached ? 1 : 0) | (c->persistent ? 2 : 0) | (c->peer_resident ? 4 : 0);
  if (smem_bytes) *smem_bytes = (int64_t)c->greedy_smem;
  return TTC_OK;
}

int tt_cross_set_timing(ttc_ctx* c, int32_t enable) {
  if (!c) return fail(TTC_ERR_ARG, "null context");
  c->timing = enable != 0;
  c->dc.phase_ns = c->timing ? c->phase_buf : nullptr;
  if (c->timing) CK(cudaMemsetAsync(c->phase_buf, 0, TTC_PHASE_WORDS * sizeof(unsigned long long), c->stream));
  return TTC_OK;
}

int tt_cross_get_phase_times(ttc_ctx* c, double* us_out, int32_t count) {
  if (!c || !us_out) return fail(TTC_ERR_ARG, "null argument");
  if (count < 12) return fail(TTC_ERR_ARG, "need 12 slots");
  if (!TTC_PHASE_CLOCKS)
    return fail(TTC_ERR_STATE, "library built without the phase clocks (TTC_PHASE_CLOCKS=0): "
                               "tools/probe_phases.py uses build/libttcross_clocks.so");
  std::vector<unsigned long long> v(TTC_PHASE_WORDS);
  CK(cudaMemcpyAsync(v.data(), c->phase_buf, sizeof(unsigned long long) * TTC_PHASE_WORDS, cudaMemcpyDeviceToHost,
                     c->stream));
  CK(cudaStreamSynchronize(c->stream));
  for (int i = 0; i < TTC_PHASE_WORDS && i < count; ++i) {
    const bool is_count = i == PH_LAUNCHES || (i >= TTC_NPHASES && (i - TTC_NPHASES) % TTC_LOG_W == PH_LAUNCHES);
    us_out[i] = is_count ? (double)v[i] : v[i] * 1e-3;
  }
  return TTC_OK;
}

void tt_cross_destroy(ttc_ctx* c) {
  if (!c) return;
  if (c->stream) cudaStreamSynchronize(c->stream);
  for (auto& r : c->evs) {
    cudaEventDestroy(r.a);
    cudaEventDestroy(r.b);
  }
  for (auto e : c->ev_pool) cudaEventDestroy(e);
  if (c->graph_exec) cudaGraphExecDestroy(c->graph_exec);
  if (c->graph) cudaGraphDestroy(c->graph);
  if (c->cap_stream) cudaStreamDestroy(c->cap_stream);
  for (int i = 0; i < 2; ++i) {
    if (c->side[i]) cudaStreamDestroy(c->side[i]);
    if (c->ev_fork[i]) cudaEventDestroy(c->ev_fork[i]);
    if (c->ev_join[i]) cudaEventDestroy(c->ev_join[i]);
  }
  for (int i = 0; i < 2; ++i)
    for (int j = 0; j < 3; ++j)
      if (c->peer_maps[i][j]) cudaIpcCloseMemHandle(c->peer_maps[i][j]);
  for (void* p : c->allocs) cudaFree(p);
  if (c->out_host) cudaFreeHost(c->out_host);
  delete c;
}

// ---------------------------------------------------------------------------------------
// cross-GPU wavefront (include/ttcross.h: tt_cross_peer_handles ... tt_cross_get_loopback)
// ---------------------------------------------------------------------------------------
static_assert(3 * sizeof(cudaIpcMemHandle_t) == TTC_PEER_HANDLE_BYTES, "TTC_PEER_HANDLE_BYTES");
int tt_cross_peer_handles(ttc_ctx* c, void* out, int64_t capacity) {
  if (!c || !out) return fail(TTC_ERR_ARG, "null argument");
  if (capacity < TTC_PEER_HANDLE_BYTES) return fail(TTC_ERR_ARG, "capacity < TTC_PEER_HANDLE_BYTES");
  if (c->cfg.world < 2) return fail(TTC_ERR_STATE, "tt_cross_peer_handles needs world > 1");
  int* bases[3] = {c->dc.rec_cur, c->dc.rank_ring, c->dc.done};
  for (int j = 0; j < 3; ++j) {
    cudaIpcMemHandle_t h;
    CK(cudaIpcGetMemHandle(&h, bases[j]));
    std::memcpy(static_cast<unsigned char*>(out) + j * sizeof(cudaIpcMemHandle_t), &h, sizeof(h));
  }
  return TTC_OK;
}

int tt_cross_peer_open(ttc_ctx* c, const void* left, const void* right) {
  if (!c) return fail(TTC_ERR_ARG, "null context");
  if (c->cfg.world < 2) return fail(TTC_ERR_STATE, "tt_cross_peer_open needs world > 1");
  if (c->dc.loopback) return fail(TTC_ERR_STATE, "loopback mode is on");
  if (!c->peer_resident)
    return fail(TTC_ERR_STATE, "no cross-GPU wavefront for this context (x-form family, or the owned superblocks' clusters "
                               "are not all resident at once)");
  if ((left != nullptr) != (c->cfg.rank > 0) || (right != nullptr) != (c->cfg.rank < c->cfg.world - 1))
    return fail(TTC_ERR_ARG, "a rank needs exactly its existing neighbours' handles (left: rank > 0, right: rank < world-1)");
  if (c->pending) return fail(TTC_ERR_STATE, "uncommitted local sweep");
  CK(cudaStreamSynchronize(c->stream));
  const void* hs[2] = {left, right};
  for (int i = 0; i < 2; ++i) {
    for (int j = 0; j < 3; ++j) {
      if (c->peer_maps[i][j]) { cudaIpcCloseMemHandle(c->peer_maps[i][j]); c->peer_maps[i][j] = nullptr; }
      if (!hs[i]) continue;
      cudaIpcMemHandle_t h;
      std::memcpy(&h, static_cast<const unsigned char*>(hs[i]) + j * sizeof(cudaIpcMemHandle_t), sizeof(h));
      void* p = nullptr;
      CK(cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess));
      c->peer_maps[i][j] = p;
    }
    c->dc.prec[i] = static_cast<int*>(c->peer_maps[i][0]);
    c->dc.pring[i] = static_cast<int*>(c->peer_maps[i][1]);
    c->dc.pdone[i] = static_cast<int*>(c->peer_maps[i][2]);
  }
  c->dc.rdone = c->dc.done;
  c->dc.rring = c->dc.rank_ring;
  c->dc.pb_lo = left ? c->kb : -1;    // this rank's first superblock: left neighbour on rank - 1
  c->dc.pb_hi = right ? c->ke : -1;   // its last (k + 1 == ke): right neighbour on rank + 1
  return TTC_OK;
}

int tt_cross_sweep_peer(ttc_ctx* c, int32_t n_sweeps) {
  if (!c) return fail(TTC_ERR_ARG, "null context");
  if (c->cfg.world < 2) return fail(TTC_ERR_STATE, "tt_cross_sweep_peer needs world > 1 (world == 1: tt_cross_sweep)");
  if (!c->dc.pdone[0] && !c->dc.pdone[1]) return fail(TTC_ERR_STATE, "tt_cross_peer_open first");
  if (n_sweeps < 1) return fail(TTC_ERR_ARG, "n_sweeps < 1");
  if (c->pending) return fail(TTC_ERR_STATE, "uncommitted local sweep");
  if (!c->peer_consistent) return fail(TTC_ERR_STATE, "tt_cross_sweep_local ran since the last reset");
  return do_sweeps_peer(c, n_sweeps);
}

int tt_cross_set_loopback(ttc_ctx* c, int32_t boundary) {
  if (!c) return fail(TTC_ERR_ARG, "null context");
  if (c->cfg.world != 1) return fail(TTC_ERR_STATE, "tt_cross_set_loopback needs world == 1");
  const int d = c->dc.d;
  if (boundary != 0 && (boundary < 1 || boundary > d - 2)) return fail(TTC_ERR_ARG, "boundary must be 0 or in [1, d-2]");
  if (boundary != 0 && !(c->persistent && c->peer_resident))
    return fail(TTC_ERR_STATE, "loopback needs the persistent sweep launch of a t-form family");
  if (c->pending) return fail(TTC_ERR_STATE, "uncommitted local sweep");
  if (boundary != 0 && !c->lb_rec) {
    if (int e = dalloc(c, &c->lb_rec, (size_t)c->rec_ints)) return e;
    if (int e = dalloc(c, &c->lb_ring, (size_t)2 * d)) return e;
    if (int e = dalloc(c, &c->lb_done, (size_t)d)) return e;
  }
  DevCtx& dc = c->dc;
  const bool on = boundary != 0;
  for (int i = 0; i < 2; ++i) {
    dc.prec[i] = on ? c->lb_rec : nullptr;
    dc.pring[i] = on ? c->lb_ring : nullptr;
    dc.pdone[i] = on ? c->lb_done : nullptr;
  }
  dc.rdone = on ? c->lb_done : dc.done;
  dc.rring = on ? c->lb_ring : dc.rank_ring;
  dc.pb_lo = on ? boundary : -1;   // superblock `boundary` sees its left neighbour as remote,
  dc.pb_hi = on ? boundary : -1;   // superblock `boundary - 1` its right neighbour
  dc.loopback = on ? 1 : 0;
  if (c->graph_exec) { cudaGraphExecDestroy(c->graph_exec); c->graph_exec = nullptr; }   // (captured kernel parameters)
  if (c->graph) { cudaGraphDestroy(c->graph); c->graph = nullptr; }
  c->graph_sweeps = -1;
  return do_reset(c);
}

int tt_cross_get_loopback(ttc_ctx* c, int32_t* rec_out, int32_t* ring_out, int32_t* done_out) {
  if (!c || !rec_out || !ring_out || !done_out) return fail(TTC_ERR_ARG, "null argument");
  if (!c->dc.loopback) return fail(TTC_ERR_STATE, "loopback mode is off");
  if (c->pending) return fail(TTC_ERR_STATE, "uncommitted local sweep");
  const int d = c->dc.d;
  CK(cudaMemcpyAsync(rec_out, c->lb_rec, sizeof(int32_t) * c->rec_ints, cudaMemcpyDeviceToHost, c->stream));
  CK(cudaMemcpyAsync(ring_out, c->lb_ring, sizeof(int32_t) * 2 * (d - 1), cudaMemcpyDeviceToHost, c->stream));
  CK(cudaMemcpyAsync(done_out, c->lb_done, sizeof(int32_t) * (d - 1), cudaMemcpyDeviceToHost, c->stream));
  int32_t flags[2] = {0, 0};
  CK(cudaMemcpyAsync(flags, c->dc.flags, sizeof(flags), cudaMemcpyDeviceToHost, c->stream));
  CK(cudaStreamSynchronize(c->stream));
  if (flags[1]) return fail(TTC_ERR_CUDA, kWaveTimeout);
  return TTC_OK;
}

}  // extern "C"
