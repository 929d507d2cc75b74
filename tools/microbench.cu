// tools/microbench.cu -- B200 latency probes that inform the k_sweep design (round 1):
//   (a) cluster barrier + DSMEM argmax round, per cluster size
//   (b) per-launch overhead of a CUDA graph of empty cluster kernels (64 CTAs)
//   (c) dependent L2 load latency (pointer chase)
//   (d) fp64 dependent-chain latencies: DADD, DMUL, IEEE division, rho, double-double x 2^e
//       product, and one whole D-family superblock entry + 16-term u.v update (the rook step's
//       per-row chain)
//   (e) st.async + mbarrier candidate exchange round (the k_sweep cluster argmax)
//   (f) warp argmax latency: REDUX (warp_argmax) vs the shuffle tree (warp_argmax_shfl)
// build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/microbench tools/microbench.cu
#include <cooperative_groups.h>
#include <climits>
#include <cstdint>
#include <cstdio>
#include <vector>
namespace cg = cooperative_groups;
#include "../paper_1903_11554_b200/csrc/ttc_common.cuh"
#include "../paper_1903_11554_b200/csrc/ttc_greedy.cuh"
using namespace ttc;

// (d) dependent chains; kind: 0 dadd, 1 dmul, 2 ddiv, 3 rho, 4 dde_mul, 5 entry + 16-term update
__global__ void k_fp64_chain(int kind, int iters, double seed, double* sink, unsigned long long* out) {
  __shared__ double vec[16], uc[16 * 32];
  __shared__ DDE fslot[4];
  for (int i = threadIdx.x; i < 16; i += blockDim.x) vec[i] = 0.5 + i * 1e-3;
  for (int i = threadIdx.x; i < 16 * 32; i += blockDim.x) uc[i] = 0.25 + i * 1e-4;
  if (threadIdx.x < 4) fslot[threadIdx.x] = {0.75 + threadIdx.x * 1e-3, 1e-18, 0, 0};
  __syncthreads();
  double x = seed + threadIdx.x * 1e-9, y = 0.999999;
  DDE p = {x, 0.0, 0, 0};
  ESum es = {12345, 678};
  unsigned long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
    if (kind == 0) x = __dadd_rn(x, y);
    else if (kind == 1) x = __dmul_rn(x, y);
    else if (kind == 2) x = __ddiv_rn(y, x);
    else if (kind == 3) x = rho(x, y) + 0.5;
    else if (kind == 4) dde_mul(p, fslot[i & 3]);
    else {
      ESum s = es;
      esum_add(s, ESum{(long long)(x * 1e3), 5});
      const double Sd = esum_round(s);
      const double SS = __dmul_rn(Sd, Sd);
      DDE q = fslot[0];
      dde_mul(q, fslot[1]);
      dde_mul(q, fslot[2]);
      dde_mul(q, fslot[3]);
      dde_mul_d(q, rho(x, y));
      double e = __ddiv_rn(dde_round(q), SS);
      for (int t = 0; t < 16; ++t) e = __dsub_rn(e, __dmul_rn(uc[t * 32 + (threadIdx.x & 31)], vec[t]));
      x = 0.5 + e * 1e-30;
    }
  }
  unsigned long long t1 = clock64();
  if (kind == 4) x = p.hi;
  sink[blockIdx.x * blockDim.x + threadIdx.x] = x;
  if (blockIdx.x == 0 && threadIdx.x == 0) *out = t1 - t0;
}

// (e) candidate exchange through st.async + mbarrier (no cluster barrier), warp 0 only
__global__ void k_xchg_rounds(int iters, unsigned long long* out) {
  cg::cluster_group cl = cg::this_cluster();
  __shared__ __align__(16) double xc[2][16][2];
  __shared__ __align__(8) unsigned long long xbar[2];
  const int G = (int)cl.num_blocks(), me = (int)cl.block_rank(), lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int q = 0; q < 2; ++q) {
      const unsigned a = (unsigned)__cvta_generic_to_shared(&xbar[q]);
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(a) : "memory");
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  cl.sync();
  unsigned long long t0 = clock64();
  double best = 0;
  for (int i = 0; i < iters; ++i) {
    if (threadIdx.x < 32) {
      const int q = i & 1;
      const unsigned bar = (unsigned)__cvta_generic_to_shared(&xbar[q]);
      if (lane == 0)
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(16 * G) : "memory");
      if (lane < G) {
        unsigned ra, rb;
        asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"((unsigned)__cvta_generic_to_shared(&xc[q][me][0])), "r"(lane));
        asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(rb) : "r"(bar), "r"(lane));
        asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v2.b64 [%0], {%1, %2}, [%3];" ::"r"(ra),
                     "l"(__double_as_longlong(best + me)), "l"((long long)i), "r"(rb) : "memory");
      }
      unsigned ok = 0;
      while (!ok)
        asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}"
                     : "=r"(ok) : "r"(bar), "r"((unsigned)(i >> 1) & 1u) : "memory");
      double v = lane < G ? xc[q][lane][0] : -1.0;
      for (int o = 16; o; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
      best = v * 1e-300;
    }
    __syncthreads();
  }
  cl.sync();
  if (blockIdx.x == 0 && threadIdx.x == 0) *out = clock64() - t0;
}

__global__ void k_cluster_rounds(int iters, unsigned long long* out) {
  cg::cluster_group cl = cg::this_cluster();
  __shared__ double cand[2];
  __shared__ double best;
  unsigned long long t0 = clock64();
  int ph = 0;
  for (int i = 0; i < iters; ++i) {
    if (threadIdx.x == 0) {
      cand[ph] = (double)(blockIdx.x ^ i);
      asm volatile("fence.acq_rel.cluster;" ::: "memory");
    }
    asm volatile("barrier.cluster.arrive.relaxed.aligned;" ::: "memory");
    asm volatile("barrier.cluster.wait.aligned;" ::: "memory");
    if (threadIdx.x < 32) {
      double v = -1;
      if (threadIdx.x < (int)cl.num_blocks()) v = cl.map_shared_rank(cand, threadIdx.x)[ph];
      for (int o = 16; o; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
      if (threadIdx.x == 0) best = v;
    }
    __syncthreads();
    ph ^= 1;
  }
  cl.sync();
  if (blockIdx.x == 0 && threadIdx.x == 0) *out = clock64() - t0;
}

__global__ void k_cta_rounds(int iters, unsigned long long* out) {
  __shared__ double red[32];
  unsigned long long t0 = clock64();
  double v = threadIdx.x;
  for (int i = 0; i < iters; ++i) {
    for (int o = 16; o; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
    __syncthreads();
    if (threadIdx.x < 32) {
      double w = threadIdx.x < (blockDim.x >> 5) ? red[threadIdx.x] : -1;
      for (int o = 16; o; o >>= 1) w = fmax(w, __shfl_xor_sync(0xffffffffu, w, o));
      if (threadIdx.x == 0) red[0] = w;
    }
    __syncthreads();
    v = red[0] + threadIdx.x;
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) *out = clock64() - t0;
}

__global__ void k_empty() {}

__global__ void k_chase(const int* next, int iters, int* sink, unsigned long long* out) {
  int p = 0;
  unsigned long long t0 = clock64();
  for (int i = 0; i < iters; ++i) p = next[p];
  *out = clock64() - t0;
  *sink = p;
}

// (f) one warp, dependent chain of warp argmaxes; kind 0 REDUX, 1 shuffle tree
__global__ void k_warp_argmax(int kind, int iters, unsigned long long* out, double* sink) {
  double v = 0.25 + 1e-3 * ((threadIdx.x * 7) & 31);
  long long f = threadIdx.x;
  unsigned long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
    double bv = v;
    long long bf = f;
    if (kind == 0) warp_argmax(bv, bf);
    else warp_argmax_shfl(bv, bf);
    v = v + bv * 1e-30;   // depends on the result
    f = (f + bf) & 31;
  }
  unsigned long long t1 = clock64();
  sink[threadIdx.x] = v + f;
  if (threadIdx.x == 0) *out = t1 - t0;
}

int main() {
  unsigned long long* d_out;
  cudaMalloc(&d_out, 8);
  unsigned long long h;
  int iters = 2000;
  for (int G : {1, 2, 4, 8, 16}) {
    cudaFuncSetAttribute(k_cluster_rounds, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    cudaLaunchConfig_t lc = {};
    lc.gridDim = dim3(4 * G);
    lc.blockDim = dim3(288);
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = G;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    lc.attrs = at;
    lc.numAttrs = 1;
    cudaLaunchKernelEx(&lc, k_cluster_rounds, iters, d_out);
    cudaLaunchKernelEx(&lc, k_cluster_rounds, iters, d_out);
    cudaDeviceSynchronize();
    cudaMemcpy(&h, d_out, 8, cudaMemcpyDeviceToHost);
    printf("{\"probe\": \"cluster_argmax_round\", \"G\": %d, \"cycles\": %.1f}\n", G, (double)h / iters);
  }
  {
    double* sink;
    cudaMalloc(&sink, 32 * sizeof(double));
    for (int kind : {0, 1}) {
      k_warp_argmax<<<1, 32>>>(kind, iters, d_out, sink);
      k_warp_argmax<<<1, 32>>>(kind, iters, d_out, sink);
      cudaDeviceSynchronize();
      cudaMemcpy(&h, d_out, 8, cudaMemcpyDeviceToHost);
      printf("{\"probe\": \"warp_argmax\", \"impl\": \"%s\", \"cycles\": %.1f}\n", kind ? "shfl_tree" : "redux",
             (double)h / iters);
    }
    cudaFree(sink);
  }
  k_cta_rounds<<<64, 288>>>(iters, d_out);
  k_cta_rounds<<<64, 288>>>(iters, d_out);
  cudaDeviceSynchronize();
  cudaMemcpy(&h, d_out, 8, cudaMemcpyDeviceToHost);
  printf("{\"probe\": \"cta_argmax_round_288\", \"cycles\": %.1f}\n", (double)h / iters);
  // graph of empty launches
  for (int G : {1, 16}) {
    cudaStream_t s;
    cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
    cudaGraph_t g;
    cudaGraphExec_t ge;
    cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal);
    for (int i = 0; i < 100; ++i) {
      cudaLaunchConfig_t lc = {};
      lc.gridDim = dim3(64);
      lc.blockDim = dim3(288);
      lc.stream = s;
      cudaLaunchAttribute at[1];
      at[0].id = cudaLaunchAttributeClusterDimension;
      at[0].val.clusterDim.x = G;
      at[0].val.clusterDim.y = 1;
      at[0].val.clusterDim.z = 1;
      lc.attrs = at;
      lc.numAttrs = 1;
      cudaLaunchKernelEx(&lc, k_empty);
    }
    cudaStreamEndCapture(s, &g);
    cudaGraphInstantiate(&ge, g, 0);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    for (int w = 0; w < 3; ++w) cudaGraphLaunch(ge, s);
    cudaEventRecord(a, s);
    for (int w = 0; w < 10; ++w) cudaGraphLaunch(ge, s);
    cudaEventRecord(b, s);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    printf("{\"probe\": \"graph_launch_empty_64ctas\", \"G\": %d, \"us_per_launch\": %.3f}\n", G, ms * 1e3 / 1000);
  }
  // L2 pointer chase (4 MB, random permutation)
  const int N = 1 << 19;
  std::vector<int> nx(N);
  for (int i = 0; i < N; ++i) nx[i] = (int)((i * 2654435761u + 12345) % N);
  int *d_next, *d_sink;
  cudaMalloc(&d_next, N * 4);
  cudaMalloc(&d_sink, 4);
  cudaMemcpy(d_next, nx.data(), N * 4, cudaMemcpyHostToDevice);
  k_chase<<<1, 1>>>(d_next, 20000, d_sink, d_out);
  k_chase<<<1, 1>>>(d_next, 20000, d_sink, d_out);
  cudaDeviceSynchronize();
  cudaMemcpy(&h, d_out, 8, cudaMemcpyDeviceToHost);
  printf("{\"probe\": \"l2_dependent_load\", \"cycles\": %.1f}\n", (double)h / 20000);
  // (d) fp64 chains: one warp per SM on 64 SMs, 288-thread blocks (the k_sweep shape)
  {
    double* d_sink;
    cudaMalloc(&d_sink, 64 * 288 * sizeof(double));
    const char* names[] = {"dadd", "dmul", "ddiv", "rho", "dde_mul", "d_entry_plus_16_updates"};
    for (int kind = 0; kind < 6; ++kind) {
      const int it = kind == 5 ? 200 : 2000;
      k_fp64_chain<<<64, 288>>>(kind, it, 0.3, d_sink, d_out);
      k_fp64_chain<<<64, 288>>>(kind, it, 0.3, d_sink, d_out);
      cudaDeviceSynchronize();
      cudaMemcpy(&h, d_out, 8, cudaMemcpyDeviceToHost);
      printf("{\"probe\": \"fp64_chain\", \"op\": \"%s\", \"cycles_per_op\": %.1f}\n", names[kind], (double)h / it);
    }
  }
  // (e) st.async exchange rounds
  for (int G : {2, 4, 8, 16}) {
    cudaFuncSetAttribute(k_xchg_rounds, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    cudaLaunchConfig_t lc = {};
    lc.gridDim = dim3(4 * G);
    lc.blockDim = dim3(288);
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = G;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    lc.attrs = at;
    lc.numAttrs = 1;
    cudaLaunchKernelEx(&lc, k_xchg_rounds, iters, d_out);
    cudaLaunchKernelEx(&lc, k_xchg_rounds, iters, d_out);
    cudaDeviceSynchronize();
    cudaMemcpy(&h, d_out, 8, cudaMemcpyDeviceToHost);
    printf("{\"probe\": \"st_async_exchange_round\", \"G\": %d, \"cycles\": %.1f}\n", G, (double)h / iters);
  }
  printf("{\"status\": \"%s\"}\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
