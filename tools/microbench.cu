// tools/microbench.cu -- B200 latency probes that inform the k_sweep design (round 1):
//   (a) cluster barrier + DSMEM argmax round, per cluster size
//   (b) per-launch overhead of a CUDA graph of empty cluster kernels (64 CTAs)
//   (c) dependent L2 load latency (pointer chase)
// build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/microbench tools/microbench.cu
#include <cooperative_groups.h>
#include <cstdio>
#include <vector>
namespace cg = cooperative_groups;

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
  printf("{\"status\": \"%s\"}\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
