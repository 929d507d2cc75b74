// tools/ext_probe.cu -- cycles per t of the phase-2 recurrence ext_rec<L> (k_sweep extension)
// in isolation: 114 CTAs x 512 threads (the D_20 launch shape), coefficients in shared memory,
// rows side (no division) and columns side (division by u_t(x_t) per t).
// build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 --fmad=false -std=c++17 -o tools/ext_probe tools/ext_probe.cu
#include <cooperative_groups.h>
#include <climits>
#include <cstdint>
#include <cstdio>
namespace cg = cooperative_groups;
#include "../paper_1903_11554_b200/csrc/ttc_common.cuh"
#include "../paper_1903_11554_b200/csrc/ttc_greedy.cuh"
using namespace ttc;

template <int L>
__global__ void __launch_bounds__(512, 1) k_rec(int r, int side, int reps, double* sink, unsigned long long* out) {
  extern __shared__ double coefL[];
  double* pdiag = s_pdiag;
  double* prcp = s_prcp;
  const int cap = 64;
  for (int e = threadIdx.x; e < cap * L * EXR_CS; e += blockDim.x) coefL[e] = 1e-3 * ((e * 7) % 13) - 0.006;
  if (threadIdx.x < 64) {
    pdiag[threadIdx.x] = 1.5 + 0.01 * threadIdx.x;
    prcp[threadIdx.x] = rcp_refined(pdiag[threadIdx.x]);
  }
  __syncthreads();
  const int lane = threadIdx.x & 31, l = threadIdx.x & (L - 1), gbase = lane & ~(L - 1);
  double acc[EXR_NS];
#pragma unroll
  for (int i = 0; i < EXR_NS; ++i) acc[i] = 1.0 + 1e-3 * i + 1e-6 * threadIdx.x;
  const unsigned long long t0 = clock64();
  for (int k = 0; k < reps; ++k) ext_rec<L>(acc, r, l, gbase, side, pdiag, prcp, coefL);
  const unsigned long long t1 = clock64();
  double s = 0;
#pragma unroll
  for (int i = 0; i < EXR_NS; ++i) s += acc[i];
  sink[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0 && blockIdx.x == 0) *out = t1 - t0;
}

int main() {
  double* sink;
  unsigned long long* d_out;
  cudaMalloc(&sink, 114 * 512 * sizeof(double));
  cudaMalloc(&d_out, 8);
  const int reps = 20;
  for (int side : {0, 1})
    for (int r : {16, 32, 55, 64}) {
      const int L = r <= 16 ? 1 : (r <= 32 ? 2 : 4);
      const int smem = 64 * L * EXR_CS * 8;
      auto f = L == 1 ? k_rec<1> : (L == 2 ? k_rec<2> : k_rec<4>);
      cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
      f<<<114, 512, smem>>>(r, side, reps, sink, d_out);
      f<<<114, 512, smem>>>(r, side, reps, sink, d_out);
      cudaDeviceSynchronize();
      unsigned long long h = 0;
      cudaMemcpy(&h, d_out, 8, cudaMemcpyDeviceToHost);
      printf("{\"probe\": \"ext_rec\", \"side\": %d, \"r\": %d, \"L\": %d, \"cycles_per_t\": %.1f, \"us_per_pass\": %.2f}\n",
             side, r, L, (double)h / reps / r, (double)h / reps / 1965.0);
    }
  printf("{\"status\": \"%s\"}\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
