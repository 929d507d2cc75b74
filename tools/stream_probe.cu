// tools/stream_probe.cu -- the rook step's factor stream in isolation: CTAs of 512 threads
// stream U[t][x] (t < r) of a D_20-sized factor matrix through the per-warp TMA ring (TmaRing of
// the sweep kernel, 16-term stages) and run the t-ascending u.v chain per row, as a column step
// does; reports the aggregate and per-CTA bandwidth for several CTA counts and ring depths.
// build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 --fmad=false -std=c++17 -o tools/stream_probe tools/stream_probe.cu
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cooperative_groups.h>
#include <climits>
#include <cstdint>
#include <cstdio>
namespace cg = cooperative_groups;
#include "../paper_1903_11554_b200/csrc/ttc_common.cuh"
#include "../paper_1903_11554_b200/csrc/ttc_greedy.cuh"
using namespace ttc;

__global__ void __launch_bounds__(512, 1) k_stream(const void* tmap, int sbn, int cap, int r, int G, int P, int reps,
                                                   int math, int tb, double* sink) {
  extern __shared__ __align__(1024) double ring[];
  __shared__ GreedySmem S;
  const int tid = threadIdx.x, T = blockDim.x;
  if (tid < 64) S.vec[tid] = 1e-3 * (tid + 1);
  tma_ring_init(&S);
  __syncthreads();
  const int job = blockIdx.x / G, cr = blockIdx.x % G;
  const int rpc = (((sbn + G - 1) / G + 1) & ~1);
  const int xb = cr * rpc, xe = min(sbn, xb + rpc);
  RingPos pos{0, 0u};
  double acc = 0.0;
  for (int k = 0; k < reps; ++k) {
    TmaRing<true> rg;
    rg.start(ring, tmap, &S, T, tid, tb, P, r, job * cap, xb, xe, pos, 0.f);
    const int nblk = (xe - xb + T - 1) / T;
    for (int j = 0; j < nblk; ++j) {
      if (math) acc += rg.dot_sub(1.0, S.vec);
      else {   // the ring only: wait for each stage, no chain
        for (int b = 0; b < rg.nb; ++b) {
          if (rg.lane == 0 && rg.is < rg.total) rg.issue();
          mbar_wait(&rg.full[rg.pos.slot], rg.pos.phase);
          acc += rg.wbuf[rg.pos.slot * tb * 32 + rg.lane];
          __syncwarp();
          if (++rg.pos.slot == rg.P) { rg.pos.slot = 0; rg.pos.phase ^= 1u; }
        }
      }
    }
    pos = rg.pos;
  }
  sink[blockIdx.x * T + tid] = acc;
}

int main() {
  const int sbn = 32832, cap = 64, nj = 19, r = 64;
  double *U, *sink;
  const size_t rows = (size_t)nj * cap;
  cudaMalloc(&U, rows * sbn * 8);
  cudaMemset(U, 0, rows * sbn * 8);
  cudaMalloc(&sink, 148 * 512 * 8);
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
  auto encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  auto make = [&](int tb) {
    CUtensorMap map;
    const cuuint64_t dims[2] = {(cuuint64_t)sbn, (cuuint64_t)rows};
    const cuuint64_t strides[1] = {(cuuint64_t)sbn * 8};
    const cuuint32_t box[2] = {32, (cuuint32_t)tb};
    const cuuint32_t es[2] = {1, 1};
    encode(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, U, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
           CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    CUtensorMap* dmap;
    cudaMalloc(&dmap, sizeof(map));
    cudaMemcpy(dmap, &map, sizeof(map), cudaMemcpyHostToDevice);
    return dmap;
  };
  cudaFuncSetAttribute(k_stream, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int reps = 8;
  struct V { int math, P, tb, smem_kb; };
  const V vs[] = {{1, 2, 16, 128}, {1, 2, 16, 192}, {0, 2, 16, 128}, {0, 2, 16, 192}, {0, 3, 16, 192},
                  {0, 2, 24, 192}, {0, 4, 8, 128}, {0, 6, 8, 192}, {0, 2, 8, 64}, {1, 4, 8, 128}};
  for (const V& v : vs)
    for (int jobs : {19, 4, 1}) {
      const int G = 6, grid = jobs * G;
      const CUtensorMap* dmap = make(v.tb);
      const int smem = v.smem_kb * 1024;
      k_stream<<<grid, 512, smem>>>(dmap, sbn, cap, r, G, v.P, reps, v.math, v.tb, sink);
      cudaEventRecord(e0);
      k_stream<<<grid, 512, smem>>>(dmap, sbn, cap, r, G, v.P, reps, v.math, v.tb, sink);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms = 0;
      cudaEventElapsedTime(&ms, e0, e1);
      const double bytes = (double)reps * jobs * sbn * r * 8.0;
      printf("{\"probe\": \"tma_stream\", \"math\": %d, \"P\": %d, \"tb\": %d, \"smem_kb\": %d, \"ctas\": %d, "
             "\"GBps\": %.1f, \"GBps_per_cta\": %.1f, \"us_per_step\": %.2f}\n",
             v.math, v.P, v.tb, v.smem_kb, grid, bytes / ms / 1e6, bytes / ms / 1e6 / grid, ms * 1e3 / reps);
    }
  printf("{\"status\": \"%s\"}\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
