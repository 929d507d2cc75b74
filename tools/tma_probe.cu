// tools/tma_probe.cu -- minimal check of 2-D TMA loads (cp.async.bulk.tensor) from a tensor map
// held in global memory vs passed as a __grid_constant__ kernel parameter, with and without a
// thread-block cluster (diagnostics for the TMA ring of the sweep kernel).
// build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/tma_probe tools/tma_probe.cu
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <vector>

__device__ __forceinline__ unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }

template <bool PARAM>
__global__ void k_probe(const __grid_constant__ CUtensorMap pmap, const CUtensorMap* gmap, int W, int TB, double* out,
                        int xoff) {
  extern __shared__ __align__(1024) double buf[];
  __shared__ __align__(8) unsigned long long bar;
  const void* map = PARAM ? (const void*)&pmap : (const void*)gmap;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const int x = blockIdx.x * W + xoff, y = 3;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&bar)), "r"(W * TB * 8)
                 : "memory");
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
            smem_u32(buf)),
        "l"(map), "r"(x), "r"(y), "r"(smem_u32(&bar))
        : "memory");
  }
  unsigned ok = 0;
  while (!ok)
    asm volatile(
        "{\n .reg .pred q;\n mbarrier.try_wait.parity.shared::cta.b64 q, [%1], %2;\n selp.u32 %0, 1, 0, q;\n}"
        : "=r"(ok) : "r"(smem_u32(&bar)), "r"(0u) : "memory");
  for (int i = threadIdx.x; i < W * TB; i += blockDim.x) out[(long long)blockIdx.x * W * TB + i] = buf[i];
}

int main() {
  const int n0 = 32832, n1 = 1216, W = 256, TB = 8, nblk = 16;
  std::vector<double> h((size_t)n0 * n1);
  for (size_t i = 0; i < h.size(); ++i) h[i] = (double)i;
  double *g, *out;
  cudaMalloc(&g, h.size() * 8);
  cudaMemcpy(g, h.data(), h.size() * 8, cudaMemcpyHostToDevice);
  cudaMalloc(&out, (size_t)nblk * W * TB * 8);
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
  auto encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  CUtensorMap map;
  const cuuint64_t dims[2] = {(cuuint64_t)n0, (cuuint64_t)n1};
  const cuuint64_t strides[1] = {(cuuint64_t)n0 * 8};
  const cuuint32_t box[2] = {(cuuint32_t)W, (cuuint32_t)TB};
  const cuuint32_t es[2] = {1, 1};
  CUresult cr = encode(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, g, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                       CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  printf("{\"encode\": %d}\n", (int)cr);
  CUtensorMap* gmap;
  cudaMalloc(&gmap, sizeof(map));
  cudaMemcpy(gmap, &map, sizeof(map), cudaMemcpyHostToDevice);
  const size_t smem = W * TB * 8;
  cudaFuncSetAttribute(k_probe<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaFuncSetAttribute(k_probe<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  for (int xoff : {0, 1, 2})
  for (int param = 1; param >= 0; --param)
    for (int cl : {1, 8}) {
      cudaLaunchConfig_t lc = {};
      lc.gridDim = dim3(nblk);
      lc.blockDim = dim3(256);
      lc.dynamicSmemBytes = smem;
      cudaLaunchAttribute at[1];
      at[0].id = cudaLaunchAttributeClusterDimension;
      at[0].val.clusterDim.x = cl;
      at[0].val.clusterDim.y = 1;
      at[0].val.clusterDim.z = 1;
      lc.attrs = at;
      lc.numAttrs = 1;
      cudaMemset(out, 0, (size_t)nblk * W * TB * 8);
      cudaError_t e = param ? cudaLaunchKernelEx(&lc, k_probe<true>, map, (const CUtensorMap*)gmap, W, TB, out, xoff)
                            : cudaLaunchKernelEx(&lc, k_probe<false>, map, (const CUtensorMap*)gmap, W, TB, out, xoff);
      cudaError_t e2 = cudaDeviceSynchronize();
      std::vector<double> o((size_t)nblk * W * TB);
      cudaMemcpy(o.data(), out, o.size() * 8, cudaMemcpyDeviceToHost);
      long bad = 0;
      for (int b = 0; b < nblk; ++b)
        for (int t = 0; t < TB; ++t)
          for (int i = 0; i < W; ++i)
            if (o[(size_t)b * W * TB + t * W + i] != h[(size_t)(3 + t) * n0 + b * W + i + xoff]) ++bad;
      printf("{\"xoff\": %d, \"param\": %d, \"cluster\": %d, \"launch\": \"%s\", \"sync\": \"%s\", \"bad\": %ld}\n", xoff, param, cl,
             cudaGetErrorString(e), cudaGetErrorString(e2), bad);
      if (e2 != cudaSuccess) return 1;
    }
  return 0;
}
