// tools/fp64_peak.cu -- measured fp64 throughput of this B200 (the denominator of the
// "% of fp64 peak" roofline, which MEASURED_PEAKS.json does not carry).
//
// Every thread runs ILP independent dependent-chains of one operation (DFMA: x = x*a + b,
// 2 flop; DMUL; DADD: 1 flop each) for `iters` iterations; grid = 148 SMs x 4 CTAs x 256
// threads.  Timed with CUDA events: "burst" = best of 10 launches of ~20 ms each (a kernel
// timed alone), "sustained" = back-to-back launches for ~4 s (a kernel inside a long step, at
// whatever clock the power cap allows).  Prints one JSON line per (op, mode).
// build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/fp64_peak tools/fp64_peak.cu
#include <cstdio>
#include <cuda_runtime.h>

#define ILP 8

template <int OP>
__global__ void __launch_bounds__(256) k_fp64(int iters, double a, double b, double* sink) {
  double x[ILP];
#pragma unroll
  for (int i = 0; i < ILP; ++i) x[i] = 1.0 + 1e-9 * (threadIdx.x + i);
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int u = 0; u < 16; ++u)
#pragma unroll
      for (int i = 0; i < ILP; ++i) {
        if (OP == 0) x[i] = fma(x[i], a, b);
        else if (OP == 1) x[i] = __dmul_rn(x[i], a);
        else x[i] = __dadd_rn(x[i], b);
      }
  }
  double s = 0.0;
#pragma unroll
  for (int i = 0; i < ILP; ++i) s += x[i];
  if (s == 12345.678) sink[blockIdx.x * blockDim.x + threadIdx.x] = s;   // (never true: keeps the chains live)
}

template <int OP>
double run(int blocks, int iters, int launches, float* ms_out, double* sink) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const double a = OP == 0 ? 0.9999999999 : 0.99999999999, b = 1e-12;
  cudaEventRecord(e0);
  for (int l = 0; l < launches; ++l) k_fp64<OP><<<blocks, 256>>>(iters, a, b, sink);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms = 0.f;
  cudaEventElapsedTime(&ms, e0, e1);
  *ms_out = ms;
  const double ops = (double)blocks * 256 * iters * 16 * ILP * launches;
  const double flop = ops * (OP == 0 ? 2.0 : 1.0);
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  return flop / (ms * 1e-3) / 1e12;
}

template <int OP>
void probe(const char* name, int blocks, double* sink) {
  float ms;
  run<OP>(blocks, 64, 1, &ms, sink);   // warm-up
  // ~20 ms per launch
  int iters = 256;
  run<OP>(blocks, iters, 1, &ms, sink);
  iters = (int)(iters * 20.0 / (ms > 0 ? ms : 1));
  double best = 0;
  for (int r = 0; r < 10; ++r) {
    const double t = run<OP>(blocks, iters, 1, &ms, sink);
    if (t > best) best = t;
  }
  printf("{\"probe\": \"fp64_peak\", \"op\": \"%s\", \"mode\": \"burst\", \"tflops\": %.3f, \"ms_per_launch\": %.2f}\n",
         name, best, ms);
  const double sus = run<OP>(blocks, iters, 200, &ms, sink);
  printf("{\"probe\": \"fp64_peak\", \"op\": \"%s\", \"mode\": \"sustained\", \"tflops\": %.3f, \"seconds\": %.2f}\n",
         name, sus, ms * 1e-3);
}

int main() {
  int dev = 0, sms = 0, clk = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev);
  const int blocks = sms * 4;
  double* sink;
  cudaMalloc(&sink, (size_t)blocks * 256 * sizeof(double));
  printf("{\"probe\": \"device\", \"sms\": %d, \"clock_khz\": %d, \"nominal_dfma_tflops\": %.3f}\n", sms, clk,
         sms * 64.0 * 2 * clk * 1e3 / 1e12);
  probe<0>("dfma", blocks, sink);
  probe<1>("dmul", blocks, sink);
  probe<2>("dadd", blocks, sink);
  printf("{\"status\": \"%s\"}\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
