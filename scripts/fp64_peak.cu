// DFMA throughput microbenchmark (the fp64 roof of K6).
// Every thread runs 8 independent FMA chains for `iters` iterations; grid =
// 148 SMs x 8 CTAs x 256 threads. Prints one JSON line with the best of 10
// launches (CUDA events):  nvcc -gencode arch=compute_100a,code=sm_100a -O3
// scripts/fp64_peak.cu -o /tmp/fp64_peak && /tmp/fp64_peak
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k_dfma(double* out, int iters, double a, double b) {
  double x[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) x[i] = threadIdx.x * 1e-3 + i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) x[i] = fma(x[i], a, b);
  }
  double s = 0.0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += x[i];
  if (s == 12345.678) out[0] = s;  // keep the chains live
}

int main() {
  int dev = 0, sms = 0, clk = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev);
  double* out;
  cudaMalloc(&out, 8);
  const int threads = 256, blocks = sms * 8, iters = 1 << 14;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  k_dfma<<<blocks, threads>>>(out, iters, 0.999999, 1e-9);
  float best = 1e30f;
  for (int r = 0; r < 10; ++r) {
    cudaEventRecord(e0);
    k_dfma<<<blocks, threads>>>(out, iters, 0.999999, 1e-9);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, e0, e1);
    if (ms < best) best = ms;
  }
  const double flops = 2.0 * 8.0 * iters * double(threads) * blocks;
  const double tf = flops / (best * 1e-3) / 1e12;
  printf("{\"dfma_tflops\": %.3f, \"best_ms\": %.4f, \"sms\": %d, \"clock_mhz_attr\": %d, "
         "\"dfma_per_clk_per_sm_at_attr_clock\": %.1f, \"how\": \"8 independent FMA chains per thread, "
         "%d CTAs x %d threads x %d iterations, best of 10, CUDA events\"}\n",
         tf, best, sms, clk / 1000, flops / 2.0 / (best * 1e-3) / sms / (clk * 1e3), blocks, threads, iters);
  cudaError_t err = cudaGetLastError();
  return err == cudaSuccess ? 0 : 1;
}
