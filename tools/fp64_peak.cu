// Sustained FP64 DFMA throughput microbenchmark (roofline denominator for the
// FP64-bound sweeps). All SMs, 8 independent FMA chains per thread, timed
// with CUDA events. Prints one JSON line.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void dfma_loop(double *out, int iters, double a, double b) {
  double x0 = threadIdx.x * 1e-9, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3;
  double x4 = x0 + 4, x5 = x0 + 5, x6 = x0 + 6, x7 = x0 + 7;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int u = 0; u < 16; ++u) {
      x0 = fma(x0, a, b); x1 = fma(x1, a, b); x2 = fma(x2, a, b); x3 = fma(x3, a, b);
      x4 = fma(x4, a, b); x5 = fma(x5, a, b); x6 = fma(x6, a, b); x7 = fma(x7, a, b);
    }
  }
  double s = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
  if (s == 1234.5) out[0] = s;
}
int main() {
  int dev = 0, nsm = 0, clk = 0;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev);
  double *out; cudaMalloc(&out, 8);
  int threads = 256, blocks = nsm * 8, iters = 4000;
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int w = 0; w < 3; ++w) dfma_loop<<<blocks, threads>>>(out, iters, 0.999999, 1e-7);
  float best = 1e30f, tot = 0; int reps = 20;
  for (int r = 0; r < reps; ++r) {
    cudaEventRecord(e0);
    dfma_loop<<<blocks, threads>>>(out, iters, 0.999999, 1e-7);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1); if (ms < best) best = ms; tot += ms;
  }
  double flops = 2.0 * 8 * 16 * (double)iters * threads * blocks;
  printf("{\"fp64_tflops_burst\": %.3f, \"fp64_tflops_mean\": %.3f, \"sms\": %d, \"clock_khz_attr\": %d, \"err\": \"%s\"}\n",
         flops / best / 1e9, flops / (tot / reps) / 1e9, nsm, clk, cudaGetErrorString(cudaGetLastError()));
  return 0;
}
