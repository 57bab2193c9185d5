// FP64 pipe latency / ILP probe: DFMA throughput on all SMs as a function of
// the independent chains per thread (ILP) and the warps per SM sub-partition
// (occupancy).  Tells how much ILP x occupancy the sweeps need to keep the
// FP64 pipe busy.  Prints one line per configuration.
#include <cstdio>
#include <cuda_runtime.h>
template <int ILP>
__global__ void chains(double *out, int iters, double a, double b) {
  double x[ILP];
#pragma unroll
  for (int c = 0; c < ILP; ++c) x[c] = threadIdx.x * 1e-9 + c;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int u = 0; u < 32; ++u)
#pragma unroll
      for (int c = 0; c < ILP; ++c) x[c] = fma(x[c], a, b);
  }
  double s = 0;
#pragma unroll
  for (int c = 0; c < ILP; ++c) s += x[c];
  if (s == 1234.5) out[0] = s;
}
template <int ILP>
void run(int nsm, double *out) {
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int wps = 1; wps <= 16; wps *= 2) {   // warps per SMSP: 4*wps warps per SM, one CTA of 128 threads = 1 warp/SMSP
    const int threads = 128, blocks = nsm * wps, iters = 2000 / ILP;
    chains<ILP><<<blocks, threads>>>(out, iters, 0.999999, 1e-7);
    cudaEventRecord(e0);
    chains<ILP><<<blocks, threads>>>(out, iters, 0.999999, 1e-7);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    const double flops = 2.0 * 32 * ILP * (double)iters * threads * blocks;
    printf("ILP %d warps/SMSP %2d: %.2f TFLOP/s\n", ILP, wps, flops / ms / 1e9);
  }
}
int main() {
  int nsm = 0; cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  double *out; cudaMalloc(&out, 8);
  run<1>(nsm, out); run<2>(nsm, out); run<4>(nsm, out); run<8>(nsm, out);
  return 0;
}
