// FP64 register-operand probe: DFMA chains whose multiplier / addend are
// (0) constants, (1) per-chain registers (no operand shared between consecutive
// instructions), (2) one register shared by all chains
#include <cstdio>
#include <cuda_runtime.h>
template <int ILP, int MODE>
__global__ void chains(double *out, int iters, double a, double b) {
  double x[ILP], y[ILP], z[ILP];
#pragma unroll
  for (int c = 0; c < ILP; ++c) { x[c] = threadIdx.x * 1e-9 + c; y[c] = a + c * 1e-12 + threadIdx.x * 1e-15; z[c] = b + c * 1e-13 + threadIdx.x * 1e-16; }
  const double ys = a + threadIdx.x * 1e-15, zs = b + threadIdx.x * 1e-16;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int u = 0; u < 32; ++u)
#pragma unroll
      for (int c = 0; c < ILP; ++c) {
        if (MODE == 0) x[c] = fma(x[c], a, b);
        else if (MODE == 1) x[c] = fma(x[c], y[c], z[c]);
        else if (MODE == 2) x[c] = fma(x[c], ys, zs);
        else if (MODE == 3) x[c] = x[c] * y[c];
        else x[c] = x[c] + z[c];
      }
  }
  double s = 0;
#pragma unroll
  for (int c = 0; c < ILP; ++c) s += x[c] + y[c] + z[c];
  if (s == 1234.5) out[0] = s;
}
template <int ILP, int MODE>
void run(int nsm, double *out) {
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int wps = 4; wps <= 16; wps *= 2) {
    const int threads = 128, blocks = nsm * wps, iters = 2000 / ILP;
    chains<ILP, MODE><<<blocks, threads>>>(out, iters, 0.999999, 1e-7);
    cudaEventRecord(e0);
    chains<ILP, MODE><<<blocks, threads>>>(out, iters, 0.999999, 1e-7);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    const double flops = 2.0 * 32 * ILP * (double)iters * threads * blocks;
    printf("mode %d ILP %d warps/SMSP %2d: %.2f TFLOP/s\n", MODE, ILP, wps, flops / ms / 1e9);
  }
}
int main() {
  int nsm = 0; cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  double *out; cudaMalloc(&out, 8);
  run<1, 0>(nsm, out); run<1, 1>(nsm, out); run<1, 2>(nsm, out);
  run<2, 0>(nsm, out); run<2, 1>(nsm, out); run<2, 2>(nsm, out);
  run<4, 0>(nsm, out); run<4, 1>(nsm, out); run<4, 2>(nsm, out); run<4, 3>(nsm, out); run<4, 4>(nsm, out);
  return 0;
}
