// PCIe probe: host<->device bandwidth of contiguous and 3D-pitched copies
// (the pf_step_io slab copies), one direction alone and both at once.
// nvcc -O2 -o tools/pcie_probe tools/pcie_probe.cu
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdlib>
int main() {
  const size_t nx = 512, ny = 512, nz = 512, pitch = 528, rows = ny + 2;   // one component of a 512^3 block
  const size_t hbytes = nx * ny * nz * 8, dbytes = pitch * rows * (nz + 2) * 8;
  double *h0, *h1, *d0, *d1;
  cudaMallocHost(&h0, hbytes); cudaMallocHost(&h1, hbytes);
  cudaMalloc(&d0, dbytes); cudaMalloc(&d1, dbytes);
  cudaStream_t s0, s1; cudaStreamCreate(&s0); cudaStreamCreate(&s1);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  auto p3 = [&](double *h, double *d, bool up, cudaStream_t s) {
    cudaMemcpy3DParms m = {};
    cudaPitchedPtr hp = make_cudaPitchedPtr(h, nx * 8, nx * 8, ny), dp = make_cudaPitchedPtr(d, pitch * 8, pitch * 8, rows);
    cudaPos hpos = make_cudaPos(0, 0, 0), dpos = make_cudaPos(32, 1, 1);
    if (up) { m.srcPtr = hp; m.srcPos = hpos; m.dstPtr = dp; m.dstPos = dpos; m.kind = cudaMemcpyHostToDevice; }
    else { m.srcPtr = dp; m.srcPos = dpos; m.dstPtr = hp; m.dstPos = hpos; m.kind = cudaMemcpyDeviceToHost; }
    m.extent = make_cudaExtent(nx * 8, ny, nz);
    cudaMemcpy3DAsync(&m, s);
  };
  auto run = [&](const char *name, int mode) {
    for (int rep = 0; rep < 2; ++rep) {
      cudaDeviceSynchronize();
      cudaEventRecord(a, 0);
      cudaStreamWaitEvent(s0, a, 0); cudaStreamWaitEvent(s1, a, 0);
      if (mode == 0) cudaMemcpyAsync(d0, h0, hbytes, cudaMemcpyHostToDevice, s0);
      if (mode == 1) cudaMemcpyAsync(h0, d0, hbytes, cudaMemcpyDeviceToHost, s0);
      if (mode == 2) { cudaMemcpyAsync(d0, h0, hbytes, cudaMemcpyHostToDevice, s0); cudaMemcpyAsync(h1, d1, hbytes, cudaMemcpyDeviceToHost, s1); }
      if (mode == 3) p3(h0, d0, true, s0);
      if (mode == 4) p3(h0, d0, false, s0);
      if (mode == 5) { p3(h0, d0, true, s0); p3(h1, d1, false, s1); }
      cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
      cudaEventRecord(e0, s0); cudaEventRecord(e1, s1);
      cudaStreamWaitEvent(0, e0, 0); cudaStreamWaitEvent(0, e1, 0);
      cudaEventRecord(b, 0); cudaEventSynchronize(b);
      float ms; cudaEventElapsedTime(&ms, a, b);
      const double gb = (mode == 2 || mode == 5 ? 2.0 : 1.0) * hbytes / 1e9;
      if (rep) printf("%-32s %8.2f ms  %6.1f GB/s total\n", name, ms, gb / (ms / 1e3));
    }
  };
  run("H2D contiguous", 0); run("D2H contiguous", 1); run("H2D + D2H contiguous", 2);
  run("H2D 3D pitched", 3); run("D2H 3D pitched", 4); run("H2D + D2H 3D pitched", 5);
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
