// pf_tile.cuh — tile geometry and async-copy helpers shared by the z-marching
// sweeps (pf_phi.cu, pf_mu.cu).
//
// CTA = TX (x) x TY (y) threads, one thread per (i,j) column, marching a chunk
// of planes in z (z is the outermost loop because T depends on
// z only; the per-plane table row is staged once per plane).  A tile plane in
// shared memory is (TX+2) x (TY+2) cells: the interior plus a one-cell ring
// (with the 4 in-plane corners, needed by the D3C19 tangential gradients).
// Planes are staged two ahead with cp.async (LDGSTS: global -> shared without
// registers), so the loads of plane k+2 overlap the compute of plane k.
#pragma once
#include "pf_kernels.cuh"

namespace pf {

constexpr int TX = 32, TY = 8, RX = TX + 2, RY = TY + 2;
constexpr int NTHR = TX * TY;
constexpr int NRING = 2 * RX + 2 * TY;  // 84 ring cells incl. the 4 in-plane corners
constexpr int NSLOT = 4;                // plane slots: k-1, k, k+1 in use, k+2 in flight

// ring cell r -> (col, row) in the (RX x RY) tile (col/row 0 = index -1)
__device__ __forceinline__ void ring_cell(int r, int &col, int &row) {
  if (r < RX) { col = r; row = 0; }
  else if (r < 2 * RX) { col = r - RX; row = RY - 1; }
  else if (r < 2 * RX + TY) { col = 0; row = r - 2 * RX + 1; }
  else { col = RX - 1; row = r - 2 * RX - TY + 1; }
}
__device__ __forceinline__ bool ring_corner(int col, int row) {
  return (col == 0 || col == RX - 1) && (row == 0 || row == RY - 1);
}

// 8-byte async copy global -> shared; !ok zero-fills (src-size 0)
__device__ __forceinline__ void cp_async8(void *smem, const double *gmem, bool ok) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(s), "l"(gmem), "r"(ok ? 8 : 0) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory"); }

// z-chunk length: enough CTAs to fill the 148 SMs several times over,
// chunks of at least 16 planes.
inline int chunk_z(int nz, int nxy_tiles) {
  int kz = nz;
  while (kz > 16 && (int64_t)nxy_tiles * ((nz + kz - 1) / kz) < 148 * 8) kz = (kz + 1) / 2;
  return kz;
}

}  // namespace pf
