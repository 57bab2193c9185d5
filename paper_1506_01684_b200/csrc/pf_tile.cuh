// pf_tile.cuh — tile geometry and async-copy helpers shared by the z-marching
// sweeps (pf_phi.cu, pf_mu.cu).
//
// CTA = TX (x) x TY (y) threads, one thread per (i,j) column, marching a chunk
// of planes in z (z is the outermost loop because T depends on
// z only; the per-plane table row is staged once per plane).  A tile plane in
// shared memory is (TX+2) x (TY+2) cells: the interior plus a one-cell ring
// (with the 4 in-plane corners, needed by the D3C19 tangential gradients).
// Planes are staged ahead by TMA bulk-tensor copies (below), so the loads of
// plane k+2 overlap the compute of plane k.
#pragma once
#include <algorithm>
#include <cmath>
#include "pf_kernels.cuh"

namespace pf {

#if !defined(PF_TILE_X) || !defined(PF_TILE_Y)
#error "define PF_TILE_X / PF_TILE_Y (the CTA tile) before including pf_tile.cuh"
#endif
constexpr int TX = PF_TILE_X, TY = PF_TILE_Y, RX = TX + 2, RY = TY + 2;
constexpr int NTHR = TX * TY;
constexpr int NRING = 2 * RX + 2 * TY;  // 84 ring cells incl. the 4 in-plane corners
constexpr int NSLOT = 4;                // plane slots: k-1, k, k+1 in use, k+2 in flight
// the thread that issues the TMA copies: lane 0 of the last warp, which has no
// far-face / ring work (warps 0-2 do), so the issue does not lengthen the
// slowest warp's path to the next CTA barrier
constexpr int ISSUER = NTHR - 32;

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

// ---------------------------------------------------------------------------
// TMA (cp.async.bulk.tensor) + mbarrier helpers.  One elected thread arms the
// plane's mbarrier with the expected byte count and issues one bulk-tensor copy
// per component box; every thread waits on the barrier's phase parity.
// ---------------------------------------------------------------------------
// A bulk-tensor box must start on a 16-byte boundary in x and land on a
// 128-byte-aligned shared address (measured: tools/tma_probe.cu), so a staged
// tile is RXS = TX + 4 doubles wide, starting one column left of the ring
// (column i0 - 2, even because XO and i0 are): tile column c (c = 0 <-> i0 - 1)
// lives at RXS-row offset c + 1.  TSZ pads the RY x RXS tile to 128 B.
constexpr int RXS = TX + 4;
constexpr int TSZ = ((RY * RXS * 8 + 127) / 128) * 128 / 8;
static_assert(RY * RXS <= TSZ && (TSZ * 8) % 128 == 0, "tile padding");
#define TILE_AT(arr, row, col) (arr)[(row) * RXS + (col) + 1]

__device__ __forceinline__ uint32_t smem_u32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_fence_init() {
  asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t *bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred P1;\n"
      "WAIT:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
      "@P1 bra.uni DONE;\n\t"
      "bra.uni WAIT;\n"
      "DONE:\n\t}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory"); }
// 3D box (x fastest) of a tensor map into shared memory
__device__ __forceinline__ void tma_load_3d(void *dst, const CUtensorMap *map, int x, int y, int z, uint64_t *bar) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];\n"
      ::"r"(smem_u32(dst)), "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(z), "r"(smem_u32(bar))
      : "memory");
}
// contiguous bytes (multiple of 16, 16-B aligned) into shared memory
__device__ __forceinline__ void bulk_load(void *dst, const void *src, uint32_t bytes, uint64_t *bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n"
               ::"r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}

// z-chunk length.  Every CTA of a sweep does nearly the same work, so the grid
// runs in waves of (SMs x resident CTAs per SM); a ragged last wave idles the
// rest of the GPU (2048 CTAs on 592 slots: 3.46 waves take 4).  The chunk is
// halved (while it is longer than 16 planes, so a chunk keeps >= 9 planes; a chunk re-stages one plane above and below)
// until the grid spans at least min_waves waves, or (fill_ok) fills its last
// wave to >= 97 % from at least one full wave.  Measured (512^3, tools/ab_*): the
// phi-sweep is fastest at ~28 waves (64-plane chunks: 3.93 ms vs 4.09 ms
// unchunked), the mu-sweep, which stages more per chunk start, at ~7 (256).
inline int chunk_z(int nz, int nxy_tiles, int slots, int min_waves, bool fill_ok) {
  int kz = nz;
  auto eff = [&](int k) {
    const double w = (double)nxy_tiles * ((nz + k - 1) / k) / slots;
    return w / std::ceil(w);
  };
  while (kz > 16) {
    const int64_t n = (int64_t)nxy_tiles * ((nz + kz - 1) / kz);
    if (n >= (int64_t)min_waves * slots || (fill_ok && n >= slots && eff(kz) >= 0.97)) break;
    kz = (kz + 1) / 2;
  }
  return kz;
}

// resident CTAs of a kernel on the whole GPU (SMs x occupancy), queried once
template <class K>
int grid_slots(K kernel, int threads, size_t smem) {
  int dev = 0, sms = 0, per = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, kernel, threads, smem);
  return std::max(1, sms * std::max(1, per));
}

}  // namespace pf
