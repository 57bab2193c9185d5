// pf_kernels.cuh — kernel declarations and launch-side structs shared by the
// runtime (pf_runtime.cu) and the kernel translation units.
#pragma once
#include <cstdint>
#include <cuda.h>
#include <cuda_runtime.h>
#include "pf_dev.cuh"

namespace pf {

constexpr int XO = 4;  // column of interior i = 0 within a padded row (i = -1 at 3)
// CTA tiles of the z-marching sweeps (pf_tile.cuh), measured best (tools/ab_*):
// 16 x 8 for the phi-sweep (128 threads, each warp two rows; 4 CTAs / SM; the
// 24 far faces of a plane fit one warp — 32 x 4: 4.16 ms, 16 x 8: 4.09 ms,
// 16 x 16: 4.21, 8 x 16: 5.4 at 512^3), 32 x 8 for the mu-sweep (2 CTAs / SM;
// 16 x 16: +4 %).  -DPF_PHI_TX/TY, -DPF_MU_TX/TY override for experiments.
#ifndef PF_PHI_TX
#define PF_PHI_TX 16
#endif
#ifndef PF_PHI_TY
#define PF_PHI_TY 8
#endif
#ifndef PF_MU_TX
#define PF_MU_TX 32
#endif
#ifndef PF_MU_TY
#define PF_MU_TY 8
#endif
// the fused mu(n) + phi(n+1) kernel (pf_fused.cu): 16 x 8 at 3 CTAs / SM
#ifndef PF_FUSED_TX
#define PF_FUSED_TX 16
#endif
#ifndef PF_FUSED_TY
#define PF_FUSED_TY 8
#endif
constexpr int FUSED_TILE_X = PF_FUSED_TX, FUSED_TILE_Y = PF_FUSED_TY;
constexpr int PHI_TILE_X = PF_PHI_TX, PHI_TILE_Y = PF_PHI_TY, MU_TILE_X = PF_MU_TX, MU_TILE_Y = PF_MU_TY;

// TMA descriptors of one block's fields in one time level (encoded on the host
// over the whole padded allocation: dims {pitch, ny+2, planes}, x fastest).
// tile: box (TX+4) x (TY+2) x 1 — interior tile + ring, x from a 16-byte boundary.
struct TmaMaps {
  CUtensorMap phi[NPH];   // phi^n,     tile box
  CUtensorMap phin[NPH];  // phi^{n+1}, tile box
  CUtensorMap mu[NMU];    // mu^n,      tile box
};

// Pointers into one block's fields, offset to interior cell (0,0,0) of the
// current window position; element (i,j,k) at p + k*plane + j*pitch + i with
// i,j,k in [-1, n].
struct BlockView {
  const double *phi[NPH];
  const double *mu[NMU];
  const double *phin[NPH];  // phi^{n+1} (mu-sweep input)
  double *out[NPH];         // phi^{n+1} (phi-sweep) or mu^{n+1} (mu-sweep)
  int nx, ny, nz;
  int64_t pitch, plane;
  const double *tab;        // table row of local plane k = 0
  int zoff;                 // allocation plane of local k = 0 (1 + window offset), for TMA
  int tile_x0, tile_y0;     // first CTA tile of a launch over a tile sub-range (mu-sweep
                            // interior / shell split, overlap mode 4); 0 otherwise
};

// Strided 3D box copy (halo exchange: local copy, pack, unpack).
struct CopyOp {
  const double *src[NPH];
  double *dst[NPH];
  int64_t ssx, ssy, ssz;    // source strides (elements)
  int64_t dsx, dsy, dsz;    // destination strides
  int ex, ey, ez;           // extents
  int ncomp;
  int64_t cta0;             // first CTA of this op in its launch (upload_ops)
  int xpad;                 // >= 0: a ghost column alone in its 32-byte sector (the other
                            // three doubles are row padding) at this slot: each cell is
                            // written as the whole sector, so DRAM sees no partial-sector
                            // read-modify-write; -1: plain copy
};
constexpr int COPY_CELLS_PER_CTA = 1024;   // 256 threads x 4 cells

struct InitSpec {
  int kind, n_seeds, nlam;
  double layer_height, W, mu_noise;
  uint64_t seed;
  int64_t NX, NY, NZ;       // global grid
  const double *sx, *sy;    // voronoi seeds (device)
  const int *sp;            // voronoi seed phases
  const int64_t *lam;       // lamella starts (nlam+1 entries)
  int planar_phase;
};

struct TabParams {
  double T0, G, v, dt, dx, T_eut, eps;
  double A0[NPH][NMU], A1[NPH][NMU], c0[NPH][NMU], m[NPH][NMU], L[NPH], D[NPH][NMU];
};
// table rows for global window planes kg = -1 .. nplanes-2 (row = kg + 1)
// d_step != nullptr: the time level is read from device memory (CUDA graph replays)
void launch_table(cudaStream_t s, double *tab, int64_t nplanes, const TabParams &tp, int64_t step, int64_t zorig,
                  const int64_t *d_step = nullptr);
void launch_step_inc(cudaStream_t s, int64_t *d_step);
void launch_phi_naive(cudaStream_t s, const KParams &kp, const BlockView &b);
void launch_mu_naive(cudaStream_t s, const KParams &kp, const BlockView &b);
void prepare_phi_tiled();   // shared-memory opt-in of the tiled sweeps (once, outside captures)
void prepare_mu_tiled();
void launch_phi_tiled(cudaStream_t s, const KParams &kp, const BlockView &b, const TmaMaps &tm);
// mu-sweep modes: the whole update (Algorithm 1), or Algorithm 2's split
// into the part without the anti-trapping current and the
// part that adds its divergence after the phi^{n+1} halo exchange
enum { MU_FULL = 0, MU_LOCAL = 1, MU_NEIGHBOR = 2 };
void launch_mu_tiled(cudaStream_t s, const KParams &kp, const BlockView &b, const TmaMaps &tm, int mode = MU_FULL);
// the mu-sweep over CTA tiles [tx0, tx1) x [ty0, ty1) of the block (b may be a
// z-slab view): bitwise the cells' values of the whole-block launch
void launch_mu_tiles(cudaStream_t s, const KParams &kp, const BlockView &b, const TmaMaps &tm, int tx0, int tx1,
                     int ty0, int ty1);
// the fused kernel (pf_fused.cu): b is the mu-sweep view of step n (phi =
// phi^n, phin = phi^{n+1}, mu = mu^n, out = mu^{n+1}, tab = step n's rows),
// tm its maps with the fused tile box; fo the phi^{n+2} output and step n+1's
// table rows.  Bitwise the mu-sweep of step n followed by the phi-sweep of n+1.
struct FusedOut {
  double *phi2[NPH];      // phi^{n+2}, offset like BlockView::out
  const double *tabp;     // table row of local plane 0 at step n+1
};
void prepare_fused();
void launch_fused(cudaStream_t s, const KParams &kp, const BlockView &b, const TmaMaps &tm, const FusedOut &fo);
int mu_tiles_x(int nx);   // CTA tiles of the mu-sweep along x / y
int mu_tiles_y(int ny);
void launch_copy(cudaStream_t s, const CopyOp *d_ops, int nops, int64_t nctas);
void launch_init(cudaStream_t s, const InitSpec &is, double *const phi[NPH], double *const mu[NMU],
                 int nx, int ny, int nz, int64_t pitch, int64_t plane, int64_t x0, int64_t y0, int64_t z0);
void launch_fill_plane(cudaStream_t s, double *const f[NPH], int ncomp, const double *vals, int nx, int ny,
                       int64_t pitch);
void launch_front(cudaStream_t s, const double *phil, int nx, int ny, int nz, int64_t pitch, int64_t plane,
                  double thr, int64_t kbase, unsigned long long *d_out);
void launch_nancheck(cudaStream_t s, const double *const f[NPH], int ncomp, int nx, int ny, int nz, int64_t pitch,
                     int64_t plane, unsigned long long *d_first);
void launch_gather(cudaStream_t s, const double *const f[NPH], int ncomp, int nx, int ny, int nz, int64_t pitch,
                   int64_t plane, double *dst, int64_t dnx, int64_t dny, int64_t dn, int64_t ox, int64_t oy, int64_t oz,
                   bool scatter, double *const fw[NPH]);
// marching-cubes case table {ntri, 3 edges per triangle} x 256 (host only)
void mesh_case_table(int8_t *out);
// marching-cubes mesh of one phase over the rank's box (pf_mesh.cu); synchronous
cudaError_t launch_mesh(cudaStream_t s, const double *const *f, int bnx, int bny, int bnz, int pbx, int pby,
                        int pbz, int64_t pitch, int64_t plane, int64_t nx, int64_t ny, int64_t nzc, int64_t X0,
                        int64_t Y0, int64_t Z0, int64_t NX, int64_t NY, int64_t zorig, double iso, double dx,
                        int64_t cap, int64_t *ids, double *pos, int64_t *ntri, void **scratch, size_t *scratch_bytes);
void launch_cvt32(cudaStream_t s, double *f, int nx, int ny, int nz, int64_t pitch, int64_t plane, float *dst,
                  int64_t dnx, int64_t dny, int64_t ox, int64_t oy, int64_t oz, bool to_fields);

}  // namespace pf
