// pf_mu.cu — production mu-sweep (Eq. (3)-(4)): z-marching
// 2.5D tiles; every staggered value M grad mu - J_at (the
// "computationally most intensive part") is evaluated once per face.
//
// Shared memory per CTA (2 CTAs / SM):
//   * phi^{n+1} tile planes k-1 .. k+2 (ring + corners: the D3C19 stencil of the
//     anti-trapping current needs tangential gradients at face neighbours,
//     PAPER.md:179), phi^n and mu tile planes k .. k+2, table rows — all staged
//     two planes ahead with cp.async;
//   * the mobility of plane k (computed once per cell);
//   * the x/y face values of plane k.
// Everything else a face needs (dphi, c^l - c^a, tangential gradients) is
// read or derived from the staged planes inside the face routine, and only
// when the exact-zero guards let the anti-trapping term through (bulk liquid
// and bulk solid faces exit after the diffusive flux).  z-faces are carried in
// registers.  All arithmetic is the pinned code of pf_dev.cuh, so results do
// not depend on tile or block boundaries.
#include "pf_tile.cuh"

namespace pf {

constexpr int NS3 = 3;  // phi^n / mu slots: k, k+1, k+2 (in flight)

struct MuSmem {
  double pn[NSLOT][NPH][RY][RX];  // phi^{n+1}, planes k-1 .. k+2
  double po[NS3][NPH][RY][RX];    // phi^n, planes k .. k+2
  double mu[NS3][NMU][RY][RX];    // mu^n,  planes k .. k+2
  double tab[NSLOT][TAB];
  double M[NMU][RY][RX];          // mobility of plane k
  double fx[NMU][TY][TX + 1];     // x-face values at i - 1/2
  double fy[NMU][TY + 1][TX];     // y-face values at j - 1/2
};

// Accessor over the staged planes for tile cell (col,row) of plane k:
// pn slots (k-1, k, k+1) = (snm, sn, snp), phi^n/mu slot s3, table row tab.
struct RawQ {
  const MuSmem &S;
  const KParams &kp;
  int snm, sn, snp, s3, col, row;
  const double *tab;
  double Mv[NMU];
  __device__ __forceinline__ double pn(int a) const { return S.pn[sn][a][row][col]; }
  __device__ __forceinline__ double dp(int a) const { return RN_SUB(S.pn[sn][a][row][col], S.po[s3][a][row][col]); }
  __device__ __forceinline__ double gt(int a, int e) const {
    if (e == 0) return cgrad(kp, S.pn[sn][a][row][col - 1], S.pn[sn][a][row][col + 1]);
    if (e == 1) return cgrad(kp, S.pn[sn][a][row - 1][col], S.pn[sn][a][row + 1][col]);
    return cgrad(kp, S.pn[snm][a][row][col], S.pn[snp][a][row][col]);
  }
  __device__ __forceinline__ double M(int c) const { return Mv[c]; }
  __device__ __forceinline__ double mu(int c) const { return S.mu[s3][c][row][col]; }
  __device__ __forceinline__ double dcl(int a, int c) const { return dcl_of(tab, a, c, mu(c)); }
};

__global__ void __launch_bounds__(NTHR, 2) mu_tiled_kernel(KParams kp, BlockView b, int kz) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  MuSmem &S = *reinterpret_cast<MuSmem *>(smem_raw);
  const int tx = threadIdx.x, ty = threadIdx.y, tid = ty * TX + tx;
  const int i0 = blockIdx.x * TX, j0 = blockIdx.y * TY;
  const int k0 = blockIdx.z * kz, k1 = min(k0 + kz, b.nz);
  const int i = i0 + tx, j = j0 + ty;
  const bool active = (i < b.nx) && (j < b.ny);
  const bool inb = (i <= b.nx) && (j <= b.ny);
  const int64_t colo = (int64_t)j * b.pitch + i;
  const int oc = tx + 1, orow = ty + 1;
  const bool ring_thr = tid < NRING;
  int rcol = 0, rrow = 0;
  if (ring_thr) ring_cell(tid, rcol, rrow);
  const bool rcorner = ring_corner(rcol, rrow);
  const int rgi = i0 - 1 + rcol, rgj = j0 - 1 + rrow;
  const bool rok = ring_thr && rgi <= b.nx && rgj <= b.ny;
  const int64_t roff = rok ? (int64_t)rgj * b.pitch + rgi : colo;

  auto slot = [&](int k) { return (k - k0 + 1) & (NSLOT - 1); };
  auto slot3 = [&](int k) { return (k - k0 + 3) % NS3; };
  // stage plane k: phi^{n+1} (tile + ring + corners) always; phi^n, mu and the
  // mu when plane k is >= k0 (the first plane whose cells we update)
  auto stage = [&](int k) {
    const int s = slot(k), s3 = slot3(k);
    const int64_t pk = (int64_t)k * b.plane;
    const bool full = k >= k0;
#pragma unroll
    for (int a = 0; a < NPH; ++a) {
      cp_async8(&S.pn[s][a][orow][oc], b.phin[a] + pk + colo, inb);
      if (ring_thr) cp_async8(&S.pn[s][a][rrow][rcol], b.phin[a] + pk + roff, rok);
      if (full) {
        cp_async8(&S.po[s3][a][orow][oc], b.phi[a] + pk + colo, inb);
        if (ring_thr && !rcorner) cp_async8(&S.po[s3][a][rrow][rcol], b.phi[a] + pk + roff, rok);
      }
    }
    if (full) {
#pragma unroll
      for (int c = 0; c < NMU; ++c) {
        cp_async8(&S.mu[s3][c][orow][oc], b.mu[c] + pk + colo, inb);
        if (ring_thr && !rcorner) cp_async8(&S.mu[s3][c][rrow][rcol], b.mu[c] + pk + roff, rok);
      }
    }
    if (tid < TAB) cp_async8(&S.tab[s][tid], b.tab + (int64_t)k * TAB + tid, true);
    cp_async_commit();
  };
  auto rawq = [&](int k, int col, int row) {
    return RawQ{S, kp, slot(k - 1), slot(k), slot(k + 1), slot3(k), col, row, S.tab[slot(k)], {0.0, 0.0}};
  };

  // ---- prologue: planes k0-1 .. k0+1 resident
  stage(k0 - 1);
  stage(k0);
  stage(k0 + 1);
  cp_async_wait<0>();
  __syncthreads();
  // z-face k0 - 1/2 from the own column's quantities at k0-1 and k0 (phi^n,
  // mu, table at k0-1 read directly from global: needed once per chunk)
  double fzm[NMU];
  {
    double po[NPH], pn[NPH], mu[NMU];
    const int64_t pk = (int64_t)(k0 - 1) * b.plane;
#pragma unroll
    for (int a = 0; a < NPH; ++a) { po[a] = inb ? __ldg(b.phi[a] + pk + colo) : 0.0; pn[a] = S.pn[slot(k0 - 1)][a][orow][oc]; }
#pragma unroll
    for (int c = 0; c < NMU; ++c) mu[c] = inb ? __ldg(b.mu[c] + pk + colo) : 0.0;
    MuQ qm;
    mu_cell_q(S.tab[slot(k0 - 1)], po, pn, mu, qm);
    const int s0 = slot(k0 - 1);
#pragma unroll
    for (int a = 0; a < NPH; ++a) {
      qm.gn[a][0] = cgrad(kp, S.pn[s0][a][orow][oc - 1], S.pn[s0][a][orow][oc + 1]);
      qm.gn[a][1] = cgrad(kp, S.pn[s0][a][orow - 1][oc], S.pn[s0][a][orow + 1][oc]);
      qm.gn[a][2] = 0.0;
    }
    RawQ hi = rawq(k0, oc, orow);
    double poc[NPH];
#pragma unroll
    for (int a = 0; a < NPH; ++a) poc[a] = S.po[slot3(k0)][a][orow][oc];
    hi.Mv[0] = mob_of(hi.tab, 0, poc);
    hi.Mv[1] = mob_of(hi.tab, 1, poc);
    mu_face_t(kp, MuQAcc{qm}, hi, 2, fzm);
  }

  for (int k = k0; k < k1; ++k) {
    const int sn = slot(k), s3 = slot3(k);
    // A: mobility of plane k (own + ring cells), then stage plane k+2
    {
      double po[NPH];
#pragma unroll
      for (int a = 0; a < NPH; ++a) po[a] = S.po[s3][a][orow][oc];
      S.M[0][orow][oc] = mob_of(S.tab[sn], 0, po);
      S.M[1][orow][oc] = mob_of(S.tab[sn], 1, po);
      if (ring_thr && !rcorner) {
#pragma unroll
        for (int a = 0; a < NPH; ++a) po[a] = S.po[s3][a][rrow][rcol];
        S.M[0][rrow][rcol] = mob_of(S.tab[sn], 0, po);
        S.M[1][rrow][rcol] = mob_of(S.tab[sn], 1, po);
      }
    }
    if (k + 2 <= k1) stage(k + 2);
    else cp_async_commit();
    cp_async_wait<1>();
    __syncthreads();  // C
    // D: faces of plane k
    double po_c[NPH], pn_c[NPH], mu_c[NMU];
    {
      double f[NMU];
      {  // own -x face
        RawQ lo = rawq(k, oc - 1, orow), hi = rawq(k, oc, orow);
        lo.Mv[0] = S.M[0][orow][oc - 1]; lo.Mv[1] = S.M[1][orow][oc - 1];
        hi.Mv[0] = S.M[0][orow][oc]; hi.Mv[1] = S.M[1][orow][oc];
        mu_face_t(kp, lo, hi, 0, f);
        S.fx[0][ty][tx] = f[0];
        S.fx[1][ty][tx] = f[1];
      }
      {  // own -y face
        RawQ lo = rawq(k, oc, orow - 1), hi = rawq(k, oc, orow);
        lo.Mv[0] = S.M[0][orow - 1][oc]; lo.Mv[1] = S.M[1][orow - 1][oc];
        hi.Mv[0] = S.M[0][orow][oc]; hi.Mv[1] = S.M[1][orow][oc];
        mu_face_t(kp, lo, hi, 1, f);
        S.fy[0][ty][tx] = f[0];
        S.fy[1][ty][tx] = f[1];
      }
      if (tid < TX + TY) {  // far faces: +y of the last row (warp 0), +x of the last column (warp 1)
        const int d = tid < TX ? 1 : 0;
        const int c0 = d == 1 ? tid + 1 : TX, r0 = d == 1 ? TY : tid - TX + 1;
        const int c1 = d == 1 ? c0 : c0 + 1, r1 = d == 1 ? r0 + 1 : r0;
        RawQ lo = rawq(k, c0, r0), hi = rawq(k, c1, r1);
        lo.Mv[0] = S.M[0][r0][c0]; lo.Mv[1] = S.M[1][r0][c0];
        hi.Mv[0] = S.M[0][r1][c1]; hi.Mv[1] = S.M[1][r1][c1];
        mu_face_t(kp, lo, hi, d, f);
        if (d == 0) { S.fx[0][r0 - 1][TX] = f[0]; S.fx[1][r0 - 1][TX] = f[1]; }
        else { S.fy[0][TY][c0 - 1] = f[0]; S.fy[1][TY][c0 - 1] = f[1]; }
      }
    }
    double fzp[NMU];
    {  // z-face k+1/2 of the own column; own values of plane k to registers
      RawQ lo = rawq(k, oc, orow), hi = rawq(k + 1, oc, orow);
      lo.Mv[0] = S.M[0][orow][oc]; lo.Mv[1] = S.M[1][orow][oc];
      double pon[NPH];
#pragma unroll
      for (int a = 0; a < NPH; ++a) {
        pon[a] = S.po[slot3(k + 1)][a][orow][oc];
        po_c[a] = S.po[s3][a][orow][oc];
        pn_c[a] = S.pn[sn][a][orow][oc];
      }
      mu_c[0] = S.mu[s3][0][orow][oc];
      mu_c[1] = S.mu[s3][1][orow][oc];
      hi.Mv[0] = mob_of(hi.tab, 0, pon);
      hi.Mv[1] = mob_of(hi.tab, 1, pon);
      mu_face_t(kp, lo, hi, 2, fzp);
    }
    __syncthreads();  // E
    // F: cell update of (i, j, k)
    if (active) {
      double divf[NMU], out[NMU];
#pragma unroll
      for (int c = 0; c < NMU; ++c)
        divf[c] = ((S.fx[c][ty][tx + 1] - S.fx[c][ty][tx]) + (S.fy[c][ty + 1][tx] - S.fy[c][ty][tx])) +
                  (fzp[c] - fzm[c]);
      mu_cell_update(kp, S.tab[sn], po_c, pn_c, mu_c, divf, out);
      const int64_t o = (int64_t)k * b.plane + colo;
      b.out[0][o] = out[0];
      b.out[1][o] = out[1];
    }
    fzm[0] = fzp[0];
    fzm[1] = fzp[1];
  }
}

void launch_mu_tiled(cudaStream_t s, const KParams &kp, const BlockView &b) {
  const int gx = (b.nx + TX - 1) / TX, gy = (b.ny + TY - 1) / TY;
  const int kz = chunk_z(b.nz, gx * gy);
  dim3 grd(gx, gy, (b.nz + kz - 1) / kz), blk(TX, TY);
  const size_t sm = sizeof(MuSmem);
  static bool attr = false;
  if (!attr) { cudaFuncSetAttribute(mu_tiled_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm); attr = true; }
  mu_tiled_kernel<<<grd, blk, sm, s>>>(kp, b, kz);
}

}  // namespace pf
