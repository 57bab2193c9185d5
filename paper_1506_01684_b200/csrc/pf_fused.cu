// pf_fused.cu — the mu-sweep of step n and the phi-sweep of step n+1 in ONE
// z-marching kernel (Algorithm 1, PAPER.md:158-174, lines 4 and 1 of
// consecutive iterations).
//
// Why they fuse: the phi-sweep reads mu at the cell centre only (D3C1,
// the grand-potential driving force is local in mu), so
// phi^{n+2}(i,j,k) needs, besides the phi^{n+1} stencil, only mu^{n+1}(i,j,k),
// which this thread has just computed.  The phi^{n+1} tiles the mu-sweep stages
// for its anti-trapping stencil (D3C19 with the in-plane corners) are exactly
// the tiles the phi-sweep of step n+1 reads, so each plane is staged once for
// both.  HBM traffic per cell: read phi^n, phi^{n+1}, mu^n, write mu^{n+1},
// phi^{n+2}: 128 B instead of 80 + 96 = 176 B for the two sweeps, and the
// latency-bound mu work interleaves with the FP64-bound phi work in the same
// warps.
//
// Per plane k (two CTA barriers, as in the mu-sweep):
//   A  stage phi^{n+1}(k+2) + both table rows, phi^n / mu^n (k+1) (TMA);
//      mobility of the tile ring; flatness vote of phi^{n+1}_l(k+1)
//   C  __syncthreads
//   D  mu faces of plane k (pf_mu.cu's code) and phi faces of plane k on
//      phi^{n+1} (pf_phi.cu's code), the own cell's centre differences
//   E  __syncthreads
//   F  mu^{n+1}(k) = mu cell update; phi^{n+2}(k) = phi cell update with that
//      mu^{n+1}; both stored
// Every face and cell routine is the pinned code of pf_dev.cuh, in the same
// expression order as the two separate sweeps: the results are bitwise those
// of pf_mu.cu followed by pf_phi.cu (tests/test_gpu_fused.py).
#include "pf_kernels.cuh"
#define PF_TILE_X FUSED_TILE_X
#define PF_TILE_Y FUSED_TILE_Y
#include "pf_tile.cuh"

namespace pf {
namespace {

#ifndef PF_FUSED_PM_SLOTS
#define PF_FUSED_PM_SLOTS 2
#endif
constexpr int FPM = PF_FUSED_PM_SLOTS;
// mu x faces: the +x face of a cell is the own -x face of the next lane in its
// TX-wide row segment of the warp (shuffle); shared memory keeps the far column
#ifndef PF_FUSED_SHFL
#define PF_FUSED_SHFL 0
#endif
constexpr bool kFShfl = PF_FUSED_SHFL != 0 && (TX == 16 || TX == 32);   // phi^n / mu slots: planes k .. k+FPM-1 (staged FPM-1 ahead)
// (3 slots measured slower: 7.67 vs 6.33 ms at 512^3 — the extra 6.6 KB costs the third CTA per SM)
template <bool ANISO>
struct __align__(128) FusedSmemT {
  double pn[NSLOT][NPH][TSZ];     // phi^{n+1}, planes k-1 .. k+2
  double po[FPM][NPH][TSZ];       // phi^n, planes k .. k+FPM-1
  double mu[FPM][NMU][TSZ];       // mu^n
  double tab[NSLOT][TAB];         // table rows of step n (mu part)
  double tabp[NSLOT][TAB];        // table rows of step n+1 (phi part)
  double M[NMU][RY][RX];          // mobility of plane k
  double fx[NMU][TY][kFShfl ? 1 : TX + 1];   // mu x-face values at i - 1/2 (kFShfl: the far column only)
  double fy[NMU][TY + 1][TX];     // mu y-face values at j - 1/2
  double pfx[NPH][TY][TX + 1];    // phi x-face fluxes
  double pfy[NPH][TY + 1][TX];    // phi y-face fluxes
  double jz[ANISO ? NPH : 1][TY][TX];   // anisotropic: the phi z-face carry (thread-private)
  uint64_t bar_pn[NSLOT];
  uint64_t bar_pm[FPM];
  uint32_t wflat[3][NTHR / 32];
};
constexpr int NBOX = RX * RY;
static_assert(NBOX <= 2 * NTHR, "flatness check covers the box in two passes");
constexpr uint32_t F_PN_BYTES = (NPH * RXS * RY + 2 * TAB) * 8;   // phi^{n+1} tiles + two table rows
constexpr uint32_t F_PM_BYTES = ((NPH + NMU) * RXS * RY) * 8;    // phi^n + mu tiles
#define T(arr, row, col) TILE_AT(arr, row, col)

// accessors over the staged planes (pf_mu.cu's RawQ / ColQ on this layout)
template <class SM>
struct FRawQ {
  const SM &S;
  int snm, sn, snp, s2, col, row;
  const double *tb;
  double Mv[NMU];
  __device__ __forceinline__ double pn(int a) const { return T(S.pn[sn][a], row, col); }
  __device__ __forceinline__ double dp(int a) const { return RN_SUB(T(S.pn[sn][a], row, col), T(S.po[s2][a], row, col)); }
  __device__ __forceinline__ double gt(int a, int e) const {
    if (e == 0) return cdiff(T(S.pn[sn][a], row, col - 1), T(S.pn[sn][a], row, col + 1));
    if (e == 1) return cdiff(T(S.pn[sn][a], row - 1, col), T(S.pn[sn][a], row + 1, col));
    return cdiff(T(S.pn[snm][a], row, col), T(S.pn[snp][a], row, col));
  }
  __device__ __forceinline__ double M(int c) const { return Mv[c]; }
  __device__ __forceinline__ double mu(int c) const { return T(S.mu[s2][c], row, col); }
  __device__ __forceinline__ double dcl(int a, int c) const { return dcl_of(tb, a, c, mu(c)); }
  __device__ __forceinline__ const double *tab() const { return tb; }
};
template <class SM>
struct FColQ {
  const SM &S;
  int sc, col, row;
  const double *tb;
  const double *po, *muv;
  double Mv[NMU];
  __device__ __forceinline__ double pn(int a) const { return T(S.pn[sc][a], row, col); }
  __device__ __forceinline__ double dp(int a) const { return RN_SUB(T(S.pn[sc][a], row, col), po[a]); }
  __device__ __forceinline__ double gt(int a, int e) const {
    if (e == 0) return cdiff(T(S.pn[sc][a], row, col - 1), T(S.pn[sc][a], row, col + 1));
    return cdiff(T(S.pn[sc][a], row - 1, col), T(S.pn[sc][a], row + 1, col));
  }
  __device__ __forceinline__ double M(int c) const { return Mv[c]; }
  __device__ __forceinline__ double mu(int c) const { return muv[c]; }
  __device__ __forceinline__ double dcl(int a, int c) const { return dcl_of(tb, a, c, muv[c]); }
  __device__ __forceinline__ const double *tab() const { return tb; }
};

#ifndef PF_FUSED_UNROLL
#define PF_FUSED_UNROLL 1
#endif
// plane-loop unroll (measured at 512^3, isotropic: 1 -> 6.36 ms, 2 -> 6.45, 4 -> 7.41)
constexpr int kFusedUnroll = PF_FUSED_UNROLL;
// the three solids of an x/y face's anti-trapping current in a rolled loop (1) or unrolled (0), as pf_mu.cu
// (here the rolled loop measured faster: 6.31 vs 6.40 ms at 512^3 — the fused kernel's code is twice the size)
#ifndef PF_FUSED_ROLL
#define PF_FUSED_ROLL 1
#endif
constexpr bool kFRoll = PF_FUSED_ROLL != 0;
// 3 CTAs of 128 threads per SM (166 registers; 2 CTAs: 7.78 ms vs 6.45)
#ifndef PF_FUSED_MINB
#define PF_FUSED_MINB (384 / NTHR)
#endif

// SC: 0 no region-shortcut code, 2 the skip-faces vote of pf_phi.cu
template <bool ANISO, int DM, int SC>
__global__ void __launch_bounds__(NTHR, PF_FUSED_MINB)
    fused_kernel(const __grid_constant__ TmaMaps tm, KParams kp, BlockView b, FusedOut fo, int kz) {
  using Smem = FusedSmemT<ANISO>;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  Smem &S = *reinterpret_cast<Smem *>(smem_raw);
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
#define PF_AN (ANISO ? 1 : 0), DM

  auto slot = [&](int k) { return (k - k0 + 1) & (NSLOT - 1); };
  auto par4 = [&](int k) { return (uint32_t)(((k - k0 + 1) >> 2) & 1); };
  auto slot2 = [&](int k) { return FPM == 2 ? (k - k0) & 1 : (k - k0) % FPM; };
  auto par2 = [&](int k) { return (uint32_t)(((k - k0) / FPM) & 1); };
  const int bx = i0 - 2 + XO, by = j0;
  auto stage_pn = [&](int k) {   // phi^{n+1} tiles + the two table rows of plane k
    const int s = slot(k);
    mbar_expect_tx(&S.bar_pn[s], F_PN_BYTES);
#pragma unroll
    for (int a = 0; a < NPH; ++a) tma_load_3d(S.pn[s][a], &tm.phin[a], bx, by, k + b.zoff, &S.bar_pn[s]);
    bulk_load(S.tab[s], b.tab + (int64_t)k * TAB, TAB * 8, &S.bar_pn[s]);
    bulk_load(S.tabp[s], fo.tabp + (int64_t)k * TAB, TAB * 8, &S.bar_pn[s]);
  };
  auto stage_pm = [&](int k) {   // phi^n and mu tiles of plane k
    const int s = slot2(k);
    mbar_expect_tx(&S.bar_pm[s], F_PM_BYTES);
#pragma unroll
    for (int a = 0; a < NPH; ++a) tma_load_3d(S.po[s][a], &tm.phi[a], bx, by, k + b.zoff, &S.bar_pm[s]);
#pragma unroll
    for (int c = 0; c < NMU; ++c) tma_load_3d(S.mu[s][c], &tm.mu[c], bx, by, k + b.zoff, &S.bar_pm[s]);
  };
  const int vq0 = tid, vq1 = tid + NTHR;
  const int vo[2] = {(vq0 / RX) * RXS + vq0 % RX + 1, (vq1 / RX) * RXS + vq1 % RX + 1};
  auto vote_flat = [&](int k, int e) {
    const double *pl = S.pn[slot(k)][LIQ];
    bool one = true, zero = true;
#pragma unroll
    for (int r = 0; r < 2; ++r) {
      if (tid + r * NTHR < NBOX) {
        const double v = pl[vo[r]];
        one = one && v == 1.0;
        zero = zero && v == 0.0;
      }
    }
    const uint32_t f = (__all_sync(0xffffffffu, one) ? 1u : 0u) | (__all_sync(0xffffffffu, zero) ? 2u : 0u);
    if ((tid & 31) == 0) S.wflat[e][tid >> 5] = f;
  };
  // (a REDUX over the warps' votes as in pf_mu.cu measured +0.4 % here)
  auto read_flat = [&](int e) {
    uint32_t f = 3u;
#pragma unroll
    for (int w = 0; w < NTHR / 32; ++w) f &= S.wflat[e][w];
    return f;
  };
  auto rawq = [&](int k, int col, int row) {
    return FRawQ<Smem>{S, slot(k - 1), slot(k), slot(k + 1), slot2(k), col, row, S.tab[slot(k)], {0.0, 0.0}};
  };
  auto own_load = [&](int k, double po[NPH], double mu[NMU]) {
    const int64_t pk = (int64_t)k * b.plane;
#pragma unroll
    for (int a = 0; a < NPH; ++a) po[a] = inb ? __ldg(b.phi[a] + pk + colo) : 0.0;
#pragma unroll
    for (int c = 0; c < NMU; ++c) mu[c] = inb ? __ldg(b.mu[c] + pk + colo) : 0.0;
  };
  auto own_q = [&](int k, const double po[NPH], const double mu[NMU], MuQ &q) {
    const int sc = slot(k);
    double pn[NPH];
#pragma unroll
    for (int a = 0; a < NPH; ++a) pn[a] = T(S.pn[sc][a], orow, oc);
    mu_cell_q(S.tab[sc], po, pn, mu, q);
#pragma unroll
    for (int a = 0; a < NPH; ++a) {
      q.gn[a][0] = cdiff(T(S.pn[sc][a], orow, oc - 1), T(S.pn[sc][a], orow, oc + 1));
      q.gn[a][1] = cdiff(T(S.pn[sc][a], orow - 1, oc), T(S.pn[sc][a], orow + 1, oc));
      q.gn[a][2] = 0.0;
    }
  };
  // phi part: raw centre differences of tile cell (col,row) of the phi^{n+1}
  // planes (component d unused), as pf_phi.cu's tan_grad
  auto tan_grad = [&](int sc, int sm, int sp, int col, int row, int d, double g[NPH][3]) {
#pragma unroll
    for (int a = 0; a < NPH; ++a) {
      g[a][0] = d == 0 ? 0.0 : cdiff(T(S.pn[sc][a], row, col - 1), T(S.pn[sc][a], row, col + 1));
      g[a][1] = d == 1 ? 0.0 : cdiff(T(S.pn[sc][a], row - 1, col), T(S.pn[sc][a], row + 1, col));
      g[a][2] = d == 2 ? 0.0 : cdiff(T(S.pn[sm][a], row, col), T(S.pn[sp][a], row, col));
    }
  };
  double gdum[NPH][3];
#pragma unroll
  for (int a = 0; a < NPH; ++a)
#pragma unroll
    for (int e = 0; e < 3; ++e) gdum[a][e] = 0.0;

  // ---- prologue
  if (tid == 0) {
    for (int q = 0; q < NSLOT; ++q) mbar_init(&S.bar_pn[q], 1);
    for (int q = 0; q < FPM; ++q) mbar_init(&S.bar_pm[q], 1);
    mbar_fence_init();
  }
  __syncthreads();
  if (tid == ISSUER) {
    stage_pn(k0 - 1);
    stage_pn(k0);
    stage_pn(k0 + 1);
    stage_pm(k0);
    if (FPM > 2 && k0 + 1 < k1) stage_pm(k0 + 1);
  }
  double fzm[NMU], po_n[NPH], mu_n[NMU], Mown[NMU];
  double jzm[NPH];   // phi z-face k - 1/2 (isotropic: registers; anisotropic: S.jz)
  {
    double pom[NPH], mum[NMU];
    own_load(k0 - 1, pom, mum);
    own_load(k0, po_n, mu_n);
    mbar_wait(&S.bar_pn[slot(k0 - 1)], par4(k0 - 1));
    mbar_wait(&S.bar_pn[slot(k0)], par4(k0));
    mbar_wait(&S.bar_pn[slot(k0 + 1)], par4(k0 + 1));
    MuQ qm, qc;
    own_q(k0 - 1, pom, mum, qm);
    own_q(k0, po_n, mu_n, qc);
    Mown[0] = qc.M[0];
    Mown[1] = qc.M[1];
    mu_face_t<true>(kp, MuQAcc{qm}, MuQAcc{qc}, 2, fzm);
    vote_flat(k0 - 1, 0);
    vote_flat(k0, 1);
    // phi z-face k0 - 1/2 on phi^{n+1}
    const int s0 = slot(k0 - 1), s1 = slot(k0);
    double lo[NPH], hi[NPH], gl[NPH][3], gh[NPH][3];
#pragma unroll
    for (int a = 0; a < NPH; ++a) { lo[a] = T(S.pn[s0][a], orow, oc); hi[a] = T(S.pn[s1][a], orow, oc); }
    if (ANISO) {
      tan_grad(s0, s0, s0, oc, orow, 2, gl);
      tan_grad(s1, s1, s1, oc, orow, 2, gh);
    }
    phi_face<PF_AN>(kp, lo, hi, ANISO ? gl : gdum, ANISO ? gh : gdum, 2, jzm);
    if (ANISO)
#pragma unroll
      for (int a = 0; a < NPH; ++a) S.jz[a][ty][tx] = jzm[a];
  }
  __syncthreads();
  uint32_t flm = read_flat(0), flc = read_flat(1), flp;
  int fe = 2;

#pragma unroll kFusedUnroll
  for (int k = k0; k < k1; ++k) {
    const int sn = slot(k), s2 = slot2(k), sm = slot(k - 1), sp = slot(k + 1);
    const bool more = k + 1 < k1;
    // A
    if (tid == ISSUER) {
      if (k + 2 <= k1) stage_pn(k + 2);
      if (FPM == 2 ? more : k + FPM - 1 < k1) stage_pm(k + FPM - 1);
    }
    double po_c[NPH], mu_c[NMU];
#pragma unroll
    for (int a = 0; a < NPH; ++a) po_c[a] = po_n[a];
#pragma unroll
    for (int c = 0; c < NMU; ++c) mu_c[c] = mu_n[c];
    own_load(k + 1, po_n, mu_n);
    mbar_wait(&S.bar_pm[s2], par2(k));
    S.M[0][orow][oc] = Mown[0];
    S.M[1][orow][oc] = Mown[1];
    if (ring_thr && !rcorner) {
      double po[NPH], M[NMU];
#pragma unroll
      for (int a = 0; a < NPH; ++a) po[a] = T(S.po[s2][a], rrow, rcol);
      mob2(S.tab[sn], po, M);
      S.M[0][rrow][rcol] = M[0];
      S.M[1][rrow][rcol] = M[1];
    }
    if (k > k0) mbar_wait(&S.bar_pn[sp], par4(k + 1));
    vote_flat(k + 1, fe);
    __syncthreads();  // C
    flp = read_flat(fe);
    fe = fe == 2 ? 0 : fe + 1;
    const bool fast_xy = ((flm & flc & flp) & 1u) || (flc & 2u);
    const bool fast_z = ((flc & flp) & 1u) || ((flc & flp) & 2u);
    flm = flc;
    flc = flp;

    // D (mu): faces of plane k
    double fxo[NMU] = {0.0, 0.0}, fyo[NMU] = {0.0, 0.0};
    if (fast_xy) {
#pragma unroll
      for (int c = 0; c < NMU; ++c) {
        fxo[c] = mu_flux_diff(kp, S.M[c][orow][oc - 1], Mown[c], T(S.mu[s2][c], orow, oc - 1), mu_c[c]);
        fyo[c] = mu_flux_diff(kp, S.M[c][orow - 1][oc], Mown[c], T(S.mu[s2][c], orow - 1, oc), mu_c[c]);
        if (!kFShfl) S.fx[c][ty][tx] = fxo[c];
        S.fy[c][ty][tx] = fyo[c];
      }
      if (tid < TX + TY) {
        const int d = tid < TX ? 1 : 0;
        const int c0 = d == 1 ? tid + 1 : TX, r0 = d == 1 ? TY : tid - TX + 1;
        const int c1 = d == 1 ? c0 : c0 + 1, r1 = d == 1 ? r0 + 1 : r0;
#pragma unroll
        for (int c = 0; c < NMU; ++c) {
          const double f = mu_flux_diff(kp, S.M[c][r0][c0], S.M[c][r1][c1], T(S.mu[s2][c], r0, c0),
                                        T(S.mu[s2][c], r1, c1));
          if (d == 0) S.fx[c][r0 - 1][kFShfl ? 0 : TX] = f;
          else S.fy[c][TY][c0 - 1] = f;
        }
      }
    } else {
      double f[NMU];
      {
        auto lo = rawq(k, oc - 1, orow), hi = rawq(k, oc, orow);
        lo.Mv[0] = S.M[0][orow][oc - 1]; lo.Mv[1] = S.M[1][orow][oc - 1];
        hi.Mv[0] = Mown[0]; hi.Mv[1] = Mown[1];
        mu_face_t<true, kFRoll>(kp, lo, hi, 0, fxo);
        if (!kFShfl) {
          S.fx[0][ty][tx] = fxo[0];
          S.fx[1][ty][tx] = fxo[1];
        }
      }
      {
        auto lo = rawq(k, oc, orow - 1), hi = rawq(k, oc, orow);
        lo.Mv[0] = S.M[0][orow - 1][oc]; lo.Mv[1] = S.M[1][orow - 1][oc];
        hi.Mv[0] = Mown[0]; hi.Mv[1] = Mown[1];
        mu_face_t<true, kFRoll>(kp, lo, hi, 1, fyo);
        S.fy[0][ty][tx] = fyo[0];
        S.fy[1][ty][tx] = fyo[1];
      }
      if (tid < TX + TY) {
        const int d = tid < TX ? 1 : 0;
        const int c0 = d == 1 ? tid + 1 : TX, r0 = d == 1 ? TY : tid - TX + 1;
        const int c1 = d == 1 ? c0 : c0 + 1, r1 = d == 1 ? r0 + 1 : r0;
        auto lo = rawq(k, c0, r0), hi = rawq(k, c1, r1);
        lo.Mv[0] = S.M[0][r0][c0]; lo.Mv[1] = S.M[1][r0][c0];
        hi.Mv[0] = S.M[0][r1][c1]; hi.Mv[1] = S.M[1][r1][c1];
        mu_face_t<true, kFRoll>(kp, lo, hi, d, f);
        if (d == 0) { S.fx[0][r0 - 1][kFShfl ? 0 : TX] = f[0]; S.fx[1][r0 - 1][kFShfl ? 0 : TX] = f[1]; }
        else { S.fy[0][TY][c0 - 1] = f[0]; S.fy[1][TY][c0 - 1] = f[1]; }
      }
    }
    double fzp[NMU], pn_c[NPH], Mnx[NMU] = {0.0, 0.0};
    if (fast_z) {
      mob2(S.tab[sp], po_n, Mnx);
#pragma unroll
      for (int c = 0; c < NMU; ++c) fzp[c] = mu_flux_diff(kp, Mown[c], Mnx[c], mu_c[c], mu_n[c]);
    } else {
      auto lo = rawq(k, oc, orow);
      lo.Mv[0] = Mown[0]; lo.Mv[1] = Mown[1];
      FColQ<Smem> hi{S, sp, oc, orow, S.tab[sp], po_n, mu_n, {0.0, 0.0}};
      mob2(S.tab[sp], po_n, hi.Mv);
      mu_face_t<true>(kp, lo, hi, 2, fzp);
      Mnx[0] = hi.Mv[0];
      Mnx[1] = hi.Mv[1];
    }
#pragma unroll
    for (int a = 0; a < NPH; ++a) pn_c[a] = T(S.pn[sn][a], orow, oc);
    double dpart[NMU], fxp[NMU];   // fxp: the +x face from the next lane (kFShfl)
#pragma unroll
    for (int c = 0; c < NMU; ++c) {
      fxp[c] = kFShfl ? __shfl_down_sync(0xffffffffu, fxo[c], 1, TX) : 0.0;
      dpart[c] = ((fzp[c] - fzm[c]) - fxo[c]) - fyo[c];
      fzm[c] = fzp[c];
      Mown[c] = Mnx[c];
    }

    // D (phi of step n+1): faces of plane k on phi^{n+1}; the own cell's centre
    // differences (read before E: slot(k-1) is refilled at A(k+1))
    // region shortcut (SC = 2, pf_set_shortcuts; pf_phi.cu's vote on phi^{n+1}):
    // a warp whose cells are simplex vertices with an identical D3C7 (D3C19)
    // neighbourhood has exactly zero own faces and keeps phi^{n+2} = phi^{n+1}
    bool skip = false;
    if (SC == 2) {
      if (__all_sync(0xffffffffu, is_vertex_bits(pn_c) || !active)) {
        auto same = [](double x, double v) { return __double_as_longlong(x) == __double_as_longlong(v); };
        bool mine = true;
#pragma unroll
        for (int a = 0; a < NPH; ++a) {
          const double v = pn_c[a];
          mine = mine && same(T(S.pn[sn][a], orow, oc - 1), v) && same(T(S.pn[sn][a], orow, oc + 1), v) &&
                 same(T(S.pn[sn][a], orow - 1, oc), v) && same(T(S.pn[sn][a], orow + 1, oc), v) &&
                 same(T(S.pn[sm][a], orow, oc), v) && same(T(S.pn[sp][a], orow, oc), v);
          if (ANISO)
            mine = mine && same(T(S.pn[sn][a], orow - 1, oc - 1), v) && same(T(S.pn[sn][a], orow - 1, oc + 1), v) &&
                   same(T(S.pn[sn][a], orow + 1, oc - 1), v) && same(T(S.pn[sn][a], orow + 1, oc + 1), v) &&
                   same(T(S.pn[sm][a], orow, oc - 1), v) && same(T(S.pn[sm][a], orow, oc + 1), v) &&
                   same(T(S.pn[sm][a], orow - 1, oc), v) && same(T(S.pn[sm][a], orow + 1, oc), v) &&
                   same(T(S.pn[sp][a], orow, oc - 1), v) && same(T(S.pn[sp][a], orow, oc + 1), v) &&
                   same(T(S.pn[sp][a], orow - 1, oc), v) && same(T(S.pn[sp][a], orow + 1, oc), v);
        }
        skip = __all_sync(0xffffffffu, mine || !active) != 0;
      }
    }
    double gc[NPH][3], jzp[NPH], dpp[NPH];
    {
      double jf[NPH], lo[NPH], hi[NPH], gl[NPH][3], gh[NPH][3];
      auto far_faces = [&]() {
        if (tid < TX + TY) {
          const int d = tid < TX ? 1 : 0;
          const int c0 = d == 1 ? tid + 1 : TX, r0 = d == 1 ? TY : tid - TX + 1;
          const int c1 = d == 1 ? c0 : c0 + 1, r1 = d == 1 ? r0 + 1 : r0;
#pragma unroll
          for (int a = 0; a < NPH; ++a) { lo[a] = T(S.pn[sn][a], r0, c0); hi[a] = T(S.pn[sn][a], r1, c1); }
          if (ANISO) {
            tan_grad(sn, sm, sp, c0, r0, d, gl);
            tan_grad(sn, sm, sp, c1, r1, d, gh);
          }
          phi_face<PF_AN>(kp, lo, hi, ANISO ? gl : gdum, ANISO ? gh : gdum, d, jf);
#pragma unroll
          for (int a = 0; a < NPH; ++a) {
            if (d == 0) S.pfx[a][r0 - 1][TX] = jf[a];
            else S.pfy[a][TY][c0 - 1] = jf[a];
          }
        }
      };
      if (SC == 2 && skip) {   // own faces exactly 0; the far faces as usual
#pragma unroll
        for (int a = 0; a < NPH; ++a) {
          jzp[a] = 0.0;
          dpp[a] = 0.0;
          if (!ANISO) jzm[a] = 0.0;
          S.pfx[a][ty][tx] = 0.0;
          S.pfy[a][ty][tx] = 0.0;
        }
        far_faces();
      } else {
      if (ANISO) tan_grad(sn, sm, sp, oc, orow, -1, gc);   // gown: the own cell's raw differences
      double pp[NPH];
#pragma unroll
      for (int a = 0; a < NPH; ++a) pp[a] = T(S.pn[sp][a], orow, oc);
      if (!ANISO) far_faces();
      if (ANISO) {
        tan_grad(sp, sp, sp, oc, orow, 2, gh);
        phi_face<PF_AN>(kp, pn_c, pp, gc, gh, 2, jzp);
      } else {
        phi_face<PF_AN>(kp, pn_c, pp, gdum, gdum, 2, jzp);
#pragma unroll
        for (int a = 0; a < NPH; ++a) {
          dpp[a] = jzp[a] - jzm[a];
          jzm[a] = jzp[a];
        }
      }
#pragma unroll
      for (int d = 0; d < 2; ++d) {
        const int lc = d == 0 ? oc - 1 : oc, lr = d == 0 ? orow : orow - 1;
#pragma unroll
        for (int a = 0; a < NPH; ++a) {
          lo[a] = T(S.pn[sn][a], lr, lc);
          hi[a] = ANISO ? T(S.pn[sn][a], orow, oc) : pn_c[a];
        }
        if (ANISO) tan_grad(sn, sm, sp, lc, lr, d, gl);
        phi_face<PF_AN>(kp, lo, hi, ANISO ? gl : gdum, ANISO ? gc : gdum, d, jf);
#pragma unroll
        for (int a = 0; a < NPH; ++a) {
          if (d == 0) S.pfx[a][ty][tx] = jf[a];
          else S.pfy[a][ty][tx] = jf[a];
          if (!ANISO) dpp[a] -= jf[a];
        }
      }
      if (ANISO) far_faces();
      if (!ANISO)
#pragma unroll
        for (int a = 0; a < NPH; ++a) {
          gc[a][0] = T(S.pn[sn][a], orow, oc + 1) - T(S.pn[sn][a], orow, oc - 1);
          gc[a][1] = T(S.pn[sn][a], orow + 1, oc) - T(S.pn[sn][a], orow - 1, oc);
          gc[a][2] = pp[a] - T(S.pn[sm][a], orow, oc);
        }
      }
    }
    __syncthreads();  // E: the faces of plane k (both fields) complete
    // F: mu^{n+1}(i,j,k), then phi^{n+2}(i,j,k) with it
    if (active) {
      double divf[NMU], mu1[NMU];
#pragma unroll
      for (int c = 0; c < NMU; ++c)
        divf[c] = dpart[c] + ((kFShfl ? (tx == TX - 1 ? S.fx[c][ty][0] : fxp[c]) : S.fx[c][ty][tx + 1]) +
                              S.fy[c][ty + 1][tx]);
      const int64_t o = (int64_t)k * b.plane + colo;
      mu_cell_update(kp, S.tab[sn], po_c, pn_c, mu_c, divf, mu1);
      st_field(&b.out[0][o], mu1[0]);
      st_field(&b.out[1][o], mu1[1]);
      if (SC == 2 && skip) {
#pragma unroll
        for (int a = 0; a < NPH; ++a) st_field(&fo.phi2[a][o], pn_c[a]);
      } else {
      const double *tp = S.tabp[sn];
      double r0[NPH], q[NPH];
      phi_cell_rhs0<PF_AN>(kp, tp, pn_c, mu1, gc, r0);
      const double c = tp[ANISO ? T_EPSTDX16 : T_EPSTDX];
      if (ANISO) {
#pragma unroll
        for (int a = 0; a < NPH; ++a) {
          dpp[a] = (jzp[a] - S.jz[a][ty][tx]) - S.pfx[a][ty][tx] - S.pfy[a][ty][tx];
          q[a] = r0[a] - c * dpp[a];
        }
      } else {
#pragma unroll
        for (int a = 0; a < NPH; ++a) q[a] = r0[a] - c * dpp[a];
      }
      double rhs[NPH], out[NPH];
#pragma unroll
      for (int a = 0; a < NPH; ++a) rhs[a] = q[a] - c * (S.pfx[a][ty][tx + 1] + S.pfy[a][ty + 1][tx]);
      phi_cell_project(kp, pn_c, rhs, out);
#pragma unroll
      for (int a = 0; a < NPH; ++a) st_field(&fo.phi2[a][o], out[a]);
      }
    }
    if (ANISO)
#pragma unroll
      for (int a = 0; a < NPH; ++a) S.jz[a][ty][tx] = jzp[a];
  }
#undef PF_AN
}
#undef T

constexpr int DM_SL = (1 << pair_of(0, LIQ)) | (1 << pair_of(1, LIQ)) | (1 << pair_of(2, LIQ));
int g_fused_slots[2] = {1, 1};

}  // namespace

void prepare_fused() {
  const int sa = (int)sizeof(FusedSmemT<true>), si = (int)sizeof(FusedSmemT<false>);
  cudaFuncSetAttribute(fused_kernel<false, -1, 0>, cudaFuncAttributeMaxDynamicSharedMemorySize, si);
  cudaFuncSetAttribute(fused_kernel<false, -1, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, si);
  cudaFuncSetAttribute(fused_kernel<true, -1, 0>, cudaFuncAttributeMaxDynamicSharedMemorySize, sa);
  cudaFuncSetAttribute(fused_kernel<true, -1, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, sa);
  cudaFuncSetAttribute(fused_kernel<true, DM_SL, 0>, cudaFuncAttributeMaxDynamicSharedMemorySize, sa);
  g_fused_slots[0] = grid_slots(fused_kernel<false, -1, 0>, NTHR, si);
  g_fused_slots[1] = grid_slots(fused_kernel<true, -1, 0>, NTHR, sa);
}

void launch_fused(cudaStream_t s, const KParams &kp, const BlockView &b, const TmaMaps &tm, const FusedOut &fo) {
  const int gx = (b.nx + TX - 1) / TX, gy = (b.ny + TY - 1) / TY;
// z-chunks for >= 16 waves of resident CTAs (measured: 8 -> 6.45 ms, 16 -> 6.39, 32 -> 6.40)
#ifndef PF_FUSED_WAVES
#define PF_FUSED_WAVES 16
#endif
  const int kz = chunk_z(b.nz, gx * gy, g_fused_slots[kp.aniso ? 1 : 0], PF_FUSED_WAVES, true);
  dim3 grd(gx, gy, (b.nz + kz - 1) / kz), blk(TX, TY);
  // shortcuts on: the vote variants, except the solid-liquid anisotropic model
  // (pf_phi.cu: its vote measured slower in every scenario; bitwise the same)
  const size_t si = sizeof(FusedSmemT<false>), sa = sizeof(FusedSmemT<true>);
  if (!kp.aniso) {
    if (kp.shortcuts) fused_kernel<false, -1, 2><<<grd, blk, si, s>>>(tm, kp, b, fo, kz);
    else fused_kernel<false, -1, 0><<<grd, blk, si, s>>>(tm, kp, b, fo, kz);
  } else if (kp.dmask == DM_SL) {
    fused_kernel<true, DM_SL, 0><<<grd, blk, sa, s>>>(tm, kp, b, fo, kz);
  } else if (kp.shortcuts) {
    fused_kernel<true, -1, 2><<<grd, blk, sa, s>>>(tm, kp, b, fo, kz);
  } else {
    fused_kernel<true, -1, 0><<<grd, blk, sa, s>>>(tm, kp, b, fo, kz);
  }
}

}  // namespace pf
