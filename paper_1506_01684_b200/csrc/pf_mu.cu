// pf_mu.cu — production mu-sweep (Eq. (3)-(4)): z-marching
// 2.5D tiles; every staggered value M grad mu - J_at (the
// "computationally most intensive part") is evaluated once per face.
//
// Shared memory per CTA (2 CTAs / SM), filled by TMA bulk-tensor copies issued
// by one thread and guarded by mbarriers:
//   * phi^{n+1} tile planes k-1 .. k+2 (interior + ring + corners: the D3C19
//     stencil of the anti-trapping current needs tangential gradients at face
//     neighbours) — staged two planes ahead, 4 slots;
//   * phi^n and mu tile planes k .. k+2 — staged two planes ahead, 3 slots;
//   * table rows; the mobility of plane k (computed once per cell); the x/y
//     face values of plane k (x faces: only the far column; the rest by shuffle).
// Everything else a face needs (dphi, c^l - c^a, tangential gradients) is
// derived from the staged planes inside the face routine, and only when the
// exact-zero guards let the anti-trapping term through.  Flat planes: when the
// staged phi^{n+1}_l tiles make every guard of a plane's faces close (pure
// liquid over planes k-1..k+1, or no liquid in the face cells), the CTA takes
// the diffusive flux only — decided CTA-uniformly per plane from the staged
// tiles, bitwise identical to the guarded path.  z-faces are carried
// in registers; the own column's phi^n / mu at k+1 (the z-face's upper cell)
// come from registers.  All arithmetic is the pinned code of pf_dev.cuh, so
// results do not depend on tile or block boundaries.
#include <type_traits>
#include "pf_kernels.cuh"
#define PF_TILE_X MU_TILE_X
#define PF_TILE_Y MU_TILE_Y
#include "pf_tile.cuh"

namespace pf {

#ifndef PF_MU_PM_SLOTS
#define PF_MU_PM_SLOTS 3
#endif
// phi^n / mu tile slots: 2 = staged one plane ahead, 3 = two planes ahead
// (measured at 512^3: with 32 x 16 tiles, one CTA per SM, the second plane of
// lead takes C4 from 3.61 to 3.42 ms; 32 x 8 with three slots fits 2 CTAs per SM
// only since the x faces travel by shuffle (kShfl, 4 KB less): C4 3.08 -> 2.97 ms)
constexpr int NPM = PF_MU_PM_SLOTS;
// x faces: with TX = 32 a warp is one tile row, so the +x face of a cell is the
// own -x face of the next lane (a shuffle) and shared memory keeps only the
// tile's far column (the +x faces of the last lane): 4 KB less per CTA
#ifndef PF_MU_SHFL
#define PF_MU_SHFL 1
#endif
constexpr bool kShfl = PF_MU_SHFL != 0 && TX == 32;
// (measured: C4 2.958 vs 2.933 ms, all-guards-open 9.37 vs 9.39: off by default)
#ifndef PF_MU_FAR_CONST
#define PF_MU_FAR_CONST 0
#endif

struct __align__(128) MuSmem {
  double pn[NSLOT][NPH][TSZ];     // phi^{n+1}, planes k-1 .. k+2
  double po[NPM][NPH][TSZ];       // phi^n, planes k .. k+NPM-1
  double mu[NPM][NMU][TSZ];       // mu^n
  double tab[NSLOT][TAB];
  double M[NMU][RY][RX];          // mobility of plane k
  double fx[NMU][TY][kShfl ? 1 : TX + 1];   // x-face values at i - 1/2 (kShfl: the far column i = TX only)
  double fy[NMU][TY + 1][TX];     // y-face values at j - 1/2
  uint64_t bar_pn[NSLOT];         // phi^{n+1} + table of a plane
  uint64_t bar_pm[NPM];           // phi^n + mu of a plane
  uint32_t wflat[3][NTHR / 32];   // per-warp flatness votes of a staged phi^{n+1}_l plane
};
#ifndef PF_MU_UNROLL
#define PF_MU_UNROLL 4
#endif
#ifndef PF_MU_ROLL
#define PF_MU_ROLL 0
#endif
// x/y faces (both cells in shared memory): PF_MU_ROLL = 1 puts the three
// solids of the anti-trapping current in a loop that is not unrolled — a
// third of the code (measured on the all-guards-open state, round 2: 13.6 ->
// 10.8 ms; C4 unchanged).  With the x faces by shuffle and the two-plane lead
// the unrolled solids measured faster on both states (C4 2.960 -> 2.933 ms,
// all-guards-open 9.86 -> 9.39 ms): 0 is the default
constexpr bool kMuRoll = PF_MU_ROLL != 0;
constexpr int kMuUnroll = PF_MU_UNROLL;   // plane-loop unroll (round 1: 2 -> 4 -0.8 %; with the rolled anti-trapping
                                          // solids and the library-call fallback, 4 spilled: C4 3.78 vs 3.15 ms; without
                                          // the fallback (R31): 4 vs 2 C4 3.104 vs 3.127, interface 9.97 vs 10.39;
                                          // 3: 3.129 / 10.46, 8: 3.46 / 11.5; 4 unrolled solids: 3.161 / 9.48)
constexpr int NBOX = RX * RY;     // staged cells of a plane tile (interior + ring + corners)
static_assert(NBOX <= 2 * NTHR, "flatness check covers the box in two passes");
#define T(arr, row, col) TILE_AT(arr, row, col)
#define FX_FAR(c, r) S.fx[c][r][kShfl ? 0 : TX]
constexpr uint32_t MU_PN_BYTES = (NPH * RXS * RY + TAB) * 8;   // phi^{n+1} tiles + table row
constexpr uint32_t MU_PM_BYTES = ((NPH + NMU) * RXS * RY) * 8;  // phi^n + mu tiles

// Accessor over the staged planes for tile cell (col,row) of plane k:
// phi^{n+1} slots (k-1, k, k+1) = (snm, sn, snp), phi^n/mu slot s2, table row.
struct RawQ {
  const MuSmem &S;
  const KParams &kp;
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

// Accessor for the own column's cell at plane k+1 (the upper cell of the
// z-face k+1/2): phi^{n+1} and its in-plane gradients from slot sc, phi^n and
// mu from registers, mobility precomputed; same pinned arithmetic as RawQ /
// mu_cell_q, so the face has the same bits however its cells were staged.
struct ColQ {
  const MuSmem &S;
  const KParams &kp;
  int sc, col, row;
  const double *tb;
  const double *po, *muv;
  double Mv[NMU];
  __device__ __forceinline__ double pn(int a) const { return T(S.pn[sc][a], row, col); }
  __device__ __forceinline__ double dp(int a) const { return RN_SUB(T(S.pn[sc][a], row, col), po[a]); }
  __device__ __forceinline__ double gt(int a, int e) const {
    if (e == 0) return cdiff(T(S.pn[sc][a], row, col - 1), T(S.pn[sc][a], row, col + 1));
    return cdiff(T(S.pn[sc][a], row - 1, col), T(S.pn[sc][a], row + 1, col));  // e == 1 (z-face: e != 2)
  }
  __device__ __forceinline__ double M(int c) const { return Mv[c]; }
  __device__ __forceinline__ double mu(int c) const { return muv[c]; }
  __device__ __forceinline__ double dcl(int a, int c) const { return dcl_of(tb, a, c, muv[c]); }
  __device__ __forceinline__ const double *tab() const { return tb; }
};

// MODE: MU_FULL the whole mu update (Algorithm 1); MU_LOCAL everything but the
// anti-trapping current, MU_NEIGHBOR only its divergence added to the
// MU_LOCAL result (Algorithm 2: the local part needs no
// phi^{n+1} ghosts, so the phi halo exchange can run beside it).
template <int MODE>
__global__ void __launch_bounds__(NTHR, 512 / NTHR) mu_tiled_kernel(const __grid_constant__ TmaMaps tm, KParams kp,
                                                           BlockView b, int kz) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  MuSmem &S = *reinterpret_cast<MuSmem *>(smem_raw);
  const int tx = threadIdx.x, ty = threadIdx.y, tid = ty * TX + tx;
  const int i0 = (blockIdx.x + b.tile_x0) * TX, j0 = (blockIdx.y + b.tile_y0) * TY;
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

  auto slot = [&](int k) { return (k - k0 + 1) & (NSLOT - 1); };
  auto par4 = [&](int k) { return (uint32_t)(((k - k0 + 1) >> 2) & 1); };
  auto slot2 = [&](int k) { return NPM == 2 ? (k - k0) & 1 : (k - k0) % NPM; };
  auto par2 = [&](int k) { return (uint32_t)(((k - k0) / NPM) & 1); };
  const int bx = i0 - 2 + XO, by = j0;  // tile box origin (16-byte aligned x)
  auto stage_pn = [&](int k) {            // phi^{n+1} tiles + table row of plane k
    const int s = slot(k);
    // no proxy fence (WAR ordered by the CTA barrier; see pf_phi.cu)
    mbar_expect_tx(&S.bar_pn[s], MU_PN_BYTES);
#pragma unroll
    for (int a = 0; a < NPH; ++a) tma_load_3d(S.pn[s][a], &tm.phin[a], bx, by, k + b.zoff, &S.bar_pn[s]);
    bulk_load(S.tab[s], b.tab + (int64_t)k * TAB, TAB * 8, &S.bar_pn[s]);
  };
  auto stage_pm = [&](int k) {            // phi^n and mu tiles of plane k
    const int s = slot2(k);
    mbar_expect_tx(&S.bar_pm[s], MU_PM_BYTES);
#pragma unroll
    for (int a = 0; a < NPH; ++a) tma_load_3d(S.po[s][a], &tm.phi[a], bx, by, k + b.zoff, &S.bar_pm[s]);
#pragma unroll
    for (int c = 0; c < NMU; ++c) tma_load_3d(S.mu[s][c], &tm.mu[c], bx, by, k + b.zoff, &S.bar_pm[s]);
  };
  // flatness vote of the staged phi^{n+1}_l tile of plane k into wflat[e]:
  // bit 0 = every cell is exactly 1 (pure liquid), bit 1 = every cell is 0
  const int vq0 = tid, vq1 = tid + NTHR;   // this thread's box cells (tile offsets)
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
  // the AND of the warps' votes: lane l reads warp (l mod nwarps)'s, one
  // warp-wide AND reduction (REDUX) instead of a load per warp in every thread
  // (measured: C4 mu 2.971 -> 2.957 ms)
#ifndef PF_FLAT_REDUX
#define PF_FLAT_REDUX 1
#endif
  auto read_flat = [&](int e) {
    if (PF_FLAT_REDUX) return __reduce_and_sync(0xffffffffu, S.wflat[e][(tid & 31) % (NTHR / 32)]);
    uint32_t f = 3u;
#pragma unroll
    for (int w = 0; w < NTHR / 32; ++w) f &= S.wflat[e][w];
    return f;
  };
  auto rawq = [&](int k, int col, int row) {
    return RawQ{S, kp, slot(k - 1), slot(k), slot(k + 1), slot2(k), col, row, S.tab[slot(k)], {0.0, 0.0}};
  };
  // own column phi^n, mu of plane k from global (registers)
  auto own_load = [&](int k, double po[NPH], double mu[NMU]) {
    const int64_t pk = (int64_t)k * b.plane;
#pragma unroll
    for (int a = 0; a < NPH; ++a) po[a] = inb ? __ldg(b.phi[a] + pk + colo) : 0.0;
#pragma unroll
    for (int c = 0; c < NMU; ++c) mu[c] = inb ? __ldg(b.mu[c] + pk + colo) : 0.0;
  };
  // own-column MuQ of plane k in registers (tangential x,y gradients from slot(k))
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

  // ---- prologue: phi^{n+1} planes k0-1 .. k0+1, phi^n / mu plane k0
  if (tid == 0) {
    for (int q = 0; q < NSLOT; ++q) mbar_init(&S.bar_pn[q], 1);
    for (int q = 0; q < NPM; ++q) mbar_init(&S.bar_pm[q], 1);
    mbar_fence_init();
  }
  __syncthreads();
  if (tid == ISSUER) {
    stage_pn(k0 - 1);
    stage_pn(k0);
    stage_pn(k0 + 1);
    stage_pm(k0);
    if (NPM > 2 && k0 + 1 < k1) stage_pm(k0 + 1);
  }
  // Mown: the own column's mobility at plane k, carried from the z-face
  // k-1/2 where it was formed as the upper cell's (same pinned mob2: same bits)
  double fzm[NMU], po_n[NPH], mu_n[NMU], Mown[NMU];
  {  // z-face k0 - 1/2 from the own column's register quantities at k0-1 and k0
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
    if (MODE == MU_LOCAL) {
#pragma unroll
      for (int c = 0; c < NMU; ++c) fzm[c] = mu_flux_diff(kp, qm.M[c], qc.M[c], qm.mu[c], qc.mu[c]);
    } else {
      mu_face_t<MODE == MU_FULL>(kp, MuQAcc{qm}, MuQAcc{qc}, 2, fzm);
    }
    vote_flat(k0 - 1, 0);
    vote_flat(k0, 1);
  }
  __syncthreads();
  uint32_t flm = read_flat(0), flc = read_flat(1), flp;   // flatness of planes k-1, k, k+1
  int fe = 2;                                              // wflat entry of plane k+1

  // unrolled by 4: the plane-slot state (phi^{n+1} slot mod 4, phi^n/mu slot mod
  // 2) becomes static and the loop-carried z-face / column values need no
  // register moves (measured: x2 -3 %, x4 another -0.8 %)
#pragma unroll kMuUnroll
  for (int k = k0; k < k1; ++k) {
    const int sn = slot(k), s2 = slot2(k);
    const bool more = k + 1 < k1;
    // A: stage phi^{n+1}(k+2) and phi^n/mu(k+1) (their slots were last read in
    // D(k-1), before barrier E(k-1)); own column of plane k+1 into registers
    if (tid == ISSUER) {
      if (k + 2 <= k1) stage_pn(k + 2);
      if (NPM == 2 ? more : k + NPM - 1 < k1) stage_pm(k + NPM - 1);
    }
    double po_c[NPH], mu_c[NMU];
#pragma unroll
    for (int a = 0; a < NPH; ++a) po_c[a] = po_n[a];
#pragma unroll
    for (int c = 0; c < NMU; ++c) mu_c[c] = mu_n[c];
    own_load(k + 1, po_n, mu_n);
    mbar_wait(&S.bar_pm[s2], par2(k));   // phi^n / mu of plane k resident
    if (MODE != MU_NEIGHBOR) {  // mobility of plane k (own: carried; ring cells)
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
    }
    // phi^{n+1}(k+1), staged at A(k-1); its flatness vote
    if (k > k0) mbar_wait(&S.bar_pn[slot(k + 1)], par4(k + 1));
    vote_flat(k + 1, fe);
    __syncthreads();  // C: M of plane k and the votes visible; faces of plane k-1 consumed
    flp = read_flat(fe);
    fe = fe == 2 ? 0 : fe + 1;
    // every x/y face of plane k has J = 0: liquid flat over k-1..k+1 (|grad phi_l|^2 = 0)
    // or no liquid in plane k (phibar_l = 0); the z-face k+1/2 likewise over k, k+1
    const bool fast_xy = MODE == MU_LOCAL || ((flm & flc & flp) & 1u) || (flc & 2u);
    const bool fast_z = MODE == MU_LOCAL || ((flc & flp) & 1u) || ((flc & flp) & 2u);
    flm = flc;
    flc = flp;
    // D: faces of plane k; the own -x / -y faces also stay in registers (fxo, fyo)
    double fxo[NMU] = {0.0, 0.0}, fyo[NMU] = {0.0, 0.0};
    if (fast_xy && MODE == MU_NEIGHBOR) {   // J = 0 on every x/y face of the plane
#pragma unroll
      for (int c = 0; c < NMU; ++c) {
        if (!kShfl) S.fx[c][ty][tx] = 0.0;
        S.fy[c][ty][tx] = 0.0;
      }
      if (tid < TX + TY) {
#pragma unroll
        for (int c = 0; c < NMU; ++c) {
          if (tid >= TX) FX_FAR(c, tid - TX) = 0.0;
          else S.fy[c][TY][tid] = 0.0;
        }
      }
    } else if (fast_xy) {
#pragma unroll
      for (int c = 0; c < NMU; ++c) {   // own mu, M from registers (inb: the staged values)
        fxo[c] = mu_flux_diff(kp, S.M[c][orow][oc - 1], Mown[c], T(S.mu[s2][c], orow, oc - 1), mu_c[c]);
        fyo[c] = mu_flux_diff(kp, S.M[c][orow - 1][oc], Mown[c], T(S.mu[s2][c], orow - 1, oc), mu_c[c]);
        if (!kShfl) S.fx[c][ty][tx] = fxo[c];
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
          if (d == 0) FX_FAR(c, r0 - 1) = f;
          else S.fy[c][TY][c0 - 1] = f;
        }
      }
    } else {
      double f[NMU];
      {  // own -x face
        RawQ lo = rawq(k, oc - 1, orow), hi = rawq(k, oc, orow);
        lo.Mv[0] = S.M[0][orow][oc - 1]; lo.Mv[1] = S.M[1][orow][oc - 1];
        hi.Mv[0] = Mown[0]; hi.Mv[1] = Mown[1];
        mu_face_t<MODE == MU_FULL, kMuRoll>(kp, lo, hi, 0, fxo);
        if (!kShfl) {
          S.fx[0][ty][tx] = fxo[0];
          S.fx[1][ty][tx] = fxo[1];
        }
      }
      {  // own -y face
        RawQ lo = rawq(k, oc, orow - 1), hi = rawq(k, oc, orow);
        lo.Mv[0] = S.M[0][orow - 1][oc]; lo.Mv[1] = S.M[1][orow - 1][oc];
        hi.Mv[0] = Mown[0]; hi.Mv[1] = Mown[1];
        mu_face_t<MODE == MU_FULL, kMuRoll>(kp, lo, hi, 1, fyo);
        S.fy[0][ty][tx] = fyo[0];
        S.fy[1][ty][tx] = fyo[1];
      }
      // far faces: +y of the last row (warp 0), +x of the last column (warp 1);
      // PF_MU_FAR_CONST: each with a compile-time direction (the face routine's
      // component and accessor selects fold away)
      auto far_face = [&](auto dc, int c0, int r0) {
        constexpr int d = decltype(dc)::value;
        const int c1 = d == 1 ? c0 : c0 + 1, r1 = d == 1 ? r0 + 1 : r0;
        RawQ lo = rawq(k, c0, r0), hi = rawq(k, c1, r1);
        lo.Mv[0] = S.M[0][r0][c0]; lo.Mv[1] = S.M[1][r0][c0];
        hi.Mv[0] = S.M[0][r1][c1]; hi.Mv[1] = S.M[1][r1][c1];
        mu_face_t<MODE == MU_FULL, kMuRoll>(kp, lo, hi, d, f);
        if (d == 0) { FX_FAR(0, r0 - 1) = f[0]; FX_FAR(1, r0 - 1) = f[1]; }
        else { S.fy[0][TY][c0 - 1] = f[0]; S.fy[1][TY][c0 - 1] = f[1]; }
      };
      if (PF_MU_FAR_CONST) {
        if (tid < TX) far_face(std::integral_constant<int, 1>{}, tid + 1, TY);
        else if (tid < TX + TY) far_face(std::integral_constant<int, 0>{}, TX, tid - TX + 1);
      } else if (tid < TX + TY) {
        const int d = tid < TX ? 1 : 0;
        const int c0 = d == 1 ? tid + 1 : TX, r0 = d == 1 ? TY : tid - TX + 1;
        const int c1 = d == 1 ? c0 : c0 + 1, r1 = d == 1 ? r0 + 1 : r0;
        RawQ lo = rawq(k, c0, r0), hi = rawq(k, c1, r1);
        lo.Mv[0] = S.M[0][r0][c0]; lo.Mv[1] = S.M[1][r0][c0];
        hi.Mv[0] = S.M[0][r1][c1]; hi.Mv[1] = S.M[1][r1][c1];
        mu_face_t<MODE == MU_FULL, kMuRoll>(kp, lo, hi, d, f);
        if (d == 0) { FX_FAR(0, r0 - 1) = f[0]; FX_FAR(1, r0 - 1) = f[1]; }
        else { S.fy[0][TY][c0 - 1] = f[0]; S.fy[1][TY][c0 - 1] = f[1]; }
      }
    }
    double fzp[NMU], pn_c[NPH], Mnx[NMU] = {0.0, 0.0};   // Mnx: own mobility at k+1
    if (fast_z && MODE == MU_NEIGHBOR) {
      fzp[0] = fzp[1] = 0.0;
#pragma unroll
      for (int a = 0; a < NPH; ++a) pn_c[a] = T(S.pn[sn][a], orow, oc);
    } else if (fast_z) {
      mob2(S.tab[slot(k + 1)], po_n, Mnx);
#pragma unroll
      for (int c = 0; c < NMU; ++c) fzp[c] = mu_flux_diff(kp, Mown[c], Mnx[c], mu_c[c], mu_n[c]);
#pragma unroll
      for (int a = 0; a < NPH; ++a) pn_c[a] = T(S.pn[sn][a], orow, oc);
    } else {  // z-face k+1/2: own cell at k (shared memory) and at k+1 (registers;
              // the anti-trapping operands are only formed if the guards open)
      RawQ lo = rawq(k, oc, orow);
      lo.Mv[0] = Mown[0]; lo.Mv[1] = Mown[1];
      const int s1 = slot(k + 1);
      ColQ hi{S, kp, s1, oc, orow, S.tab[s1], po_n, mu_n, {0.0, 0.0}};
      if (MODE == MU_FULL) mob2(S.tab[s1], po_n, hi.Mv);
      mu_face_t<MODE == MU_FULL>(kp, lo, hi, 2, fzp);
      Mnx[0] = hi.Mv[0];
      Mnx[1] = hi.Mv[1];
#pragma unroll
      for (int a = 0; a < NPH; ++a) pn_c[a] = T(S.pn[sn][a], orow, oc);
    }
    // the divergence's own-face part before the barrier (the oracle's O5.9
    // sum in another order: equal up to rounding)
    double dpart[NMU], fxp[NMU];   // fxp: the +x face from the next lane (kShfl)
#pragma unroll
    for (int c = 0; c < NMU; ++c) {
      fxp[c] = kShfl ? __shfl_down_sync(0xffffffffu, fxo[c], 1) : 0.0;
      dpart[c] = ((fzp[c] - fzm[c]) - fxo[c]) - fyo[c];
      fzm[c] = fzp[c];
      Mown[c] = Mnx[c];
    }
    __syncthreads();  // E
    // F: cell update of (i, j, k)
    if (active) {
      double divf[NMU], out[NMU];
#pragma unroll
      for (int c = 0; c < NMU; ++c)
        divf[c] = dpart[c] + ((kShfl ? (tx == TX - 1 ? FX_FAR(c, ty) : fxp[c]) : S.fx[c][ty][tx + 1]) +
                              S.fy[c][ty + 1][tx]);
      const int64_t o = (int64_t)k * b.plane + colo;
      if (MODE != MU_NEIGHBOR) {
        mu_cell_update(kp, S.tab[sn], po_c, pn_c, mu_c, divf, out);
        st_field(&b.out[0][o], out[0]);
        st_field(&b.out[1][o], out[1]);
      } else if (divf[0] != 0.0 || divf[1] != 0.0) {   // divj = 0: mu_loc stands, bit for bit
        const double loc[NMU] = {b.out[0][o], b.out[1][o]};
        mu_cell_add_j(kp, S.tab[sn], pn_c, loc, divf, out);
        st_field(&b.out[0][o], out[0]);
        st_field(&b.out[1][o], out[1]);
      }
    }
  }
#undef T
}

// Opt-in to > 48 KB of dynamic shared memory, once per process (pf_create;
// not inside a stream capture).
static int g_mu_slots = 1;   // resident CTAs on the GPU

void prepare_mu_tiled() {
  const int sm = (int)sizeof(MuSmem);
  cudaFuncSetAttribute(mu_tiled_kernel<MU_FULL>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm);
  cudaFuncSetAttribute(mu_tiled_kernel<MU_LOCAL>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm);
  cudaFuncSetAttribute(mu_tiled_kernel<MU_NEIGHBOR>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm);
  g_mu_slots = grid_slots(mu_tiled_kernel<MU_FULL>, NTHR, sm);
}

template <int MODE>
void launch_mu_mode(cudaStream_t s, const KParams &kp, const BlockView &b, const TmaMaps &tm) {
  const int gx = (b.nx + TX - 1) / TX, gy = (b.ny + TY - 1) / TY;
// >= 8 waves or a >= 97 % full last one: 256-plane chunks at 512^3 (measured
// with the two-plane lead: 256 -> 2.958 ms, 128 -> 2.966, 64 -> 2.995, 32 -> 3.059)
#ifndef PF_MU_WAVES
#define PF_MU_WAVES 8
#endif
  int kz = chunk_z(b.nz, gx * gy, g_mu_slots, PF_MU_WAVES, true);
#ifdef PF_MU_KZ
  kz = std::min(kz, PF_MU_KZ);
#endif
  dim3 grd(gx, gy, (b.nz + kz - 1) / kz), blk(TX, TY);
  mu_tiled_kernel<MODE><<<grd, blk, sizeof(MuSmem), s>>>(tm, kp, b, kz);
}

int mu_tiles_x(int nx) { return (nx + TX - 1) / TX; }
int mu_tiles_y(int ny) { return (ny + TY - 1) / TY; }

void launch_mu_tiles(cudaStream_t s, const KParams &kp, const BlockView &b, const TmaMaps &tm, int tx0, int tx1,
                     int ty0, int ty1) {
  if (tx1 <= tx0 || ty1 <= ty0 || b.nz <= 0) return;
  BlockView v = b;
  v.tile_x0 = tx0;
  v.tile_y0 = ty0;
  const int kz = chunk_z(b.nz, (tx1 - tx0) * (ty1 - ty0), g_mu_slots, 8, true);
  dim3 grd(tx1 - tx0, ty1 - ty0, (b.nz + kz - 1) / kz), blk(TX, TY);
  mu_tiled_kernel<MU_FULL><<<grd, blk, sizeof(MuSmem), s>>>(tm, kp, v, kz);
}

void launch_mu_tiled(cudaStream_t s, const KParams &kp, const BlockView &b, const TmaMaps &tm, int mode) {
  if (mode == MU_LOCAL) launch_mu_mode<MU_LOCAL>(s, kp, b, tm);
  else if (mode == MU_NEIGHBOR) launch_mu_mode<MU_NEIGHBOR>(s, kp, b, tm);
  else launch_mu_mode<MU_FULL>(s, kp, b, tm);
}

}  // namespace pf
