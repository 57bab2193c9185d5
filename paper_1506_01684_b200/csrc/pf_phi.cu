// pf_phi.cu — production phi-sweep (Eq. (1)-(2)): z-marching
// 2.5D tiles with every staggered face flux (PAPER.md:299-317,
// fig:staggeredBuffer) evaluated exactly once:
//   * x- and y-faces of plane k: each thread evaluates its -x and -y face, warp
//     0 the tile's far +y / +x faces; results go to shared memory (buffers
//     alternating with the plane's parity) and are read by both adjacent cells;
//   * z-faces: carried in registers from k-1/2 to k+1/2 (the paper's Nx x Ny
//     staggered buffer becomes one register set per column; anisotropic: a
//     thread-private shared-memory slot).
// Data movement: per plane, one elected thread issues TMA bulk-tensor copies of
// the 4 phi tiles (interior + ring + corners) and a bulk copy of the table row,
// two planes ahead, into 4 rotating slots guarded by mbarriers; mu (the cell's
// own value only) comes from global memory one plane ahead.  One CTA barrier
// per plane.  The face and gradient routines are the pinned ones of pf_dev.cuh:
// a face evaluated at a tile / chunk / block edge has the same bits as mid-tile.
#include <type_traits>
#include "pf_kernels.cuh"
#define PF_TILE_X PHI_TILE_X
#define PF_TILE_Y PHI_TILE_Y
#include "pf_tile.cuh"

namespace pf {

#ifndef PF_PHI_NS
#define PF_PHI_NS 4
#endif
// phi^n tile slots: 4 = planes k-1..k+1 resident and k+2 staged at the top of
// iteration k; 3 = k+2 staged into k-1's slot right after the barrier (with
// the z-face carry only in the anisotropic layout, the isotropic kernel then
// fits 5 CTAs per SM at 96 registers: measured 3.68 ms vs 3.55 at 512^3, 3.78
// at 4 CTAs — the shorter lead costs more than the occupancy gains)
constexpr int PNS = PF_PHI_NS;
#ifndef PF_PHI_FAR_SPLIT
#define PF_PHI_FAR_SPLIT 1
#endif
#ifndef PF_PHI_FAR_SPLIT_ISO
#define PF_PHI_FAR_SPLIT_ISO 0
#endif
template <bool ANISO>
struct __align__(128) PhiSmemT {
  double p[PNS][NPH][TSZ];         // phi^n tile planes, (row, col) at row * RX + col
  double tab[PNS][TAB];            // per-plane table rows
  double fx[2][NPH][TY][TX + 1];   // x-face fluxes at i - 1/2, i = 0..TX (plane parity)
  double fy[2][NPH][TY + 1][TX];   // y-face fluxes at j - 1/2, j = 0..TY
  uint64_t bar[PNS];               // one mbarrier per slot
  double jz[ANISO ? NPH : 1][TY][TX];   // anisotropic: the z-face carry, thread-private (measured: frees
                                   // registers the D3C19 faces use; isotropic keeps it in registers)
};

constexpr uint32_t PHI_STAGE_BYTES = (NPH * RXS * RY + TAB) * 8;

// SC: 0 no shortcut code, 1 the round-1 vote (run-time flag), 2 skip-faces shortcuts;
// DM: the anisotropic kernel's cubic-pair mask at compile time (-1: kp.dmask)
template <bool ANISO, int SC, int DM = -1>
#ifndef PF_PHI_MINB
#define PF_PHI_MINB (512 / NTHR)
#endif
#ifndef PF_PHI_MINB_ISO
#define PF_PHI_MINB_ISO PF_PHI_MINB
#endif
__global__ void __launch_bounds__(NTHR, ANISO ? PF_PHI_MINB : PF_PHI_MINB_ISO)
    phi_tiled_kernel(const __grid_constant__ TmaMaps tm, KParams kp, BlockView b, int kz) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  PhiSmemT<ANISO> &S = *reinterpret_cast<PhiSmemT<ANISO> *>(smem_raw);
  const int tx = threadIdx.x, ty = threadIdx.y, tid = ty * TX + tx;
  const int i0 = blockIdx.x * TX, j0 = blockIdx.y * TY;
  const int k0 = blockIdx.z * kz, k1 = min(k0 + kz, b.nz);
  const int i = i0 + tx, j = j0 + ty;
  const bool active = (i < b.nx) && (j < b.ny);   // owns an interior cell
  const int64_t colo = (int64_t)j * b.pitch + i;
  const int oc = tx + 1, orow = ty + 1;            // own tile coordinates
#define T(arr, row, col) TILE_AT(arr, row, col)
// the face and cell routines specialised for this kernel's model: each of the
// two kernels carries only its own code (measured: iso -1.8 %, aniso -6 %;
// 35 % less code, fewer instruction-fetch stalls)
#define PF_AN (ANISO ? 1 : 0), DM

  auto slot = [&](int k) { return PNS == 4 ? (k - k0 + 1) & 3 : (k - k0 + 1) % PNS; };
  auto parity = [&](int k) { return (uint32_t)(((k - k0 + 1) / PNS) & 1); };
  // plane k -> its slot: 4 phi tiles, 2 mu interior boxes, the table row
  auto stage = [&](int k) {
    const int s = slot(k);
    // no proxy fence: the slot's last (generic) reads are ordered before this
    // (async) refill by the CTA barrier; a fence here costs a MEMBAR that waits
    // for the issuing warp's outstanding global stores
    mbar_expect_tx(&S.bar[s], PHI_STAGE_BYTES);
    const int z = k + b.zoff;
#pragma unroll
    for (int a = 0; a < NPH; ++a) tma_load_3d(S.p[s][a], &tm.phi[a], i0 - 2 + XO, j0, z, &S.bar[s]);
    bulk_load(S.tab[s], b.tab + (int64_t)k * TAB, TAB * 8, &S.bar[s]);
  };
  auto wait = [&](int k) { mbar_wait(&S.bar[slot(k)], parity(k)); };
  // tangential raw centre differences of tile cell (col,row) in slot sc
  // (component d unused); z-tangential from slots sm/sp
  auto tan_grad = [&](int sc, int sm, int sp, int col, int row, int d, double g[NPH][3]) {
#pragma unroll
    for (int a = 0; a < NPH; ++a) {
      g[a][0] = d == 0 ? 0.0 : cdiff(T(S.p[sc][a], row, col - 1), T(S.p[sc][a], row, col + 1));
      g[a][1] = d == 1 ? 0.0 : cdiff(T(S.p[sc][a], row - 1, col), T(S.p[sc][a], row + 1, col));
      g[a][2] = d == 2 ? 0.0 : cdiff(T(S.p[sm][a], row, col), T(S.p[sp][a], row, col));
    }
  };
  double gdum[NPH][3];
#pragma unroll
  for (int a = 0; a < NPH; ++a)
#pragma unroll
    for (int e = 0; e < 3; ++e) gdum[a][e] = 0.0;

  // ---- prologue: planes k0-1, k0, k0+1 resident, z-face k0 - 1/2
  if (tid == 0) {
    for (int s = 0; s < PNS; ++s) mbar_init(&S.bar[s], 1);
    mbar_fence_init();
  }
  __syncthreads();
  if (tid == ISSUER) {
    stage(k0 - 1);
    stage(k0);
    stage(k0 + 1);
  }
  wait(k0 - 1);
  wait(k0);
  double jzm[NPH];
  {
    const int s0 = slot(k0 - 1), s1 = slot(k0);
    double lo[NPH], hi[NPH], gl[NPH][3], gh[NPH][3];
#pragma unroll
    for (int a = 0; a < NPH; ++a) { lo[a] = T(S.p[s0][a], orow, oc); hi[a] = T(S.p[s1][a], orow, oc); }
    if (ANISO) {
      tan_grad(s0, s0, s0, oc, orow, 2, gl);
      tan_grad(s1, s1, s1, oc, orow, 2, gh);
    }
    phi_face<PF_AN>(kp, lo, hi, ANISO ? gl : gdum, ANISO ? gh : gdum, 2, jzm);
    if (ANISO)
#pragma unroll
      for (int a = 0; a < NPH; ++a) S.jz[a][ty][tx] = jzm[a];
  }

  // One CTA barrier per plane (B): the face buffers alternate by plane parity,
  // so D(k) never overwrites faces another thread may still read in F(k-1);
  // buffer (k & 1) was last read in F(k-2), which every thread finished before
  // reaching B(k-1).  TMA refills slot(k+2) = slot(k-2), last read in D(k-1),
  // likewise before B(k-1).  mu (D3C1: the cell's own value) comes straight
  // from global memory one plane ahead, which keeps the shared footprint at
  // 4 CTAs / SM.
  double mu_n[NMU];
#pragma unroll
  for (int c = 0; c < NMU; ++c) mu_n[c] = active ? __ldg(b.mu[c] + (int64_t)k0 * b.plane + colo) : 0.0;
  for (int k = k0; k < k1; ++k) {
    // A: stage plane k+2 (needed from iteration k+1 on); wait for plane k+1
    if (PNS == 4 && tid == ISSUER && k + 2 <= k1) stage(k + 2);
    double mu_c[NMU];
#pragma unroll
    for (int c = 0; c < NMU; ++c) {
      mu_c[c] = mu_n[c];
      mu_n[c] = (active && k + 1 < k1) ? __ldg(b.mu[c] + (int64_t)(k + 1) * b.plane + colo) : 0.0;
    }
    wait(k + 1);
    const int sc = slot(k), sm = slot(k - 1), sp = slot(k + 1);
    const int fb = (k - k0) & 1;
    // D: faces of plane k.  The own column's values are read from shared memory
    // once (the LSU pipe, not the FP64 pipe, was the busier one: ncu v14 72 %
    // vs 58 %) and, isotropic, the cell's own faces enter its divergence from
    // registers before the barrier:
    //   dpart = ((jz+ - jz-) - jx-) - jy-,   rhs = (r0 - c dpart) - c (jx+ + jy+)
    // with c = eps T / dx (the oracle's O4.6 sum in another order: equal up to
    // rounding; the anisotropic kernel forms dpart after the barrier).
    // region shortcut, SC = 2 (NEXT-1): voted
    // before the faces with integer compares on the bits (a double compare is
    // an FP64-pipe instruction), in two stages (own cell a simplex vertex, then
    // its D3C7 / D3C19 neighbours identical).  A shortcut warp's own faces are
    // exactly 0 (2x2 determinants and differences of equal 0/1 values), so it
    // writes zeros instead of evaluating them and keeps phi^{n+1} = phi^n,
    // bitwise what the full update returns (is_vertex).  Slots k-1..k+1 are
    // resident; slot(k-1) is refilled only after barrier B(k).
    bool skip2 = false;
    if (SC == 2) {
      double pcv[NPH];
#pragma unroll
      for (int a = 0; a < NPH; ++a) pcv[a] = T(S.p[sc][a], orow, oc);
      if (__all_sync(0xffffffffu, is_vertex_bits(pcv) || !active)) {
        auto same = [](double x, double v) { return __double_as_longlong(x) == __double_as_longlong(v); };
        bool mine = true;
#pragma unroll
        for (int a = 0; a < NPH; ++a) {
          const double v = pcv[a];
          mine = mine && same(T(S.p[sc][a], orow, oc - 1), v) && same(T(S.p[sc][a], orow, oc + 1), v) &&
                 same(T(S.p[sc][a], orow - 1, oc), v) && same(T(S.p[sc][a], orow + 1, oc), v) &&
                 same(T(S.p[sm][a], orow, oc), v) && same(T(S.p[sp][a], orow, oc), v);
          if (ANISO)
            mine = mine && same(T(S.p[sc][a], orow - 1, oc - 1), v) && same(T(S.p[sc][a], orow - 1, oc + 1), v) &&
                   same(T(S.p[sc][a], orow + 1, oc - 1), v) && same(T(S.p[sc][a], orow + 1, oc + 1), v) &&
                   same(T(S.p[sm][a], orow, oc - 1), v) && same(T(S.p[sm][a], orow, oc + 1), v) &&
                   same(T(S.p[sm][a], orow - 1, oc), v) && same(T(S.p[sm][a], orow + 1, oc), v) &&
                   same(T(S.p[sp][a], orow, oc - 1), v) && same(T(S.p[sp][a], orow, oc + 1), v) &&
                   same(T(S.p[sp][a], orow - 1, oc), v) && same(T(S.p[sp][a], orow + 1, oc), v);
        }
        skip2 = __all_sync(0xffffffffu, mine || !active) != 0;
      }
    }
    double pc[NPH], pp[NPH], jzp[NPH], dpart[NPH];
    if (!ANISO)
#pragma unroll
      for (int a = 0; a < NPH; ++a) pc[a] = T(S.p[sc][a], orow, oc);
    // anisotropic: the own cell's raw centre differences once (the hi side of
    // its -x / -y faces and the cell update's gradients; pinned: same bits)
    double gown[NPH][3];
    if (ANISO) tan_grad(sc, sm, sp, oc, orow, -1, gown);
    {
      double jf[NPH], lo[NPH], hi[NPH], gl[NPH][3], gh[NPH][3];
      // far faces: +y of the last row, +x of the last column (warp 0); the
      // isotropic kernel issues them first, the anisotropic one after its own
      // faces (measured: iso -1.1 %, aniso +5 % the other way round)
      // PF_PHI_FAR_SPLIT (anisotropic): +y far faces on warp 0, +x far faces on
      // warp 1, each with a compile-time direction (no run-time-d arrays in
      // local memory — the kernel's 48-byte stack frame — no direction selects):
      // C5-model phi 6.113 -> 5.944 ms at 512^3, bitwise the same fields; the
      // isotropic face has no direction-dependent operands and measured slower
      // split (3.64 vs 3.55 ms: PF_PHI_FAR_SPLIT_ISO off)
      auto far_face_d = [&](auto dc, int c0, int r0) {
        constexpr int d = decltype(dc)::value;
        const int c1 = d == 1 ? c0 : c0 + 1, r1 = d == 1 ? r0 + 1 : r0;
#pragma unroll
        for (int a = 0; a < NPH; ++a) { lo[a] = T(S.p[sc][a], r0, c0); hi[a] = T(S.p[sc][a], r1, c1); }
        if (ANISO) {
          tan_grad(sc, sm, sp, c0, r0, d, gl);
          tan_grad(sc, sm, sp, c1, r1, d, gh);
        }
        phi_face<PF_AN>(kp, lo, hi, ANISO ? gl : gdum, ANISO ? gh : gdum, d, jf);
#pragma unroll
        for (int a = 0; a < NPH; ++a) {
          if (d == 0) S.fx[fb][a][r0 - 1][TX] = jf[a];
          else S.fy[fb][a][TY][c0 - 1] = jf[a];
        }
      };
      auto far_faces = [&]() {
        if ((ANISO && PF_PHI_FAR_SPLIT) || (!ANISO && PF_PHI_FAR_SPLIT_ISO)) {
          const int w = tid >> 5, l = tid & 31;
          if (w == 0 && l < TX) far_face_d(std::integral_constant<int, 1>{}, l + 1, TY);
          else if (w == 1 && l < TY) far_face_d(std::integral_constant<int, 0>{}, TX, l + 1);
        } else if (tid < TX + TY) {
          const int d = tid < TX ? 1 : 0;
          const int c0 = d == 1 ? tid + 1 : TX, r0 = d == 1 ? TY : tid - TX + 1;
          const int c1 = d == 1 ? c0 : c0 + 1, r1 = d == 1 ? r0 + 1 : r0;
#pragma unroll
          for (int a = 0; a < NPH; ++a) { lo[a] = T(S.p[sc][a], r0, c0); hi[a] = T(S.p[sc][a], r1, c1); }
          if (ANISO) {
            tan_grad(sc, sm, sp, c0, r0, d, gl);
            tan_grad(sc, sm, sp, c1, r1, d, gh);
          }
          phi_face<PF_AN>(kp, lo, hi, ANISO ? gl : gdum, ANISO ? gh : gdum, d, jf);
#pragma unroll
          for (int a = 0; a < NPH; ++a) {
            if (d == 0) S.fx[fb][a][r0 - 1][TX] = jf[a];
            else S.fy[fb][a][TY][c0 - 1] = jf[a];
          }
        }
      };
      if (SC == 2 && skip2) {   // a shortcut warp: its own faces are exactly 0; the far faces as usual
#pragma unroll
        for (int a = 0; a < NPH; ++a) {
          pc[a] = T(S.p[sc][a], orow, oc);
          jzp[a] = 0.0;
          dpart[a] = 0.0;
          if (!ANISO) jzm[a] = 0.0;
          S.fx[fb][a][ty][tx] = 0.0;
          S.fy[fb][a][ty][tx] = 0.0;
        }
        far_faces();
      } else {
      if (!ANISO) far_faces();
      if (ANISO) {   // anisotropic: the z-face k+1/2 first too (its dpart is formed after the barrier; -0.4 %)
#pragma unroll
        for (int a = 0; a < NPH; ++a) {
          pp[a] = T(S.p[sp][a], orow, oc);
          pc[a] = T(S.p[sc][a], orow, oc);
        }
        tan_grad(sp, sp, sp, oc, orow, 2, gh);   // lo side: the own cell's gown
        phi_face<PF_AN>(kp, pc, pp, gown, gh, 2, jzp);
      }
      if (!ANISO) {   // isotropic: the z-face k+1/2 next (measured -0.8 % against last)
#pragma unroll
        for (int a = 0; a < NPH; ++a) pp[a] = T(S.p[sp][a], orow, oc);
        phi_face<PF_AN>(kp, pc, pp, gdum, gdum, 2, jzp);
#pragma unroll
        for (int a = 0; a < NPH; ++a) {
          dpart[a] = jzp[a] - jzm[a];
          jzm[a] = jzp[a];
        }
      }
#pragma unroll
      for (int d = 0; d < 2; ++d) {   // own -x (d = 0) and -y (d = 1) face
        const int lc = d == 0 ? oc - 1 : oc, lr = d == 0 ? orow : orow - 1;
#pragma unroll
        for (int a = 0; a < NPH; ++a) {
          lo[a] = T(S.p[sc][a], lr, lc);
          hi[a] = ANISO ? T(S.p[sc][a], orow, oc) : pc[a];   // anisotropic: re-read (registers)
        }
        if (ANISO) tan_grad(sc, sm, sp, lc, lr, d, gl);
        phi_face<PF_AN>(kp, lo, hi, ANISO ? gl : gdum, ANISO ? gown : gdum, d, jf);
#pragma unroll
        for (int a = 0; a < NPH; ++a) {
          if (d == 0) S.fx[fb][a][ty][tx] = jf[a];
          else S.fy[fb][a][ty][tx] = jf[a];
          if (!ANISO) dpart[a] -= jf[a];
        }
      }
      if (ANISO) far_faces();
      }
    }
    // region shortcut (NEXT-1): a warp whose cells
    // are all simplex vertices with an identical D3C7 (D3C19) neighbourhood
    // keeps phi^{n+1} = phi^n — bitwise what the full update returns (is_vertex)
    auto bulk_warp = [&]() {
      if (SC != 1 || !kp.shortcuts) return false;   // SC = 0: the check compiled out
      bool mine = is_vertex(pc);
#pragma unroll
      for (int a = 0; a < NPH; ++a) {
        const double v = pc[a];
        mine = mine && T(S.p[sc][a], orow, oc - 1) == v && T(S.p[sc][a], orow, oc + 1) == v &&
               T(S.p[sc][a], orow - 1, oc) == v && T(S.p[sc][a], orow + 1, oc) == v &&
               T(S.p[sm][a], orow, oc) == v && pp[a] == v;
        if (ANISO)
          mine = mine && T(S.p[sc][a], orow - 1, oc - 1) == v && T(S.p[sc][a], orow - 1, oc + 1) == v &&
                 T(S.p[sc][a], orow + 1, oc - 1) == v && T(S.p[sc][a], orow + 1, oc + 1) == v &&
                 T(S.p[sm][a], orow, oc - 1) == v && T(S.p[sm][a], orow, oc + 1) == v &&
                 T(S.p[sm][a], orow - 1, oc) == v && T(S.p[sm][a], orow + 1, oc) == v &&
                 T(S.p[sp][a], orow, oc - 1) == v && T(S.p[sp][a], orow, oc + 1) == v &&
                 T(S.p[sp][a], orow - 1, oc) == v && T(S.p[sp][a], orow + 1, oc) == v;
      }
      return __all_sync(0xffffffffu, mine || !active) != 0;
    };
    // the vote reads slot(k-1), which stage(k+3) refills right after B(k): it
    // is taken before the barrier in both kernels
    const bool skip = SC == 2 ? skip2 : bulk_warp();
    // isotropic: the cell terms that need no face flux (phi_cell_rhs0, on the
    // raw centre differences) are formed before the barrier, where the tile
    // values are still at hand; the anisotropic kernel has no registers to
    // spare for that and forms them after it
    double q[NPH];   // r0 - c dpart
    if (!ANISO && active && !skip) {
      double r0[NPH], gc[NPH][3];
#pragma unroll
      for (int a = 0; a < NPH; ++a) {
        gc[a][0] = T(S.p[sc][a], orow, oc + 1) - T(S.p[sc][a], orow, oc - 1);
        gc[a][1] = T(S.p[sc][a], orow + 1, oc) - T(S.p[sc][a], orow - 1, oc);
        gc[a][2] = pp[a] - T(S.p[sm][a], orow, oc);
      }
      phi_cell_rhs0<PF_AN>(kp, S.tab[sc], pc, mu_c, gc, r0);
      const double c = S.tab[sc][T_EPSTDX];
#pragma unroll
      for (int a = 0; a < NPH; ++a) q[a] = r0[a] - c * dpart[a];
    }
    __syncthreads();  // B: faces of plane k complete
    // three slots: plane k+2 into plane k-1's slot, whose last reads (the vote,
    // the z differences, the anisotropic gradients) came before B(k)
    if (PNS == 3 && tid == ISSUER && k + 2 <= k1) stage(k + 2);
    if (active && skip) {
      const int64_t o = (int64_t)k * b.plane + colo;
#pragma unroll
      for (int a = 0; a < NPH; ++a) st_field(&b.out[a][o], pc[a]);
    } else if (active) {
      const double c = S.tab[sc][ANISO ? T_EPSTDX16 : T_EPSTDX];   // anisotropic fluxes: 16 dx j
      if (ANISO) {
        double r0[NPH];
        phi_cell_rhs0<PF_AN>(kp, S.tab[sc], pc, mu_c, gown, r0);
#pragma unroll
        for (int a = 0; a < NPH; ++a) {
          dpart[a] = (jzp[a] - S.jz[a][ty][tx]) - S.fx[fb][a][ty][tx] - S.fy[fb][a][ty][tx];
          q[a] = r0[a] - c * dpart[a];
        }
      }
      double rhs[NPH], out[NPH];
#pragma unroll
      for (int a = 0; a < NPH; ++a) rhs[a] = q[a] - c * (S.fx[fb][a][ty][tx + 1] + S.fy[fb][a][ty + 1][tx]);
      phi_cell_project(kp, pc, rhs, out);
      const int64_t o = (int64_t)k * b.plane + colo;
#pragma unroll
      for (int a = 0; a < NPH; ++a) st_field(&b.out[a][o], out[a]);
    }
    if (ANISO)
#pragma unroll
      for (int a = 0; a < NPH; ++a) S.jz[a][ty][tx] = jzp[a];   // thread-private slot
  }
#undef T
#undef PF_AN
}

// Opt-in to > 48 KB of dynamic shared memory, once per process (pf_create;
// not inside a stream capture).
static int g_phi_slots[2] = {1, 1};   // resident CTAs on the GPU, [ANISO]

// the cubic pairs of the solid-liquid interfaces only (pairs (a, l): p = 2, 4, 5),
// the model of C5 (delta_sl): compiled without the per-pair mask test
constexpr int DM_SL = (1 << pair_of(0, LIQ)) | (1 << pair_of(1, LIQ)) | (1 << pair_of(2, LIQ));

void prepare_phi_tiled() {
  const int sa = (int)sizeof(PhiSmemT<true>), si = (int)sizeof(PhiSmemT<false>);
  cudaFuncSetAttribute(phi_tiled_kernel<true, 0>, cudaFuncAttributeMaxDynamicSharedMemorySize, sa);
  cudaFuncSetAttribute(phi_tiled_kernel<true, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, sa);
  cudaFuncSetAttribute(phi_tiled_kernel<true, 0, DM_SL>, cudaFuncAttributeMaxDynamicSharedMemorySize, sa);
  cudaFuncSetAttribute(phi_tiled_kernel<false, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, si);
  cudaFuncSetAttribute(phi_tiled_kernel<false, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, si);
  g_phi_slots[0] = grid_slots(phi_tiled_kernel<false, 1>, NTHR, si);
  g_phi_slots[1] = grid_slots(phi_tiled_kernel<true, 0>, NTHR, sa);
}

void launch_phi_tiled(cudaStream_t s, const KParams &kp, const BlockView &b, const TmaMaps &tm) {
  const int gx = (b.nx + TX - 1) / TX, gy = (b.ny + TY - 1) / TY;
#ifndef PF_PHI_WAVES
#define PF_PHI_WAVES 16
#endif
  const int kz = chunk_z(b.nz, gx * gy, g_phi_slots[kp.aniso ? 1 : 0], PF_PHI_WAVES, false);
  dim3 grd(gx, gy, (b.nz + kz - 1) / kz), blk(TX, TY);
  const size_t sm = kp.aniso ? sizeof(PhiSmemT<true>) : sizeof(PhiSmemT<false>);
  // shortcuts on: the skip-faces kernels (SC = 2).  Off: the anisotropic kernel
  // without any shortcut code (-3 %), the isotropic one with the round-1
  // run-time check compiled in (its code without it, or with the SC = 2 vote
  // in the same kernel, measured +1.7 %: the compiler's schedule, not the
  // check, decides there)
  // the solid-liquid anisotropic kernel runs without the vote even with
  // shortcuts on: its skip-faces variant measured slower in every scenario
  // (256^3 interface / solid / liquid: 0.89 / 0.92 / 0.85 vs 0.80 / 0.81 / 0.79
  // ms, profiles/r02_scenarios_aniso.md) — bitwise the same results either way
  const bool sl = kp.dmask == DM_SL;
  if (kp.shortcuts && !(kp.aniso && sl)) {
    if (kp.aniso) phi_tiled_kernel<true, 2><<<grd, blk, sm, s>>>(tm, kp, b, kz);
    else phi_tiled_kernel<false, 2><<<grd, blk, sm, s>>>(tm, kp, b, kz);
  } else if (kp.aniso && sl) {
    phi_tiled_kernel<true, 0, DM_SL><<<grd, blk, sm, s>>>(tm, kp, b, kz);
  } else if (kp.aniso) {
    phi_tiled_kernel<true, 0><<<grd, blk, sm, s>>>(tm, kp, b, kz);
  } else {
    phi_tiled_kernel<false, 1><<<grd, blk, sm, s>>>(tm, kp, b, kz);
  }
}

}  // namespace pf
