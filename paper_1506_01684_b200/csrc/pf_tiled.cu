// pf_tiled.cu — the production sweeps: z-marching 2.5D tiles.
//
// CTA = 32 (x) x 8 (y) threads, one thread per (i,j) column, marching a chunk
// of KZ planes in z (z is the outermost loop because T depends
// on z only; the table row is read once per plane).  Staggered face values
// (fig:staggeredBuffer) are evaluated exactly once per face:
//   * x- and y-faces of plane k: one per thread (its -x / -y face) plus the
//     tile's far faces, written to shared memory and read back by both cells;
//   * z-faces: carried in registers from plane k-1/2 to k+1/2 (the paper's
//     Nx x Ny staggered buffer becomes a per-thread register).
// The face routines are the pinned ones of pf_dev.cuh, so a face evaluated at
// a tile / chunk / block edge has the same bits as mid-tile (decomposition
// invariance, solute conservation).
#include "pf_kernels.cuh"

namespace pf {

constexpr int TX = 32, TY = 8, RX = TX + 2, RY = TY + 2;
constexpr int NTHR = TX * TY;
constexpr int NRING = 2 * RX + 2 * TY;  // 84 ring cells incl. the 4 in-plane corners

// ring cell r -> (col, row) in the (RX x RY) tile (col/row 0 = index -1)
__device__ __forceinline__ void ring_cell(int r, int &col, int &row) {
  if (r < RX) { col = r; row = 0; }
  else if (r < 2 * RX) { col = r - RX; row = RY - 1; }
  else if (r < 2 * RX + TY) { col = 0; row = r - 2 * RX + 1; }
  else { col = RX - 1; row = r - 2 * RX - TY + 1; }
}

// ===========================================================================
// phi-sweep
// ===========================================================================
template <bool ANISO>
struct PhiSmem {
  static constexpr int NPL = ANISO ? 3 : 1;
  double p[NPL][NPH][RY][RX];     // phi^n tile planes (ring + corners)
  double fx[NPH][TY][TX + 1];     // x-face fluxes at i - 1/2, i = 0..TX
  double fy[NPH][TY + 1][TX];     // y-face fluxes at j - 1/2, j = 0..TY
};

template <bool ANISO>
__global__ void __launch_bounds__(NTHR, ANISO ? 1 : 2) phi_tiled_kernel(KParams kp, BlockView b, int kz) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  PhiSmem<ANISO> &S = *reinterpret_cast<PhiSmem<ANISO> *>(smem_raw);
  constexpr int NPL = PhiSmem<ANISO>::NPL;
  const int tx = threadIdx.x, ty = threadIdx.y, tid = ty * TX + tx;
  const int i0 = blockIdx.x * TX, j0 = blockIdx.y * TY;
  const int k0 = blockIdx.z * kz, k1 = min(k0 + kz, b.nz);
  const int i = i0 + tx, j = j0 + ty;
  const bool active = (i < b.nx) && (j < b.ny);    // owns an interior cell
  const bool inb = (i <= b.nx) && (j <= b.ny);      // interior or ghost column
  const int64_t colo = (int64_t)j * b.pitch + i;   // own column offset

  // load one tile cell (col,row in tile coords) of plane k into smem buffer s
  auto load_cell = [&](int s, int col, int row, int k) {
    const int gi = i0 - 1 + col, gj = j0 - 1 + row;
    const bool ok = gi <= b.nx && gj <= b.ny;
    const int64_t o = (int64_t)k * b.plane + (int64_t)gj * b.pitch + gi;
#pragma unroll
    for (int a = 0; a < NPH; ++a) S.p[s][a][row][col] = ok ? __ldg(b.phi[a] + o) : 0.0;
  };
  auto load_plane = [&](int s, int k) {  // whole tile + ring of plane k
    load_cell(s, tx + 1, ty + 1, k);
    for (int r = tid; r < NRING; r += NTHR) {
      int col, row;
      ring_cell(r, col, row);
      load_cell(s, col, row, k);
    }
  };

  // own-column registers: phi at k-1, k, k+1 and the z-face flux at k-1/2
  double pm[NPH], pc[NPH], pp[NPH], jzm[NPH], jzp[NPH];
  double gdum[NPH][3];
#pragma unroll
  for (int a = 0; a < NPH; ++a) {
    pm[a] = inb ? __ldg(b.phi[a] + (int64_t)(k0 - 1) * b.plane + colo) : 0.0;
    pc[a] = inb ? __ldg(b.phi[a] + (int64_t)k0 * b.plane + colo) : 0.0;
#pragma unroll
    for (int e = 0; e < 3; ++e) gdum[a][e] = 0.0;
  }
  int sm = 0, sc = 1, sp = 2;  // aniso plane slots (k-1, k, k+1)
  if (ANISO) {
    load_plane(sm, k0 - 1);
    load_plane(sc, k0);
    __syncthreads();
    // z-face at k0 - 1/2 between planes k0-1 and k0: tangential (x,y) gradients
    double glo[NPH][3], ghi[NPH][3];
#pragma unroll
    for (int a = 0; a < NPH; ++a) {
      glo[a][0] = cgrad(kp, S.p[sm][a][ty + 1][tx], S.p[sm][a][ty + 1][tx + 2]);
      glo[a][1] = cgrad(kp, S.p[sm][a][ty][tx + 1], S.p[sm][a][ty + 2][tx + 1]);
      ghi[a][0] = cgrad(kp, S.p[sc][a][ty + 1][tx], S.p[sc][a][ty + 1][tx + 2]);
      ghi[a][1] = cgrad(kp, S.p[sc][a][ty][tx + 1], S.p[sc][a][ty + 2][tx + 1]);
      glo[a][2] = ghi[a][2] = 0.0;
    }
    phi_face(kp, pm, pc, glo, ghi, 2, jzm);
  } else {
    phi_face(kp, pm, pc, gdum, gdum, 2, jzm);
  }

  for (int k = k0; k < k1; ++k) {
    const double *tab = b.tab + (int64_t)k * TAB;
#pragma unroll
    for (int a = 0; a < NPH; ++a) pp[a] = inb ? __ldg(b.phi[a] + (int64_t)(k + 1) * b.plane + colo) : 0.0;
    double mu[NMU];
    mu[0] = active ? __ldg(b.mu[0] + (int64_t)k * b.plane + colo) : 0.0;
    mu[1] = active ? __ldg(b.mu[1] + (int64_t)k * b.plane + colo) : 0.0;
    if (ANISO) {
      load_plane(sp, k + 1);
    } else {
#pragma unroll
      for (int a = 0; a < NPH; ++a) S.p[0][a][ty + 1][tx + 1] = pc[a];
      for (int r = tid; r < NRING; r += NTHR) {
        int col, row;
        ring_cell(r, col, row);
        if ((col == 0 || col == RX - 1) && (row == 0 || row == RY - 1)) continue;  // corners unused
        load_cell(0, col, row, k);
      }
    }
    __syncthreads();
    const int cs = ANISO ? sc : 0;
    // ---- faces of plane k: own -x and -y faces, then the tile's far faces
    {
      double jf[NPH], lo[NPH], hi[NPH], gl[NPH][3], gh[NPH][3];
#pragma unroll
      for (int pass = 0; pass < 2; ++pass) {
        const int d = pass;  // 0: x-face (i-1/2), 1: y-face (j-1/2)
        const int lc = d == 0 ? tx : tx + 1, lr = d == 0 ? ty + 1 : ty;
#pragma unroll
        for (int a = 0; a < NPH; ++a) { lo[a] = S.p[cs][a][lr][lc]; hi[a] = S.p[cs][a][ty + 1][tx + 1]; }
        if (ANISO) {
#pragma unroll
          for (int a = 0; a < NPH; ++a) {
            // tangential gradients of the two cells (component d unused)
            gl[a][0] = d == 0 ? 0.0 : cgrad(kp, S.p[cs][a][lr][lc - 1], S.p[cs][a][lr][lc + 1]);
            gl[a][1] = d == 1 ? 0.0 : cgrad(kp, S.p[cs][a][lr - 1][lc], S.p[cs][a][lr + 1][lc]);
            gl[a][2] = cgrad(kp, S.p[sm][a][lr][lc], S.p[sp][a][lr][lc]);
            gh[a][0] = d == 0 ? 0.0 : cgrad(kp, S.p[cs][a][ty + 1][tx], S.p[cs][a][ty + 1][tx + 2]);
            gh[a][1] = d == 1 ? 0.0 : cgrad(kp, S.p[cs][a][ty][tx + 1], S.p[cs][a][ty + 2][tx + 1]);
            gh[a][2] = cgrad(kp, S.p[sm][a][ty + 1][tx + 1], S.p[sp][a][ty + 1][tx + 1]);
          }
        }
        phi_face(kp, lo, hi, ANISO ? gl : gdum, ANISO ? gh : gdum, d, jf);
#pragma unroll
        for (int a = 0; a < NPH; ++a) {
          if (d == 0) S.fx[a][ty][tx] = jf[a];
          else S.fy[a][ty][tx] = jf[a];
        }
      }
      // far faces: +y faces of the last row (warp 0), +x faces of the last column (warp 1)
      if (tid < TX + TY) {
        const int d = tid < TX ? 1 : 0;
        const int c0 = d == 1 ? tid + 1 : TX, r0 = d == 1 ? TY : tid - TX + 1;   // low cell (tile coords)
        const int c1 = d == 1 ? c0 : c0 + 1, r1 = d == 1 ? r0 + 1 : r0;           // high cell
#pragma unroll
        for (int a = 0; a < NPH; ++a) { lo[a] = S.p[cs][a][r0][c0]; hi[a] = S.p[cs][a][r1][c1]; }
        if (ANISO) {
#pragma unroll
          for (int a = 0; a < NPH; ++a) {
            gl[a][0] = d == 0 ? 0.0 : cgrad(kp, S.p[cs][a][r0][c0 - 1], S.p[cs][a][r0][c0 + 1]);
            gl[a][1] = d == 1 ? 0.0 : cgrad(kp, S.p[cs][a][r0 - 1][c0], S.p[cs][a][r0 + 1][c0]);
            gl[a][2] = cgrad(kp, S.p[sm][a][r0][c0], S.p[sp][a][r0][c0]);
            gh[a][0] = d == 0 ? 0.0 : cgrad(kp, S.p[cs][a][r1][c1 - 1], S.p[cs][a][r1][c1 + 1]);
            gh[a][1] = d == 1 ? 0.0 : cgrad(kp, S.p[cs][a][r1 - 1][c1], S.p[cs][a][r1 + 1][c1]);
            gh[a][2] = cgrad(kp, S.p[sm][a][r1][c1], S.p[sp][a][r1][c1]);
          }
        }
        phi_face(kp, lo, hi, ANISO ? gl : gdum, ANISO ? gh : gdum, d, jf);
#pragma unroll
        for (int a = 0; a < NPH; ++a) {
          if (d == 0) S.fx[a][r0 - 1][TX] = jf[a];
          else S.fy[a][TY][c0 - 1] = jf[a];
        }
      }
      // z-face k+1/2 (own column, registers)
      if (ANISO) {
#pragma unroll
        for (int a = 0; a < NPH; ++a) {
          gl[a][0] = cgrad(kp, S.p[cs][a][ty + 1][tx], S.p[cs][a][ty + 1][tx + 2]);
          gl[a][1] = cgrad(kp, S.p[cs][a][ty][tx + 1], S.p[cs][a][ty + 2][tx + 1]);
          gh[a][0] = cgrad(kp, S.p[sp][a][ty + 1][tx], S.p[sp][a][ty + 1][tx + 2]);
          gh[a][1] = cgrad(kp, S.p[sp][a][ty][tx + 1], S.p[sp][a][ty + 2][tx + 1]);
          gl[a][2] = gh[a][2] = 0.0;
        }
      }
      phi_face(kp, pc, pp, ANISO ? gl : gdum, ANISO ? gh : gdum, 2, jzp);
    }
    __syncthreads();
    // ---- cell update of (i, j, k)
    if (active) {
      double gc[NPH][3], jm[3][NPH], jp[3][NPH], out[NPH];
#pragma unroll
      for (int a = 0; a < NPH; ++a) {
        gc[a][0] = cgrad(kp, S.p[cs][a][ty + 1][tx], S.p[cs][a][ty + 1][tx + 2]);
        gc[a][1] = cgrad(kp, S.p[cs][a][ty][tx + 1], S.p[cs][a][ty + 2][tx + 1]);
        gc[a][2] = cgrad(kp, pm[a], pp[a]);
        jm[0][a] = S.fx[a][ty][tx];
        jp[0][a] = S.fx[a][ty][tx + 1];
        jm[1][a] = S.fy[a][ty][tx];
        jp[1][a] = S.fy[a][ty + 1][tx];
        jm[2][a] = jzm[a];
        jp[2][a] = jzp[a];
      }
      phi_cell_update(kp, tab, pc, mu, gc, jm, jp, out);
      const int64_t o = (int64_t)k * b.plane + colo;
#pragma unroll
      for (int a = 0; a < NPH; ++a) b.out[a][o] = out[a];
    }
#pragma unroll
    for (int a = 0; a < NPH; ++a) { pm[a] = pc[a]; pc[a] = pp[a]; jzm[a] = jzp[a]; }
    if (ANISO) { const int t = sm; sm = sc; sc = sp; sp = t; }
    __syncthreads();
  }
}

static int chunk_z(int nz, int nxy_tiles) {
  // enough CTAs to fill the machine several times, chunks >= 16 planes
  int kz = nz;
  while (kz > 16 && (int64_t)nxy_tiles * ((nz + kz - 1) / kz) < 148 * 8) kz = (kz + 1) / 2;
  return kz;
}

void launch_phi_tiled(cudaStream_t s, const KParams &kp, const BlockView &b) {
  const int gx = (b.nx + TX - 1) / TX, gy = (b.ny + TY - 1) / TY;
  const int kz = chunk_z(b.nz, gx * gy);
  dim3 grd(gx, gy, (b.nz + kz - 1) / kz), blk(TX, TY);
  if (kp.aniso) {
    const size_t sm = sizeof(PhiSmem<true>);
    static bool attr = false;
    if (!attr) { cudaFuncSetAttribute(phi_tiled_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm); attr = true; }
    phi_tiled_kernel<true><<<grd, blk, sm, s>>>(kp, b, kz);
  } else {
    const size_t sm = sizeof(PhiSmem<false>);
    phi_tiled_kernel<false><<<grd, blk, sm, s>>>(kp, b, kz);
  }
}

// ===========================================================================
// mu-sweep
// ===========================================================================
// Per plane k the CTA stages phi^{n+1} for planes k-1, k, k+1 (tile + ring +
// corners, for the tangential gradients of the D3C19 anti-trapping faces,
// PAPER.md:179) and the per-cell quantities of plane k (mobility, c^l - c^a,
// dphi, mu: computed once per cell), then evaluates every
// x/y face of the plane once and the z-face k+1/2 per column.
struct MuSmem {
  double pn[3][NPH][RY][RX];
  double M[NMU][RY][RX];
  double dcl[3][NMU][RY][RX];
  double dp[3][RY][RX];
  double mu[NMU][RY][RX];
  double fx[NMU][TY][TX + 1];
  double fy[NMU][TY + 1][TX];
};

__device__ __forceinline__ void q_to_smem(MuSmem &S, int col, int row, const MuQ &q) {
#pragma unroll
  for (int c = 0; c < NMU; ++c) {
    S.M[c][row][col] = q.M[c];
    S.mu[c][row][col] = q.mu[c];
#pragma unroll
    for (int a = 0; a < 3; ++a) S.dcl[a][c][row][col] = q.dcl[a][c];
  }
#pragma unroll
  for (int a = 0; a < 3; ++a) S.dp[a][row][col] = q.dp[a];
}

// MuQ of tile cell (col,row) of plane slot sc from smem; tangential gradients
// (all but component d) from the phi^{n+1} planes sm, sc, sp.
__device__ __forceinline__ void q_from_smem(const KParams &kp, const MuSmem &S, int sm, int sc, int sp, int col,
                                            int row, int d, MuQ &q) {
#pragma unroll
  for (int c = 0; c < NMU; ++c) {
    q.M[c] = S.M[c][row][col];
    q.mu[c] = S.mu[c][row][col];
#pragma unroll
    for (int a = 0; a < 3; ++a) q.dcl[a][c] = S.dcl[a][c][row][col];
  }
#pragma unroll
  for (int a = 0; a < NPH; ++a) {
    q.pn[a] = S.pn[sc][a][row][col];
    q.dp[a] = a < 3 ? S.dp[a][row][col] : 0.0;
    q.gn[a][0] = d == 0 ? 0.0 : cgrad(kp, S.pn[sc][a][row][col - 1], S.pn[sc][a][row][col + 1]);
    q.gn[a][1] = d == 1 ? 0.0 : cgrad(kp, S.pn[sc][a][row - 1][col], S.pn[sc][a][row + 1][col]);
    q.gn[a][2] = d == 2 ? 0.0 : cgrad(kp, S.pn[sm][a][row][col], S.pn[sp][a][row][col]);
  }
}

__global__ void __launch_bounds__(NTHR, 1) mu_tiled_kernel(KParams kp, BlockView b, int kz) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  MuSmem &S = *reinterpret_cast<MuSmem *>(smem_raw);
  const int tx = threadIdx.x, ty = threadIdx.y, tid = ty * TX + tx;
  const int i0 = blockIdx.x * TX, j0 = blockIdx.y * TY;
  const int k0 = blockIdx.z * kz, k1 = min(k0 + kz, b.nz);
  const int i = i0 + tx, j = j0 + ty;
  const bool active = (i < b.nx) && (j < b.ny);
  const bool inb = (i <= b.nx) && (j <= b.ny);
  const int64_t colo = (int64_t)j * b.pitch + i;

  auto gload = [&](const double *p, int gi, int gj, int k, bool ok) -> double {
    return ok ? __ldg(p + (int64_t)k * b.plane + (int64_t)gj * b.pitch + gi) : 0.0;
  };
  auto load_pn_plane = [&](int s, int k) {
    for (int r = tid; r < RX * RY; r += NTHR) {
      const int col = r % RX, row = r / RX;
      const int gi = i0 - 1 + col, gj = j0 - 1 + row;
      const bool ok = gi <= b.nx && gj <= b.ny;
#pragma unroll
      for (int a = 0; a < NPH; ++a) S.pn[s][a][row][col] = gload(b.phin[a], gi, gj, k, ok);
    }
  };
  // per-cell quantities of own column at plane k (registers)
  auto own_q = [&](int k, const double pn[NPH], MuQ &q, double po[NPH], double mu[NMU]) {
#pragma unroll
    for (int a = 0; a < NPH; ++a) po[a] = inb ? __ldg(b.phi[a] + (int64_t)k * b.plane + colo) : 0.0;
#pragma unroll
    for (int c = 0; c < NMU; ++c) mu[c] = inb ? __ldg(b.mu[c] + (int64_t)k * b.plane + colo) : 0.0;
    mu_cell_q(b.tab + (int64_t)k * TAB, po, pn, mu, q);
  };

  int sm = 0, sc = 1, sp = 2;
  load_pn_plane(sm, k0 - 1);
  load_pn_plane(sc, k0);
  // own column: quantities at k0-1 and k0, z-face at k0 - 1/2
  double po_c[NPH], pn_c[NPH], mu_c[NMU], fzm[NMU];
  {
    double po_m[NPH], pn_m[NPH], mu_m[NMU];
#pragma unroll
    for (int a = 0; a < NPH; ++a) {
      pn_m[a] = inb ? __ldg(b.phin[a] + (int64_t)(k0 - 1) * b.plane + colo) : 0.0;
      pn_c[a] = inb ? __ldg(b.phin[a] + (int64_t)k0 * b.plane + colo) : 0.0;
    }
    MuQ qm, qc;
    own_q(k0 - 1, pn_m, qm, po_m, mu_m);
    own_q(k0, pn_c, qc, po_c, mu_c);
    __syncthreads();
#pragma unroll
    for (int a = 0; a < NPH; ++a) {
      qm.gn[a][0] = cgrad(kp, S.pn[sm][a][ty + 1][tx], S.pn[sm][a][ty + 1][tx + 2]);
      qm.gn[a][1] = cgrad(kp, S.pn[sm][a][ty][tx + 1], S.pn[sm][a][ty + 2][tx + 1]);
      qc.gn[a][0] = cgrad(kp, S.pn[sc][a][ty + 1][tx], S.pn[sc][a][ty + 1][tx + 2]);
      qc.gn[a][1] = cgrad(kp, S.pn[sc][a][ty][tx + 1], S.pn[sc][a][ty + 2][tx + 1]);
      qm.gn[a][2] = qc.gn[a][2] = 0.0;
    }
    mu_face(kp, qm, qc, 2, fzm);
  }

  for (int k = k0; k < k1; ++k) {
    const double *tab = b.tab + (int64_t)k * TAB;
    // phi^{n+1} plane k+1 (tile + ring + corners)
    load_pn_plane(sp, k + 1);
    // per-cell quantities of plane k: own cell ...
    {
      MuQ q;
      mu_cell_q(tab, po_c, pn_c, mu_c, q);
      q_to_smem(S, tx + 1, ty + 1, q);
    }
    // ... and the ring (no corners); phi^{n+1}(k) of the ring is in slot sc
    for (int r = tid; r < NRING; r += NTHR) {
      int col, row;
      ring_cell(r, col, row);
      if ((col == 0 || col == RX - 1) && (row == 0 || row == RY - 1)) continue;
      const int gi = i0 - 1 + col, gj = j0 - 1 + row;
      const bool ok = gi <= b.nx && gj <= b.ny;
      double po[NPH], pn[NPH], mu[NMU];
#pragma unroll
      for (int a = 0; a < NPH; ++a) { po[a] = gload(b.phi[a], gi, gj, k, ok); pn[a] = S.pn[sc][a][row][col]; }
#pragma unroll
      for (int c = 0; c < NMU; ++c) mu[c] = gload(b.mu[c], gi, gj, k, ok);
      MuQ q;
      mu_cell_q(tab, po, pn, mu, q);
      q_to_smem(S, col, row, q);
    }
    // own column at k+1 (for the z-face k+1/2 and the next iteration)
    double po_n[NPH], pn_n[NPH], mu_n[NMU];
#pragma unroll
    for (int a = 0; a < NPH; ++a) pn_n[a] = inb ? __ldg(b.phin[a] + (int64_t)(k + 1) * b.plane + colo) : 0.0;
    MuQ qn;
    own_q(k + 1, pn_n, qn, po_n, mu_n);
    __syncthreads();
    // ---- faces of plane k
    {
      double f[NMU];
      MuQ ql, qh;
      // own -x face
      q_from_smem(kp, S, sm, sc, sp, tx, ty + 1, 0, ql);
      q_from_smem(kp, S, sm, sc, sp, tx + 1, ty + 1, 0, qh);
      mu_face(kp, ql, qh, 0, f);
      S.fx[0][ty][tx] = f[0];
      S.fx[1][ty][tx] = f[1];
      // own -y face
      q_from_smem(kp, S, sm, sc, sp, tx + 1, ty, 1, ql);
      q_from_smem(kp, S, sm, sc, sp, tx + 1, ty + 1, 1, qh);
      mu_face(kp, ql, qh, 1, f);
      S.fy[0][ty][tx] = f[0];
      S.fy[1][ty][tx] = f[1];
      // far faces: +y of the last row (warp 0), +x of the last column (warp 1)
      if (tid < TX) {
        q_from_smem(kp, S, sm, sc, sp, tid + 1, TY, 1, ql);
        q_from_smem(kp, S, sm, sc, sp, tid + 1, TY + 1, 1, qh);
        mu_face(kp, ql, qh, 1, f);
        S.fy[0][TY][tid] = f[0];
        S.fy[1][TY][tid] = f[1];
      } else if (tid < TX + TY) {
        const int r = tid - TX + 1;
        q_from_smem(kp, S, sm, sc, sp, TX, r, 0, ql);
        q_from_smem(kp, S, sm, sc, sp, TX + 1, r, 0, qh);
        mu_face(kp, ql, qh, 0, f);
        S.fx[0][r - 1][TX] = f[0];
        S.fx[1][r - 1][TX] = f[1];
      }
    }
    // z-face k+1/2: own cell (k, from smem) and (k+1, registers)
    double fzp[NMU];
    {
      MuQ qc;
      q_from_smem(kp, S, sm, sc, sp, tx + 1, ty + 1, 2, qc);
#pragma unroll
      for (int a = 0; a < NPH; ++a) {
        qn.gn[a][0] = cgrad(kp, S.pn[sp][a][ty + 1][tx], S.pn[sp][a][ty + 1][tx + 2]);
        qn.gn[a][1] = cgrad(kp, S.pn[sp][a][ty][tx + 1], S.pn[sp][a][ty + 2][tx + 1]);
        qn.gn[a][2] = 0.0;
      }
      mu_face(kp, qc, qn, 2, fzp);
    }
    __syncthreads();
    // ---- cell update of (i, j, k)
    if (active) {
      double divf[NMU], out[NMU];
#pragma unroll
      for (int c = 0; c < NMU; ++c)
        divf[c] = ((S.fx[c][ty][tx + 1] - S.fx[c][ty][tx]) + (S.fy[c][ty + 1][tx] - S.fy[c][ty][tx])) +
                  (fzp[c] - fzm[c]);
      mu_cell_update(kp, tab, po_c, pn_c, mu_c, divf, out);
      const int64_t o = (int64_t)k * b.plane + colo;
      b.out[0][o] = out[0];
      b.out[1][o] = out[1];
    }
#pragma unroll
    for (int a = 0; a < NPH; ++a) { po_c[a] = po_n[a]; pn_c[a] = pn_n[a]; }
#pragma unroll
    for (int c = 0; c < NMU; ++c) { mu_c[c] = mu_n[c]; fzm[c] = fzp[c]; }
    { const int t = sm; sm = sc; sc = sp; sp = t; }
    __syncthreads();
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
