// pf_kernels.cu — per-plane table, naive (reference-variant) sweeps, halo box
// copies, device initial condition, window front reduction, NaN check and
// gather/scatter between the padded ghost layout and the public SoA layout.
#include <algorithm>
#include <cmath>
#include "pf_kernels.cuh"

namespace pf {

// ---------------------------------------------------------------------------
// a1: per-plane coefficient table.  One thread per
// global window plane kg = -1..NZ; T = T0 + G((kg + zorig + 1/2) dx - v n dt).
// ---------------------------------------------------------------------------
__global__ void table_kernel(double *tab, int64_t nplanes, TabParams tp, int64_t step, int64_t zorig,
                             const int64_t *d_step) {
  const int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (r >= nplanes) return;
  if (d_step) step = *d_step;   // graph replays: the time level lives on the device
  const int64_t kg = r - 1;
  const double z = ((double)(kg + zorig) + 0.5) * tp.dx;
  const double T = tp.T0 + tp.G * (z - tp.v * ((double)step * tp.dt));
  const double th = T - tp.T_eut;
  double *row = tab + r * TAB;
  row[T_T] = T;
  row[T_EPST] = tp.eps * T;
  row[T_TEPS] = T / tp.eps;
  row[T_EPSTDX] = tp.eps * T / tp.dx;
  row[T_EPSTDX16] = tp.eps * T / (16.0 * tp.dx * tp.dx);
  for (int a = 0; a < NPH; ++a) {
    row[T_B + a] = tp.L[a] * th / tp.T_eut;
    for (int c = 0; c < NMU; ++c) {
      const double A = tp.A0[a][c] + tp.A1[a][c] * th;
      const double i2a = 1.0 / (2.0 * A);
      row[T_INV2A + a * 2 + c] = i2a;
      row[T_INV4A + a * 2 + c] = 0.5 * i2a;
      row[T_CHAT + a * 2 + c] = tp.c0[a][c] + tp.m[a][c] * th;
      row[T_KAPPA + a * 2 + c] = 2.0 * tp.A1[a][c] * i2a * i2a;
      row[T_MC + a * 2 + c] = tp.D[a][c] * i2a;
    }
  }
  for (int a = 0; a < 3; ++a)
    for (int c = 0; c < NMU; ++c) {
      row[T_DI2A + a * 2 + c] = row[T_INV2A + LIQ * 2 + c] - row[T_INV2A + a * 2 + c];
      row[T_DCHAT + a * 2 + c] = row[T_CHAT + LIQ * 2 + c] - row[T_CHAT + a * 2 + c];
      row[T_DCHAT2 + a * 2 + c] = 2.0 * row[T_DCHAT + a * 2 + c];   // exact
    }
}

void launch_table(cudaStream_t s, double *tab, int64_t nplanes, const TabParams &tp, int64_t step, int64_t zorig,
                  const int64_t *d_step) {
  table_kernel<<<(unsigned)((nplanes + 127) / 128), 128, 0, s>>>(tab, nplanes, tp, step, zorig, d_step);
}

__global__ void step_inc_kernel(int64_t *d_step) { *d_step += 1; }
void launch_step_inc(cudaStream_t s, int64_t *d_step) { step_inc_kernel<<<1, 1, 0, s>>>(d_step); }

// ---------------------------------------------------------------------------
// Naive phi-sweep: one thread per cell, every neighbour read from global
// memory, each face evaluated from both of its cells (identical bits thanks
// to the pinned face routine).  Reference variant for the tiled kernel.
// ---------------------------------------------------------------------------
__device__ __forceinline__ void load_phi(const BlockView &b, int64_t o, double v[NPH]) {
#pragma unroll
  for (int a = 0; a < NPH; ++a) v[a] = __ldg(b.phi[a] + o);
}

// raw centre differences phi(c+e) - phi(c-e) of all phases (the convention of
// phi_face and phi_cell_rhs0); component `skip` (the face normal of a
// neighbour cell, never used) is set to 0 instead of reading 2 cells away.
__device__ __forceinline__ void centre_diffs(const double *const f[NPH], int64_t o, const int64_t st[3],
                                             double g[NPH][3], int skip = -1) {
#pragma unroll
  for (int e = 0; e < 3; ++e)
#pragma unroll
    for (int a = 0; a < NPH; ++a)
      g[a][e] = (e == skip) ? 0.0 : cdiff(__ldg(f[a] + o - st[e]), __ldg(f[a] + o + st[e]));
}

__global__ void __launch_bounds__(128) phi_naive_kernel(KParams kp, BlockView b) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  const int j = blockIdx.y * blockDim.y + threadIdx.y;
  const int k = blockIdx.z;
  if (i >= b.nx || j >= b.ny) return;
  const int64_t st[3] = {1, b.pitch, b.plane};
  const int64_t o = k * b.plane + j * b.pitch + i;
  double ph[NPH], mu[NMU], gc[NPH][3], jm[3][NPH], jp[3][NPH], out[NPH];
  load_phi(b, o, ph);
  mu[0] = __ldg(b.mu[0] + o);
  mu[1] = __ldg(b.mu[1] + o);
  centre_diffs(b.phi, o, st, gc);
#pragma unroll
  for (int d = 0; d < 3; ++d) {
    double pl[NPH], pu[NPH], gl[NPH][3], gu[NPH][3];
    load_phi(b, o - st[d], pl);
    load_phi(b, o + st[d], pu);
    if (kp.aniso) {
      centre_diffs(b.phi, o - st[d], st, gl, d);
      centre_diffs(b.phi, o + st[d], st, gu, d);
    }
    phi_face(kp, pl, ph, gl, gc, d, jm[d]);
    phi_face(kp, ph, pu, gc, gu, d, jp[d]);
  }
  phi_cell_update(kp, b.tab + (int64_t)k * TAB, ph, mu, gc, jm, jp, out);
#pragma unroll
  for (int a = 0; a < NPH; ++a) b.out[a][o] = out[a];
}

void launch_phi_naive(cudaStream_t s, const KParams &kp, const BlockView &b) {
  dim3 blk(32, 4, 1), grd((b.nx + 31) / 32, (b.ny + 3) / 4, b.nz);
  phi_naive_kernel<<<grd, blk, 0, s>>>(kp, b);
}

// ---------------------------------------------------------------------------
// Naive mu-sweep.
// ---------------------------------------------------------------------------
__device__ __forceinline__ void load_muq(const KParams &kp, const BlockView &b, int64_t o, const int64_t st[3],
                                         const double *tabrow, MuQ &q, int skip = -1) {
  double po[NPH], pn[NPH], mu[NMU];
#pragma unroll
  for (int a = 0; a < NPH; ++a) { po[a] = __ldg(b.phi[a] + o); pn[a] = __ldg(b.phin[a] + o); }
  mu[0] = __ldg(b.mu[0] + o);
  mu[1] = __ldg(b.mu[1] + o);
  mu_cell_q(tabrow, po, pn, mu, q);
#pragma unroll
  for (int e = 0; e < 3; ++e)   // raw centre differences (mu_face_t is scale-free in them)
#pragma unroll
    for (int a = 0; a < NPH; ++a)
      q.gn[a][e] = (e == skip) ? 0.0 : cdiff(__ldg(b.phin[a] + o - st[e]), __ldg(b.phin[a] + o + st[e]));
}

__global__ void __launch_bounds__(128) mu_naive_kernel(KParams kp, BlockView b) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  const int j = blockIdx.y * blockDim.y + threadIdx.y;
  const int k = blockIdx.z;
  if (i >= b.nx || j >= b.ny) return;
  const int64_t st[3] = {1, b.pitch, b.plane};
  const int64_t o = k * b.plane + j * b.pitch + i;
  const double *tab = b.tab + (int64_t)k * TAB;
  MuQ qc;
  load_muq(kp, b, o, st, tab, qc);
  double divf[NMU] = {0.0, 0.0};
#pragma unroll 1
  for (int d = 0; d < 3; ++d) {
    MuQ ql, qu;
    load_muq(kp, b, o - st[d], st, d == 2 ? tab - TAB : tab, ql, d);
    load_muq(kp, b, o + st[d], st, d == 2 ? tab + TAB : tab, qu, d);
    double fm[NMU], fp[NMU];
    mu_face(kp, ql, qc, d, fm);
    mu_face(kp, qc, qu, d, fp);
    divf[0] += fp[0] - fm[0];
    divf[1] += fp[1] - fm[1];
  }
  double po[NPH], out[NMU];
#pragma unroll
  for (int a = 0; a < NPH; ++a) po[a] = __ldg(b.phi[a] + o);
  mu_cell_update(kp, tab, po, qc.pn, qc.mu, divf, out);
  b.out[0][o] = out[0];
  b.out[1][o] = out[1];
}

void launch_mu_naive(cudaStream_t s, const KParams &kp, const BlockView &b) {
  dim3 blk(32, 4, 1), grd((b.nx + 31) / 32, (b.ny + 3) / 4, b.nz);
  mu_naive_kernel<<<grd, blk, 0, s>>>(kp, b);
}

// ---------------------------------------------------------------------------
// Halo: strided 3D box copies (local copy, pack into / unpack from NCCL
// buffers).  blockIdx.y = op index.
// ---------------------------------------------------------------------------
// One launch copies a list of boxes; op q owns CTAs [cta0_q, cta0_{q+1}),
// each CTA 1024 cells of it.  A box is at most a face of a block (< 2^32
// cells), so the index split uses 32-bit division.
__global__ void copy_kernel(const CopyOp *__restrict__ ops, int nops) {
  int q = 0;
  while (q + 1 < nops && __ldg(&ops[q + 1].cta0) <= (int64_t)blockIdx.x) ++q;
  const CopyOp op = ops[q];
  const uint32_t ex = (uint32_t)op.ex, ey = (uint32_t)op.ey;
  const uint32_t n = ex * ey * (uint32_t)op.ez;
  const uint32_t base = (uint32_t)(blockIdx.x - op.cta0) * COPY_CELLS_PER_CTA;
#pragma unroll
  for (int e = 0; e < COPY_CELLS_PER_CTA / 256; ++e) {
    const uint32_t t = base + e * 256 + threadIdx.x;
    if (t >= n) break;
    const uint32_t r = t / ex, x = t - r * ex, z = r / ey, y = r - z * ey;
    const int64_t so = x * op.ssx + y * op.ssy + z * op.ssz;
    const int64_t dof = x * op.dsx + y * op.dsy + z * op.dsz;
    // all components' loads first (the source and destination pointers could
    // alias as far as the compiler knows): four reads in flight per thread
    double v[NPH];
#pragma unroll
    for (int c = 0; c < NPH; ++c) v[c] = c < op.ncomp ? op.src[c][so] : 0.0;
    if (op.xpad >= 0) {
#pragma unroll
      for (int c = 0; c < NPH; ++c) {
        if (c >= op.ncomp) break;
        double2 *sec = reinterpret_cast<double2 *>(op.dst[c] + dof - op.xpad);
        sec[0] = make_double2(op.xpad == 0 ? v[c] : 0.0, op.xpad == 1 ? v[c] : 0.0);
        sec[1] = make_double2(op.xpad == 2 ? v[c] : 0.0, op.xpad == 3 ? v[c] : 0.0);
      }
    } else {
#pragma unroll
      for (int c = 0; c < NPH; ++c)
        if (c < op.ncomp) op.dst[c][dof] = v[c];
    }
  }
}

void launch_copy(cudaStream_t s, const CopyOp *d_ops, int nops, int64_t nctas) {
  if (nops <= 0 || nctas <= 0) return;
  copy_kernel<<<(unsigned)nctas, 256, 0, s>>>(d_ops, nops);
}

// ---------------------------------------------------------------------------
// Initial condition (recipe DESIGN.md §3).  Same counter-
// based splitmix64 generator as the shared input module, implemented here
// independently.
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint64_t mix64(uint64_t z) {
  z += 0x9E3779B97F4A7C15ULL;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}
__device__ __forceinline__ double u01(uint64_t seed, uint64_t stream, uint64_t idx) {
  const uint64_t r = mix64(mix64(seed ^ (stream * 0xD1B54A32D192ED03ULL)) ^ idx);
  return (double)(r >> 11) * 0x1.0p-53;
}
__device__ __forceinline__ double ramp(double d, double W) {
  if (d >= 0.5 * W) return 1.0;
  if (d <= -0.5 * W) return 0.0;
  return 0.5 * (1.0 + sin(M_PI * d / W));
}
__device__ __forceinline__ double min_image(double d, double n) {
  if (d > 0.5 * n) d -= n;
  else if (d < -0.5 * n) d += n;
  return d;
}

__global__ void init_kernel(InitSpec is, BlockView b, int64_t x0, int64_t y0, int64_t z0) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  const int j = blockIdx.y * blockDim.y + threadIdx.y;
  if (i >= b.nx || j >= b.ny) return;
  const int64_t gi = x0 + i, gj = y0 + j;
  int p1, p2;
  double r = 1.0;
  if (is.kind == 0) {
    const double x = gi + 0.5, y = gj + 0.5;
    int best = -1, other = -1;
    double bd = 0, brx = 0, bry = 0, od = 0, orx = 0, ory = 0;
    for (int q = 0; q < is.n_seeds; ++q) {
      const double rx = min_image(x - is.sx[q], (double)is.NX), ry = min_image(y - is.sy[q], (double)is.NY);
      const double d = rx * rx + ry * ry;
      if (best < 0 || d < bd) { best = q; bd = d; brx = rx; bry = ry; }
    }
    p1 = p2 = is.sp[best];
    for (int q = 0; q < is.n_seeds; ++q) {
      if (is.sp[q] == p1) continue;
      const double rx = min_image(x - is.sx[q], (double)is.NX), ry = min_image(y - is.sy[q], (double)is.NY);
      const double d = rx * rx + ry * ry;
      if (other < 0 || d < od) { other = q; od = d; orx = rx; ory = ry; }
    }
    if (other >= 0) {
      const double ex = brx - orx, ey = bry - ory, sep = sqrt(ex * ex + ey * ey);
      if (sep > 0) { p2 = is.sp[other]; r = ramp((od - bd) / (2.0 * sep), is.W); }
    }
  } else if (is.kind == 1) {
    int l = 0;
    while (l + 1 < is.nlam && is.lam[l + 1] <= gi) ++l;
    const double x = gi + 0.5, dl = x - (double)is.lam[l], dr = (double)is.lam[l + 1] - x;
    const int nb = dl < dr ? (l - 1 + is.nlam) % is.nlam : (l + 1) % is.nlam;
    p1 = l % 3;
    p2 = nb % 3;
    if (p1 != p2) r = ramp(dl < dr ? dl : dr, is.W);
  } else {
    p1 = p2 = is.planar_phase;
  }
  for (int k = 0; k < b.nz; ++k) {
    const int64_t kg = z0 + k;
    const int64_t o = k * b.plane + j * b.pitch + i;
    const double sol = ramp(is.layer_height - (kg + 0.5), is.W);
    double ph[NPH] = {0, 0, 0, 0};
    ph[p1] += sol * r;
    ph[p2] += sol * (1.0 - r);
    ph[LIQ] = 1.0 - sol;
#pragma unroll
    for (int a = 0; a < NPH; ++a) b.out[a][o] = ph[a];
    const uint64_t g = (uint64_t)((kg * is.NY + gj) * is.NX + gi);
    for (int c = 0; c < NMU; ++c)
      const_cast<double *>(b.mu[c])[o] = is.mu_noise == 0.0 ? 0.0 : is.mu_noise * (2.0 * u01(is.seed, 8 + c, g) - 1.0);
  }
}

void launch_init(cudaStream_t s, const InitSpec &is, double *const phi[NPH], double *const mu[NMU], int nx, int ny,
                 int nz, int64_t pitch, int64_t plane, int64_t x0, int64_t y0, int64_t z0) {
  BlockView b{};
  for (int a = 0; a < NPH; ++a) b.out[a] = phi[a];
  for (int c = 0; c < NMU; ++c) b.mu[c] = mu[c];
  b.nx = nx; b.ny = ny; b.nz = nz; b.pitch = pitch; b.plane = plane;
  dim3 blk(32, 4), grd((nx + 31) / 32, (ny + 3) / 4);
  init_kernel<<<grd, blk, 0, s>>>(is, b, x0, y0, z0);
}

// fill interior plane (i in [0,nx), j in [0,ny)) of ncomp arrays with vals[c]
__global__ void fill_plane_kernel(double *f0, double *f1, double *f2, double *f3, int ncomp, double v0, double v1,
                                  double v2, double v3, int nx, int ny, int64_t pitch) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x, j = blockIdx.y;
  if (i >= nx) return;
  const int64_t o = j * pitch + i;
  f0[o] = v0;
  f1[o] = v1;
  if (ncomp > 2) { f2[o] = v2; f3[o] = v3; }
}

void launch_fill_plane(cudaStream_t s, double *const f[NPH], int ncomp, const double *vals, int nx, int ny,
                       int64_t pitch) {
  fill_plane_kernel<<<dim3((nx + 127) / 128, ny), 128, 0, s>>>(f[0], f[1], ncomp > 2 ? f[2] : nullptr,
                                                                ncomp > 2 ? f[3] : nullptr, ncomp, vals[0], vals[1],
                                                                ncomp > 2 ? vals[2] : 0.0, ncomp > 2 ? vals[3] : 0.0,
                                                                nx, ny, pitch);
}

// ---------------------------------------------------------------------------
// Window front (reading R16): highest plane with phi_l < thr, and highest
// plane with phi_l < 1.  d_out[0] = max (k+kbase+1) for phi_l < thr, d_out[1]
// the same for phi_l < 1 (0 = none).  One block per plane.
// ---------------------------------------------------------------------------
__global__ void front_kernel(const double *phil, int nx, int ny, int64_t pitch, int64_t plane, double thr,
                             int64_t kbase, unsigned long long *out) {
  const int k = blockIdx.x;
  int below = 0, nonliq = 0;
  for (int t = threadIdx.x; t < nx * ny; t += blockDim.x) {
    const int i = t % nx, j = t / nx;
    const double v = phil[k * plane + j * pitch + i];
    below |= (v < thr);
    nonliq |= (v < 1.0);
  }
  below = __syncthreads_or(below);
  nonliq = __syncthreads_or(nonliq);
  if (threadIdx.x == 0) {
    if (below) atomicMax(out + 0, (unsigned long long)(k + kbase + 1));
    if (nonliq) atomicMax(out + 1, (unsigned long long)(k + kbase + 1));
  }
}

void launch_front(cudaStream_t s, const double *phil, int nx, int ny, int nz, int64_t pitch, int64_t plane,
                  double thr, int64_t kbase, unsigned long long *d_out) {
  front_kernel<<<nz, 256, 0, s>>>(phil, nx, ny, pitch, plane, thr, kbase, d_out);
}

// NaN/Inf check: d_first = min linear (comp, k, j, i) index of a non-finite value
__global__ void nancheck_kernel(const double *f0, const double *f1, const double *f2, const double *f3, int ncomp,
                                int nx, int ny, int nz, int64_t pitch, int64_t plane, unsigned long long *first) {
  const int64_t n = (int64_t)nx * ny * nz;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n; t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = t % nx, j = (t / nx) % ny, k = t / ((int64_t)nx * ny);
    const int64_t o = k * plane + j * pitch + i;
    const double *fs[4] = {f0, f1, f2, f3};
    for (int c = 0; c < ncomp; ++c)
      if (!isfinite(fs[c][o])) atomicMin(first, (unsigned long long)(c * n + t));
  }
}

void launch_nancheck(cudaStream_t s, const double *const f[NPH], int ncomp, int nx, int ny, int nz, int64_t pitch,
                     int64_t plane, unsigned long long *d_first) {
  nancheck_kernel<<<148 * 8, 256, 0, s>>>(f[0], f[1], ncomp > 2 ? f[2] : nullptr, ncomp > 2 ? f[3] : nullptr, ncomp,
                                          nx, ny, nz, pitch, plane, d_first);
}

// gather (padded field -> compact SoA box inside a larger compact array) or
// scatter.  One CTA per x-row (grid-stride over the ny*nz rows), threads along
// the row: coalesced on both sides, the index split once per row.
__global__ void gather_kernel(const double *f0, const double *f1, const double *f2, const double *f3, double *w0,
                              double *w1, double *w2, double *w3, int ncomp, int nx, int ny, int nz, int64_t pitch,
                              int64_t plane, double *dst, int64_t dnx, int64_t dny, int64_t dn, int64_t ox,
                              int64_t oy, int64_t oz, int scatter) {
  const double *fs[4] = {f0, f1, f2, f3};
  double *ws[4] = {w0, w1, w2, w3};
  const int64_t rows = (int64_t)ny * nz;
  for (int64_t r = blockIdx.x; r < rows; r += gridDim.x) {
    const int64_t j = r % ny, k = r / ny;
    const int64_t o = k * plane + j * pitch;
    const int64_t d = ((oz + k) * dny + (oy + j)) * dnx + ox;
    for (int i = threadIdx.x; i < nx; i += blockDim.x) {
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        if (c >= ncomp) break;
        if (scatter) ws[c][o + i] = dst[c * dn + d + i];
        else dst[c * dn + d + i] = fs[c][o + i];
      }
    }
  }
}

void launch_gather(cudaStream_t s, const double *const f[NPH], int ncomp, int nx, int ny, int nz, int64_t pitch,
                   int64_t plane, double *dst, int64_t dnx, int64_t dny, int64_t dn, int64_t ox, int64_t oy, int64_t oz,
                   bool scatter, double *const fw[NPH]) {
  const double *z = nullptr;
  double *w[4] = {nullptr, nullptr, nullptr, nullptr};
  if (scatter) for (int c = 0; c < ncomp; ++c) w[c] = fw[c];
  const double *r[4] = {z, z, z, z};
  if (!scatter) for (int c = 0; c < ncomp; ++c) r[c] = f[c];
  const int64_t rows = (int64_t)ny * nz;
  const unsigned grid = (unsigned)std::min<int64_t>(rows, 148 * 16);
  gather_kernel<<<grid, 256, 0, s>>>(r[0], r[1], r[2], r[3], w[0], w[1], w[2], w[3], ncomp, nx, ny, nz, pitch, plane,
                                     dst, dnx, dny, dn, ox, oy, oz, scatter ? 1 : 0);
}

// FP32 checkpoint conversion: one padded binary64 component
// <-> a compact binary32 box (x fastest) at offset (ox, oy, oz) inside a
// dnx*dny*... array.  double -> float is the IEEE round-to-nearest-even cast,
// float -> double is exact.
__global__ void cvt32_kernel(double *f, int nx, int ny, int nz, int64_t pitch, int64_t plane, float *dst,
                             int64_t dnx, int64_t dny, int64_t ox, int64_t oy, int64_t oz, int to_fields) {
  const int64_t rows = (int64_t)ny * nz;   // one CTA per x-row, as gather_kernel
  for (int64_t r = blockIdx.x; r < rows; r += gridDim.x) {
    const int64_t j = r % ny, k = r / ny;
    const int64_t o = k * plane + j * pitch;
    const int64_t d = ((oz + k) * dny + (oy + j)) * dnx + ox;
    for (int i = threadIdx.x; i < nx; i += blockDim.x) {
      if (to_fields) f[o + i] = (double)dst[d + i];
      else dst[d + i] = __double2float_rn(f[o + i]);
    }
  }
}

void launch_cvt32(cudaStream_t s, double *f, int nx, int ny, int nz, int64_t pitch, int64_t plane, float *dst,
                  int64_t dnx, int64_t dny, int64_t ox, int64_t oy, int64_t oz, bool to_fields) {
  const int64_t rows = (int64_t)ny * nz;
  const unsigned grid = (unsigned)std::min<int64_t>(rows, 148 * 16);
  cvt32_kernel<<<grid, 256, 0, s>>>(f, nx, ny, nz, pitch, plane, dst, dnx, dny, ox, oy, oz, to_fields ? 1 : 0);
}

}  // namespace pf
