// pf_mesh.cu — marching-cubes interface meshes on the device (NEXT-4;
// "a custom marching cubes algorithm based on
// [lorensen1987marching] ... generates meshes locally on each block, using the
// phi values as input.  For each phase, a mesh is generated ...  The marching
// cubes algorithm extends to the ghost regions such that the local meshes can
// be stitched together").  The cube variant is reading R26:
// samples at cell centres, a corner is inside when phi_a > iso, the surface of
// a cube is assembled from per-face segments (so two cubes sharing a face
// always agree: watertight), cycles are fanned from an apex that puts no fan
// diagonal into a cube face, vertices are identified by their global grid
// edge.  The 256-case table is generated here from those rules.
//
// Device work per call, deterministic order (cubes by (k, j, i), triangles in
// table order — the order a serial sweep would emit them):
//   1. count: one warp per cube row (y, z), lanes over x, triangle counts of
//      the row's cubes summed;
//   2. exclusive scan of the row counts (cub);
//   3. emit: one warp per row again, a warp scan of the per-cube counts gives
//      each cube its slot; vertices are interpolated with the same
//      IEEE-rounded operations as a scalar evaluation.
// Cube corners are read straight from the blocks' fields: the corner at the
// upper face of a block is its ghost layer (periodic wrap or the neighbour's
// data after the step's halo exchange), which is what "extends to the ghost
// regions" means.
#include <cub/cub.cuh>
#include <cstring>
#include "pf_kernels.cuh"

namespace pf {

namespace {

// cube edges: lower corner, upper corner, axis.  Corner c = dx + 2 dy + 4 dz.
// Edges 0-3 run along x at (dy, dz) = (e & 1, e >> 1), 4-7 along y at (dx, dz),
// 8-11 along z at (dx, dy).
struct Edge { int c0, c1, axis; };

Edge cube_edge(int e) {
  const int p = e & 1, q = (e >> 1) & 1, ax = e >> 2;
  if (ax == 0) return {2 * p + 4 * q, 2 * p + 4 * q + 1, 0};
  if (ax == 1) return {p + 4 * q, p + 4 * q + 2, 1};
  return {p + 2 * q, p + 2 * q + 4, 2};
}

int edge_between(int a, int b) {
  for (int e = 0; e < 12; ++e) {
    const Edge E = cube_edge(e);
    if ((E.c0 == a && E.c1 == b) || (E.c0 == b && E.c1 == a)) return e;
  }
  return -1;
}

// the six faces, corners counter-clockwise seen from outside
void cube_faces(int F[6][4]) {
  for (int a = 0; a < 3; ++a) {
    const int u = (a + 1) % 3, v = (a + 2) % 3;   // e_u x e_v = +e_a
    for (int side = 0; side < 2; ++side) {
      static const int uv[4][2] = {{0, 0}, {1, 0}, {1, 1}, {0, 1}};
      for (int r = 0; r < 4; ++r) {
        const int q = side == 1 ? r : 3 - r;        // outward normal -e_a: reversed
        int d[3];
        d[a] = side; d[u] = uv[q][0]; d[v] = uv[q][1];
        F[2 * a + side][r] = d[0] + 2 * d[1] + 4 * d[2];
      }
    }
  }
}

bool edges_share_face(int e0, int e1, const int F[6][4]) {
  const Edge A = cube_edge(e0), B = cube_edge(e1);
  const int cs[4] = {A.c0, A.c1, B.c0, B.c1};
  for (int f = 0; f < 6; ++f) {
    bool all = true;
    for (int c : cs) {
      bool in = false;
      for (int r = 0; r < 4; ++r) in = in || F[f][r] == c;
      all = all && in;
    }
    if (all) return true;
  }
  return false;
}

// table[case] = {ntri, e00, e01, e02, e10, ...}: at most 5 triangles
constexpr int MC_MAXT = 5;
void build_table(int8_t tab[256][1 + 3 * MC_MAXT]) {
  int F[6][4];
  cube_faces(F);
  for (int cs = 0; cs < 256; ++cs) {
    bool ins[8];
    for (int c = 0; c < 8; ++c) ins[c] = (cs >> c) & 1;
    int nxt[12];
    for (int e = 0; e < 12; ++e) nxt[e] = -1;
    // per face: every maximal run of inside corners q_a..q_b gives a segment
    // from its entry edge (q_a-1, q_a) to its exit edge (q_b, q_b+1)
    for (int f = 0; f < 6; ++f) {
      bool fi[4];
      int nin = 0;
      for (int r = 0; r < 4; ++r) { fi[r] = ins[F[f][r]]; nin += fi[r]; }
      if (nin == 0 || nin == 4) continue;
      for (int a = 0; a < 4; ++a) {
        if (!fi[a] || fi[(a + 3) & 3]) continue;
        int b = a;
        while (fi[(b + 1) & 3]) b = (b + 1) & 3;
        nxt[edge_between(F[f][(a + 3) & 3], F[f][a])] = edge_between(F[f][b], F[f][(b + 1) & 3]);
      }
    }
    int nt = 0;
    bool seen[12] = {};
    for (int start = 0; start < 12; ++start) {   // cycles in order of their smallest edge
      if (nxt[start] < 0 || seen[start]) continue;
      int cyc[12], m = 0;
      for (int e = start; !seen[e]; e = nxt[e]) { seen[e] = true; cyc[m++] = e; }
      // apex: smallest edge sharing no cube face with a non-adjacent cycle vertex
      int best = -1;
      for (int r = 0; r < m; ++r) {
        bool ok = true;
        for (int t = 2; t < m - 1; ++t) ok = ok && !edges_share_face(cyc[r], cyc[(r + t) % m], F);
        if (ok && (best < 0 || cyc[r] < cyc[best])) best = r;
      }
      for (int t = 1; t < m - 1; ++t) {
        tab[cs][1 + 3 * nt + 0] = (int8_t)cyc[best];
        tab[cs][1 + 3 * nt + 1] = (int8_t)cyc[(best + t) % m];
        tab[cs][1 + 3 * nt + 2] = (int8_t)cyc[(best + t + 1) % m];
        ++nt;
      }
    }
    tab[cs][0] = (int8_t)nt;
  }
}

__constant__ int8_t c_mc[256][1 + 3 * MC_MAXT];

struct MeshArgs {
  const double *const *f;   // per block of the rank: phi_a at interior (0,0,0), current state
  int bnx, bny, bnz;        // block interior size
  int pbx, pby, pbz;        // blocks per axis in the rank's box
  int64_t pitch, plane;
  int64_t nx, ny, nzc;      // cubes per axis (x, y: the box; z: cube layers)
  int64_t X0, Y0, Z0, NX, NY, zorig;
  double iso, dx;
  int64_t cap;
};

// The four field rows (y + dy, z + dz) a cube row (y, z) reads.  One block
// per rank (the usual case): plain row pointers.  Several blocks: per corner
// the block along x is looked up (the position one past a block's last cell
// is its ghost layer).
struct CubeRow {
  const double *r[4];   // row (dy, dz) at index dy + 2 dz, element x (one block) / block-row base (several)
  int64_t off[4];       // several blocks: in-block offset of the row
  int q[4];             // several blocks: block index of x-block 0
};

__device__ __forceinline__ CubeRow cube_row(const MeshArgs &m, int64_t y, int64_t z) {
  CubeRow R;
#pragma unroll
  for (int c = 0; c < 4; ++c) {
    const int64_t yy = y + (c & 1), zz = z + (c >> 1);
    const int by = (int)min(yy / m.bny, (int64_t)m.pby - 1), bz = (int)min(zz / m.bnz, (int64_t)m.pbz - 1);
    R.q[c] = m.pbx * (by + m.pby * bz);
    R.off[c] = (zz - (int64_t)bz * m.bnz) * m.plane + (yy - (int64_t)by * m.bny) * m.pitch;
    R.r[c] = m.f[R.q[c]] + R.off[c];
  }
  return R;
}

template <bool ONE>
__device__ __forceinline__ int cube_case(const MeshArgs &m, const CubeRow &R, int x, double v[8]) {
  int cs = 0;
#pragma unroll
  for (int c = 0; c < 8; ++c) {
    const int xx = x + (c & 1), row = c >> 1;
    if (ONE) {
      v[c] = __ldg(R.r[row] + xx);
    } else {
      const int bx = min(xx / m.bnx, m.pbx - 1);
      v[c] = __ldg(m.f[R.q[row] + bx] + R.off[row] + (xx - bx * m.bnx));
    }
    cs |= (v[c] > m.iso) << c;
  }
  return cs;
}

template <bool ONE>
__global__ void mc_count_kernel(MeshArgs m, int64_t *row_cnt) {
  const int64_t row = (int64_t)blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32;
  const int lane = threadIdx.x & 31;
  if (row >= m.ny * m.nzc) return;
  const int64_t y = row % m.ny, z = row / m.ny;
  const CubeRow R = cube_row(m, y, z);
  int n = 0;
  for (int x = lane; x < m.nx; x += 32) {
    double v[8];
    n += c_mc[cube_case<ONE>(m, R, x, v)][0];
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) n += __shfl_xor_sync(0xffffffffu, n, o);
  if (lane == 0) row_cnt[row] = n;
}

template <bool ONE>
__global__ void mc_emit_kernel(MeshArgs m, const int64_t *row_off, int64_t *ids, double *pos) {
  const int64_t row = (int64_t)blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32;
  const int lane = threadIdx.x & 31;
  if (row >= m.ny * m.nzc) return;
  const int64_t y = row % m.ny, z = row / m.ny;
  const CubeRow R = cube_row(m, y, z);
  int64_t base = row_off[row];
  for (int x0 = 0; x0 < m.nx; x0 += 32) {
    const int x = x0 + lane;
    double v[8];
    const int cs = x < m.nx ? cube_case<ONE>(m, R, x, v) : 0;
    const int nt = c_mc[cs][0];
    int incl = nt;   // warp inclusive scan of the per-cube counts
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int t = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += t;
    }
    const int64_t first = base + incl - nt;
    for (int t = 0; t < nt; ++t) {
      const int64_t tri = first + t;
      if (tri >= m.cap) break;
      for (int q = 0; q < 3; ++q) {
        const int e = c_mc[cs][1 + 3 * t + q];
        const int p = e & 1, r = (e >> 1) & 1, ax = e >> 2;
        // lower corner of the edge (cube-local offsets)
        const int ox = ax == 0 ? 0 : p, oy = ax == 1 ? 0 : (ax == 0 ? p : r), oz = ax == 2 ? 0 : r;
        const int c0 = ox + 2 * oy + 4 * oz, c1 = c0 + (ax == 0 ? 1 : ax == 1 ? 2 : 4);
        const int64_t gx = (m.X0 + x + ox) % m.NX, gy = (m.Y0 + y + oy) % m.NY, gz = m.Z0 + z + oz;
        ids[3 * tri + q] = 3 * (gx + m.NX * (gy + m.NY * gz)) + ax;
        // t = (iso - f0) / (f1 - f0); position ((g + 1/2) + t) dx along the edge, (g + 1/2) dx across
        const double tt = __ddiv_rn(__dsub_rn(m.iso, v[c0]), __dsub_rn(v[c1], v[c0]));
        const double g[3] = {(double)gx, (double)gy, (double)(gz + m.zorig)};
#pragma unroll
        for (int d = 0; d < 3; ++d) {
          const double h = __dadd_rn(g[d], 0.5);
          pos[9 * tri + 3 * q + d] = __dmul_rn(d == ax ? __dadd_rn(h, tt) : h, m.dx);
        }
      }
    }
    base += __shfl_sync(0xffffffffu, incl, 31);
  }
}

}  // namespace

void mesh_case_table(int8_t *out) {
  static int8_t tab[256][1 + 3 * MC_MAXT];
  build_table(tab);
  memcpy(out, tab, sizeof(tab));
}

// Host side: table upload on first use, then count -> scan -> emit.  `f` is a
// device array of the rank's block pointers; `scratch` grows as needed.
cudaError_t launch_mesh(cudaStream_t s, const double *const *f, int bnx, int bny, int bnz, int pbx, int pby,
                        int pbz, int64_t pitch, int64_t plane, int64_t nx, int64_t ny, int64_t nzc, int64_t X0, int64_t Y0,
                        int64_t Z0, int64_t NX, int64_t NY, int64_t zorig, double iso, double dx, int64_t cap,
                        int64_t *ids, double *pos, int64_t *ntri, void **scratch, size_t *scratch_bytes) {
  static bool table_ready = false;
  if (!table_ready) {
    static int8_t tab[256][1 + 3 * MC_MAXT];
    build_table(tab);
    cudaError_t e = cudaMemcpyToSymbol(c_mc, tab, sizeof(tab));
    if (e != cudaSuccess) return e;
    table_ready = true;
  }
  *ntri = 0;
  const int64_t rows = ny * nzc;
  if (rows <= 0 || nx <= 0) return cudaSuccess;
  MeshArgs m{f, bnx, bny, bnz, pbx, pby, pbz, pitch, plane, nx, ny, nzc, X0, Y0, Z0, NX, NY, zorig, iso, dx, cap};
  // scratch: row counts (rows + 1), row offsets (rows + 1), cub temp
  size_t cub_bytes = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, cub_bytes, (int64_t *)nullptr, (int64_t *)nullptr, rows + 1, s);
  const size_t need = 2 * (size_t)(rows + 1) * sizeof(int64_t) + cub_bytes + 256;
  if (*scratch_bytes < need) {
    if (*scratch) cudaFree(*scratch);
    cudaError_t e = cudaMalloc(scratch, need);
    if (e != cudaSuccess) { *scratch = nullptr; *scratch_bytes = 0; return e; }
    *scratch_bytes = need;
  }
  int64_t *cnt = (int64_t *)*scratch, *off = cnt + rows + 1;
  void *tmp = (void *)(((uintptr_t)(off + rows + 1) + 255) & ~(uintptr_t)255);
  const int wpb = 8;   // warps (rows) per CTA
  const unsigned grid = (unsigned)((rows + wpb - 1) / wpb);
  cudaMemsetAsync(cnt + rows, 0, sizeof(int64_t), s);
  const bool one = pbx == 1 && pby == 1 && pbz == 1;
  if (one) mc_count_kernel<true><<<grid, 32 * wpb, 0, s>>>(m, cnt);
  else mc_count_kernel<false><<<grid, 32 * wpb, 0, s>>>(m, cnt);
  cub::DeviceScan::ExclusiveSum(tmp, cub_bytes, cnt, off, rows + 1, s);
  cudaError_t e = cudaMemcpyAsync(ntri, off + rows, sizeof(int64_t), cudaMemcpyDeviceToHost, s);
  if (e != cudaSuccess) return e;
  if (cap > 0 && one) mc_emit_kernel<true><<<grid, 32 * wpb, 0, s>>>(m, off, ids, pos);
  if (cap > 0 && !one) mc_emit_kernel<false><<<grid, 32 * wpb, 0, s>>>(m, off, ids, pos);
  e = cudaStreamSynchronize(s);
  if (e != cudaSuccess) return e;
  return cudaGetLastError();
}

}  // namespace pf
