// pf_runtime.cu — host runtime behind the C ABI of include/pf.h.
//
// Owns: the block decomposition ("equal-size blocks", one per
// GPU rank or several per GPU), the fields (FP64, SoA, padded rows, one full
// ghost layer: the 12 edges the D3C19 stencil needs, and the 8
// corners the marching cubes read), the
// per-plane table, the halo plans (local device copies + NCCL grouped
// send/recv), the moving window and the
// NaN watchdog ("no silent NaN propagation").
#include <cuda_runtime.h>
#include <fcntl.h>
#include <nccl.h>
#include <sys/stat.h>
#include <unistd.h>

#include <cerrno>
#include <algorithm>
#include <array>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <map>
#include <string>
#include <vector>

#include "../../include/pf.h"
#include "pf_kernels.cuh"

using namespace pf;

namespace {

thread_local std::string g_create_error;

struct Block {
  int bx, by, bz;            // block coordinates
  int nx, ny, nz;
  int64_t x0, y0, z0;        // global offset of the interior
  int64_t pitch, plane, nplanes_alloc;
  double *phi[3][NPH];       // two copies (src/dst), allocation bases; a third for the
                             // fused kernel's phi^{n+2} (pf_set_fusion), rotated with them
  double *mu[2][NMU];
  int woff;                  // window offset (planes)
  CUtensorMap tphi[3][NPH];  // TMA maps per time level: phi tile box (phi-sweep tile),
  CUtensorMap tphim[3][NPH]; //   phi tile box (mu-sweep tile),
  CUtensorMap tmu[2][NMU];   //   mu tile box (mu-sweep tile)
  CUtensorMap tphif[3][NPH]; //   phi / mu tile boxes of the fused kernel
  CUtensorMap tmuf[2][NMU];
};

struct Plan {                // halo plan of one field in one copy
  CopyOp *d_local = nullptr;   // pack into the send buffer + local copies (one launch)
  CopyOp *d_unpack = nullptr;  // unpack from the receive buffer (one launch, after the exchange)
  int nlocal = 0, nunpack = 0;
  int64_t ctas_local = 0, ctas_unpack = 0;   // CTAs of the two launches (upload_ops)
};

struct Peer {
  int rank;
  int64_t send_off, send_cnt, recv_off, recv_cnt;  // in doubles, per field
};

}  // namespace

struct pf_ctx {
  pf_grid g{};
  pf_params p{};
  KParams kp{};
  TabParams tp{};
  int nblocks_total = 0;
  std::vector<Block> blocks;       // blocks owned by this rank
  int cur = 0;                     // index of the src copy
  cudaStream_t stream = nullptr;
  bool own_stream = false;
  // mu-halo overlap: the mu^{n+1} ghost exchange runs on
  // cstream (with its own communicator) while the next phi-sweep runs on stream
  cudaStream_t cstream = nullptr;
  cudaEvent_t ev_mu_done = nullptr, ev_mu_halo = nullptr;
  cudaEvent_t ev_phi_done = nullptr, ev_phi_halo = nullptr;   // Algorithm 2's phi halo hiding
  cudaEvent_t ev_copy = nullptr, ev_stage[2] = {nullptr, nullptr};  // pf_read / pf_write staging
  bool mu_pending = false;
  ncclComm_t comm_mu = nullptr;
  double *d_tab = nullptr;
  int64_t tab_planes = 0;
  Plan plan[2][3];                 // [field 0=phi 1=mu][copy] (copy 2: phi only, with fusion)
  // fused mu(n) + phi(n+1) steps (pf_set_fusion): a third phi copy, the table
  // rows of the next step
  bool fusion = false, phi3 = false;
  double *d_tab2 = nullptr;
  std::vector<Peer> peers[2];      // per field
  double *d_send[2] = {nullptr, nullptr}, *d_recv[2] = {nullptr, nullptr};
  int64_t send_total[2] = {0, 0}, recv_total[2] = {0, 0};
  ncclComm_t comm = nullptr;
  unsigned long long *d_red = nullptr;  // reductions scratch (4 x u64)
  double *d_stage = nullptr;            // read/write staging
  int64_t stage_elems = 0;
  int64_t step = 0, zorig = 0, shifts = 0, last_front = -1, next_check = 0;
  int slack = 0;
  bool initialized = false;
  bool plans_woff0 = false;  // the halo plans are current and were built with every woff = 0
  pf_status status = PF_OK;
  std::string err;
  // timing
  bool timing = false;
  std::vector<cudaEvent_t> ev;     // pool
  size_t ev_used = 0;
  struct Span { int kind; size_t e0, e1; int nlaunch; };
  std::vector<Span> spans;
  double ms[5] = {0, 0, 0, 0, 0};  // phi, mu, halo, other, fused
  int64_t launches = 0, phi_launches = 0, mu_launches = 0, fused_launches = 0;
  // box of this rank
  int64_t box_nx = 0, box_ny = 0, box_nz = 0, box_x0 = 0, box_y0 = 0, box_z0 = 0;
  // marching cubes (pf_mesh): block pointer table, scan scratch, host-output staging
  const double **d_mesh_f = nullptr;
  void *mesh_scratch = nullptr;
  size_t mesh_scratch_bytes = 0;
  void *mesh_out = nullptr;
  size_t mesh_out_bytes = 0;
  // CUDA graphs of one step (single-rank, timing off): one per parity of the
  // src copy, invalidated whenever the halo plans, the window or the origin change
  cudaGraphExec_t gexec[2] = {nullptr, nullptr};
  int64_t graph_launches[2] = {0, 0};
  int64_t *d_step = nullptr;       // device copy of the time level for the table kernel
  // pf_step_io on a single-block context: the block cut into z-slabs, ghost
  // copy lists per slab (both fields, both copies), per-slab events, the
  // upload and download streams
  struct SlabIO {
    int H = 0, S = 0;                      // slab height, slab count
    int woff = 0;                          // window offset the copy lists were built for
    const double *phi0[2] = {nullptr, nullptr};   // and the phi copies' addresses
    std::vector<CopyOp *> ops[2][2];       // [field][copy][slab]
    std::vector<int> nops[2][2];
    std::vector<int64_t> nctas[2][2];
    std::vector<CopyOp *> ops_x[2];        // phi^{n+1} ghosts of slab s + the next slab's first plane, [copy][slab]
    std::vector<int> nops_x[2];
    std::vector<int64_t> nctas_x[2];
    std::vector<cudaEvent_t> ev_up, ev_mu;
    cudaStream_t up = nullptr, dn = nullptr;
  } sio;
};

namespace {

pf_status fail(pf_ctx *c, pf_status st, const char *fmt, ...) {
  char buf[1024];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  if (c) {
    if (c->status == PF_OK) { c->status = st; c->err = buf; }
  } else {
    g_create_error = buf;
  }
  return st;
}

#define CK(call)                                                                                       \
  do {                                                                                                 \
    cudaError_t e_ = (call);                                                                           \
    if (e_ != cudaSuccess)                                                                             \
      return fail(c, PF_ERR_CUDA, "%s failed: %s (%s:%d)", #call, cudaGetErrorString(e_), __FILE__, __LINE__); \
  } while (0)
#define CKN(call)                                                                                      \
  do {                                                                                                 \
    ncclResult_t r_ = (call);                                                                          \
    if (r_ != ncclSuccess)                                                                             \
      return fail(c, PF_ERR_COMM, "%s failed: %s (%s:%d)", #call, ncclGetErrorString(r_), __FILE__, __LINE__); \
  } while (0)
#define CKS(expr)                    \
  do {                               \
    pf_status s_ = (expr);           \
    if (s_ != PF_OK) return s_;      \
  } while (0)

inline double *field_ptr(const Block &b, int field, int copy, int comp) {
  return field == 0 ? b.phi[copy][comp] : b.mu[copy][comp];
}
// address of interior (i,j,k) of a component base
inline int64_t cell_off(const Block &b, int64_t i, int64_t j, int64_t k) {
  return (k + 1 + b.woff) * b.plane + (j + 1) * b.pitch + (i + XO);
}

int block_id(const pf_ctx *c, int bx, int by, int bz) { return bx + c->g.px * (by + c->g.py * bz); }
int owner_rank(const pf_ctx *c, int bid) { return c->g.nranks == 1 ? 0 : bid; }

// the 26 ghost directions: faces and edges (the D3C19 stencil) and corners (one
// cell each; the marching cubes at a block's far corner read them)
std::vector<std::array<int, 3>> ghost_dirs() {
  std::vector<std::array<int, 3>> v;
  for (int dz = -1; dz <= 1; ++dz)
    for (int dy = -1; dy <= 1; ++dy)
      for (int dx = -1; dx <= 1; ++dx) {
        const int m = std::abs(dx) + std::abs(dy) + std::abs(dz);
        if (m >= 1) v.push_back({dx, dy, dz});
      }
  return v;
}

struct Region {   // one ghost region of a receiving block and where it comes from
  int dst_bid, src_bid;
  int64_t ds[3], ss[3];   // start indices (dest in receiver, source in sender)
  int64_t ext[3];
};

// Ghost region of block (bx,by,bz) in direction d and its source (periodic
// x/y, zero-gradient z at the global walls; reading R13).
Region ghost_region(const pf_ctx *c, int bx, int by, int bz, const std::array<int, 3> &d, int nx, int ny, int nz) {
  const int P[3] = {c->g.px, c->g.py, c->g.pz};
  const int b[3] = {bx, by, bz};
  const int64_t n[3] = {nx, ny, nz};
  Region r;
  int s[3];
  for (int a = 0; a < 3; ++a) {
    int dp = d[a];
    if (a == 2 && (b[2] + d[2] < 0 || b[2] + d[2] >= P[2])) dp = 0;  // wall: clamp
    s[a] = ((b[a] + dp) % P[a] + P[a]) % P[a];
    r.ds[a] = d[a] == -1 ? -1 : (d[a] == 1 ? n[a] : 0);
    r.ext[a] = d[a] == 0 ? n[a] : 1;
    if (dp == -1) r.ss[a] = n[a] - 1;
    else if (dp == 1) r.ss[a] = 0;
    else r.ss[a] = d[a] == -1 ? 0 : (d[a] == 1 ? n[a] - 1 : 0);
  }
  r.dst_bid = block_id(c, bx, by, bz);
  r.src_bid = block_id(c, s[0], s[1], s[2]);
  return r;
}

int local_index(const pf_ctx *c, int bid) {
  for (size_t q = 0; q < c->blocks.size(); ++q)
    if (block_id(c, c->blocks[q].bx, c->blocks[q].by, c->blocks[q].bz) == bid) return (int)q;
  return -1;
}

// Ghost column of an x-direction region whose 32-byte sector holds no interior
// cell (the other doubles are row padding): the slot of the ghost in that
// sector, else -1.  i = -1 sits at column XO-1 = 3, the end of the row's first
// sector; i = nx at column XO+nx, the start of a sector when nx % 4 == 0.
int ghost_xpad(const Region &r, int nx) {
  static_assert(XO == 4, "row padding layout");
  if (r.ext[0] != 1) return -1;
  if (r.ds[0] == -1) return 3;
  if (r.ds[0] == nx && (XO + nx) % 4 == 0) return 0;
  return -1;
}

// Upload a copy list; each op gets CTAs in proportion to its size (first CTA
// in cta0), *nctas = the launch's CTA count: a 12-edge + 6-face halo is then a
// few thousand CTAs, not 18 x the largest face's.
pf_status upload_ops(pf_ctx *c, std::vector<CopyOp> ops, CopyOp **d, int64_t *nctas) {
  if (*d) { cudaFree(*d); *d = nullptr; }
  *nctas = 0;
  if (ops.empty()) return PF_OK;
  for (auto &op : ops) {
    op.cta0 = *nctas;
    *nctas += ((int64_t)op.ex * op.ey * op.ez + COPY_CELLS_PER_CTA - 1) / COPY_CELLS_PER_CTA;
  }
  CK(cudaMalloc(d, ops.size() * sizeof(CopyOp)));
  CK(cudaMemcpy(*d, ops.data(), ops.size() * sizeof(CopyOp), cudaMemcpyHostToDevice));
  return PF_OK;
}

// TMA descriptor over a whole padded component allocation: dims {pitch,
// ny+2, planes}, x fastest, FP64, box bx x by x 1, out-of-range boxes zero-filled.
typedef CUresult (*EncodeTiledFn)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *, const cuuint64_t *,
                                  const cuuint64_t *, const cuuint32_t *, const cuuint32_t *, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

pf_status encode_map(pf_ctx *c, CUtensorMap *m, double *base, const Block &b, int bx, int by) {
  static EncodeTiledFn fn = nullptr;
  if (!fn) {
    void *p = nullptr;
    cudaDriverEntryPointQueryResult q;
    CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q));
    if (!p || q != cudaDriverEntryPointSuccess) return fail(c, PF_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
    fn = (EncodeTiledFn)p;
  }
  const cuuint64_t dims[3] = {(cuuint64_t)b.pitch, (cuuint64_t)(b.ny + 2), (cuuint64_t)b.nplanes_alloc};
  const cuuint64_t strides[2] = {(cuuint64_t)b.pitch * 8, (cuuint64_t)b.plane * 8};
  const cuuint32_t box[3] = {(cuuint32_t)bx, (cuuint32_t)by, 1}, es[3] = {1, 1, 1};
  const CUresult r = fn(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, base, dims, strides, box, es,
                        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(c, PF_ERR_CUDA, "cuTensorMapEncodeTiled failed (%d)", (int)r);
  return PF_OK;
}

pf_status encode_maps(pf_ctx *c, Block &b) {
  for (int cp = 0; cp < 3; ++cp) {
    if (!b.phi[cp][0]) continue;
    for (int a = 0; a < NPH; ++a)
      CKS(encode_map(c, &b.tphif[cp][a], b.phi[cp][a], b, FUSED_TILE_X + 4, FUSED_TILE_Y + 2));
    if (cp < 2)
      for (int q = 0; q < NMU; ++q)
        CKS(encode_map(c, &b.tmuf[cp][q], b.mu[cp][q], b, FUSED_TILE_X + 4, FUSED_TILE_Y + 2));
  }
  for (int cp = 0; cp < 3; ++cp) {
    if (!b.phi[cp][0]) continue;
    // tile boxes start one column left of the ring (16-byte aligned x): tile width + 4;
    // phi-sweep tiles are PHI_TILE_Y high, mu-sweep tiles MU_TILE_Y
    for (int a = 0; a < NPH; ++a) {
      CKS(encode_map(c, &b.tphi[cp][a], b.phi[cp][a], b, PHI_TILE_X + 4, PHI_TILE_Y + 2));
      CKS(encode_map(c, &b.tphim[cp][a], b.phi[cp][a], b, MU_TILE_X + 4, MU_TILE_Y + 2));
    }
    for (int q = 0; q < NMU && cp < 2; ++q) {
      CKS(encode_map(c, &b.tmu[cp][q], b.mu[cp][q], b, MU_TILE_X + 4, MU_TILE_Y + 2));
    }
  }
  return PF_OK;
}

// descriptors of the current time levels for the phi-sweep (field 0) or the
// mu-sweep (field 1)
TmaMaps maps_of(const pf_ctx *c, const Block &b, int field) {
  TmaMaps t;
  const int s = c->cur, d = c->cur ^ 1;
  for (int a = 0; a < NPH; ++a) {
    t.phi[a] = field == 0 ? b.tphi[s][a] : b.tphim[s][a];
    t.phin[a] = b.tphim[d][a];
  }
  for (int q = 0; q < NMU; ++q) t.mu[q] = b.tmu[s][q];
  return t;
}

// maps of the fused kernel at the current state: phi^n, phi^{n+1}, mu^n
TmaMaps maps_fused(const pf_ctx *c, const Block &b) {
  TmaMaps t;
  const int s = c->cur, d = c->cur ^ 1;
  for (int a = 0; a < NPH; ++a) { t.phi[a] = b.tphif[s][a]; t.phin[a] = b.tphif[d][a]; }
  for (int q = 0; q < NMU; ++q) t.mu[q] = b.tmuf[s][q];
  return t;
}

// Build the halo plans of both fields and both copies.
void invalidate_graphs(pf_ctx *c) {
  for (int q = 0; q < 2; ++q)
    if (c->gexec[q]) { cudaGraphExecDestroy(c->gexec[q]); c->gexec[q] = nullptr; }
}

pf_status build_plans(pf_ctx *c) {
  invalidate_graphs(c);   // captured launches hold the plans' device pointers
  const auto dirs = ghost_dirs();
  const int nb = c->nblocks_total;
  const Block &b0 = c->blocks[0];
  const int nx = b0.nx, ny = b0.ny, nz = b0.nz;
  const int me = c->g.rank;
  for (int field = 0; field < 2; ++field) {
    const int ncomp = field == 0 ? NPH : NMU;
    // peers: message layout per (peer) = receiver's regions in dir order
    std::map<int, Peer> peers;
    std::vector<Region> recv_regions, send_regions;  // with peer ordering
    for (int bid = 0; bid < nb; ++bid) {
      const int bx = bid % c->g.px, by = (bid / c->g.px) % c->g.py, bz = bid / (c->g.px * c->g.py);
      for (const auto &d : dirs) {
        const Region r = ghost_region(c, bx, by, bz, d, nx, ny, nz);
        const int rdst = owner_rank(c, r.dst_bid), rsrc = owner_rank(c, r.src_bid);
        if (rdst == me && rsrc != me) recv_regions.push_back(r);
        if (rsrc == me && rdst != me) send_regions.push_back(r);
      }
    }
    // order messages by peer rank, regions within a peer in enumeration order
    int64_t off = 0;
    for (int pr = 0; pr < c->g.nranks; ++pr) {
      int64_t cnt = 0;
      for (const auto &r : recv_regions)
        if (owner_rank(c, r.src_bid) == pr) cnt += r.ext[0] * r.ext[1] * r.ext[2] * ncomp;
      if (cnt) { Peer &p = peers[pr]; p.rank = pr; p.recv_off = off; p.recv_cnt = cnt; off += cnt; }
    }
    c->recv_total[field] = off;
    off = 0;
    for (int pr = 0; pr < c->g.nranks; ++pr) {
      int64_t cnt = 0;
      for (const auto &r : send_regions)
        if (owner_rank(c, r.dst_bid) == pr) cnt += r.ext[0] * r.ext[1] * r.ext[2] * ncomp;
      if (cnt) {
        Peer &p = peers[pr];
        p.rank = pr; p.send_off = off; p.send_cnt = cnt; off += cnt;
      }
    }
    c->send_total[field] = off;
    c->peers[field].clear();
    for (auto &kv : peers) c->peers[field].push_back(kv.second);
    if (c->d_send[field]) { cudaFree(c->d_send[field]); c->d_send[field] = nullptr; }
    if (c->d_recv[field]) { cudaFree(c->d_recv[field]); c->d_recv[field] = nullptr; }
    if (c->send_total[field]) CK(cudaMalloc(&c->d_send[field], c->send_total[field] * sizeof(double)));
    if (c->recv_total[field]) CK(cudaMalloc(&c->d_recv[field], c->recv_total[field] * sizeof(double)));

    for (int copy = 0; copy < (field == 0 && c->phi3 ? 3 : 2); ++copy) {
      std::vector<CopyOp> local, pack, unpack;
      Plan &pl = c->plan[field][copy];
      // local copies: both ends on this rank
      for (size_t q = 0; q < c->blocks.size(); ++q) {
        const Block &B = c->blocks[q];
        for (const auto &d : dirs) {
          const Region r = ghost_region(c, B.bx, B.by, B.bz, d, nx, ny, nz);
          if (owner_rank(c, r.src_bid) != me) continue;
          const Block &S = c->blocks[local_index(c, r.src_bid)];
          CopyOp op{};
          for (int cc = 0; cc < ncomp; ++cc) {
            op.src[cc] = field_ptr(S, field, copy, cc) + cell_off(S, r.ss[0], r.ss[1], r.ss[2]);
            op.dst[cc] = field_ptr(B, field, copy, cc) + cell_off(B, r.ds[0], r.ds[1], r.ds[2]);
          }
          op.ssx = op.dsx = 1; op.ssy = op.dsy = B.pitch; op.ssz = op.dsz = B.plane;
          op.ex = (int)r.ext[0]; op.ey = (int)r.ext[1]; op.ez = (int)r.ext[2]; op.ncomp = ncomp;
          op.xpad = ghost_xpad(r, nx);
          local.push_back(op);
        }
      }
      // pack: regions this rank sends, per peer in the receiver's order
      for (const Peer &p : c->peers[field]) {
        int64_t o = p.send_off;
        for (const auto &r : send_regions) {
          if (owner_rank(c, r.dst_bid) != p.rank) continue;
          const Block &S = c->blocks[local_index(c, r.src_bid)];
          const int64_t n = r.ext[0] * r.ext[1] * r.ext[2];
          CopyOp op{};
          for (int cc = 0; cc < ncomp; ++cc) {
            op.src[cc] = field_ptr(S, field, copy, cc) + cell_off(S, r.ss[0], r.ss[1], r.ss[2]);
            op.dst[cc] = c->d_send[field] + o + cc * n;
          }
          op.ssx = 1; op.ssy = S.pitch; op.ssz = S.plane;
          op.dsx = 1; op.dsy = r.ext[0]; op.dsz = r.ext[0] * r.ext[1];
          op.ex = (int)r.ext[0]; op.ey = (int)r.ext[1]; op.ez = (int)r.ext[2]; op.ncomp = ncomp;
          op.xpad = -1;
          pack.push_back(op);
          o += n * ncomp;
        }
        int64_t o2 = p.recv_off;
        for (const auto &r : recv_regions) {
          if (owner_rank(c, r.src_bid) != p.rank) continue;
          const Block &B = c->blocks[local_index(c, r.dst_bid)];
          const int64_t n = r.ext[0] * r.ext[1] * r.ext[2];
          CopyOp op{};
          for (int cc = 0; cc < ncomp; ++cc) {
            op.src[cc] = c->d_recv[field] + o2 + cc * n;
            op.dst[cc] = field_ptr(B, field, copy, cc) + cell_off(B, r.ds[0], r.ds[1], r.ds[2]);
          }
          op.ssx = 1; op.ssy = r.ext[0]; op.ssz = r.ext[0] * r.ext[1];
          op.dsx = 1; op.dsy = B.pitch; op.dsz = B.plane;
          op.ex = (int)r.ext[0]; op.ey = (int)r.ext[1]; op.ez = (int)r.ext[2]; op.ncomp = ncomp;
          op.xpad = ghost_xpad(r, nx);
          unpack.push_back(op);
          o2 += n * ncomp;
        }
      }
      // local copies go with the pack launch (no dependency on communication)
      std::vector<CopyOp> first = pack;
      first.insert(first.end(), local.begin(), local.end());
      pl.nlocal = (int)first.size();
      CKS(upload_ops(c, first, &pl.d_local, &pl.ctas_local));
      pl.nunpack = (int)unpack.size();
      CKS(upload_ops(c, unpack, &pl.d_unpack, &pl.ctas_unpack));
    }
  }
  c->plans_woff0 = true;
  for (const auto &b : c->blocks) if (b.woff != 0) c->plans_woff0 = false;
  return PF_OK;
}

size_t ev_next(pf_ctx *c) {
  if (c->ev_used == c->ev.size()) {
    cudaEvent_t e;
    cudaEventCreate(&e);
    c->ev.push_back(e);
  }
  return c->ev_used++;
}

struct TimedSpan {  // records an event pair around a group of launches (kind < 0: untimed)
  pf_ctx *c; int kind; size_t e0; int n;
  TimedSpan(pf_ctx *c_, int kind_, int n_) : c(c_), kind(kind_), e0(0), n(n_) {
    if (c->timing && kind >= 0) { e0 = ev_next(c); cudaEventRecord(c->ev[e0], c->stream); }
  }
  ~TimedSpan() {
    if (c->timing && kind >= 0) {
      const size_t e1 = ev_next(c);
      cudaEventRecord(c->ev[e1], c->stream);
      c->spans.push_back({kind, e0, e1, n});
    }
  }
};

// Exchange the ghosts of one field in one copy, on the
// main stream, or — `overlap` — on the comm stream with its own communicator
// (the mu^{n+1} exchange overlapping the next phi-sweep).
pf_status exchange(pf_ctx *c, int field, int copy, bool overlap = false) {
  const Plan &pl = c->plan[field][copy];
  cudaStream_t st = overlap ? c->cstream : c->stream;
  ncclComm_t comm = overlap ? c->comm_mu : c->comm;
  TimedSpan ts(c, overlap ? -1 : 2, 0);
  if (pl.nlocal) { launch_copy(st, pl.d_local, pl.nlocal, pl.ctas_local); c->launches++; }
  if (c->g.nranks > 1 && !c->peers[field].empty()) {
    CKN(ncclGroupStart());
    for (const Peer &p : c->peers[field]) {
      if (p.send_cnt) CKN(ncclSend(c->d_send[field] + p.send_off, (size_t)p.send_cnt, ncclDouble, p.rank, comm, st));
      if (p.recv_cnt) CKN(ncclRecv(c->d_recv[field] + p.recv_off, (size_t)p.recv_cnt, ncclDouble, p.rank, comm, st));
    }
    CKN(ncclGroupEnd());
  }
  if (pl.nunpack) { launch_copy(st, pl.d_unpack, pl.nunpack, pl.ctas_unpack); c->launches++; }
  CK(cudaGetLastError());
  return PF_OK;
}

// Make the main stream wait for a pending overlapped mu exchange.
pf_status join_mu(pf_ctx *c) {
  if (!c->mu_pending) return PF_OK;
  CK(cudaStreamWaitEvent(c->stream, c->ev_mu_halo, 0));
  c->mu_pending = false;
  return PF_OK;
}

BlockView view(const pf_ctx *c, const Block &b, int field_out) {
  BlockView v{};
  const int s = c->cur, d = c->cur ^ 1;
  const int64_t o = cell_off(b, 0, 0, 0);
  for (int a = 0; a < NPH; ++a) { v.phi[a] = b.phi[s][a] + o; v.phin[a] = b.phi[d][a] + o; }
  for (int q = 0; q < NMU; ++q) v.mu[q] = b.mu[s][q] + o;
  if (field_out == 0) for (int a = 0; a < NPH; ++a) v.out[a] = b.phi[d][a] + o;
  else for (int q = 0; q < NMU; ++q) v.out[q] = b.mu[d][q] + o;
  v.nx = b.nx; v.ny = b.ny; v.nz = b.nz; v.pitch = b.pitch; v.plane = b.plane;
  v.tab = c->d_tab + (b.z0 + 1) * TAB;
  v.zoff = 1 + b.woff;
  return v;
}

pf_status collect_timing(pf_ctx *c) {
  if (!c->timing) return PF_OK;
  CK(cudaStreamSynchronize(c->stream));
  for (const auto &s : c->spans) {
    float ms = 0;
    CK(cudaEventElapsedTime(&ms, c->ev[s.e0], c->ev[s.e1]));
    c->ms[s.kind] += ms;
    if (s.kind == 0) c->phi_launches += s.nlaunch;
    if (s.kind == 1) c->mu_launches += s.nlaunch;
    if (s.kind == 4) c->fused_launches += s.nlaunch;
  }
  c->spans.clear();
  c->ev_used = 0;
  return PF_OK;
}

pf_status window_compact(pf_ctx *c) {
  // copy planes [woff, woff + nz + 2) of the src copy into [0, nz + 2) of the
  // dst copy (scratch between steps), then swap
  for (auto &b : c->blocks) {
    const size_t bytes = (size_t)(b.nz + 2) * b.plane * sizeof(double);
    for (int a = 0; a < NPH; ++a)
      CK(cudaMemcpyAsync(b.phi[c->cur ^ 1][a], b.phi[c->cur][a] + (int64_t)b.woff * b.plane, bytes,
                         cudaMemcpyDeviceToDevice, c->stream));
    for (int q = 0; q < NMU; ++q)
      CK(cudaMemcpyAsync(b.mu[c->cur ^ 1][q], b.mu[c->cur][q] + (int64_t)b.woff * b.plane, bytes,
                         cudaMemcpyDeviceToDevice, c->stream));
    b.woff = 0;
  }
  c->cur ^= 1;
  return PF_OK;
}

// Moving window (reading R16): decide after the step whether the
// front reached ceil(frac * NZ); shift one plane (ring offset) if so.
pf_status window_check(pf_ctx *c) {
  if (!c->p.window) return PF_OK;
  if (c->step < c->next_check) return PF_OK;
  CK(cudaMemsetAsync(c->d_red, 0, 2 * sizeof(unsigned long long), c->stream));
  for (const auto &b : c->blocks) {
    const double *phil = b.phi[c->cur][LIQ] + cell_off(b, 0, 0, 0);
    launch_front(c->stream, phil, b.nx, b.ny, b.nz, b.pitch, b.plane, c->p.window_phi_l, b.z0, c->d_red);
    c->launches++;
  }
  if (c->g.nranks > 1) CKN(ncclAllReduce(c->d_red, c->d_red, 2, ncclUint64, ncclMax, c->comm, c->stream));
  unsigned long long h[2];
  CK(cudaMemcpyAsync(h, c->d_red, sizeof(h), cudaMemcpyDeviceToHost, c->stream));
  CK(cudaStreamSynchronize(c->stream));
  const int64_t front = (int64_t)h[0] - 1, k1 = (int64_t)h[1] - 1;
  c->last_front = front;
  const int64_t trig = (int64_t)std::ceil(c->p.window_frac * (double)c->g.nz);
  if (front >= trig) {
    bool need_compact = false;
    for (auto &b : c->blocks) if (b.woff >= c->slack) need_compact = true;
    if (need_compact) CKS(window_compact(c));
    for (auto &b : c->blocks) b.woff += 1;
    // top blocks: new top interior plane = liquid (phi = e_l, mu = 0)
    for (auto &b : c->blocks) {
      if (b.bz != c->g.pz - 1) continue;
      double *fp[NPH], *fm[NPH] = {nullptr, nullptr, nullptr, nullptr};
      for (int a = 0; a < NPH; ++a) fp[a] = b.phi[c->cur][a] + cell_off(b, 0, 0, b.nz - 1);
      for (int q = 0; q < NMU; ++q) fm[q] = b.mu[c->cur][q] + cell_off(b, 0, 0, b.nz - 1);
      const double liq[4] = {0.0, 0.0, 0.0, 1.0}, zero[4] = {0, 0, 0, 0};
      launch_fill_plane(c->stream, fp, NPH, liq, b.nx, b.ny, b.pitch);
      launch_fill_plane(c->stream, fm, NMU, zero, b.nx, b.ny, b.pitch);
      c->launches += 2;
    }
    c->zorig += 1;
    c->shifts += 1;
    CKS(build_plans(c));
    CKS(exchange(c, 0, c->cur));
    CKS(exchange(c, 1, c->cur));
    c->next_check = c->step + 1;
  } else {
    // phi_l < 1 reaches at most one plane further per step (D3C7/D3C19 reach
    // 1): no shift is possible before k1 can reach the trigger
    c->next_check = c->step + std::max<int64_t>(1, trig - k1 - 1);
  }
  return PF_OK;
}

pf_status nan_check(pf_ctx *c) {
  CK(cudaMemsetAsync(c->d_red + 2, 0xff, 2 * sizeof(unsigned long long), c->stream));
  for (size_t q = 0; q < c->blocks.size(); ++q) {
    const Block &b = c->blocks[q];
    const double *fp[NPH], *fm[NPH] = {nullptr, nullptr, nullptr, nullptr};
    for (int a = 0; a < NPH; ++a) fp[a] = b.phi[c->cur][a] + cell_off(b, 0, 0, 0);
    for (int m = 0; m < NMU; ++m) fm[m] = b.mu[c->cur][m] + cell_off(b, 0, 0, 0);
    launch_nancheck(c->stream, fp, NPH, b.nx, b.ny, b.nz, b.pitch, b.plane, c->d_red + 2);
    launch_nancheck(c->stream, fm, NMU, b.nx, b.ny, b.nz, b.pitch, b.plane, c->d_red + 3);
    unsigned long long h[2];
    CK(cudaMemcpyAsync(h, c->d_red + 2, sizeof(h), cudaMemcpyDeviceToHost, c->stream));
    CK(cudaStreamSynchronize(c->stream));
    for (int f = 0; f < 2; ++f) {
      if (h[f] == ~0ULL) continue;
      const int64_t n = (int64_t)b.nx * b.ny * b.nz;
      const int64_t comp = (int64_t)(h[f] / n), t = (int64_t)(h[f] % n);
      const int64_t i = t % b.nx, j = (t / b.nx) % b.ny, k = t / ((int64_t)b.nx * b.ny);
      return fail(c, PF_ERR_NUMERICAL, "non-finite %s[%lld] at step %lld, global cell (%lld, %lld, %lld)",
                  f == 0 ? "phi" : "mu", (long long)comp, (long long)c->step, (long long)(b.x0 + i),
                  (long long)(b.y0 + j), (long long)(b.z0 + k));
    }
  }
  return PF_OK;
}

// ---------------------------------------------------------------------------
// pf_step_io: one step from a host state to a host state on a single-block
// context, cut into z-slabs so that the upload of slab s+1, the sweeps of the
// slabs before it and the download of finished slabs overlap (PCIe is full
// duplex; the step's compute is a few percent of its transfer time).  Every
// kernel is the one pf_step launches, on a view shifted to the slab's planes;
// chunk edges do not change a face's bits (pinned rounding), so the result is
// pf_write + pf_step(1) + pf_read bit for bit.
// ---------------------------------------------------------------------------
BlockView slab_view(BlockView v, int field_out, int z0, int z1) {
  const int64_t o = (int64_t)z0 * v.plane;
  for (int a = 0; a < NPH; ++a) { v.phi[a] += o; v.phin[a] += o; }
  for (int q = 0; q < NMU; ++q) v.mu[q] += o;
  for (int a = 0; a < (field_out == 0 ? NPH : NMU); ++a) v.out[a] += o;
  v.nz = z1 - z0;
  v.zoff += z0;
  v.tab += (int64_t)z0 * TAB;
  return v;
}

// ghost copies of one field / copy restricted to planes [z0, z1) of the single
// block: the 26 directions, the wall planes only with the first / last slab
pf_status slab_ops(pf_ctx *c, int field, int copy, int z0, int z1, CopyOp **d, int *nops, int64_t *nctas) {
  const Block &B = c->blocks[0];
  const int ncomp = field == 0 ? NPH : NMU;
  std::vector<CopyOp> ops;
  for (const auto &dir : ghost_dirs()) {
    Region r = ghost_region(c, B.bx, B.by, B.bz, dir, B.nx, B.ny, B.nz);
    if (dir[2] == 0) { r.ds[2] = r.ss[2] = z0; r.ext[2] = z1 - z0; }
    else if ((dir[2] < 0 && z0 != 0) || (dir[2] > 0 && z1 != B.nz)) continue;
    CopyOp op{};
    for (int cc = 0; cc < ncomp; ++cc) {
      op.src[cc] = field_ptr(B, field, copy, cc) + cell_off(B, r.ss[0], r.ss[1], r.ss[2]);
      op.dst[cc] = field_ptr(B, field, copy, cc) + cell_off(B, r.ds[0], r.ds[1], r.ds[2]);
    }
    op.ssx = op.dsx = 1; op.ssy = op.dsy = B.pitch; op.ssz = op.dsz = B.plane;
    op.ex = (int)r.ext[0]; op.ey = (int)r.ext[1]; op.ez = (int)r.ext[2]; op.ncomp = ncomp;
    op.xpad = ghost_xpad(r, B.nx);
    ops.push_back(op);
  }
  *nops = (int)ops.size();
  *d = nullptr;
  return upload_ops(c, ops, d, nctas);
}

void slab_free(pf_ctx *c);

pf_status slab_setup(pf_ctx *c) {
  auto &io = c->sio;
  const Block &b0 = c->blocks[0];
  if (io.S && io.woff == b0.woff && io.phi0[0] == b0.phi[0][0] && io.phi0[1] == b0.phi[1][0]) return PF_OK;
  if (io.S) slab_free(c);   // the window moved since: the copy lists hold plane addresses
  io.woff = b0.woff;
  io.phi0[0] = b0.phi[0][0];   // the copy lists hold field addresses: fusion rotates the phi copies
  io.phi0[1] = b0.phi[1][0];
  const int nz = c->blocks[0].nz;
#ifndef PF_SLABS
#define PF_SLABS 32   // measured at 512^3: 16 -> 146.1, 32 -> 144.4, 64 -> 146.1 ms per step
#endif
  // ~PF_SLABS slabs: the download of slab s waits for the upload of slab s+1,
  // so the pipeline's fill + drain cost ~2 slabs of one-way transfer time
  io.H = std::max(4, (nz + PF_SLABS - 1) / PF_SLABS);
  io.S = (nz + io.H - 1) / io.H;
  CK(cudaStreamCreateWithFlags(&io.up, cudaStreamNonBlocking));
  CK(cudaStreamCreateWithFlags(&io.dn, cudaStreamNonBlocking));
  io.ev_up.assign(io.S, nullptr);
  io.ev_mu.assign(io.S, nullptr);
  for (int s = 0; s < io.S; ++s) {
    CK(cudaEventCreateWithFlags(&io.ev_up[s], cudaEventDisableTiming));
    CK(cudaEventCreateWithFlags(&io.ev_mu[s], cudaEventDisableTiming));
  }
  for (int f = 0; f < 2; ++f)
    for (int cp = 0; cp < 2; ++cp) {
      io.ops[f][cp].assign(io.S, nullptr);
      io.nops[f][cp].assign(io.S, 0);
      io.nctas[f][cp].assign(io.S, 0);
      for (int s = 0; s < io.S; ++s)
        CKS(slab_ops(c, f, cp, s * io.H, std::min(nz, (s + 1) * io.H), &io.ops[f][cp][s], &io.nops[f][cp][s],
                     &io.nctas[f][cp][s]));
    }
  for (int cp = 0; cp < 2; ++cp) {
    io.ops_x[cp].assign(io.S, nullptr);
    io.nops_x[cp].assign(io.S, 0);
    io.nctas_x[cp].assign(io.S, 0);
    for (int s = 0; s < io.S; ++s)
      CKS(slab_ops(c, 0, cp, s * io.H, std::min(nz, (s + 1) * io.H + 1), &io.ops_x[cp][s], &io.nops_x[cp][s],
                   &io.nctas_x[cp][s]));
  }
  return PF_OK;
}

void slab_free(pf_ctx *c) {
  auto &io = c->sio;
  for (int f = 0; f < 2; ++f)
    for (int cp = 0; cp < 2; ++cp)
      for (auto *p : io.ops[f][cp]) if (p) cudaFree(p);
  for (int cp = 0; cp < 2; ++cp)
    for (auto *p : io.ops_x[cp]) if (p) cudaFree(p);
  for (auto e : io.ev_up) if (e) cudaEventDestroy(e);
  for (auto e : io.ev_mu) if (e) cudaEventDestroy(e);
  if (io.up) { cudaStreamSynchronize(io.up); cudaStreamDestroy(io.up); }
  if (io.dn) { cudaStreamSynchronize(io.dn); cudaStreamDestroy(io.dn); }
  io = pf_ctx::SlabIO{};
}

// interior planes [z0, z1) of copy `copy` <-> the compact host state (DMA
// straight into / out of the padded layout: one 3D copy per component)
pf_status slab_copy(pf_ctx *c, int copy, const double *phi, const double *mu, int z0, int z1, bool up,
                    cudaStream_t st) {
  const Block &b = c->blocks[0];
  const int64_t n = (int64_t)b.nx * b.ny * b.nz;
  for (int field = 0; field < 2; ++field)
    for (int q = 0; q < (field == 0 ? NPH : NMU); ++q) {
      double *h = const_cast<double *>(field == 0 ? phi : mu) + q * n;
      double *dv = field_ptr(b, field, copy, q);
      cudaPitchedPtr hp = make_cudaPitchedPtr(h, (size_t)b.nx * 8, (size_t)b.nx * 8, (size_t)b.ny);
      cudaPitchedPtr dp = make_cudaPitchedPtr(dv, (size_t)b.pitch * 8, (size_t)b.pitch * 8, (size_t)b.ny + 2);
      const cudaPos hpos = make_cudaPos(0, 0, (size_t)z0), dpos = make_cudaPos(XO * 8, 1, (size_t)(z0 + 1 + b.woff));
      cudaMemcpy3DParms m = {};
      if (up) { m.srcPtr = hp; m.srcPos = hpos; m.dstPtr = dp; m.dstPos = dpos; m.kind = cudaMemcpyHostToDevice; }
      else { m.srcPtr = dp; m.srcPos = dpos; m.dstPtr = hp; m.dstPos = hpos; m.kind = cudaMemcpyDeviceToHost; }
      m.extent = make_cudaExtent((size_t)b.nx * 8, (size_t)b.ny, (size_t)(z1 - z0));
      CK(cudaMemcpy3DAsync(&m, st));
    }
  return PF_OK;
}

pf_status fill_all_ghosts(pf_ctx *c) {
  CKS(exchange(c, 0, c->cur));
  CKS(exchange(c, 1, c->cur));
  return PF_OK;
}

pf_status check_state(pf_ctx *c, bool need_init) {
  if (!c) return PF_ERR_ARG;
  if (c->status != PF_OK) return PF_ERR_STATE;
  if (need_init && !c->initialized) return fail(c, PF_ERR_STATE, "pf_step/pf_read before pf_init/pf_write");
  CK(cudaSetDevice(c->g.device));
  return PF_OK;
}

bool is_device_ptr(const void *p) {
  cudaPointerAttributes a;
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) { cudaGetLastError(); return false; }
  return a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged;
}

// copy the rank box between the public compact layout (user, host/device) and the fields
pf_status move_state(pf_ctx *c, double *phi, double *mu, bool to_fields) {
  const int64_t n = c->box_nx * c->box_ny * c->box_nz;
  // host buffers: component by component through two device staging buffers,
  // the PCIe copy of one component (comm stream) overlapping the layout kernel
  // of the other (main stream)
  int q_all = 0;
  for (int field = 0; field < 2; ++field) {
    double *user = field == 0 ? phi : mu;
    const int ncomp = field == 0 ? NPH : NMU;
    const bool dev = is_device_ptr(user);
    if (!dev && !c->d_stage) {  // two components of staging, allocated on first host transfer
      c->stage_elems = n;
      CK(cudaMalloc(&c->d_stage, 2 * (size_t)n * sizeof(double)));
    }
    for (int q = 0; q < ncomp; ++q, ++q_all) {
      const int sb = q_all & 1;
      double *buf = dev ? user + (int64_t)q * n : c->d_stage + sb * n;
      double *hbuf = user + (int64_t)q * n;
      if (!dev) {   // staging buffer sb free: its previous user (component q_all - 2) is done
        CK(cudaStreamWaitEvent(to_fields ? c->cstream : c->stream, c->ev_stage[sb], 0));
      }
      if (to_fields && !dev) {
        CK(cudaMemcpyAsync(buf, hbuf, (size_t)n * sizeof(double), cudaMemcpyHostToDevice, c->cstream));
        CK(cudaEventRecord(c->ev_copy, c->cstream));
        CK(cudaStreamWaitEvent(c->stream, c->ev_copy, 0));
      }
      for (const auto &b : c->blocks) {
        double *base = field_ptr(b, field, c->cur, q) + cell_off(b, 0, 0, 0);
        const double *f[NPH] = {base, nullptr, nullptr, nullptr};
        double *w[NPH] = {base, nullptr, nullptr, nullptr};
        launch_gather(c->stream, f, 1, b.nx, b.ny, b.nz, b.pitch, b.plane, buf, c->box_nx, c->box_ny, n,
                      b.x0 - c->box_x0, b.y0 - c->box_y0, b.z0 - c->box_z0, to_fields, w);
      }
      CK(cudaGetLastError());
      if (dev) continue;
      if (to_fields) {
        CK(cudaEventRecord(c->ev_stage[sb], c->stream));                 // scatter done: buffer free
      } else {
        CK(cudaEventRecord(c->ev_copy, c->stream));                      // gather done
        CK(cudaStreamWaitEvent(c->cstream, c->ev_copy, 0));
        CK(cudaMemcpyAsync(hbuf, buf, (size_t)n * sizeof(double), cudaMemcpyDeviceToHost, c->cstream));
        CK(cudaEventRecord(c->ev_stage[sb], c->cstream));                // copy-out done: buffer free
      }
    }
  }
  CK(cudaStreamSynchronize(c->cstream));
  CK(cudaStreamSynchronize(c->stream));
  return PF_OK;
}

// ---------------------------------------------------------------------------
// FP32 checkpoints: "four phi values and two mu values per
// cell ... checkpoints use only single precision".  File = 72-byte header
// (magic "PFCP0001", u64 NX NY NZ, u32 N, u32 K-1, f64 dx, f64 t, u64 step,
// u64 window origin; little endian) + component-major binary32 body (all
// phi_0, ..., phi_3, mu_0, mu_1; each x fastest over the global grid;
// SPEC.md:462-466).  Every rank converts its blocks on the device in z-chunks
// and writes / reads its own rows with pwrite / pread, the host I/O of chunk
// i overlapping the conversion + PCIe copy of chunk i+1.
// ---------------------------------------------------------------------------
static_assert(__BYTE_ORDER__ == __ORDER_LITTLE_ENDIAN__, "checkpoint format is little endian");
constexpr int64_t CKPT_HDR = 72;
constexpr int64_t CKPT_CHUNK = 8 << 20;  // floats per conversion chunk (32 MB)

// I/O and format errors do not poison the context (message in pf_last_error)
pf_status io_fail(pf_ctx *c, const char *fmt, ...) {
  char buf[1024];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  if (c->status == PF_OK) c->err = buf;
  return PF_ERR_IO;
}

// collective "did any rank fail?" (an allreduce(max) of the local error flag);
// also orders the ranks' file accesses
pf_status io_agree(pf_ctx *c, pf_status local) {
  if (c->g.nranks == 1) return local;
  const unsigned long long flag = local != PF_OK;
  CK(cudaMemcpyAsync(c->d_red + 3, &flag, sizeof(flag), cudaMemcpyHostToDevice, c->stream));
  CKN(ncclAllReduce(c->d_red + 3, c->d_red + 3, 1, ncclUint64, ncclMax, c->comm, c->stream));
  unsigned long long any = 0;
  CK(cudaMemcpyAsync(&any, c->d_red + 3, sizeof(any), cudaMemcpyDeviceToHost, c->stream));
  CK(cudaStreamSynchronize(c->stream));
  if (local != PF_OK) return local;
  return any ? io_fail(c, "checkpoint I/O failed on another rank") : PF_OK;
}

struct CkptChunk { int blk, q; int kz0, nzc; };

std::vector<CkptChunk> ckpt_chunks(const pf_ctx *c) {
  std::vector<CkptChunk> v;
  for (int q = 0; q < NPH + NMU; ++q)
    for (int bi = 0; bi < (int)c->blocks.size(); ++bi) {
      const Block &b = c->blocks[bi];
      const int nzc = (int)std::max<int64_t>(1, CKPT_CHUNK / ((int64_t)b.nx * b.ny));
      for (int k = 0; k < b.nz; k += nzc) v.push_back({bi, q, k, std::min(nzc, b.nz - k)});
    }
  return v;
}

// pwrite / pread the rows of one chunk (host buffer compact, x fastest),
// merging rows that are contiguous in the file
bool ckpt_rows(const pf_ctx *c, int fd, const CkptChunk &ch, float *h, bool write) {
  const Block &b = c->blocks[ch.blk];
  const int64_t NX = c->g.nx, NY = c->g.ny, NXYZ = NX * NY * c->g.nz;
  const int64_t rows = (int64_t)ch.nzc * b.ny, rowb = (int64_t)b.nx * 4;
  int64_t r = 0;
  while (r < rows) {
    auto off = [&](int64_t row) {
      const int64_t k = row / b.ny, j = row % b.ny;
      return CKPT_HDR + 4 * ((int64_t)ch.q * NXYZ + ((b.z0 + ch.kz0 + k) * NY + (b.y0 + j)) * NX + b.x0);
    };
    int64_t r1 = r + 1;
    while (r1 < rows && off(r1) == off(r) + (r1 - r) * rowb) ++r1;
    char *p = reinterpret_cast<char *>(h + r * b.nx);
    int64_t len = (r1 - r) * rowb, o = off(r);
    while (len > 0) {
      const ssize_t d = write ? pwrite(fd, p, (size_t)len, o) : pread(fd, p, (size_t)len, o);
      if (d <= 0) return false;
      p += d; o += d; len -= d;
    }
    r = r1;
  }
  return true;
}

struct CkptBuffers {  // two pinned host chunk buffers + one device chunk buffer
  float *h[2] = {nullptr, nullptr}, *d = nullptr;
  cudaEvent_t ev[2] = {nullptr, nullptr};
  ~CkptBuffers() {
    for (int s = 0; s < 2; ++s) { if (h[s]) cudaFreeHost(h[s]); if (ev[s]) cudaEventDestroy(ev[s]); }
    if (d) cudaFree(d);
  }
};

pf_status ckpt_alloc(pf_ctx *c, CkptBuffers &cb) {
  int64_t m = 1;
  for (const auto &b : c->blocks)
    m = std::max(m, std::min<int64_t>((int64_t)b.nx * b.ny * b.nz,
                                      std::max<int64_t>(CKPT_CHUNK / ((int64_t)b.nx * b.ny), 1) * b.nx * b.ny));
  for (int s = 0; s < 2; ++s) {
    CK(cudaMallocHost(&cb.h[s], (size_t)m * 4));
    CK(cudaEventCreateWithFlags(&cb.ev[s], cudaEventDisableTiming));
  }
  CK(cudaMalloc(&cb.d, (size_t)m * 4));
  return PF_OK;
}

void ckpt_convert(pf_ctx *c, const CkptChunk &ch, float *d, bool to_fields) {
  const Block &b = c->blocks[ch.blk];
  double *f = field_ptr(b, ch.q < NPH ? 0 : 1, c->cur, ch.q < NPH ? ch.q : ch.q - NPH) + cell_off(b, 0, 0, ch.kz0);
  launch_cvt32(c->stream, f, b.nx, b.ny, ch.nzc, b.pitch, b.plane, d, b.nx, b.ny, 0, 0, 0, to_fields);
}

// Explicit Euler is stable only for
// dt <= min(dx^2 / (6 D_mu), dx^2 / (6 D_phi)) (reading R29):
//   D_mu  = max_{a,c} D_c^a * max A / min A  (M/chi = sum phi D/(2A) /
//           sum h/(2A) <= D_max A_max/A_min on the simplex, 7-point Laplacian);
//   D_phi = 2 gamma_max T_max / tau_min  (the face flux of phase a carries
//           2 sum_b gamma_ab phibar_b^2 grad phi_a, and Eq. (1) divides eps T
//           by tau eps).
// Checked with A(T) > 0 (the parabolas' curvature, reading R7) over the
// temperatures T0 + G (z dx - v t) at the corners of z in [zlo, zhi] (plane
// indices incl. window origin), t in [tlo, thi].
bool t_range_ok(const pf_params &p, double zlo, double zhi, double tlo, double thi, char *why, size_t nwhy) {
  double Tmin = 1e300, Tmax = -1e300;
  for (double z : {zlo, zhi})
    for (double t : {tlo, thi}) {
      const double T = p.T0 + p.G * ((z + 0.5) * p.dx - p.v * t);
      Tmin = std::min(Tmin, T);
      Tmax = std::max(Tmax, T);
    }
  double Amin = 1e300, Amax = 0.0, Dmax = 0.0, gmax = 0.0, taumin = 1e300;
  for (double T : {Tmin, Tmax})
    for (int a = 0; a < 4; ++a)
      for (int q = 0; q < 2; ++q) {
        const double A = p.A0[a][q] + p.A1[a][q] * (T - p.T_eut);
        if (!(A > 0)) {
          snprintf(why, nwhy, "A[%d][%d](T=%g) <= 0 (temperatures %g..%g over z %g..%g, t %g..%g)", a, q, T, Tmin,
                   Tmax, zlo, zhi, tlo, thi);
          return false;
        }
        Amin = std::min(Amin, A);
        Amax = std::max(Amax, A);
      }
  for (int a = 0; a < 4; ++a) {
    taumin = std::min(taumin, p.tau[a]);
    for (int q = 0; q < 2; ++q) Dmax = std::max(Dmax, p.D[a][q]);
    for (int b = 0; b < 4; ++b) if (a != b) gmax = std::max(gmax, p.gamma[a][b]);
  }
  const double Dmu = Dmax * Amax / Amin, Dphi = 2.0 * gmax * std::max(Tmax, 0.0) / taumin;
  const double lim = p.dx * p.dx / (6.0 * std::max(Dmu, Dphi));
  if (!(p.dt <= lim)) {
    snprintf(why, nwhy, "dt = %g above the explicit-Euler bound %g (D_mu %g, D_phi %g; DESIGN.md R29)", p.dt, lim,
             Dmu, Dphi);
    return false;
  }
  return true;
}

pf_status validate(const pf_grid *g, const pf_params *p) {
  pf_ctx *c = nullptr;
  const int64_t n[3] = {g->nx, g->ny, g->nz};
  const int P[3] = {g->px, g->py, g->pz};
  const char *ax = "xyz";
  for (int a = 0; a < 3; ++a) {
    if (n[a] <= 0 || P[a] <= 0) return fail(c, PF_ERR_CONFIG, "axis %c: non-positive size or block count", ax[a]);
    if (n[a] % P[a] != 0)
      return fail(c, PF_ERR_CONFIG, "axis %c: %lld cells not divisible by %d blocks", ax[a], (long long)n[a], P[a]);
    if (n[a] / P[a] < 2) return fail(c, PF_ERR_CONFIG, "axis %c: blocks must be >= 2 cells", ax[a]);
  }
  const int nb = P[0] * P[1] * P[2];
  if (g->nranks != 1 && g->nranks != nb)
    return fail(c, PF_ERR_CONFIG, "nranks (%d) must be 1 or px*py*pz (%d)", g->nranks, nb);
  if (g->rank < 0 || g->rank >= g->nranks) return fail(c, PF_ERR_CONFIG, "rank %d out of range", g->rank);
  for (int a = 0; a < 4; ++a)
    for (int b = 0; b < 4; ++b) {
      if (p->gamma[a][b] != p->gamma[b][a] || p->delta[a][b] != p->delta[b][a])
        return fail(c, PF_ERR_CONFIG, "gamma/delta not symmetric at (%d,%d)", a, b);
      if (a != b && !(p->gamma[a][b] > 0)) return fail(c, PF_ERR_CONFIG, "gamma[%d][%d] must be > 0", a, b);
    }
  if (!(p->dt > 0) || !(p->dx > 0) || !(p->eps > 0)) return fail(c, PF_ERR_CONFIG, "dt, dx, eps must be > 0");
  for (int a = 0; a < 4; ++a)
    if (!(p->tau[a] > 0)) return fail(c, PF_ERR_CONFIG, "tau[%d] must be > 0", a);
  // A(T) > 0 and the explicit-Euler step bound over the initial window's
  // temperatures (z in [-1, NZ+1], t = 0); pf_step re-checks both over the
  // temperatures the requested steps reach (the isotherm's v t drift, the
  // window's origin)
  {
    char why[256];
    if (!t_range_ok(*p, -1.0, (double)g->nz + 1.0, 0.0, 0.0, why, sizeof(why)))
      return fail(c, PF_ERR_CONFIG, "%s", why);
  }
  if (p->window && !(p->window_frac > 0 && p->window_frac <= 1)) return fail(c, PF_ERR_CONFIG, "window_frac");
  if (p->overlap < 0 || p->overlap > 4) return fail(c, PF_ERR_CONFIG, "overlap must be 0..4");
  return PF_OK;
}

}  // namespace

// ===========================================================================
// C ABI
// ===========================================================================
extern "C" {

pf_status pf_nccl_unique_id(uint8_t out[128]) {
  if (!out) return PF_ERR_ARG;
  static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId size");
  ncclUniqueId id;
  if (ncclGetUniqueId(&id) != ncclSuccess) return PF_ERR_COMM;
  memcpy(out, &id, 128);
  return PF_OK;
}

pf_status pf_halo_plan(const pf_grid *g, int32_t field, int64_t *send_counts, int64_t *recv_counts) {
  if (!g || !send_counts || !recv_counts || (field != 0 && field != 1)) return PF_ERR_ARG;
  if (g->px <= 0 || g->py <= 0 || g->pz <= 0 || g->nx % g->px || g->ny % g->py || g->nz % g->pz) return PF_ERR_CONFIG;
  const int nb = g->px * g->py * g->pz;
  if ((g->nranks != 1 && g->nranks != nb) || g->rank < 0 || g->rank >= g->nranks) return PF_ERR_CONFIG;
  pf_ctx tmp;  // host-only: the region enumeration reads the grid alone
  tmp.g = *g;
  tmp.nblocks_total = nb;
  const int nx = (int)(g->nx / g->px), ny = (int)(g->ny / g->py), nz = (int)(g->nz / g->pz);
  const int ncomp = field == 0 ? NPH : NMU;
  for (int r = 0; r < g->nranks; ++r) send_counts[r] = recv_counts[r] = 0;
  for (int bid = 0; bid < nb; ++bid) {
    const int bx = bid % g->px, by = (bid / g->px) % g->py, bz = bid / (g->px * g->py);
    for (const auto &d : ghost_dirs()) {
      const Region r = ghost_region(&tmp, bx, by, bz, d, nx, ny, nz);
      const int rdst = owner_rank(&tmp, r.dst_bid), rsrc = owner_rank(&tmp, r.src_bid);
      const int64_t n = r.ext[0] * r.ext[1] * r.ext[2] * ncomp;
      if (rdst == g->rank && rsrc != g->rank) recv_counts[rsrc] += n;
      if (rsrc == g->rank && rdst != g->rank) send_counts[rdst] += n;
    }
  }
  return PF_OK;
}

pf_status pf_create(const pf_grid *g, const pf_params *p, pf_ctx **out) {
  g_create_error.clear();
  if (!g || !p || !out) return fail(nullptr, PF_ERR_ARG, "NULL argument");
  *out = nullptr;
  CKS(validate(g, p));
  pf_ctx *c = new pf_ctx();
  c->g = *g;
  c->p = *p;
  auto bail = [&](pf_status st) {
    g_create_error = c->err;
    pf_destroy(c);
    return st;
  };
  if (cudaSetDevice(g->device) != cudaSuccess) {
    cudaGetLastError();
    fail(c, PF_ERR_CUDA, "cudaSetDevice(%d) failed (no GPU?)", g->device);
    return bail(PF_ERR_CUDA);
  }
  // kernel constants
  KParams &kp = c->kp;
  kp.dt = p->dt; kp.inv_dt = 1.0 / p->dt; kp.inv_dx = 1.0 / p->dx; kp.inv_2dx = 1.0 / (2.0 * p->dx);
  for (int a = 0; a < 4; ++a) {
    kp.dt_taueps[a] = p->dt / (p->tau[a] * p->eps);
    kp.g3[a] = p->gamma3[a];
  }
  for (int q = 0; q < 6; ++q) {
    kp.g2[q] = 2.0 * p->gamma[pair_a(q)][pair_b(q)];
    kp.gf2[q] = kp.g2[q] * 0.5 / p->dx;
    kp.g2c[q] = kp.g2[q] * kp.inv_2dx * kp.inv_2dx;
    kp.omp[q] = 16.0 / (M_PI * M_PI) * p->gamma[pair_a(q)][pair_b(q)];
    kp.delta16[q] = p->aniso ? 16.0 * p->delta[pair_a(q)][pair_b(q)] : 0.0;
  }
  kp.dmask = 0;
  for (int q = 0; q < 6; ++q) kp.dmask |= (kp.delta16[q] != 0.0 ? 1 : 0) << q;
  kp.pi_eps_16dt = M_PI * p->eps / (16.0 * p->dt);
  kp.Gv = p->G * p->v;
  kp.aniso = p->aniso ? 1 : 0;
  kp.shortcuts = p->shortcuts ? 1 : 0;
  TabParams &tp = c->tp;
  tp.T0 = p->T0; tp.G = p->G; tp.v = p->v; tp.dt = p->dt; tp.dx = p->dx; tp.T_eut = p->T_eut; tp.eps = p->eps;
  for (int a = 0; a < 4; ++a) {
    tp.L[a] = p->L[a];
    for (int q = 0; q < 2; ++q) {
      tp.A0[a][q] = p->A0[a][q]; tp.A1[a][q] = p->A1[a][q]; tp.c0[a][q] = p->c0[a][q];
      tp.m[a][q] = p->m[a][q]; tp.D[a][q] = p->D[a][q];
      kp.mch[a][q] = p->m[a][q];
    }
  }
  // decomposition
  c->nblocks_total = g->px * g->py * g->pz;
  const int nx = (int)(g->nx / g->px), ny = (int)(g->ny / g->py), nz = (int)(g->nz / g->pz);
  c->slack = p->window ? 16 : 0;
  std::vector<int> mine;
  if (g->nranks == 1) for (int b = 0; b < c->nblocks_total; ++b) mine.push_back(b);
  else mine.push_back(g->rank);
  for (int bid : mine) {
    Block b{};
    b.bx = bid % g->px; b.by = (bid / g->px) % g->py; b.bz = bid / (g->px * g->py);
    b.nx = nx; b.ny = ny; b.nz = nz;
    b.x0 = (int64_t)b.bx * nx; b.y0 = (int64_t)b.by * ny; b.z0 = (int64_t)b.bz * nz;
    b.pitch = ((nx + XO + 1) + 15) / 16 * 16;
    b.plane = b.pitch * (ny + 2);
    b.nplanes_alloc = nz + 2 + c->slack;
    b.woff = 0;
    const size_t bytes = (size_t)b.plane * b.nplanes_alloc * sizeof(double);
    for (int cp = 0; cp < 2; ++cp) {
      for (int a = 0; a < NPH; ++a) {
        if (cudaMalloc(&b.phi[cp][a], bytes) != cudaSuccess) { cudaGetLastError(); c->blocks.push_back(b); fail(c, PF_ERR_CUDA, "out of device memory (%zu B)", bytes); return bail(PF_ERR_CUDA); }
        cudaMemset(b.phi[cp][a], 0, bytes);
      }
      for (int q = 0; q < NMU; ++q) {
        if (cudaMalloc(&b.mu[cp][q], bytes) != cudaSuccess) { cudaGetLastError(); c->blocks.push_back(b); fail(c, PF_ERR_CUDA, "out of device memory (%zu B)", bytes); return bail(PF_ERR_CUDA); }
        cudaMemset(b.mu[cp][q], 0, bytes);
      }
    }
    c->blocks.push_back(b);
    if (encode_maps(c, c->blocks.back()) != PF_OK) return bail(c->status);
  }
  // rank box
  {
    int64_t x1 = 0, y1 = 0, z1 = 0;
    c->box_x0 = c->box_y0 = c->box_z0 = INT64_MAX;
    for (auto &b : c->blocks) {
      c->box_x0 = std::min(c->box_x0, b.x0); c->box_y0 = std::min(c->box_y0, b.y0); c->box_z0 = std::min(c->box_z0, b.z0);
      x1 = std::max(x1, b.x0 + b.nx); y1 = std::max(y1, b.y0 + b.ny); z1 = std::max(z1, b.z0 + b.nz);
    }
    c->box_nx = x1 - c->box_x0; c->box_ny = y1 - c->box_y0; c->box_nz = z1 - c->box_z0;
  }
  if (g->stream) { c->stream = (cudaStream_t)g->stream; c->own_stream = false; }
  else {
    if (cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking) != cudaSuccess) { fail(c, PF_ERR_CUDA, "stream"); return bail(PF_ERR_CUDA); }
    c->own_stream = true;
  }
  if (cudaStreamCreateWithFlags(&c->cstream, cudaStreamNonBlocking) != cudaSuccess ||
      cudaEventCreateWithFlags(&c->ev_mu_done, cudaEventDisableTiming) != cudaSuccess ||
      cudaEventCreateWithFlags(&c->ev_mu_halo, cudaEventDisableTiming) != cudaSuccess ||
      cudaEventCreateWithFlags(&c->ev_phi_done, cudaEventDisableTiming) != cudaSuccess ||
      cudaEventCreateWithFlags(&c->ev_phi_halo, cudaEventDisableTiming) != cudaSuccess ||
      cudaEventCreateWithFlags(&c->ev_copy, cudaEventDisableTiming) != cudaSuccess ||
      cudaEventCreateWithFlags(&c->ev_stage[0], cudaEventDisableTiming) != cudaSuccess ||
      cudaEventCreateWithFlags(&c->ev_stage[1], cudaEventDisableTiming) != cudaSuccess) {
    fail(c, PF_ERR_CUDA, "comm stream / events");
    return bail(PF_ERR_CUDA);
  }
  c->tab_planes = g->nz + 2;
  if (cudaMalloc(&c->d_tab, (size_t)c->tab_planes * TAB * sizeof(double)) != cudaSuccess ||
      cudaMalloc(&c->d_red, 4 * sizeof(unsigned long long)) != cudaSuccess ||
      cudaMalloc(&c->d_step, sizeof(int64_t)) != cudaSuccess) {
    fail(c, PF_ERR_CUDA, "alloc table"); return bail(PF_ERR_CUDA);
  }
  if (g->nranks > 1) {
    ncclUniqueId id;
    memcpy(&id, g->nccl_id, 128);
    ncclResult_t r = ncclCommInitRank(&c->comm, g->nranks, id, g->rank);
    if (r != ncclSuccess) { fail(c, PF_ERR_COMM, "ncclCommInitRank: %s", ncclGetErrorString(r)); return bail(PF_ERR_COMM); }
    // a second communicator for the mu exchange, which runs on its own stream
    // concurrently with the phi-sweep / phi exchange of the next step
    r = ncclCommSplit(c->comm, 0, g->rank, &c->comm_mu, nullptr);
    if (r != ncclSuccess) { fail(c, PF_ERR_COMM, "ncclCommSplit: %s", ncclGetErrorString(r)); return bail(PF_ERR_COMM); }
  }
  if (build_plans(c) != PF_OK) return bail(c->status);
  prepare_phi_tiled();
  prepare_mu_tiled();
  prepare_fused();
  if (cudaDeviceSynchronize() != cudaSuccess) { fail(c, PF_ERR_CUDA, "setup sync"); return bail(PF_ERR_CUDA); }
  *out = c;
  return PF_OK;
}

pf_status pf_init(pf_ctx *c, uint64_t seed) {
  CKS(check_state(c, false));
  const pf_params &p = c->p;
  InitSpec is{};
  is.kind = p.init_kind; is.n_seeds = p.init_n_seeds; is.layer_height = p.init_layer_height;
  is.W = p.init_iface_width; is.mu_noise = p.init_mu_noise; is.seed = seed;
  is.NX = c->g.nx; is.NY = c->g.ny; is.NZ = c->g.nz; is.planar_phase = p.init_planar_phase;
  // host side: seeds / lamellae from the same counter-based generator
  auto mix = [](uint64_t z) {
    z += 0x9E3779B97F4A7C15ULL;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
  };
  auto u01 = [&](uint64_t stream, uint64_t idx) {
    return (double)(mix(mix(seed ^ (stream * 0xD1B54A32D192ED03ULL)) ^ idx) >> 11) * 0x1.0p-53;
  };
  std::vector<double> sx, sy;
  std::vector<int> sp;
  std::vector<int64_t> lam;
  double *d_sx = nullptr, *d_sy = nullptr;
  int *d_sp = nullptr;
  int64_t *d_lam = nullptr;
  if (p.init_kind == 0) {
    if (p.init_n_seeds <= 0) return fail(c, PF_ERR_CONFIG, "init_n_seeds must be > 0");
    for (int q = 0; q < p.init_n_seeds; ++q) {
      sx.push_back(u01(1, q) * (double)c->g.nx);
      sy.push_back(u01(2, q) * (double)c->g.ny);
      sp.push_back(std::min(2, (int)(u01(3, q) * 3.0)));
    }
    CK(cudaMalloc(&d_sx, sx.size() * sizeof(double)));
    CK(cudaMalloc(&d_sy, sy.size() * sizeof(double)));
    CK(cudaMalloc(&d_sp, sp.size() * sizeof(int)));
    CK(cudaMemcpy(d_sx, sx.data(), sx.size() * sizeof(double), cudaMemcpyHostToDevice));
    CK(cudaMemcpy(d_sy, sy.data(), sy.size() * sizeof(double), cudaMemcpyHostToDevice));
    CK(cudaMemcpy(d_sp, sp.data(), sp.size() * sizeof(int), cudaMemcpyHostToDevice));
  } else if (p.init_kind == 1) {
    int64_t x = 0, n = 0;
    while (x < c->g.nx) {
      lam.push_back(x);
      x += p.init_lam_wmin + (int64_t)(u01(4, (uint64_t)n) * (double)(p.init_lam_wmax - p.init_lam_wmin + 1));
      ++n;
    }
    lam.push_back(c->g.nx);
    is.nlam = (int)n;
    CK(cudaMalloc(&d_lam, lam.size() * sizeof(int64_t)));
    CK(cudaMemcpy(d_lam, lam.data(), lam.size() * sizeof(int64_t), cudaMemcpyHostToDevice));
  }
  is.sx = d_sx; is.sy = d_sy; is.sp = d_sp; is.lam = d_lam;
  for (auto &b : c->blocks) b.woff = 0;
  c->cur = 0;
  CKS(build_plans(c));
  for (auto &b : c->blocks) {
    double *fp[NPH], *fm[NMU];
    for (int a = 0; a < NPH; ++a) fp[a] = b.phi[c->cur][a] + cell_off(b, 0, 0, 0);
    for (int q = 0; q < NMU; ++q) fm[q] = b.mu[c->cur][q] + cell_off(b, 0, 0, 0);
    launch_init(c->stream, is, fp, fm, b.nx, b.ny, b.nz, b.pitch, b.plane, b.x0, b.y0, b.z0);
  }
  CK(cudaGetLastError());
  CKS(fill_all_ghosts(c));
  CK(cudaStreamSynchronize(c->stream));
  cudaFree(d_sx); cudaFree(d_sy); cudaFree(d_sp); cudaFree(d_lam);
  c->step = 0; c->zorig = 0; c->shifts = 0; c->next_check = 0; c->last_front = -1;
  c->initialized = true;
  return PF_OK;
}

pf_status pf_write(pf_ctx *c, const double *phi, const double *mu) {
  CKS(check_state(c, false));
  if (!phi || !mu) return fail(c, PF_ERR_ARG, "NULL state pointer");
  // the plans are rebuilt only if a window shift moved a block's ring offset
  // (pf_step_io's multi-block fallback writes every step)
  bool fresh = c->plans_woff0;
  for (auto &b : c->blocks) { fresh = fresh && b.woff == 0; b.woff = 0; }
  c->cur = 0;
  if (!fresh) CKS(build_plans(c));
  CKS(move_state(c, const_cast<double *>(phi), const_cast<double *>(mu), true));
  CKS(fill_all_ghosts(c));
  CK(cudaStreamSynchronize(c->stream));
  c->next_check = c->step;
  c->initialized = true;
  return PF_OK;
}

pf_status pf_set_time(pf_ctx *c, int64_t step, int64_t z_origin) {
  CKS(check_state(c, false));
  c->step = step;
  c->zorig = z_origin;
  c->next_check = step;
  invalidate_graphs(c);   // the origin is a captured table argument
  return PF_OK;
}

// Enqueue one time step (Algorithm 1 / 2) on the
// context's streams: table, phi-sweep, phi halo, mu-sweep(s), mu halo.
// graph = true while capturing a CUDA graph: the table reads the time level
// from d_step (incremented at the end) and the mu halo is exchanged in order
// on the main stream (results identical to the hidden exchange).
pf_status enqueue_step(pf_ctx *c, bool graph) {
  {
    TimedSpan ts(c, 3, 0);
    launch_table(c->stream, c->d_tab, c->tab_planes, c->tp, c->step, c->zorig, graph ? c->d_step : nullptr);
    c->launches++;
  }
  {  // phi-sweep (Algorithm 1 line 1)
    TimedSpan ts(c, 0, (int)c->blocks.size());
    for (const auto &b : c->blocks) {
      const BlockView v = view(c, b, 0);
      if (c->p.variant == 1) launch_phi_naive(c->stream, c->kp, v);
      else launch_phi_tiled(c->stream, c->kp, v, maps_of(c, b, 0));
      c->launches++;
    }
  }
  CK(cudaGetLastError());
  const int ov = c->p.overlap;
  const bool hide_phi = (ov == 2 || ov == 3) && c->p.variant != 1, hide_mu = (ov == 0 || ov == 3 || ov == 4) && !graph;
  auto mu_sweep = [&](int mode) -> pf_status {
    TimedSpan ts(c, 1, (int)c->blocks.size());
    for (const auto &b : c->blocks) {
      const BlockView v = view(c, b, 1);
      if (c->p.variant == 1) launch_mu_naive(c->stream, c->kp, v);
      else launch_mu_tiled(c->stream, c->kp, v, maps_of(c, b, 1), mode);
      c->launches++;
    }
    CK(cudaGetLastError());
    return PF_OK;
  };
  if (ov == 4 && c->p.variant != 1) {
    // the phi_dst exchange hidden without Algorithm 2's second pass: the
    // mu-sweep over the tiles whose stencil reads no ghost (off the x/y block
    // faces, planes 1 .. nz-2) runs beside it, the shell (the boundary tile
    // rows / columns, the two cap planes) after it.  Bitwise the cells' values
    // of the plain mu-sweep (pinned face arithmetic).
    CK(cudaEventRecord(c->ev_phi_done, c->stream));
    CK(cudaStreamWaitEvent(c->cstream, c->ev_phi_done, 0));
    CKS(exchange(c, 0, c->cur ^ 1, true));
    CK(cudaEventRecord(c->ev_phi_halo, c->cstream));
    CKS(join_mu(c));
    {
      TimedSpan ts(c, 1, (int)c->blocks.size());
      for (const auto &b : c->blocks) {
        const int gx = mu_tiles_x(b.nx), gy = mu_tiles_y(b.ny);
        if (gx >= 3 && gy >= 3 && b.nz >= 3) {
          launch_mu_tiles(c->stream, c->kp, slab_view(view(c, b, 1), 1, 1, b.nz - 1), maps_of(c, b, 1), 1, gx - 1, 1,
                          gy - 1);
          c->launches++;
        }
      }
      CK(cudaGetLastError());
    }
    CK(cudaStreamWaitEvent(c->stream, c->ev_phi_halo, 0));
    {
      TimedSpan ts(c, 1, (int)c->blocks.size());
      for (const auto &b : c->blocks) {
        const int gx = mu_tiles_x(b.nx), gy = mu_tiles_y(b.ny);
        const BlockView v = view(c, b, 1);
        if (gx >= 3 && gy >= 3 && b.nz >= 3) {
          launch_mu_tiles(c->stream, c->kp, v, maps_of(c, b, 1), 0, gx, 0, 1);            // y = 0 row of tiles
          launch_mu_tiles(c->stream, c->kp, v, maps_of(c, b, 1), 0, gx, gy - 1, gy);      // last row
          launch_mu_tiles(c->stream, c->kp, v, maps_of(c, b, 1), 0, 1, 1, gy - 1);        // x = 0 column
          launch_mu_tiles(c->stream, c->kp, v, maps_of(c, b, 1), gx - 1, gx, 1, gy - 1);  // last column
          launch_mu_tiles(c->stream, c->kp, slab_view(v, 1, 0, 1), maps_of(c, b, 1), 1, gx - 1, 1, gy - 1);
          launch_mu_tiles(c->stream, c->kp, slab_view(v, 1, b.nz - 1, b.nz), maps_of(c, b, 1), 1, gx - 1, 1, gy - 1);
          c->launches += 6;
        } else {
          launch_mu_tiled(c->stream, c->kp, v, maps_of(c, b, 1), MU_FULL);
          c->launches++;
        }
      }
      CK(cudaGetLastError());
    }
  } else if (hide_phi) {
    // Algorithm 2: phi_dst ghosts on the comm stream while
    // mu-sweep-local (no anti-trapping current: phi_dst needed at the cell
    // only) runs; mu-sweep-neighbor adds the current once the ghosts are in
    CK(cudaEventRecord(c->ev_phi_done, c->stream));
    CK(cudaStreamWaitEvent(c->cstream, c->ev_phi_done, 0));
    CKS(exchange(c, 0, c->cur ^ 1, true));
    CK(cudaEventRecord(c->ev_phi_halo, c->cstream));
    CKS(join_mu(c));                  // mu_src ghosts (previous step's exchange)
    CKS(mu_sweep(MU_LOCAL));
    CK(cudaStreamWaitEvent(c->stream, c->ev_phi_halo, 0));
    CKS(mu_sweep(MU_NEIGHBOR));
  } else {
    CKS(exchange(c, 0, c->cur ^ 1));  // lines 2-3: phi_dst ghosts + boundary
    CKS(join_mu(c));                  // mu_src ghosts (previous step's overlapped exchange)
    CKS(mu_sweep(MU_FULL));           // line 4
  }
  // lines 5-6: mu_dst ghosts + boundary.  The next phi-sweep reads mu at the
  // cell centre only (D3C1), so this exchange can overlap
  // it on the comm stream (the paper's mu communication hiding)
  if (hide_mu) {
    CK(cudaEventRecord(c->ev_mu_done, c->stream));
    CK(cudaStreamWaitEvent(c->cstream, c->ev_mu_done, 0));
    CKS(exchange(c, 1, c->cur ^ 1, true));
    CK(cudaEventRecord(c->ev_mu_halo, c->cstream));
    c->mu_pending = true;
  } else {
    CKS(exchange(c, 1, c->cur ^ 1));
  }
  if (graph) { launch_step_inc(c->stream, c->d_step); c->launches++; }
  return PF_OK;
}

// ---- fused steps (pf_set_fusion): the mu-sweep of step n and the phi-sweep
// of step n+1 in one kernel (pf_fused.cu).  A run of steps becomes
//   phi-half(n0), fused(n0) .. fused(n1-2), mu-half(n1-1)
// and every state a caller, the window check or the NaN watchdog sees is a
// complete time level (the run is cut there).  Bitwise the plain sequence.
bool fusable(const pf_ctx *c) {
  return c->fusion && c->phi3 && c->p.variant != 1 && (c->p.overlap == 0 || c->p.overlap == 1) && !c->p.graph;
}

// swap phi copy `a` with the third copy: addresses, TMA maps, the phi halo plan
void rotate_phi(pf_ctx *c, int a) {
  for (auto &b : c->blocks)
    for (int q = 0; q < NPH; ++q) {
      std::swap(b.phi[a][q], b.phi[2][q]);
      std::swap(b.tphi[a][q], b.tphi[2][q]);
      std::swap(b.tphim[a][q], b.tphim[2][q]);
      std::swap(b.tphif[a][q], b.tphif[2][q]);
    }
  std::swap(c->plan[0][a], c->plan[0][2]);
  invalidate_graphs(c);   // captured launches hold addresses
}

// Algorithm 1 lines 1-3: table rows of step n, phi-sweep, phi^{n+1} ghosts
pf_status enqueue_phi_half(pf_ctx *c) {
  {
    TimedSpan ts(c, 3, 0);
    launch_table(c->stream, c->d_tab, c->tab_planes, c->tp, c->step, c->zorig, nullptr);
    c->launches++;
  }
  {
    TimedSpan ts(c, 0, (int)c->blocks.size());
    for (const auto &b : c->blocks) {
      launch_phi_tiled(c->stream, c->kp, view(c, b, 0), maps_of(c, b, 0));
      c->launches++;
    }
  }
  CK(cudaGetLastError());
  return exchange(c, 0, c->cur ^ 1);
}

// lines 4-6: mu-sweep, mu^{n+1} ghosts (mode 0: beside what follows)
pf_status enqueue_mu_half(pf_ctx *c) {
  CKS(join_mu(c));
  {
    TimedSpan ts(c, 1, (int)c->blocks.size());
    for (const auto &b : c->blocks) {
      launch_mu_tiled(c->stream, c->kp, view(c, b, 1), maps_of(c, b, 1), MU_FULL);
      c->launches++;
    }
  }
  CK(cudaGetLastError());
  if (c->p.overlap != 0) return exchange(c, 1, c->cur ^ 1);
  CK(cudaEventRecord(c->ev_mu_done, c->stream));
  CK(cudaStreamWaitEvent(c->cstream, c->ev_mu_done, 0));
  CKS(exchange(c, 1, c->cur ^ 1, true));
  CK(cudaEventRecord(c->ev_mu_halo, c->cstream));
  c->mu_pending = true;
  return PF_OK;
}

// lines 4-6 of step n and 1-3 of step n+1: one fused kernel per block, then the
// mu^{n+1} and phi^{n+2} ghosts (the next fused kernel reads both stencils)
pf_status enqueue_fused(pf_ctx *c) {
  CKS(join_mu(c));
  {
    TimedSpan ts(c, 3, 0);
    launch_table(c->stream, c->d_tab2, c->tab_planes, c->tp, c->step + 1, c->zorig, nullptr);
    c->launches++;
  }
  {
    TimedSpan ts(c, 4, (int)c->blocks.size());
    for (const auto &b : c->blocks) {
      FusedOut fo;
      const int64_t o = cell_off(b, 0, 0, 0);
      for (int a = 0; a < NPH; ++a) fo.phi2[a] = b.phi[2][a] + o;
      fo.tabp = c->d_tab2 + (b.z0 + 1) * TAB;
      launch_fused(c->stream, c->kp, view(c, b, 1), maps_fused(c, b), fo);
      c->launches++;
    }
  }
  CK(cudaGetLastError());
  const int c0 = c->cur;
  rotate_phi(c, c0);                // phi^{n+2} takes the place of the dead phi^n
  std::swap(c->d_tab, c->d_tab2);   // step n+1's rows become the current ones
  CKS(exchange(c, 1, c0 ^ 1));
  return exchange(c, 0, c0);
}

// Capture one step from src copy c->cur into c->gexec[c->cur].
pf_status capture_step(pf_ctx *c) {
  cudaGraph_t g = nullptr;
  const int64_t l0 = c->launches;
  CK(cudaStreamBeginCapture(c->stream, cudaStreamCaptureModeThreadLocal));
  const pf_status st = enqueue_step(c, true);
  const cudaError_t e = cudaStreamEndCapture(c->stream, &g);
  if (st != PF_OK) { if (g) cudaGraphDestroy(g); return st; }
  CK(e);
  const cudaError_t ei = cudaGraphInstantiate(&c->gexec[c->cur], g, 0);
  cudaGraphDestroy(g);
  CK(ei);
  c->graph_launches[c->cur] = c->launches - l0;
  c->launches = l0;
  return PF_OK;
}

pf_status pf_step(pf_ctx *c, int64_t n) {
  CKS(check_state(c, true));
  if (n < 0) return fail(c, PF_ERR_ARG, "negative step count");
  {  // the temperatures these n steps reach: the isotherm's drift over t, and
     // with the window one origin shift per step at most (reading R16)
    char why[256];
    const double z0 = (double)c->zorig - 1.0;
    const double z1 = (double)(c->zorig + (c->p.window ? n : 0) + c->g.nz) + 1.0;
    if (!t_range_ok(c->p, z0, z1, (double)c->step * c->p.dt, (double)(c->step + n) * c->p.dt, why, sizeof(why))) {
      c->err = std::string("pf_step(") + std::to_string((long long)n) + "): " + why;
      return PF_ERR_CONFIG;   // nothing ran: the context stays usable (no poisoning)
    }
  }
  // CUDA graphs (pf_params.graph = 1) for single-rank runs without per-sweep
  // timing: one launch per step instead of five-plus — same results, bit for bit
  if (fusable(c) && n >= 2) {
    bool ahead = false;   // phi^{n+1} of the current step computed (and its ghosts)
    for (int64_t s = 0; s < n; ++s) {
      const int64_t nx1 = c->step + 1;
      const bool nan_due = c->p.nan_check_every > 0 && nx1 % c->p.nan_check_every == 0;
      const bool end = s == n - 1 || nan_due || (c->p.window && nx1 >= c->next_check);
      if (!ahead) CKS(enqueue_phi_half(c));
      if (end) CKS(enqueue_mu_half(c));
      else CKS(enqueue_fused(c));
      ahead = !end;
      c->cur ^= 1;
      c->step += 1;
      if (end) {
        if ((c->p.window && c->step >= c->next_check) || nan_due) CKS(join_mu(c));
        CKS(window_check(c));
        if (nan_due) CKS(nan_check(c));
      }
      if (c->timing && c->spans.size() > 4096) CKS(collect_timing(c));
    }
    CKS(join_mu(c));
    CK(cudaStreamSynchronize(c->stream));
    CK(cudaGetLastError());
    return collect_timing(c);
  }
  const bool use_graph = !c->timing && c->g.nranks == 1 && c->p.graph && n > 0;
  if (use_graph) {
    CKS(join_mu(c));
    CK(cudaMemcpyAsync(c->d_step, &c->step, sizeof(int64_t), cudaMemcpyHostToDevice, c->stream));
  }
  for (int64_t s = 0; s < n; ++s) {
    if (use_graph) {
      if (!c->gexec[c->cur]) CKS(capture_step(c));
      CK(cudaGraphLaunch(c->gexec[c->cur], c->stream));
      c->launches += c->graph_launches[c->cur];
    } else {
      CKS(enqueue_step(c, false));
    }
    c->cur ^= 1;                        // line 7: swap
    c->step += 1;
    const bool nan_due = c->p.nan_check_every > 0 && c->step % c->p.nan_check_every == 0;
    if ((c->p.window && c->step >= c->next_check) || nan_due) CKS(join_mu(c));
    CKS(window_check(c));
    if (nan_due) CKS(nan_check(c));
    if (c->timing && c->spans.size() > 4096) CKS(collect_timing(c));
  }
  CKS(join_mu(c));
  CK(cudaStreamSynchronize(c->stream));
  CK(cudaGetLastError());
  CKS(collect_timing(c));
  return PF_OK;
}

pf_status pf_step_io(pf_ctx *c, const double *phi_in, const double *mu_in, double *phi_out, double *mu_out) {
  CKS(check_state(c, false));
  if (!phi_in || !mu_in || !phi_out || !mu_out) return fail(c, PF_ERR_ARG, "NULL state pointer");
  const bool host = !is_device_ptr(phi_in) && !is_device_ptr(mu_in) && !is_device_ptr(phi_out) &&
                    !is_device_ptr(mu_out);
  // the slab pipeline covers one block per process, no window, the tiled
  // sweeps and the Algorithm-1 mu update (overlap 0 / 1 are bitwise equal);
  // anything else is the same sequence of calls without the overlap
  if (!host || c->g.nranks != 1 || c->blocks.size() != 1 || c->p.variant == 1 ||
      (c->p.overlap != 0 && c->p.overlap != 1)) {
    CKS(pf_write(c, phi_in, mu_in));
    CKS(pf_step(c, 1));
    return pf_read(c, phi_out, mu_out);
  }
  CKS(join_mu(c));
  CK(cudaStreamSynchronize(c->stream));
  CK(cudaStreamSynchronize(c->cstream));
  CKS(slab_setup(c));
  auto &io = c->sio;
  Block &b = c->blocks[0];
  const int src = c->cur, dst = c->cur ^ 1, S = io.S;
  auto zs = [&](int s) { return std::min(b.nz, s * io.H); };
  for (int s = 0; s < S; ++s) {   // every upload back to back
    CKS(slab_copy(c, src, phi_in, mu_in, zs(s), zs(s + 1), true, io.up));
    CK(cudaEventRecord(io.ev_up[s], io.up));
  }
  launch_table(c->stream, c->d_tab, c->tab_planes, c->tp, c->step, c->zorig, nullptr);
  c->launches++;
  // iteration s: ghosts of input slab s; then slab s-1: its phi-sweep, extended
  // by the first plane of slab s (needs input planes up to z_s + 1, in slab s)
  // so that its mu-sweep (phi^{n+1} up to plane z_s) and its download follow at
  // once — the download of slab s-1 waits for the upload of slab s only.  The
  // extra plane is computed again, to the same bits, by the next slab's sweep.
  for (int s = 0; s <= S; ++s) {
    if (s < S) {
      CK(cudaStreamWaitEvent(c->stream, io.ev_up[s], 0));
      for (int f = 0; f < 2; ++f) {
        launch_copy(c->stream, io.ops[f][src][s], io.nops[f][src][s], io.nctas[f][src][s]);
        c->launches++;
      }
    }
    if (s >= 1) {
      const int z0 = zs(s - 1), z1 = zs(s), z1x = std::min(b.nz, z1 + 1);
      launch_phi_tiled(c->stream, c->kp, slab_view(view(c, b, 0), 0, z0, z1x), maps_of(c, b, 0));
      launch_copy(c->stream, io.ops_x[dst][s - 1], io.nops_x[dst][s - 1], io.nctas_x[dst][s - 1]);
      launch_mu_tiled(c->stream, c->kp, slab_view(view(c, b, 1), 1, z0, z1), maps_of(c, b, 1), MU_FULL);
      c->launches += 3;
      CK(cudaEventRecord(io.ev_mu[s - 1], c->stream));
      CK(cudaStreamWaitEvent(io.dn, io.ev_mu[s - 1], 0));
      CKS(slab_copy(c, dst, phi_out, mu_out, z0, z1, false, io.dn));
    }
    CK(cudaGetLastError());
  }
  CKS(exchange(c, 1, dst));   // mu^{n+1} ghosts: the device keeps a complete time level
  CK(cudaStreamSynchronize(io.dn));
  CK(cudaStreamSynchronize(c->stream));
  c->cur ^= 1;
  c->step += 1;
  c->initialized = true;
  // moving window (a new state: the front is checked now, as after pf_write +
  // pf_step): a shift changes the state after its download, which is then
  // read again — the rare step pays one more transfer
  c->next_check = c->step;
  const int64_t shifts = c->shifts;
  CKS(window_check(c));
  if (c->shifts != shifts) CKS(move_state(c, phi_out, mu_out, false));
  if (c->p.nan_check_every > 0 && c->step % c->p.nan_check_every == 0) CKS(nan_check(c));
  return PF_OK;
}

pf_status pf_read(pf_ctx *c, double *phi, double *mu) {
  CKS(check_state(c, true));
  if (!phi || !mu) return fail(c, PF_ERR_ARG, "NULL state pointer");
  return move_state(c, phi, mu, false);
}

pf_status pf_save(pf_ctx *c, const char *path) {
  CKS(check_state(c, true));
  if (!path) return fail(c, PF_ERR_ARG, "NULL path");
  CKS(join_mu(c));
  pf_status st = PF_OK;
  if (c->g.rank == 0) {  // header + full-length file, before any rank writes rows
    unsigned char hdr[CKPT_HDR];
    const uint64_t dims[3] = {(uint64_t)c->g.nx, (uint64_t)c->g.ny, (uint64_t)c->g.nz};
    const uint32_t counts[2] = {NPH, NMU};
    const double dx = c->p.dx, t = (double)c->step * c->p.dt;
    const uint64_t tail[2] = {(uint64_t)c->step, (uint64_t)c->zorig};
    memcpy(hdr, "PFCP0001", 8);
    memcpy(hdr + 8, dims, 24);
    memcpy(hdr + 32, counts, 8);
    memcpy(hdr + 40, &dx, 8);
    memcpy(hdr + 48, &t, 8);
    memcpy(hdr + 56, tail, 16);
    const int64_t total = CKPT_HDR + (int64_t)(NPH + NMU) * c->g.nx * c->g.ny * c->g.nz * 4;
    const int fd = open(path, O_WRONLY | O_CREAT | O_TRUNC, 0644);
    if (fd < 0) st = io_fail(c, "pf_save: cannot create %s: %s", path, strerror(errno));
    else {
      if (pwrite(fd, hdr, CKPT_HDR, 0) != CKPT_HDR || ftruncate(fd, total) != 0)
        st = io_fail(c, "pf_save: writing %s: %s", path, strerror(errno));
      close(fd);
    }
  }
  CKS(io_agree(c, st));
  CkptBuffers cb;
  CKS(ckpt_alloc(c, cb));
  const int fd = open(path, O_WRONLY);
  if (fd < 0) st = io_fail(c, "pf_save: cannot open %s: %s", path, strerror(errno));
  const auto chunks = ckpt_chunks(c);
  for (size_t i = 0; i <= chunks.size() && st == PF_OK; ++i) {
    if (i < chunks.size()) {  // device: FP64 -> FP32 + copy out of chunk i into slot i % 2
      const CkptChunk &ch = chunks[i];
      const Block &b = c->blocks[ch.blk];
      ckpt_convert(c, ch, cb.d, false);
      CK(cudaMemcpyAsync(cb.h[i & 1], cb.d, (size_t)b.nx * b.ny * ch.nzc * 4, cudaMemcpyDeviceToHost, c->stream));
      CK(cudaEventRecord(cb.ev[i & 1], c->stream));
    }
    if (i > 0) {  // host: write chunk i - 1 while the device works on chunk i
      CK(cudaEventSynchronize(cb.ev[(i - 1) & 1]));
      if (!ckpt_rows(c, fd, chunks[i - 1], cb.h[(i - 1) & 1], true))
        st = io_fail(c, "pf_save: writing %s: %s", path, strerror(errno));
    }
  }
  CK(cudaStreamSynchronize(c->stream));
  if (fd >= 0 && close(fd) != 0 && st == PF_OK) st = io_fail(c, "pf_save: closing %s: %s", path, strerror(errno));
  return io_agree(c, st);
}

pf_status pf_load(pf_ctx *c, const char *path) {
  CKS(check_state(c, false));
  if (!path) return fail(c, PF_ERR_ARG, "NULL path");
  CKS(join_mu(c));
  pf_status st = PF_OK;
  uint64_t step = 0, zorig = 0;
  const int fd = open(path, O_RDONLY);
  if (fd < 0) st = io_fail(c, "pf_load: cannot open %s: %s", path, strerror(errno));
  else {
    unsigned char hdr[CKPT_HDR];
    uint64_t dims[3];
    uint32_t counts[2];
    double dx;
    struct stat sb;
    const int64_t total = CKPT_HDR + (int64_t)(NPH + NMU) * c->g.nx * c->g.ny * c->g.nz * 4;
    if (pread(fd, hdr, CKPT_HDR, 0) != CKPT_HDR || fstat(fd, &sb) != 0)
      st = io_fail(c, "pf_load: %s: truncated header", path);
    else if (memcmp(hdr, "PFCP0001", 8) != 0)
      st = io_fail(c, "pf_load: %s: bad magic (not a PFCP0001 checkpoint)", path);
    else {
      memcpy(dims, hdr + 8, 24);
      memcpy(counts, hdr + 32, 8);
      memcpy(&dx, hdr + 40, 8);
      memcpy(&step, hdr + 56, 8);
      memcpy(&zorig, hdr + 64, 8);
      if (dims[0] != (uint64_t)c->g.nx || dims[1] != (uint64_t)c->g.ny || dims[2] != (uint64_t)c->g.nz)
        st = io_fail(c, "pf_load: %s: grid %llux%llux%llu does not match the context's %lldx%lldx%lld", path,
                     (unsigned long long)dims[0], (unsigned long long)dims[1], (unsigned long long)dims[2],
                     (long long)c->g.nx, (long long)c->g.ny, (long long)c->g.nz);
      else if (counts[0] != NPH || counts[1] != NMU)
        st = io_fail(c, "pf_load: %s: %u phases / %u potentials, expected %d / %d", path, counts[0], counts[1], NPH, NMU);
      else if (dx != c->p.dx)
        st = io_fail(c, "pf_load: %s: dx %.17g differs from the context's %.17g", path, dx, c->p.dx);
      else if ((int64_t)sb.st_size < total)
        st = io_fail(c, "pf_load: %s: truncated body (%lld of %lld bytes)", path, (long long)sb.st_size,
                     (long long)total);
    }
  }
  st = io_agree(c, st);
  if (st != PF_OK) { if (fd >= 0) close(fd); return st; }
  // the fields are overwritten from here on: a failure leaves no valid state
  c->initialized = false;
  for (auto &b : c->blocks) b.woff = 0;
  c->cur = 0;
  CKS(build_plans(c));
  CkptBuffers cb;
  CKS(ckpt_alloc(c, cb));
  const auto chunks = ckpt_chunks(c);
  for (size_t i = 0; i < chunks.size() && st == PF_OK; ++i) {
    const CkptChunk &ch = chunks[i];
    const Block &b = c->blocks[ch.blk];
    if (i >= 2) CK(cudaEventSynchronize(cb.ev[i & 1]));  // slot free: its copy-in finished
    // host: read chunk i while the device converts chunk i - 1
    if (!ckpt_rows(c, fd, ch, cb.h[i & 1], false)) { st = io_fail(c, "pf_load: reading %s failed", path); break; }
    CK(cudaMemcpyAsync(cb.d, cb.h[i & 1], (size_t)b.nx * b.ny * ch.nzc * 4, cudaMemcpyHostToDevice, c->stream));
    CK(cudaEventRecord(cb.ev[i & 1], c->stream));
    ckpt_convert(c, ch, cb.d, true);
  }
  close(fd);
  CK(cudaStreamSynchronize(c->stream));
  CK(cudaGetLastError());
  CKS(io_agree(c, st));
  CKS(fill_all_ghosts(c));
  CK(cudaStreamSynchronize(c->stream));
  c->step = (int64_t)step;
  c->zorig = (int64_t)zorig;
  invalidate_graphs(c);
  c->next_check = c->step;
  c->last_front = -1;
  c->initialized = true;
  return PF_OK;
}

pf_status pf_set_timing(pf_ctx *c, int32_t on) {
  CKS(check_state(c, false));
  CKS(collect_timing(c));
  c->timing = on != 0;
  for (double &m : c->ms) m = 0;
  c->phi_launches = c->mu_launches = c->fused_launches = 0;
  return PF_OK;
}

pf_status pf_set_fusion(pf_ctx *c, int32_t on) {
  CKS(check_state(c, false));
  if (on && !c->phi3) {
    // the third phi copy (and the second table): allocated once, on first use
    CKS(join_mu(c));
    CK(cudaStreamSynchronize(c->stream));
    bool ok = cudaMalloc(&c->d_tab2, (size_t)c->tab_planes * TAB * sizeof(double)) == cudaSuccess;
    for (auto &b : c->blocks) {
      const size_t bytes = (size_t)b.plane * b.nplanes_alloc * sizeof(double);
      for (int a = 0; a < NPH && ok; ++a) {
        ok = cudaMalloc(&b.phi[2][a], bytes) == cudaSuccess;
        if (ok) ok = cudaMemset(b.phi[2][a], 0, bytes) == cudaSuccess;
      }
    }
    if (!ok) {   // not enough device memory: fusion stays off, the context stays usable
      cudaGetLastError();
      for (auto &b : c->blocks)
        for (int a = 0; a < NPH; ++a) if (b.phi[2][a]) { cudaFree(b.phi[2][a]); b.phi[2][a] = nullptr; }
      if (c->d_tab2) { cudaFree(c->d_tab2); c->d_tab2 = nullptr; }
      c->err = "pf_set_fusion: no device memory for the third phi copy";
      return PF_ERR_CUDA;
    }
    c->phi3 = true;
    for (auto &b : c->blocks) CKS(encode_maps(c, b));
    CKS(build_plans(c));
  }
  if (!on && c->phi3) {   // off releases the third phi copy and the second table
    CKS(join_mu(c));
    CK(cudaStreamSynchronize(c->stream));
    for (auto &b : c->blocks)
      for (int a = 0; a < NPH; ++a) { cudaFree(b.phi[2][a]); b.phi[2][a] = nullptr; }
    Plan &pl = c->plan[0][2];
    if (pl.d_local) cudaFree(pl.d_local);
    if (pl.d_unpack) cudaFree(pl.d_unpack);
    pl = Plan{};
    cudaFree(c->d_tab2);
    c->d_tab2 = nullptr;
    c->phi3 = false;
  }
  c->fusion = on != 0;
  return PF_OK;
}

pf_status pf_set_shortcuts(pf_ctx *c, int32_t on) {
  CKS(check_state(c, false));
  c->p.shortcuts = on ? 1 : 0;
  c->kp.shortcuts = on ? 1 : 0;
  invalidate_graphs(c);   // the kernel choice and its arguments are captured
  return PF_OK;
}

pf_status pf_info(pf_ctx *c, pf_info_t *o) {
  if (!c || !o) return PF_ERR_ARG;
  memset(o, 0, sizeof(*o));
  o->nx_l = c->box_nx; o->ny_l = c->box_ny; o->nz_l = c->box_nz;
  o->x0 = c->box_x0; o->y0 = c->box_y0; o->z0 = c->box_z0;
  o->step = c->step; o->z_origin = c->zorig; o->shifts = c->shifts; o->last_front = c->last_front;
  o->nblocks_local = (int32_t)c->blocks.size();
  o->timing = c->timing;
  o->ms_phi = c->ms[0]; o->ms_mu = c->ms[1]; o->ms_halo = c->ms[2]; o->ms_other = c->ms[3];
  o->launches = c->launches; o->phi_launches = c->phi_launches; o->mu_launches = c->mu_launches;
  o->ms_fused = c->ms[4]; o->fused_launches = c->fused_launches; o->fusion = c->fusion ? 1 : 0;
  return c->status == PF_OK ? PF_OK : PF_ERR_STATE;
}

const char *pf_last_error(const pf_ctx *c) {
  if (!c) return g_create_error.c_str();
  return c->err.c_str();
}

// Marching-cubes mesh of one phase over this rank's box (PAPER.md:246-251,
// reading R26; kernels in pf_mesh.cu).  Cubes whose lower corner lies in the
// box, the upper corners in the blocks' ghost layers ("extends to the ghost
// regions"); in z only cubes below the global top plane (no cube reaches into
// the zero-flux ghost), so the ranks' meshes together are the global mesh.
pf_status pf_mesh(pf_ctx *c, int32_t phase, double iso, int64_t cap, int64_t *ids, double *pos, int64_t *ntri) {
  CKS(check_state(c, true));
  if (phase < 0 || phase >= NPH) return fail(c, PF_ERR_ARG, "phase %d out of range", (int)phase);
  if (!ntri || cap < 0 || (cap > 0 && (!ids || !pos))) return fail(c, PF_ERR_ARG, "NULL output or negative cap");
  CKS(join_mu(c));
  const Block &b0 = c->blocks[0];
  const int pbx = (int)(c->box_nx / b0.nx), pby = (int)(c->box_ny / b0.ny), pbz = (int)(c->box_nz / b0.nz);
  // block pointers in box order (blocks of one rank are in block-id order)
  std::vector<const double *> f(c->blocks.size());
  for (const auto &b : c->blocks) {
    const int q = (int)((b.x0 - c->box_x0) / b0.nx + pbx * ((b.y0 - c->box_y0) / b0.ny + pby * ((b.z0 - c->box_z0) / b0.nz)));
    f[q] = field_ptr(b, 0, c->cur, phase) + cell_off(b, 0, 0, 0);
  }
  if (!c->d_mesh_f) CK(cudaMalloc(&c->d_mesh_f, f.size() * sizeof(double *)));
  CK(cudaMemcpyAsync(c->d_mesh_f, f.data(), f.size() * sizeof(double *), cudaMemcpyHostToDevice, c->stream));
  const int64_t nzc = std::min(c->box_nz, c->g.nz - 1 - c->box_z0);   // cube layers
  const bool dev = cap > 0 && is_device_ptr(ids) && is_device_ptr(pos);
  int64_t *d_ids = ids;
  double *d_pos = pos;
  if (cap > 0 && !dev) {  // host output: count first, then stage at most cap triangles
    int64_t total = 0;
    CK(launch_mesh(c->stream, c->d_mesh_f, b0.nx, b0.ny, b0.nz, pbx, pby, pbz, b0.pitch, b0.plane, c->box_nx,
                   c->box_ny, nzc, c->box_x0, c->box_y0, c->box_z0, c->g.nx, c->g.ny, c->zorig, iso, c->p.dx, 0,
                   nullptr, nullptr, &total, &c->mesh_scratch, &c->mesh_scratch_bytes));
    const int64_t nt = std::min(total, cap);
    const size_t need = (size_t)nt * (3 * sizeof(int64_t) + 9 * sizeof(double));
    if (c->mesh_out_bytes < need) {
      if (c->mesh_out) cudaFree(c->mesh_out);
      c->mesh_out = nullptr;
      c->mesh_out_bytes = 0;
      CK(cudaMalloc(&c->mesh_out, need));
      c->mesh_out_bytes = need;
    }
    d_ids = (int64_t *)c->mesh_out;
    d_pos = (double *)(d_ids + 3 * nt);
    cap = nt;
  }
  CK(launch_mesh(c->stream, c->d_mesh_f, b0.nx, b0.ny, b0.nz, pbx, pby, pbz, b0.pitch, b0.plane, c->box_nx, c->box_ny,
                 nzc, c->box_x0, c->box_y0, c->box_z0, c->g.nx, c->g.ny, c->zorig, iso, c->p.dx, cap, d_ids, d_pos,
                 ntri, &c->mesh_scratch, &c->mesh_scratch_bytes));
  if (cap > 0 && !dev) {
    CK(cudaMemcpy(ids, d_ids, (size_t)cap * 3 * sizeof(int64_t), cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(pos, d_pos, (size_t)cap * 9 * sizeof(double), cudaMemcpyDeviceToHost));
  }
  c->launches += cap > 0 ? 2 : 1;
  return PF_OK;
}

pf_status pf_mesh_table(int8_t *out) {
  if (!out) return PF_ERR_ARG;
  mesh_case_table(out);
  return PF_OK;
}

void pf_destroy(pf_ctx *c) {
  if (!c) return;
  cudaSetDevice(c->g.device);
  if (c->stream) cudaStreamSynchronize(c->stream);
  for (auto &b : c->blocks) {
    for (int cp = 0; cp < 3; ++cp) {
      for (int a = 0; a < NPH; ++a) if (b.phi[cp][a]) cudaFree(b.phi[cp][a]);
      for (int q = 0; q < NMU && cp < 2; ++q) if (b.mu[cp][q]) cudaFree(b.mu[cp][q]);
    }
  }
  for (int f = 0; f < 2; ++f) {
    for (int cp = 0; cp < 3; ++cp) {
      if (c->plan[f][cp].d_local) cudaFree(c->plan[f][cp].d_local);
      if (c->plan[f][cp].d_unpack) cudaFree(c->plan[f][cp].d_unpack);
    }
    if (c->d_send[f]) cudaFree(c->d_send[f]);
    if (c->d_recv[f]) cudaFree(c->d_recv[f]);
  }
  slab_free(c);
  if (c->d_tab) cudaFree(c->d_tab);
  if (c->d_tab2) cudaFree(c->d_tab2);
  if (c->d_red) cudaFree(c->d_red);
  if (c->d_step) cudaFree(c->d_step);
  invalidate_graphs(c);
  if (c->d_stage) cudaFree(c->d_stage);
  if (c->d_mesh_f) cudaFree(c->d_mesh_f);
  if (c->mesh_scratch) cudaFree(c->mesh_scratch);
  if (c->mesh_out) cudaFree(c->mesh_out);
  for (auto e : c->ev) cudaEventDestroy(e);
  if (c->cstream) cudaStreamSynchronize(c->cstream);
  if (c->comm_mu) ncclCommDestroy(c->comm_mu);
  if (c->comm) ncclCommDestroy(c->comm);
  if (c->ev_mu_done) cudaEventDestroy(c->ev_mu_done);
  if (c->ev_mu_halo) cudaEventDestroy(c->ev_mu_halo);
  if (c->ev_phi_done) cudaEventDestroy(c->ev_phi_done);
  if (c->ev_phi_halo) cudaEventDestroy(c->ev_phi_halo);
  if (c->ev_copy) cudaEventDestroy(c->ev_copy);
  for (auto e : c->ev_stage) if (e) cudaEventDestroy(e);
  if (c->cstream) cudaStreamDestroy(c->cstream);
  if (c->own_stream && c->stream) cudaStreamDestroy(c->stream);
  cudaGetLastError();
  delete c;
}

}  // extern "C"
