/* pf.h — C ABI of libpf.so, the B200 (sm_100a) explicit time step of the
 * grand-potential phase-field model for ternary eutectic directional
 * solidification (Bauer et al., SC'15, arXiv 1506.01684).
 *
 * One call of pf_step(ctx, 1) is Algorithm 1 of the paper (PAPER.md:158-174,
 * §Phase-field Algorithm):
 *     phi_dst <- phi-kernel(phi_src, mu_src)           Eq. (1)-(2)
 *     phi_dst ghost-layer exchange + boundary handling
 *     mu_dst  <- mu-kernel(mu_src, phi_src, phi_dst)   Eq. (3)-(4)
 *     mu_dst  ghost-layer exchange + boundary handling
 *     swap src <-> dst
 * followed, when enabled, by the moving-window shift.  The
 * problem statement the entry points follow is pf_create(grid, params),
 * pf_init(seed), pf_step(n), pf_read(phi, mu) (BASELINE.json north_star).
 *
 * Conventions
 *  - Fields are IEEE binary64 ("all computations are carried out
 *    in double precision").  Phases a = 0..3 = alpha, beta, gamma, liquid
 *    (N = 4); chemical potentials c = 0,1 (K-1 = 2).
 *  - Host-visible layout of a state (pf_read / pf_write): the rank's local
 *    interior box only, structure of arrays, x fastest:
 *        phi[a*n + (k*ny_l + j)*nx_l + i],  mu[c*n + (k*ny_l + j)*nx_l + i],
 *    n = nx_l*ny_l*nz_l.  Pointers may be host or device memory (detected).
 *  - Boundaries: periodic in x and y, zero-flux (zero-gradient ghosts) in z.
 *  - Every function returns pf_status; no C++ exception crosses the ABI.  After
 *    any error except PF_ERR_IO the context is poisoned: later calls return
 *    PF_ERR_STATE, and
 *    pf_last_error() describes the first failure.  A context is
 *    single-thread-affine.
 *  - Ownership: the context owns every device allocation (fields, halo
 *    buffers, per-plane table, events) and the NCCL communicator it creates.
 *    The caller owns the structs passed to pf_create (copied) and the buffers
 *    passed to pf_read / pf_write.  A borrowed stream must outlive the context.
 */
#ifndef PF_H_
#define PF_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  PF_OK = 0,
  PF_ERR_CONFIG = -1,    /* invalid grid / decomposition / parameters            */
  PF_ERR_NUMERICAL = -2, /* NaN or Inf found by the periodic device check          */
  PF_ERR_CUDA = -3,      /* a CUDA runtime error (message in pf_last_error)        */
  PF_ERR_COMM = -4,      /* an NCCL error                                          */
  PF_ERR_STATE = -5,     /* call out of order (step before init) or after an error */
  PF_ERR_ARG = -6,       /* NULL or out-of-range argument                          */
  PF_ERR_IO = -7         /* checkpoint file error (open/read/write, bad magic,
                            header not matching the grid, truncated body); does
                            NOT poison the context (see pf_save / pf_load)       */
} pf_status;

/* Grid and decomposition (copied by pf_create).  The global nx*ny*nz interior
 * is split into px*py*pz equal blocks (nx % px == 0 etc., else PF_ERR_CONFIG
 * naming the axis).  Block b = ix + px*(iy + py*iz).  Either
 * nranks == 1 (all blocks on this GPU; blocks exchange halos in device memory)
 * or nranks == px*py*pz (block b on rank b, halos over NCCL send/recv). */
typedef struct {
  int64_t nx, ny, nz;
  int32_t px, py, pz;
  int32_t rank, nranks;
  int32_t device;        /* CUDA ordinal of this process's GPU                     */
  uint8_t nccl_id[128];  /* ncclUniqueId from pf_nccl_unique_id() on rank 0,
                            broadcast by the caller (torch.distributed); ignored
                            when nranks == 1                                      */
  void *stream;          /* cudaStream_t to run on, or NULL for a library stream   */
} pf_grid;

/* Model parameters (copied).  Symbols of PAPER.md Eq. (1)-(4); their values
 * are not in the paper (PAPER.md:197 defers to [hoetzer15]); params/v1.json is
 * the builder's PARAMS-v1 set. */
typedef struct {
  double dx, dt, eps;         /* grid spacing, time step, interface parameter eps  */
  double tau[4];              /* relaxation tau_a (Eq. 1)                          */
  double gamma[4][4];         /* pairwise gradient/obstacle coefficient gamma_ab   */
  double gamma3[4];           /* higher-order obstacle coefficient of the triple
                                 that EXCLUDES phase x (x = 3: alpha-beta-gamma)   */
  double delta[4][4];         /* cubic anisotropy strength of pair ab (aniso only) */
  double T_eut, G, v, T0;     /* frozen T(z,t) = T0 + G (z - v t)  */
  double A0[4][2], A1[4][2];  /* parabola curvature A = A0 + A1 (T - T_eut)        */
  double c0[4][2], m[4][2];   /* c-hat = c0 + m (T - T_eut)                        */
  double L[4];                /* driving offset B = L (T - T_eut) / T_eut          */
  double D[4][2];             /* diffusivities (mobility M = sum phi D / 2A)       */
  int32_t aniso;              /* 0: isotropic gradient energy (D3C7); 1: cubic
                                 anisotropy (D3C19 phi stencil)                     */
  int32_t window;             /* 1: moving window along z           */
  double window_frac;         /* shift when the front reaches ceil(frac * NZ)      */
  double window_phi_l;        /* front = highest plane with some phi_l < this      */
  int32_t nan_check_every;    /* check phi/mu for NaN/Inf every k steps (0 = off)  */
  int32_t variant;            /* 0: tiled kernels (default); 1: naive per-cell
                                 kernels (every face evaluated from both cells)     */
  /* initial condition recipe for pf_init */
  int32_t init_kind;          /* 0 voronoi, 1 lamellar, 2 planar                   */
  int32_t init_n_seeds;
  int32_t init_lam_wmin, init_lam_wmax, init_planar_phase;
  int32_t shortcuts;          /* 1: region shortcuts —
                                 a warp of bulk cells (pure phase, identical D3C7
                                 (D3C19 if aniso) neighbourhood) skips the phi
                                 update, whose result is then its input bit for
                                 bit; results identical to shortcuts = 0         */
  double init_layer_height, init_iface_width, init_mu_noise;
  int32_t overlap;            /* communication hiding:
                                 0 (default): the mu^{n+1} halo exchange runs beside
                                   the next phi-sweep (which reads mu at the cell
                                   only) — the paper's best variant;
                                 1: none (Algorithm 1 in order);
                                 2: the phi^{n+1} halo exchange runs beside
                                   mu-sweep-local (the mu update without the
                                   anti-trapping current), then mu-sweep-neighbor
                                   adds its divergence (Algorithm 2's split); the
                                   mu halo is not hidden;
                                 3: both (Algorithm 2);
                                 4: both without Algorithm 2's second pass: the
                                   mu-sweep over the tiles that read no ghost
                                   beside the phi halo, the shell (boundary tiles,
                                   cap planes) after it; the mu halo as in 0.
                                 Results of 2/3 differ from 0/1 by rounding only;
                                 4 equals 0/1 bit for bit. */
  int32_t graph;              /* 1: single-rank runs without per-sweep timing replay
                                 each step as a CUDA graph (one launch per step);
                                 0 (default): launch the kernels one by one, which
                                 keeps the mu halo beside the next phi-sweep and
                                 measured as fast or faster.
                                 Results are identical. */
} pf_params;

/* Run-time information about a context. */
typedef struct {
  int64_t nx_l, ny_l, nz_l;   /* this rank's interior box                          */
  int64_t x0, y0, z0;         /* its global offset                                 */
  int64_t step;               /* time level n of the current state                 */
  int64_t z_origin;           /* moving-window origin (global plane of k = 0)      */
  int64_t shifts;             /* window shifts so far                              */
  int64_t last_front;         /* last front plane seen (-1: none / not computed)   */
  int32_t nblocks_local;
  int32_t timing;             /* 1 if per-sweep timing is enabled                  */
  double ms_phi, ms_mu, ms_halo, ms_other; /* accumulated device time per kernel
                                 family (CUDA events on the launching stream)      */
  int64_t launches;           /* kernels launched by pf_step so far                */
  int64_t phi_launches, mu_launches; /* sweep launches counted in ms_phi / ms_mu   */
  double ms_fused;            /* accumulated device time of the fused kernel       */
  int64_t fused_launches;     /* fused launches counted in ms_fused                */
  int32_t fusion;             /* 1 if pf_set_fusion is on                          */
  int32_t pad_;
} pf_info_t;

typedef struct pf_ctx pf_ctx;

/* Fill out[128] with a fresh ncclUniqueId (call on rank 0 only). */
pf_status pf_nccl_unique_id(uint8_t out[128]);

/* Host-only query of the halo message plan (no GPU needed): for rank g->rank,
 * the number of doubles it sends to (send_counts[r]) and receives from
 * (recv_counts[r]) every rank r in one ghost-layer exchange of `field`
 * (0 = phi, 4 components; 1 = mu, 2 components).  Faces, the 12 edges (the
 * D3C19 stencil) and the 8 corner cells (marching cubes,
 * PAPER.md:249-250) of every block; periodic x/y, zero-flux z.  Both arrays hold
 * g->nranks entries (caller-owned).  Errors: PF_ERR_ARG, PF_ERR_CONFIG. */
pf_status pf_halo_plan(const pf_grid *g, int32_t field, int64_t *send_counts, int64_t *recv_counts);

/* Validate grid and parameters, select the device, allocate fields and
 * buffers, create the communicator (nranks > 1; collective over all ranks).
 * Errors: PF_ERR_CONFIG (divisibility, gamma not symmetric / non-positive,
 * A(T) <= 0 over the initial window's temperatures, dt above the explicit-Euler
 * bound min(dx^2/(6 D_mu), dx^2/(6 D_phi)) of PAPER.md:84-86 — D_mu = D_max
 * A_max/A_min, D_phi = 2 gamma_max T_max/tau_min, reading R29),
 * PF_ERR_ARG, PF_ERR_CUDA, PF_ERR_COMM.  On success *out owns everything. */
pf_status pf_create(const pf_grid *g, const pf_params *p, pf_ctx **out);

/* Deterministic, decomposition-independent initial state from `seed` and the
 * init_* recipe (Voronoi / lamellar / planar solid layer under liquid,
 * PAPER.md:195-197), generated on the device; resets step and z_origin to 0
 * and fills all ghosts. */
pf_status pf_init(pf_ctx *c, uint64_t seed);

/* Load a state (layout above; host or device pointers), fill all ghosts. */
pf_status pf_write(pf_ctx *c, const double *phi, const double *mu);

/* Set the time level n (t = n dt) and the window origin of the current state. */
pf_status pf_set_time(pf_ctx *c, int64_t step, int64_t z_origin);

/* Advance n explicit steps (Algorithm 1 + window).  Blocking: returns after
 * the last step completed on the device.  Errors: PF_ERR_STATE before
 * pf_init/pf_write, PF_ERR_NUMERICAL with step, global cell and field in
 * pf_last_error when the NaN check trips, PF_ERR_CUDA / PF_ERR_COMM.
 * PF_ERR_CONFIG before any work if the temperatures the n steps reach (t up to
 * (step + n) dt, z over the window incl. up to n origin shifts) make some
 * A(T) <= 0 or break the dt bound of pf_create; that rejection does not poison
 * the context (message in pf_last_error). */
pf_status pf_step(pf_ctx *c, int64_t n);

/* Copy the rank's interior state out (layout above; host or device). */
pf_status pf_read(pf_ctx *c, double *phi, double *mu);

/* One step (Algorithm 1) from a host state to a host state:
 * the result equals pf_write(phi_in, mu_in) + pf_step(1) + pf_read(phi_out,
 * mu_out) bit for bit, including the state left on the device (time level
 * n+1, all ghosts filled).  Layout above; the in and out arrays may be the
 * same (in place).  On a context with one block per process, the tiled
 * sweeps and overlap 0 or 1, the block is cut into ~32 z-slabs: the
 * upload of slab s+1, the sweeps of the slabs below it and the download of
 * finished slabs overlap (PCIe is full duplex; pinned host memory reaches its
 * bandwidth); a moving-window shift after the step reads the shifted state
 * once more.  Otherwise it runs those three calls in order.  Does not need a
 * prior pf_init/pf_write.  Blocking.  Errors: PF_ERR_ARG (NULL pointer), as
 * pf_write / pf_step / pf_read. */
pf_status pf_step_io(pf_ctx *c, const double *phi_in, const double *mu_in, double *phi_out, double *mu_out);

/* FP32 checkpoint of the current state (§Input/Output: "the
 * complete simulation state ... four phi values and two mu values per cell ...
 * checkpoints use only single precision").  Collective over the context's
 * ranks; every rank writes its own rows of the one shared file `path`
 * (created / truncated by rank 0).  Format, little endian:
 *     bytes  0..7   magic "PFCP0001"
 *            8..31  u64 NX, NY, NZ (global interior)
 *           32..39  u32 N = 4 phases, u32 K-1 = 2 potentials
 *           40..55  f64 dx, f64 t = step * dt
 *           56..71  u64 step, u64 window origin (global plane of k = 0)
 *     body          binary32, component-major: phi_0..phi_3 then mu_0, mu_1,
 *                   each NX*NY*NZ values x fastest, (k*NY + j)*NX + i
 * Values are the IEEE round-to-nearest-even binary32 casts of the binary64
 * state.  Errors: PF_ERR_STATE before pf_init/pf_write/pf_load, PF_ERR_ARG,
 * PF_ERR_IO (context still usable; a partial file may remain), PF_ERR_CUDA /
 * PF_ERR_COMM. */
pf_status pf_save(pf_ctx *c, const char *path);

/* Restore a checkpoint written by pf_save (any decomposition): the state
 * becomes the binary64 widening of the stored binary32 values (exact), step
 * and window origin come from the header (t is not read back: t = step * dt);
 * all ghosts are filled.  Collective.  The header must match the context
 * (NX, NY, NZ, N, K-1, dx bit for bit) and the body be complete, else
 * PF_ERR_IO with the state untouched; a read failure after the header checks
 * returns PF_ERR_IO and leaves the context uninitialized (pf_step returns
 * PF_ERR_STATE until the next pf_init / pf_write / pf_load). */
pf_status pf_load(pf_ctx *c, const char *path);

/* Marching-cubes interface mesh of phase `phase` (0..3) over this rank's box
 * ("a custom marching cubes algorithm ... generates meshes
 * locally on each block, using the phi values as input.  For each phase, a
 * mesh is generated ... extends to the ghost regions such that the local
 * meshes can be stitched"; the variant is reading R26 of DESIGN.md §2).
 *   Samples at cell centres; cube (i,j,k) has corners (i..i+1, j..j+1,
 *   k..k+1), lower corner (global window index) in this rank's box, x/y
 *   periodic, k <= NZ-2.  A corner is inside when phi > iso.  Cubes are taken
 *   in (k, j, i) order, their triangles in case-table order: the output is
 *   deterministic and identical to a serial sweep of the box.
 *   ids [3*t + v]      int64 global grid-edge id of vertex v of triangle t:
 *                      3*(i + NX*(j + NY*k)) + axis, (i,j,k) the edge's lower
 *                      corner (x, y wrapped), axis 0/1/2 = x/y/z;
 *   pos [9*t + 3*v + q] binary64 vertex position (x, y, z): ((g + 1/2) + s) dx
 *                      along the edge, (g + 1/2) dx across it, g the global
 *                      index (z from the window origin, plus z_origin), s =
 *                      (iso - f0)/(f1 - f0) IEEE-rounded;
 *   triangles are right-handed about the normal pointing out of the phase.
 * At most `cap` triangles are written (cap = 0: count only; ids/pos may then
 * be NULL); *ntri receives the total.  ids/pos are host or device pointers
 * (auto-detected).  Collective only in the sense that every rank meshes its
 * own box.  Errors: PF_ERR_STATE before pf_init/pf_write/pf_load, PF_ERR_ARG
 * (phase out of range, NULL outputs with cap > 0, cap < 0), PF_ERR_CUDA. */
pf_status pf_mesh(pf_ctx *c, int32_t phase, double iso, int64_t cap, int64_t *ids, double *pos, int64_t *ntri);

/* Host-only query (no context, no GPU): the marching-cubes case table pf_mesh
 * uses, out[16*case + 0] = triangle count (<= 5), out[16*case + 1 + 3*t + v] =
 * cube edge of vertex v of triangle t (edges 0-3 along x at (dy,dz) =
 * (e&1, e>>1), 4-7 along y at (dx,dz), 8-11 along z at (dx,dy); corner bit c
 * = dx + 2dy + 4dz of `case` set when inside).  out: 256*16 int8 (caller
 * owned).  Errors: PF_ERR_ARG on NULL. */
pf_status pf_mesh_table(int8_t *out);

/* Enable (1) / disable (0) per-sweep CUDA-event timing; resets the timers. */
pf_status pf_set_timing(pf_ctx *c, int32_t on);

/* Switch the region shortcuts (pf_params.shortcuts, NEXT-1: PAPER.md:281-290,
 * 483-492) on (1) or off (0) for the following steps.  Results are bitwise the
 * same either way (tests/test_gpu_parity.py, test_gpu_trajectories.py); on is
 * faster on every measured block type (profiles/r02_scenarios.md), off is the
 * configuration whose FLOP count per cell is exact.
 * Errors: PF_ERR_ARG (NULL), PF_ERR_STATE after an error. */
pf_status pf_set_shortcuts(pf_ctx *c, int32_t on);

/* Fused steps on (1) or off (0) for the following pf_step calls.  On: within
 * one pf_step(n), n >= 2, the mu-sweep of step k and the phi-sweep of step k+1
 * (Algorithm 1 lines 4 and 1 of consecutive iterations) run
 * as ONE kernel: the phi-sweep reads mu at the cell centre only (D3C1,
 * PAPER.md:176-177), which that kernel has just computed, and both read the
 * same phi^{k+1} tiles — 128 B of HBM traffic per cell and step instead of
 * 176.  Every state the caller (or the moving-window check, the NaN watchdog)
 * sees is a complete time level, and results are bitwise those of fusion off
 * (tests/test_gpu_fused.py).  Applies to the tiled sweeps with overlap 0 / 1
 * and graph = 0, region shortcuts on or off; otherwise pf_step runs the
 * separate sweeps.  Default off, like the region shortcuts (an opt-in speed setting
 * with bitwise the same results): measured at 512^3 the
 * isotropic step is 3 % faster fused, the anisotropic one 19 % slower (its
 * fused kernel is register-bound).
 * on = 1 allocates a third phi copy (4 doubles per cell of the block, ghosts
 * and window slack included); on = 0 releases it.
 * Errors: PF_ERR_ARG (NULL), PF_ERR_STATE after an error, PF_ERR_CUDA if that
 * copy does not fit (fusion stays off; the context stays usable). */
pf_status pf_set_fusion(pf_ctx *c, int32_t on);

pf_status pf_info(pf_ctx *c, pf_info_t *out);

/* Message describing the first error on c (or a create failure when c is
 * NULL); valid until the next call on c. */
const char *pf_last_error(const pf_ctx *c);

/* Release every resource; c may be NULL. */
void pf_destroy(pf_ctx *c);

#ifdef __cplusplus
}
#endif
#endif /* PF_H_ */
