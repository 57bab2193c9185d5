/* pfgen.c — seeded synthetic initial states (shared input generator).
 *
 * This module is the ONLY code shared by the oracle side (tests) and the CUDA
 * side (which receives the state through pf_write).  It holds none of the
 * method's arithmetic (no phi/mu update, no thermodynamics): it only lays out
 * an initial condition, following the recipe of SURVEY.md §8(c) A17 / DESIGN.md
 * §3 for the initial setup of PAPER.md:195-197 ("solid nuclei at the bottom of
 * a liquid filled domain ... created by a Voronoi tesselation").
 *
 * Layout of the output (interior cells only, no ghosts):
 *   phi[a*n + (k*by + j)*bx + i]   a = 0..3  (alpha, beta, gamma, liquid)
 *   mu [c*n + (k*by + j)*bx + i]   c = 0..1
 * with n = bx*by*bz for the requested box [x0,x0+bx) x [y0,y0+by) x [z0,z0+bz)
 * of the global nx*ny*nz domain.  Every value is a pure function of
 * (spec, global cell), so any box decomposition yields identical bits.
 *
 * Random numbers: counter-based splitmix64 (pfgen_rng), keyed by
 * (seed, stream, index).  The CUDA pf_init implements the same generator.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

typedef struct {
  int32_t kind;          /* 0 voronoi, 1 lamellar, 2 planar (one solid phase) */
  int32_t n_seeds;       /* voronoi: number of seeds                          */
  int32_t lam_wmin, lam_wmax; /* lamellar: width range (cells, inclusive)     */
  int32_t planar_phase;  /* planar: which solid phase fills the layer         */
  int32_t pad_;
  double layer_height;   /* solid for z_centre < layer_height (cells)         */
  double iface_width;    /* W of the sine ramp (cells)                        */
  double mu_noise;       /* mu = mu_noise * U(-1,1)                           */
  uint64_t seed;
} pfgen_spec;

enum { STREAM_SEED_X = 1, STREAM_SEED_Y = 2, STREAM_SEED_PHASE = 3,
       STREAM_LAMELLA = 4, STREAM_MU0 = 8 };

static uint64_t mix64(uint64_t z) {
  z += 0x9E3779B97F4A7C15ULL;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}

uint64_t pfgen_rng(uint64_t seed, uint64_t stream, uint64_t idx) {
  return mix64(mix64(seed ^ (stream * 0xD1B54A32D192ED03ULL)) ^ idx);
}

double pfgen_u01(uint64_t seed, uint64_t stream, uint64_t idx) {
  return (double)(pfgen_rng(seed, stream, idx) >> 11) * 0x1.0p-53;
}

/* sine ramp of width W: 0 for d <= -W/2, 1 for d >= W/2 */
double pfgen_ramp(double d, double W) {
  if (d >= 0.5 * W) return 1.0;
  if (d <= -0.5 * W) return 0.0;
  return 0.5 * (1.0 + sin(M_PI * d / W));
}

static double min_image(double d, double n) {
  if (d > 0.5 * n) d -= n;
  else if (d < -0.5 * n) d += n;
  return d;
}

/* Per-column solid composition: phase p1 with weight r, p2 with weight 1-r. */
typedef struct { int p1, p2; double r; } column_mix;

static column_mix voronoi_column(const pfgen_spec *s, const double *sx, const double *sy,
                                 const int *sp, int64_t nx, int64_t ny, int64_t i, int64_t j) {
  column_mix m;
  double x = i + 0.5, y = j + 0.5;
  int best = -1; double bd = 0, brx = 0, bry = 0;
  for (int q = 0; q < s->n_seeds; ++q) {
    double rx = min_image(x - sx[q], (double)nx), ry = min_image(y - sy[q], (double)ny);
    double d = rx * rx + ry * ry;
    if (best < 0 || d < bd) { best = q; bd = d; brx = rx; bry = ry; }
  }
  m.p1 = sp[best]; m.p2 = sp[best]; m.r = 1.0;
  int other = -1; double od = 0, orx = 0, ory = 0;
  for (int q = 0; q < s->n_seeds; ++q) {
    if (sp[q] == sp[best]) continue;
    double rx = min_image(x - sx[q], (double)nx), ry = min_image(y - sy[q], (double)ny);
    double d = rx * rx + ry * ry;
    if (other < 0 || d < od) { other = q; od = d; orx = rx; ory = ry; }
  }
  if (other >= 0) {
    double ex = brx - orx, ey = bry - ory;           /* s2 - s1 as seen from x */
    double sep = sqrt(ex * ex + ey * ey);
    if (sep > 0) {
      double db = (od - bd) / (2.0 * sep);             /* distance to bisector   */
      m.p2 = sp[other];
      m.r = pfgen_ramp(db, s->iface_width);
    }
  }
  return m;
}

/* lamellae along x: widths uniform in [wmin, wmax], phases cycling 0,1,2 */
static int lamella_bounds(const pfgen_spec *s, int64_t nx, int64_t **starts_out) {
  int64_t cap = nx + 2, n = 0, x = 0;
  int64_t *st = (int64_t *)malloc(sizeof(int64_t) * (size_t)(cap + 1));
  while (x < nx) {
    st[n] = x;
    int64_t w = s->lam_wmin + (int64_t)(pfgen_u01(s->seed, STREAM_LAMELLA, (uint64_t)n) *
                                        (double)(s->lam_wmax - s->lam_wmin + 1));
    x += w; ++n;
  }
  st[n] = nx;  /* last lamella truncated at nx */
  *starts_out = st;
  return (int)n;
}

static column_mix lamellar_column(const pfgen_spec *s, const int64_t *st, int nl, int64_t i) {
  column_mix m;
  double x = i + 0.5;
  int l = 0;
  while (l + 1 < nl && st[l + 1] <= i) ++l;
  double dl = x - (double)st[l], dr = (double)st[l + 1] - x;
  int nb = dl < dr ? (l - 1 + nl) % nl : (l + 1) % nl;
  double d = dl < dr ? dl : dr;
  m.p1 = l % 3; m.p2 = nb % 3;
  m.r = (m.p1 == m.p2) ? 1.0 : pfgen_ramp(d, s->iface_width);
  return m;
}

int pfgen_box(const pfgen_spec *s, int64_t nx, int64_t ny, int64_t nz,
              int64_t x0, int64_t y0, int64_t z0, int64_t bx, int64_t by, int64_t bz,
              double *phi, double *mu) {
  if (x0 < 0 || y0 < 0 || z0 < 0 || x0 + bx > nx || y0 + by > ny || z0 + bz > nz) return -1;
  const int64_t n = bx * by * bz;
  double *sx = NULL, *sy = NULL; int *sp = NULL; int64_t *st = NULL; int nl = 0;
  if (s->kind == 0) {
    if (s->n_seeds <= 0) return -2;
    sx = (double *)malloc(sizeof(double) * (size_t)s->n_seeds);
    sy = (double *)malloc(sizeof(double) * (size_t)s->n_seeds);
    sp = (int *)malloc(sizeof(int) * (size_t)s->n_seeds);
    for (int q = 0; q < s->n_seeds; ++q) {
      sx[q] = pfgen_u01(s->seed, STREAM_SEED_X, (uint64_t)q) * (double)nx;
      sy[q] = pfgen_u01(s->seed, STREAM_SEED_Y, (uint64_t)q) * (double)ny;
      int p = (int)(pfgen_u01(s->seed, STREAM_SEED_PHASE, (uint64_t)q) * 3.0);
      sp[q] = p > 2 ? 2 : p;
    }
  } else if (s->kind == 1) {
    nl = lamella_bounds(s, nx, &st);
  }
#pragma omp parallel for collapse(2) schedule(static)
  for (int64_t j = 0; j < by; ++j)
    for (int64_t i = 0; i < bx; ++i) {
      column_mix m;
      if (s->kind == 0) m = voronoi_column(s, sx, sy, sp, nx, ny, x0 + i, y0 + j);
      else if (s->kind == 1) m = lamellar_column(s, st, nl, x0 + i);
      else { m.p1 = m.p2 = s->planar_phase; m.r = 1.0; }
      for (int64_t k = 0; k < bz; ++k) {
        const int64_t kg = z0 + k, loc = (k * by + j) * bx + i;
        const double sol = pfgen_ramp(s->layer_height - (kg + 0.5), s->iface_width);
        double ph[4] = {0, 0, 0, 0};
        ph[m.p1] += sol * m.r;
        ph[m.p2] += sol * (1.0 - m.r);
        ph[3] = 1.0 - sol;
        for (int a = 0; a < 4; ++a) phi[a * n + loc] = ph[a];
        const uint64_t g = (uint64_t)((kg * ny + (y0 + j)) * nx + (x0 + i));
        for (int c = 0; c < 2; ++c)
          mu[c * n + loc] = s->mu_noise == 0.0 ? 0.0
              : s->mu_noise * (2.0 * pfgen_u01(s->seed, STREAM_MU0 + (uint64_t)c, g) - 1.0);
      }
    }
  free(sx); free(sy); free(sp); free(st);
  return 0;
}
