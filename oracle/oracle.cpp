/* oracle.cpp — plain, slow, scalar CPU oracle of one explicit time step of the
 * grand-potential phase-field model of Bauer et al. (arXiv 1506.01684).
 *
 * TEST INFRASTRUCTURE.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load this library.  It shares no
 * code, header, table or constant generator with the CUDA path
 * (paper_1506_01684_b200/csrc); neither includes the other.
 *
 * It loops over the GLOBAL domain (no blocks, no halos, no staging): a ghost
 * neighbour is reached through index functions, periodic in x/y and clamped
 * (zero-gradient) in z (reading R13).
 * Build: -O2 -fno-fast-math -ffp-contract=off (IEEE binary64, no contraction).
 *
 * Notation (§Model, lines 81-146): phases a = 0..3 = alpha, beta,
 * gamma, liquid (N = 4, liquid index L = 3); independent components c = 0,1
 * (K-1 = 2); directions d = x,y,z.  Every function cites the passage it follows
 * and the DESIGN.md reading (R1..R25 = SURVEY.md §8(c) A1..A25) where the
 * paper is silent.
 *
 * All cell and face arithmetic is templated over the scalar type R: R = double
 * is the oracle; R = Counted counts the floating-point operations (+ - * / sqrt
 * = 1 each) on cell data, which gives the algorithmic FLOP/LUP of DESIGN.md §6
 * from the same source.  Quantities that depend on T only (the per-plane
 * values) are plain doubles and are not counted.
 *
 * Pins (tests/test_oracle_pins.py): P1 analytic profile, P2 textbook binary
 * reduction, P3 simplex + active-set enumeration, P4 solute conservation,
 * P5 Fourier decay, P6 permutation symmetry, P7 bulk fixed point, P8 term
 * identities, P10 anti-trapping zeros, P11 single-face anti-trapping
 * properties, P12 undercooling sign, P13 cubic symmetry, P17 window
 * transparency, P18 mirror symmetry, P19 dc/dT source vs the exact solution
 * of a temperature-driven liquid (kappa and m terms), P20 face gradients exact
 * on linear fields (D3C19 tangential averages in J_at and the anisotropic phi
 * faces), P21 homogeneity of the cubic gradient energy.  The coupled
 * multi-phase phi-mu-J_at regime beyond those pins is guarded by the second,
 * independent NumPy coding (oracle/oracle_np.py, tests/test_oracle_second_coding.py)
 * and by tools/oracle_mutants.py (every listed slip fails a pin).
 */
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <vector>

extern "C" {
/* Parameters (PARAMS layout of params/*.json).  gamma3[x] = coefficient of
 * the phase triple that excludes phase x. */
typedef struct {
  double dx, dt, eps;
  double tau[4];
  double gamma[4][4];
  double gamma3[4];
  double delta[4][4];
  double T_eut, G, v, T0;
  double A0[4][2], A1[4][2], c0[4][2], m[4][2], L[4], D[4][2];
  int32_t aniso;
  int32_t pad_;
} or_params;

typedef struct {
  int64_t nx, ny, nz;  /* global interior cells                          */
  int64_t step;        /* time level n of the input state (t_n = n*dt)    */
  int64_t zorig;       /* moving-window origin: global plane of k = 0     */
} or_dims;
}

namespace {

constexpr int N = 4;    /* phases            */
constexpr int NC = 2;   /* K-1 components    */
constexpr int LIQ = 3;  /* liquid index      */

/* ------------------------------------------------------------------------ */
/* Operation counter (only used by or_count_flops).                           */
/* ------------------------------------------------------------------------ */
static thread_local int64_t g_ops = 0;
static thread_local bool g_counting = true;

struct Counted {
  double v;
  Counted() : v(0) {}
  Counted(double x) : v(x) {}
};
inline Counted op(double x) { if (g_counting) ++g_ops; return Counted(x); }
inline Counted operator+(Counted a, Counted b) { return op(a.v + b.v); }
inline Counted operator-(Counted a, Counted b) { return op(a.v - b.v); }
inline Counted operator*(Counted a, Counted b) { return op(a.v * b.v); }
inline Counted operator/(Counted a, Counted b) { return op(a.v / b.v); }
inline bool operator==(Counted a, double b) { return a.v == b; }
inline Counted sqrt(Counted a) { return op(std::sqrt(a.v)); }
inline Counted max0(Counted a) { return a.v > 0.0 ? a : Counted(0.0); }
inline double val(Counted a) { return a.v; }

inline double max0(double a) { return a > 0.0 ? a : 0.0; }
inline double val(double a) { return a; }
using std::sqrt;

struct NoCount {  /* scope guard: stop counting */
  bool saved;
  NoCount() : saved(g_counting) { g_counting = false; }
  ~NoCount() { g_counting = saved; }
};

/* ------------------------------------------------------------------------ */
/* Grid access: periodic x/y, zero-gradient z (reading R13).   */
/* A field accessor returns component a at global (i, j, k); the caller may    */
/* pass unwrapped / unclamped indices.                                         */
/* ------------------------------------------------------------------------ */
inline int64_t wrap(int64_t i, int64_t n) { i %= n; return i < 0 ? i + n : i; }
inline int64_t clampz(int64_t k, int64_t n) { return k < 0 ? 0 : (k >= n ? n - 1 : k); }
inline int64_t ncell(const or_dims &g) { return g.nx * g.ny * g.nz; }
inline int64_t lin(const or_dims &g, int64_t i, int64_t j, int64_t k) {
  return (clampz(k, g.nz) * g.ny + wrap(j, g.ny)) * g.nx + wrap(i, g.nx);
}

struct GlobalField {  /* SoA global array, interior cells only */
  const double *p; const or_dims *g;
  double get(int a, int64_t i, int64_t j, int64_t k) const { return p[a * ncell(*g) + lin(*g, i, j, k)]; }
};
struct BoxField {     /* values on offsets [-2,2]^3 around (ci,cj,ck), ghost rules pre-applied */
  const double *p; int64_t ci, cj, ck;
  static constexpr int R = 2, B = 5, BN = 125;
  double get(int a, int64_t i, int64_t j, int64_t k) const {
    const int64_t l = ((k - ck + R) * B + (j - cj + R)) * B + (i - ci + R);
    return p[a * BN + l];
  }
};

template <class R, class F>
inline void load4(const F &f, int64_t i, int64_t j, int64_t k, R out[N]) {
  for (int a = 0; a < N; ++a) out[a] = R(f.get(a, i, j, k));
}
template <class R, class F>
inline void load2(const F &f, int64_t i, int64_t j, int64_t k, R out[NC]) {
  for (int c = 0; c < NC; ++c) out[c] = R(f.get(c, i, j, k));
}
inline void unit(int d, int64_t &di, int64_t &dj, int64_t &dk) { di = d == 0; dj = d == 1; dk = d == 2; }

/* ------------------------------------------------------------------------ */
/* O1 Temperature: frozen T(z,t) = T0 + G (z - v t), constant per x-y slice    */
/* (reading R12: cell-centre z = (k+zorig+1/2)dx; a     */
/* ghost plane uses its own unclamped z).                                      */
/* ------------------------------------------------------------------------ */
inline double temperature(const or_params &p, const or_dims &g, int64_t k) {
  const double z = ((double)(k + g.zorig) + 0.5) * p.dx;
  const double t = (double)g.step * p.dt;
  return p.T0 + p.G * (z - p.v * t);
}

/* ------------------------------------------------------------------------ */
/* O2 Thermodynamics: parabolic grand potentials (PAPER.md:108-111, 278-279;   */
/* SPEC.md:154-162; reading R7: A, c-hat linear in Theta = T - T_eut).         */
/* ------------------------------------------------------------------------ */
inline double A_of(const or_params &p, int a, int c, double T) { return p.A0[a][c] + p.A1[a][c] * (T - p.T_eut); }
inline double chat_of(const or_params &p, int a, int c, double T) { return p.c0[a][c] + p.m[a][c] * (T - p.T_eut); }
inline double B_of(const or_params &p, int a, double T) { return p.L[a] * (T - p.T_eut) / p.T_eut; }
/* c_c^a(mu,T) = mu_c / (2 A_c^a) + chat_c^a */
template <class R> inline R conc(const or_params &p, int a, int c, R mu_c, double T) {
  return mu_c / R(2.0 * A_of(p, a, c, T)) + R(chat_of(p, a, c, T));
}
/* psi_a(mu,T) = -sum_c [ mu_c^2/(4 A_c^a) + mu_c chat_c^a ] + B^a(T) */
template <class R> inline R psi(const or_params &p, int a, const R mu[NC], double T) {
  R s = R(0.0);
  for (int c = 0; c < NC; ++c)
    s = s + (mu[c] * mu[c] / R(4.0 * A_of(p, a, c, T)) + mu[c] * R(chat_of(p, a, c, T)));
  return R(B_of(p, a, T)) - s;
}
/* h_a = phi_a^2 / sum_b phi_b^2 (PAPER.md:135 [moelans2011]; reading R6) */
template <class R> inline void interp_h(const R ph[N], R h[N]) {
  R S = ph[0] * ph[0];
  for (int b = 1; b < N; ++b) S = S + ph[b] * ph[b];
  for (int a = 0; a < N; ++a) h[a] = ph[a] * ph[a] / S;
}

/* ------------------------------------------------------------------------ */
/* Gradient energy a = sum_{a<b} gamma_ab a_c(q_ab)^2 |q_ab|^2,                */
/* q_ab = phi_a grad phi_b - phi_b grad phi_a (reading R3);       */
/* e(q) and g(q) = de/dq.  a_c = 1 - delta(3-4Q4/|q|^4) */
/* ------------------------------------------------------------------------ */
/* Cubic anisotropy a_c depends on q/|q| only, so e is homogeneous of degree 2
 * and g of degree 1 in q.  Both are evaluated on u = q 2^-s, max|u_d| in
 * [1/2, 1) (s from frexp), and scaled back by 2^(2s) / 2^s: a power-of-two
 * scaling is exact, so in the normal range the result has the bits of the
 * unscaled formula, and q^6 no longer under- or overflows for tiny or huge
 * |q| (g(q) -> 0 continuously as q -> 0). */
inline double ldexp_r(double x, int s) { return std::ldexp(x, s); }
inline Counted ldexp_r(Counted x, int s) { return Counted(std::ldexp(x.v, s)); }  /* exact: not a FLOP */
template <class R> inline int pow2_scale(const R q[3]) {
  const double m = std::max(std::fabs(val(q[0])), std::max(std::fabs(val(q[1])), std::fabs(val(q[2]))));
  int s = 0;
  std::frexp(m, &s);
  return s;
}
template <class R> inline R pair_energy(const or_params &p, int a, int b, const R q_[3]) {
  if (q_[0] == 0.0 && q_[1] == 0.0 && q_[2] == 0.0) return R(0.0);
  const int s = p.aniso ? pow2_scale(q_) : 0;
  R q[3];
  for (int d = 0; d < 3; ++d) q[d] = ldexp_r(q_[d], -s);
  const R q2 = q[0] * q[0] + q[1] * q[1] + q[2] * q[2];
  R ac = R(1.0);
  if (p.aniso) {
    const R Q4 = q[0] * q[0] * q[0] * q[0] + q[1] * q[1] * q[1] * q[1] + q[2] * q[2] * q[2] * q[2];
    ac = R(1.0) - R(p.delta[a][b]) * (R(3.0) - R(4.0) * Q4 / (q2 * q2));
  }
  return ldexp_r(R(p.gamma[a][b]) * ac * ac * q2, 2 * s);
}
/* Components d in [d0, d1) of g_ab(q) (the face fluxes need only the normal
 * component d, the centre term all three). */
template <class R> inline void pair_grad_range(const or_params &p, int a, int b, const R q_[3], R gq[3], int d0, int d1) {
  /* e = gamma |q|^2  ->  g = 2 gamma q; also for a pair without anisotropy
     (delta_ab = 0: a_c = 1 identically, reading R3), so a model with cubic
     anisotropy on some pairs only is counted with the others isotropic */
  if (!p.aniso || p.delta[a][b] == 0.0) {
    for (int d = d0; d < d1; ++d) gq[d] = R(2.0 * p.gamma[a][b]) * q_[d];
    return;
  }
  if (q_[0] == 0.0 && q_[1] == 0.0 && q_[2] == 0.0) {  /* g(0) = 0 */
    for (int d = d0; d < d1; ++d) gq[d] = R(0.0);
    return;
  }
  const int s = pow2_scale(q_);
  R q[3];
  for (int d = 0; d < 3; ++d) q[d] = ldexp_r(q_[d], -s);
  const R q2 = q[0] * q[0] + q[1] * q[1] + q[2] * q[2];
  /* d a_c / d q_d = 16 delta (q_d^3/|q|^4 - Q4 q_d/|q|^6);
     g_d = 2 gamma a_c ( |q|^2 d a_c/d q_d + a_c q_d ) */
  const R Q4 = q[0] * q[0] * q[0] * q[0] + q[1] * q[1] * q[1] * q[1] + q[2] * q[2] * q[2] * q[2];
  const R q4 = q2 * q2;
  const R ac = R(1.0) - R(p.delta[a][b]) * (R(3.0) - R(4.0) * Q4 / q4);
  for (int d = d0; d < d1; ++d) {
    const R dac = R(16.0 * p.delta[a][b]) * (q[d] * q[d] * q[d] / q4 - Q4 * q[d] / (q4 * q2));
    gq[d] = ldexp_r(R(2.0 * p.gamma[a][b]) * ac * (q2 * dac + ac * q[d]), s);
  }
}
template <class R> inline void pair_grad(const or_params &p, int a, int b, const R q[3], R gq[3]) {
  pair_grad_range(p, a, b, q, gq, 0, 3);
}

/* O4.7 multi-obstacle potential (reading
 * R5: pairwise 16/pi^2 term + higher-order triple term, north_star). */
inline int triple_other(int a, int x, int which) {  /* the two phases != a, != x */
  int r[2], n = 0;
  for (int b = 0; b < N; ++b) if (b != a && b != x) r[n++] = b;
  return r[which];
}
template <class R> inline R omega(const or_params &p, const R ph[N]) {
  R w = R(0.0);
  for (int a = 0; a < N; ++a)
    for (int b = a + 1; b < N; ++b) w = w + R(16.0 / (M_PI * M_PI) * p.gamma[a][b]) * ph[a] * ph[b];
  for (int x = 0; x < N; ++x) {  /* triple excluding x */
    R t = R(p.gamma3[x]);
    for (int b = 0; b < N; ++b) if (b != x) t = t * ph[b];
    w = w + t;
  }
  return w;
}
template <class R> inline R domega(const or_params &p, const R ph[N], int a) {
  R s = R(0.0);
  for (int b = 0; b < N; ++b)
    if (b != a) s = s + R(16.0 / (M_PI * M_PI) * p.gamma[a][b]) * ph[b];
  for (int x = 0; x < N; ++x) {
    if (x == a) continue;  /* the triples containing a exclude some x != a */
    const int b = triple_other(a, x, 0), e = triple_other(a, x, 1);
    s = s + R(p.gamma3[x]) * ph[b] * ph[e];
  }
  return s;
}

/* O4.8 driving force d psi / d phi_a = sum_b psi_b dh_b/dphi_a
 *      = (2 phi_a / S)(psi_a - psibar), psibar = sum_b h_b psi_b,
 *      S and psibar formed once per cell */
template <class R> inline void dpsi_dphi_all(const R ph[N], const R ps[N], R out[N]) {
  R S = ph[0] * ph[0];
  for (int b = 1; b < N; ++b) S = S + ph[b] * ph[b];
  R pbar = R(0.0);
  for (int b = 0; b < N; ++b) pbar = pbar + ph[b] * ph[b] / S * ps[b];
  for (int a = 0; a < N; ++a) out[a] = R(2.0) * ph[a] / S * (ps[a] - pbar);
}

/* O4.1 centre gradients (D3C7 central differences) of all phases */
template <class R, class F>
inline void centre_grad(const or_params &p, const F &phi, int64_t i, int64_t j, int64_t k, R gr[N][3]) {
  for (int d = 0; d < 3; ++d) {
    int64_t di, dj, dk; unit(d, di, dj, dk);
    R lo[N], hi[N];
    load4(phi, i - di, j - dj, k - dk, lo);
    load4(phi, i + di, j + dj, k + dk, hi);
    for (int a = 0; a < N; ++a) gr[a][d] = (hi[a] - lo[a]) / R(2.0 * p.dx);
  }
}

/* O4.5 phi face flux between cell lo and hi = lo + e_d:
 *   phibar = (phi(lo)+phi(hi))/2; grad_f: normal 2-point difference, tangential
 *   = mean of the two centre gradients (anisotropic only; reading R4, D3C19);
 *   j_a = (d a / d grad phi_a)_d = -sum_{b != a} g_ab,d(q^f_ab) phibar_b.
 * This is the staggered quantity the paper buffers. */
template <class R>
inline void phi_face(const or_params &p, const R plo[N], const R phi_[N],
                     const R glo[N][3], const R ghi[N][3], int d, R jf[N]) {
  R pb[N], gf[N][3];
  for (int a = 0; a < N; ++a) {
    pb[a] = (plo[a] + phi_[a]) / R(2.0);
    for (int e = 0; e < 3; ++e) {
      if (e == d) gf[a][e] = (phi_[a] - plo[a]) / R(p.dx);
      else if (p.aniso) gf[a][e] = (glo[a][e] + ghi[a][e]) / R(2.0);
      else gf[a][e] = R(0.0);  /* isotropic g_d depends on q_d only */
    }
  }
  for (int a = 0; a < N; ++a) jf[a] = R(0.0);
  for (int a = 0; a < N; ++a)
    for (int b = a + 1; b < N; ++b) {
      R q[3], gq[3];
      if (p.aniso) {
        for (int e = 0; e < 3; ++e) q[e] = pb[a] * gf[b][e] - pb[b] * gf[a][e];
        pair_grad_range(p, a, b, q, gq, d, d + 1);   /* the flux needs g_d only */
      } else {  /* isotropic: only the normal component of q and g is needed */
        gq[d] = R(2.0 * p.gamma[a][b]) * (pb[a] * gf[b][d] - pb[b] * gf[a][d]);
      }
      /* d e_ab / d grad phi_a = -phibar_b g ;  d e_ab / d grad phi_b = +phibar_a g */
      jf[a] = jf[a] - gq[d] * pb[b];
      jf[b] = jf[b] + gq[d] * pb[a];
    }
}

/* O4.11 Euclidean projection onto the Gibbs simplex {sum phi = 1, phi >= 0}
 * (reading R14):
 * sort descending, rho = max{j : u_j - (sum_{r<=j} u_r - 1)/j > 0},
 * theta = (sum_{r<=rho} u_r - 1)/rho, phi = max(x - theta, 0). */
template <class R> inline void project_simplex(const R x[N], R out[N]) {
  R u[N];
  for (int a = 0; a < N; ++a) u[a] = x[a];
  std::sort(u, u + N, [](R l, R r) { return val(r) < val(l); });
  R cum = R(0.0), theta = R(0.0);
  for (int jdx = 0; jdx < N; ++jdx) {
    cum = cum + u[jdx];
    const R t = (cum - R(1.0)) / R((double)(jdx + 1));
    if (val(u[jdx]) - val(t) > 0.0) theta = t;
  }
  for (int a = 0; a < N; ++a) out[a] = max0(x[a] - theta);
}

/* O4 phi-sweep at one cell: Eq. (1)-(2), sign of Eq. (1)
 * read as minus (reading R1), Lagrange mean over all N phases (R2). */
template <class R, class F>
void phi_cell(const or_params &p, const or_dims &g, const F &phi, const F &mu,
              int64_t i, int64_t j, int64_t k, R out[N], bool count_faces = true) {
  const double T = temperature(p, g, k);
  R ph[N], m[NC], gc[N][3];
  load4(phi, i, j, k, ph);
  load2(mu, i, j, k, m);
  centre_grad(p, phi, i, j, k, gc);                               /* O4.1 */

  /* O4.2-4: d a / d phi_a = sum_{b != a} g_ab(q_ab) . grad phi_b */
  R dadphi[N];
  for (int a = 0; a < N; ++a) dadphi[a] = R(0.0);
  for (int a = 0; a < N; ++a)
    for (int b = a + 1; b < N; ++b) {
      R q[3], gq[3];
      for (int d = 0; d < 3; ++d) q[d] = ph[a] * gc[b][d] - ph[b] * gc[a][d];
      pair_grad(p, a, b, q, gq);
      for (int d = 0; d < 3; ++d) {
        dadphi[a] = dadphi[a] + gq[d] * gc[b][d];   /* d q_ab / d phi_a = grad phi_b  */
        dadphi[b] = dadphi[b] - gq[d] * gc[a][d];   /* d q_ab / d phi_b = -grad phi_a */
      }
    }

  /* O4.5-6: divergence of the face fluxes (each face evaluated from both
     cells with identical operands, so the divergence telescopes exactly) */
  R div[N];
  for (int a = 0; a < N; ++a) div[a] = R(0.0);
  {
    const bool saved = g_counting;
    if (!count_faces) g_counting = false;
    for (int d = 0; d < 3; ++d) {
      int64_t di, dj, dk; unit(d, di, dj, dk);
      R pl[N], pu[N], gl[N][3], gu[N][3], jm[N], jp[N];
      for (int a = 0; a < N; ++a) for (int e = 0; e < 3; ++e) gl[a][e] = gu[a][e] = R(0.0);
      load4(phi, i - di, j - dj, k - dk, pl);
      load4(phi, i + di, j + dj, k + dk, pu);
      if (p.aniso) {
        NoCount nc;  /* neighbours' centre gradients: charged once per cell */
        centre_grad(p, phi, i - di, j - dj, k - dk, gl);
        centre_grad(p, phi, i + di, j + dj, k + dk, gu);
      }
      phi_face(p, pl, ph, gl, gc, d, jm);   /* face (c - e_d, c) */
      phi_face(p, ph, pu, gc, gu, d, jp);   /* face (c, c + e_d) */
      for (int a = 0; a < N; ++a) div[a] = div[a] + (jp[a] - jm[a]) / R(p.dx);
    }
    g_counting = saved;
  }

  /* O4.7-9: rhs_a = eps T (da/dphi_a - div_a) + (T/eps) domega_a + dpsi_a */
  R ps[N], dps[N], rhs[N];
  for (int a = 0; a < N; ++a) ps[a] = psi(p, a, m, T);
  dpsi_dphi_all(ph, ps, dps);
  for (int a = 0; a < N; ++a)
    rhs[a] = R(p.eps * T) * (dadphi[a] - div[a]) + R(T / p.eps) * domega(p, ph, a) + dps[a];

  /* O4.10: explicit Euler of Eq. (1) (minus sign), mean over all N phases */
  R mean = R(0.0);
  for (int a = 0; a < N; ++a) mean = mean + rhs[a];
  mean = mean / R((double)N);
  R star[N];
  for (int a = 0; a < N; ++a) star[a] = ph[a] - R(p.dt / (p.tau[a] * p.eps)) * (rhs[a] - mean);

  project_simplex(star, out);                                     /* O4.11 */
}

/* ------------------------------------------------------------------------ */
/* O5 mu-sweep (Eq. (3)-(4); readings R8-R11).              */
/* ------------------------------------------------------------------------ */
template <class R> struct MuCellQ {  /* per-cell quantities */
  R M[NC];            /* mobility sum_a phi^n_a D_c^a / (2 A_c^a(T))    (R11) */
  R cc[N][NC];        /* c_c^a(mu^n, T)                                       */
  R dphi[N];          /* phi^{n+1}_a - phi^n_a                                */
  R pn[N];            /* phi^{n+1}                                            */
  R po[N];            /* phi^n                                                */
  R gn[N][3];         /* centre gradient of phi^{n+1}                         */
  R mu[NC];           /* mu^n                                                 */
};

template <class R, class FO, class FN, class FM>
void mu_cell_q(const or_params &p, const or_dims &g, const FO &phi_old, const FN &phi_new,
               const FM &mu, int64_t i, int64_t j, int64_t k, MuCellQ<R> &q) {
  const double T = temperature(p, g, k);  /* the cell's own plane (unclamped) */
  load4(phi_old, i, j, k, q.po);
  load4(phi_new, i, j, k, q.pn);
  load2(mu, i, j, k, q.mu);
  for (int c = 0; c < NC; ++c) {
    q.M[c] = R(0.0);
    for (int a = 0; a < N; ++a) q.M[c] = q.M[c] + q.po[a] * R(p.D[a][c] / (2.0 * A_of(p, a, c, T)));
  }
  for (int a = 0; a < N; ++a) {
    q.dphi[a] = q.pn[a] - q.po[a];
    for (int c = 0; c < NC; ++c) q.cc[a][c] = conc(p, a, c, q.mu[c], T);
  }
  centre_grad(p, phi_new, i, j, k, q.gn);
}

/* Face value of (M grad mu)_c and (J_at)_c at the face (lo, hi = lo + e_d).
 * Diffusive part: arithmetic-mean mobility times the 2-point difference (R11).
 * Anti-trapping part, Eq. (4) with g_a = phi_a (reading R10): face values by
 * arithmetic averaging, normals from the face gradient of phi^{n+1}, exact-zero
 * guards ("testing critical subexpressions for zeros"). */
template <class R>
void mu_face(const or_params &p, const MuCellQ<R> &lo, const MuCellQ<R> &hi, int d, R F[NC], R J[NC]) {
  for (int c = 0; c < NC; ++c)
    F[c] = (lo.M[c] + hi.M[c]) / R(2.0) * (hi.mu[c] - lo.mu[c]) / R(p.dx);
  R pb[N], gf[N][3];
  for (int a = 0; a < N; ++a) {
    pb[a] = (lo.pn[a] + hi.pn[a]) / R(2.0);
    for (int e = 0; e < 3; ++e)
      gf[a][e] = (e == d) ? (hi.pn[a] - lo.pn[a]) / R(p.dx) : (lo.gn[a][e] + hi.gn[a][e]) / R(2.0);
  }
  R S = pb[0] * pb[0];
  for (int b = 1; b < N; ++b) S = S + pb[b] * pb[b];
  const R hl = pb[LIQ] * pb[LIQ] / S;
  const R gl2 = gf[LIQ][0] * gf[LIQ][0] + gf[LIQ][1] * gf[LIQ][1] + gf[LIQ][2] * gf[LIQ][2];
  R nl[3];   /* liquid normal, once per face (only used when gl2 != 0) */
  if (!(gl2 == 0.0)) {
    const R nl_abs = sqrt(gl2);
    for (int e = 0; e < 3; ++e) nl[e] = gf[LIQ][e] / nl_abs;
  }
  for (int c = 0; c < NC; ++c) J[c] = R(0.0);
  for (int a = 0; a < N; ++a) {
    if (a == LIQ) continue;  /* sum over solids only (reading R24) */
    const R pd = (lo.dphi[a] + hi.dphi[a]) / R(2.0) / R(p.dt);   /* face d phi_a / dt */
    const R pal = pb[a] * pb[LIQ];
    const R ga2 = gf[a][0] * gf[a][0] + gf[a][1] * gf[a][1] + gf[a][2] * gf[a][2];
    if (pal == 0.0 || ga2 == 0.0 || gl2 == 0.0 || pd == 0.0) continue;
    const R na_abs = sqrt(ga2);
    R na[3];
    for (int e = 0; e < 3; ++e) na[e] = gf[a][e] / na_abs;
    R dot = R(0.0);
    for (int e = 0; e < 3; ++e) dot = dot + na[e] * nl[e];
    /* (pi eps / 4) g_a h_l / sqrt(phi_a phi_l) dphi_a/dt (n_a . n_l) n_a,d */
    const R w = R(M_PI * p.eps / 4.0) * (pb[a] * hl / sqrt(pal)) * pd * dot * na[d];
    for (int c = 0; c < NC; ++c) {
      /* (c^l - c^a) averaged over the two cells */
      const R dc = ((lo.cc[LIQ][c] - lo.cc[a][c]) + (hi.cc[LIQ][c] - hi.cc[a][c])) / R(2.0);
      J[c] = J[c] + w * dc;
    }
  }
}

template <class R, class FO, class FN, class FM>
void mu_cell(const or_params &p, const or_dims &g, const FO &phi_old, const FN &phi_new, const FM &mu,
             int64_t i, int64_t j, int64_t k, R out[NC], bool count_faces = true) {
  const double T = temperature(p, g, k);
  MuCellQ<R> q;
  mu_cell_q(p, g, phi_old, phi_new, mu, i, j, k, q);
  R hn[N], ho[N];
  interp_h(q.po, ho);
  interp_h(q.pn, hn);

  R div[NC] = {R(0.0), R(0.0)};
  {
    const bool saved = g_counting;
    if (!count_faces) g_counting = false;
    for (int d = 0; d < 3; ++d) {
      int64_t di, dj, dk; unit(d, di, dj, dk);
      MuCellQ<R> qm, qp;
      { NoCount nc; mu_cell_q(p, g, phi_old, phi_new, mu, i - di, j - dj, k - dk, qm); }
      { NoCount nc; mu_cell_q(p, g, phi_old, phi_new, mu, i + di, j + dj, k + dk, qp); }
      R Fm[NC], Jm[NC], Fp[NC], Jp[NC];
      mu_face(p, qm, q, d, Fm, Jm);
      mu_face(p, q, qp, d, Fp, Jp);
      for (int c = 0; c < NC; ++c) div[c] = div[c] + ((Fp[c] - Jp[c]) - (Fm[c] - Jm[c])) / R(p.dx);
    }
    g_counting = saved;
  }

  const double Tdot = -p.G * p.v;  /* dT/dt of the frozen temperature */
  for (int c = 0; c < NC; ++c) {
    /* O5.3 chi_c = sum_a h^{n+1}_a / (2 A_c^a) — susceptibility (R8) */
    R chi = R(0.0);
    for (int a = 0; a < N; ++a) chi = chi + hn[a] / R(2.0 * A_of(p, a, c, T));
    /* O5.4 s_c = -sum_a c_c^a(mu^n) (h^{n+1}_a - h^n_a) / dt  (R8) */
    R s = R(0.0);
    for (int a = 0; a < N; ++a) s = s - q.cc[a][c] * (hn[a] - ho[a]) / R(p.dt);
    /* O5.5 dc/dT = sum_a h^{n+1}_a (m_c^a - mu_c 2 A1_c^a / (2 A_c^a)^2) */
    R dcdT = R(0.0);
    for (int a = 0; a < N; ++a) {
      const double twoA = 2.0 * A_of(p, a, c, T);
      dcdT = dcdT + hn[a] * (R(p.m[a][c]) - q.mu[c] * R(2.0 * p.A1[a][c] / (twoA * twoA)));
    }
    /* O5.9 mu^{n+1} = mu^n + dt/chi [ s - dc/dT dT/dt + div(M grad mu - J_at) ] (Eq. 3) */
    out[c] = q.mu[c] + R(p.dt) / chi * (s - dcdT * R(Tdot) + div[c]);
  }
}

}  // namespace

/* ========================================================================== */
/* C ABI (consumed by tests/ through oracle/oracle.py)                         */
/* ========================================================================== */
extern "C" {

/* O4 over the whole domain: phi_out = phi-sweep(phi^n, mu^n). */
int or_phi_sweep(const or_params *p, const or_dims *g, const double *phi, const double *mu, double *phi_out) {
  const int64_t n = ncell(*g);
  const GlobalField F{phi, g}, M{mu, g};
#pragma omp parallel for schedule(static)
  for (int64_t k = 0; k < g->nz; ++k)
    for (int64_t j = 0; j < g->ny; ++j)
      for (int64_t i = 0; i < g->nx; ++i) {
        double o[N];
        phi_cell<double>(*p, *g, F, M, i, j, k, o);
        const int64_t c = lin(*g, i, j, k);
        for (int a = 0; a < N; ++a) phi_out[a * n + c] = o[a];
      }
  return 0;
}

/* O5 over the whole domain: mu_out = mu-sweep(mu^n, phi^n, phi^{n+1}). */
int or_mu_sweep(const or_params *p, const or_dims *g, const double *phi_old, const double *phi_new,
                const double *mu, double *mu_out) {
  const int64_t n = ncell(*g);
  const GlobalField FO{phi_old, g}, FN{phi_new, g}, M{mu, g};
#pragma omp parallel for schedule(static)
  for (int64_t k = 0; k < g->nz; ++k)
    for (int64_t j = 0; j < g->ny; ++j)
      for (int64_t i = 0; i < g->nx; ++i) {
        double o[NC];
        mu_cell<double>(*p, *g, FO, FN, M, i, j, k, o);
        const int64_t c = lin(*g, i, j, k);
        for (int q = 0; q < NC; ++q) mu_out[q * n + c] = o[q];
      }
  return 0;
}

/* Highest plane k with some phi_l < thr, or -1 (O7 front, reading R16). */
int64_t or_front(const or_dims *g, double thr, const double *phi) {
  const int64_t n = ncell(*g), plane = g->nx * g->ny;
  int64_t front = -1;
  for (int64_t k = 0; k < g->nz; ++k)
    for (int64_t c = 0; c < plane; ++c)
      if (phi[LIQ * n + k * plane + c] < thr) { front = k; break; }
  return front;
}

/* O7 moving window (reading R16).  If the front reaches
 * ceil(frac * nz): drop plane 0, move every plane down one, fill the top plane
 * with phi = e_l, mu = 0, return 1 (caller increments z_origin); else 0. */
int or_window(const or_dims *g, double frac, double front_phi_l, double *phi, double *mu) {
  const int64_t n = ncell(*g), plane = g->nx * g->ny;
  const int64_t front = or_front(g, front_phi_l, phi);
  const int64_t trig = (int64_t)std::ceil(frac * (double)g->nz);
  if (front < trig) return 0;
  for (int a = 0; a < N; ++a) {
    std::memmove(phi + a * n, phi + a * n + plane, sizeof(double) * (size_t)(n - plane));
    for (int64_t c = 0; c < plane; ++c) phi[a * n + n - plane + c] = (a == LIQ) ? 1.0 : 0.0;
  }
  for (int c = 0; c < NC; ++c) {
    std::memmove(mu + c * n, mu + c * n + plane, sizeof(double) * (size_t)(n - plane));
    for (int64_t q = 0; q < plane; ++q) mu[c * n + n - plane + q] = 0.0;
  }
  return 1;
}

/* One-step map (O4 then O5) at a list of cells given by global linear index
 * c = (k*ny + j)*nx + i.  phi^{n+1} is recomputed cell by cell on the
 * 2-neighbourhood the mu update needs.  phi_out[a*ncells + s], mu_out[c*ncells + s]. */
int or_step_cells(const or_params *p, const or_dims *g, const double *phi, const double *mu,
                  int64_t ncells, const int64_t *cells, double *phi_out, double *mu_out) {
  const GlobalField F{phi, g}, M{mu, g};
#pragma omp parallel for schedule(dynamic, 1)
  for (int64_t s = 0; s < ncells; ++s) {
    const int64_t c = cells[s];
    const int64_t i = c % g->nx, j = (c / g->nx) % g->ny, k = c / (g->nx * g->ny);
    std::vector<double> box(N * BoxField::BN, NAN);
    for (int64_t dz = -2; dz <= 2; ++dz)
      for (int64_t dy = -2; dy <= 2; ++dy)
        for (int64_t dx = -2; dx <= 2; ++dx) {
          if (std::llabs(dx) + std::llabs(dy) + std::llabs(dz) > 2) continue;
          double o[N];  /* ghost cells are copies of the wrapped / clamped cell */
          phi_cell<double>(*p, *g, F, M, wrap(i + dx, g->nx), wrap(j + dy, g->ny), clampz(k + dz, g->nz), o);
          const int64_t l = ((dz + 2) * 5 + (dy + 2)) * 5 + (dx + 2);
          for (int a = 0; a < N; ++a) box[a * BoxField::BN + l] = o[a];
        }
    const BoxField FN{box.data(), i, j, k};
    double mo[NC];
    mu_cell<double>(*p, *g, F, FN, M, i, j, k, mo);
    for (int a = 0; a < N; ++a) phi_out[a * ncells + s] = FN.get(a, i, j, k);
    for (int q = 0; q < NC; ++q) mu_out[q * ncells + s] = mo[q];
  }
  return 0;
}

/* ---- term-level entry points for the pins (P8, P11) ---------------------- */
double or_psi(const or_params *p, int a, const double mu[2], double T) { return psi<double>(*p, a, mu, T); }
double or_conc(const or_params *p, int a, int c, double mu_c, double T) { return conc<double>(*p, a, c, mu_c, T); }
void or_interp_h(const double ph[4], double h[4]) { interp_h<double>(ph, h); }
double or_omega(const or_params *p, const double ph[4]) { return omega<double>(*p, ph); }
double or_domega(const or_params *p, const double ph[4], int a) { return domega<double>(*p, ph, a); }
double or_dpsi_dphi(const or_params *p, const double ph[4], const double mu[2], double T, int a) {
  double ps[N], out[N];
  for (int b = 0; b < N; ++b) ps[b] = psi<double>(*p, b, mu, T);
  dpsi_dphi_all<double>(ph, ps, out);
  return out[a];
}
double or_pair_energy(const or_params *p, int a, int b, const double q[3]) { return pair_energy<double>(*p, a, b, q); }
void or_pair_grad(const or_params *p, int a, int b, const double q[3], double gq[3]) { pair_grad<double>(*p, a, b, q, gq); }
void or_project(const double x[4], double out[4]) { project_simplex<double>(x, out); }

/* phi face flux j_a (O4.5) between global cell (i,j,k) and (i,j,k)+e_d, with
 * both cells' centre gradients (the anisotropic tangential components). */
int or_phi_face(const or_params *p, const or_dims *g, const double *phi, int64_t i, int64_t j, int64_t k,
                int d, double jf[4]) {
  const GlobalField F{phi, g};
  int64_t di, dj, dk; unit(d, di, dj, dk);
  double lo[N], hi[N], gl[N][3], gh[N][3];
  load4(F, i, j, k, lo);
  load4(F, i + di, j + dj, k + dk, hi);
  centre_grad(*p, F, i, j, k, gl);
  centre_grad(*p, F, i + di, j + dj, k + dk, gh);
  phi_face<double>(*p, lo, hi, gl, gh, d, jf);
  return 0;
}

/* Face (M grad mu) and J_at between global cell (i,j,k) and (i,j,k)+e_d. */
int or_mu_face(const or_params *p, const or_dims *g, const double *phi_old, const double *phi_new,
               const double *mu, int64_t i, int64_t j, int64_t k, int d, double F[2], double J[2]) {
  const GlobalField FO{phi_old, g}, FN{phi_new, g}, M{mu, g};
  int64_t di, dj, dk; unit(d, di, dj, dk);
  MuCellQ<double> lo, hi;
  mu_cell_q(*p, *g, FO, FN, M, i, j, k, lo);
  mu_cell_q(*p, *g, FO, FN, M, i + di, j + dj, k + dk, hi);
  mu_face(*p, lo, hi, d, F, J);
  return 0;
}

/* Algorithmic FLOP counts per cell update: + - * / sqrt = 1,
 * each face charged once (3 per cell), per-cell quantities charged once,
 * T-only (per-plane) values free, no shortcuts.  Evaluated
 * on a generic 3^3 state with every phase present and every guard open.
 * out[0] = phi cell part, out[1] = phi face, out[2] = mu cell part, out[3] = mu
 * face; out[4] = phi total, out[5] = mu total. */
int or_count_flops(const or_params *p, int64_t out[6]) {
  const or_dims g = {3, 3, 3, 0, 0};
  const int64_t n = 27;
  std::vector<double> po(4 * n), pn(4 * n), mu(2 * n);
  for (int64_t c = 0; c < n; ++c) {
    double w[4], s = 0;
    for (int a = 0; a < 4; ++a) { w[a] = 1.0 + 0.37 * a + 0.11 * (double)((c * (a + 3)) % 7); s += w[a]; }
    for (int a = 0; a < 4; ++a) { po[a * n + c] = w[a] / s; pn[a * n + c] = 0.9 * w[a] / s + 0.1 * (a == 3 ? 0.0 : 1.0 / 3.0); }
    mu[c] = 0.01 * (double)(c % 5); mu[n + c] = -0.02 * (double)(c % 3);
  }
  const GlobalField FO{po.data(), &g}, FN{pn.data(), &g}, M{mu.data(), &g};
  /* phi cell part (faces excluded) */
  g_ops = 0; g_counting = true;
  { Counted o[N]; phi_cell<Counted>(*p, g, FO, M, 1, 1, 1, o, false); }
  out[0] = g_ops;
  /* one phi face (z face between (1,1,1) and (1,1,2)); neighbour gradients free */
  {
    Counted pl[N], pu[N], gl[N][3], gu[N][3], jf[N];
    { NoCount nc; load4(FO, 1, 1, 1, pl); load4(FO, 1, 1, 2, pu);
      centre_grad(*p, FO, 1, 1, 1, gl); centre_grad(*p, FO, 1, 1, 2, gu); }
    g_ops = 0;
    phi_face(*p, pl, pu, gl, gu, 2, jf);
    out[1] = g_ops;
  }
  /* mu cell part (faces excluded; includes the cell's own per-cell quantities) */
  g_ops = 0;
  { Counted o[NC]; mu_cell<Counted>(*p, g, FO, FN, M, 1, 1, 1, o, false); }
  out[2] = g_ops;
  {
    MuCellQ<Counted> lo, hi;
    { NoCount nc; mu_cell_q(*p, g, FO, FN, M, 1, 1, 1, lo); mu_cell_q(*p, g, FO, FN, M, 1, 1, 2, hi); }
    Counted F[NC], J[NC];
    g_ops = 0;
    mu_face(*p, lo, hi, 2, F, J);
    out[3] = g_ops;
  }
  g_counting = true;
  out[4] = out[0] + 3 * out[1];
  out[5] = out[2] + 3 * out[3];
  return 0;
}

}  // extern "C"
