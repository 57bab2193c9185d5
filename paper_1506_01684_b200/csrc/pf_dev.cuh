// pf_dev.cuh — device-side model arithmetic of the phi- and mu-sweeps
// (Eq. (1)-(4), lines 89-135; readings R1-R25 of DESIGN.md §2).
//
// Rounding discipline: every quantity that two different threads / code
// locations must reproduce bit for bit — a face flux (PAPER.md:299-317
// "staggered positions"), the per-cell quantities the faces are built from,
// the centre gradients — is written with explicit round-to-nearest intrinsics
// (__dadd_rn / __dmul_rn / __fma_rn ...), so nvcc cannot contract it
// differently at different call sites.  This gives (i) exact telescoping of the
// flux-form divergence (solute conservation, DESIGN.md pin P4) and (ii) bitwise
// decomposition invariance (P9): a face evaluated at a tile or block edge has
// the same bits as the same face evaluated mid-tile.  Cell-local updates are
// free for the compiler to contract.
#pragma once
#include <cstdint>

namespace pf {

#define RN_ADD __dadd_rn
#define RN_SUB __dsub_rn
#define RN_MUL __dmul_rn
#define RN_FMA __fma_rn

constexpr int NPH = 4;   // phases alpha, beta, gamma, liquid
constexpr int NMU = 2;   // independent chemical potentials (K-1)
constexpr int LIQ = 3;

// pair index p of (a<b): (0,1)=0 (0,2)=1 (0,3)=2 (1,2)=3 (1,3)=4 (2,3)=5
__host__ __device__ constexpr int pair_a(int p) { return p < 3 ? 0 : (p < 5 ? 1 : 2); }
__host__ __device__ constexpr int pair_b(int p) { return p < 3 ? p + 1 : (p < 5 ? p - 1 : 3); }
// pair index of {a, b}, a != b
__host__ __device__ constexpr int pair_of(int a, int b) {
  return a < b ? (a == 0 ? b - 1 : a + b) : (b == 0 ? a - 1 : a + b);
}

// Output stores of the sweeps: the fields are gigabytes, never re-read from L2
// by the next kernel, so they are written with the evict-first (streaming)
// policy and leave L2 to the tile rings neighbouring CTAs re-read (measured at
// 512^3: the sweeps unchanged within 0.05 %, the fused kernel -0.4 %)
#ifndef PF_STCS
#define PF_STCS 1
#endif
__device__ __forceinline__ void st_field(double *p, double v) {
  if (PF_STCS) __stcs(p, v);
  else *p = v;
}

// Per-step constants (kernel argument, lives in the constant bank).
struct KParams {
  double dt, inv_dt, inv_dx, inv_2dx;
  double pad0_;            // the round-1 layout (a fifth scalar here): with the arrays
                           // at other offsets the phi-sweep needs 4 more registers and
                           // spills (measured; -2 % phi time with this layout)
  double dt_taueps[NPH];   // dt / (tau_a eps)
  double g2[6];            // 2 gamma_ab per pair
  double g2c[6];           // 2 gamma_ab / (2 dx)^2 per pair: isotropic Gram of raw centre differences
  double gf2[6];           // gamma_ab / dx per pair: isotropic face flux on the lo/hi determinant
  double omp[6];           // 16/pi^2 gamma_ab per pair
  double delta16[6];       // 16 delta_ab per pair (cubic anisotropy; the pair gradient's 16 delta, exact)
  double g3[NPH];          // triple coefficient of the triple excluding x
  double mch[NPH][NMU];    // m_a,c: the (T-independent) slope of c-hat, O5.5
  double pi_eps_16dt;      // pi eps / (16 dt): the anti-trapping weight on face sums (mu_face_t)
  double Gv;               // G v = -dT/dt
  int aniso;
  int shortcuts;           // region shortcuts (NEXT-1): skip the phi update of bulk warps
  int dmask;               // bit p set: delta of pair p is not 0 (the cubic g applies)
  int pad1_;
};

// 1/s to within an ulp (faithful, not correctly rounded): the hardware
// approximation refined by two Newton steps (each doubles the correct bits),
// without the IEEE division's special-case branch.  For s > 0 normal; exact
// where 1/s is a power of two (s = 1 gives 1).
__device__ __forceinline__ double rcp_nr(double s) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(s));
  double e = __fma_rn(-s, r, 1.0);
  r = __fma_rn(r, e, r);
  e = __fma_rn(-s, r, 1.0);
  return __fma_rn(r, e, r);
}

// x == +-0 as an integer test on the bits (a double compare is an FP64-pipe
// instruction); false for NaN, like x == 0.0
__device__ __forceinline__ bool is_zero_bits(double x) { return (__double_as_longlong(x) << 1) == 0ll; }
// |x| outside [2^-e, 2^e) or zero / subnormal / inf / NaN, from the exponent bits
__device__ __forceinline__ bool exp_outside(double x, int e) {
  const int ex = (__double2hiint(x) >> 20) & 0x7ff;   // biased exponent
  return (unsigned)(ex - (1023 - e)) >= (unsigned)(2 * e);
}

// 1/sqrt(x) for x in [2^-1000, 2^1000]: the hardware approximation refined by
// two Newton steps r += r (1 - x r^2) / 2 (pinned; a few ulp, not correctly
// rounded) — the library rsqrt's special-case handling is 17 instructions.
__device__ __forceinline__ double rsqrt_nr(double x) {
  double r;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
  double e = RN_FMA(-RN_MUL(x, r), r, 1.0);
  r = RN_FMA(RN_MUL(0.5, r), e, r);
  e = RN_FMA(-RN_MUL(x, r), r, 1.0);
  return RN_FMA(RN_MUL(0.5, r), e, r);
}

// A cell whose phase vector is a simplex vertex (one component exactly 1, the
// others exactly 0).  With an identical neighbourhood its phi update returns
// it unchanged bit for bit: every gradient and face flux is exactly 0, the
// driving force vanishes (S = 1, psi-bar = psi_p), and the projection maps
// 1 + dt/(tau eps) mean back to exactly 1 (Sterbenz) and the pushed-down
// absent phases to exactly 0 — so skipping it is exact.
// the same test on the bits (integer pipe): one component 1.0, the others +-0
__device__ __forceinline__ bool is_vertex_bits(const double p[NPH]) {
  int ones = 0, zeros = 0;
#pragma unroll
  for (int a = 0; a < NPH; ++a) {
    const unsigned long long v = __double_as_longlong(p[a]);
    ones += v == 0x3FF0000000000000ull;
    zeros += (v << 1) == 0ull;
  }
  return ones == 1 && zeros == NPH - 1;
}
__device__ __forceinline__ bool is_vertex(const double p[NPH]) {
  int ones = 0, zeros = 0;
#pragma unroll
  for (int a = 0; a < NPH; ++a) { ones += p[a] == 1.0; zeros += p[a] == 0.0; }
  return ones == 1 && zeros == NPH - 1;
}

// Per-plane table (T-only subexpressions once per
// x-y slice).  TAB doubles per plane, index = global window plane + 1.
enum {
  T_T = 0, T_EPST = 1, T_TEPS = 2,
  T_EPSTDX = 3,   // eps T / dx (the face-flux divergence factor)
  // per (phase a, component c) pairs at base + a*2 + c; every base is even so
  // the (c = 0, 1) pair of a phase is one 16-byte load (tab2)
  T_INV2A = 4,    // 1/(2A)
  T_CHAT = 12,    // c-hat
  T_INV4A = 20,   // 1/(4A)
  T_KAPPA = 28,   // 2 A1 / (2A)^2
  T_MC = 36,      // D / (2A)
  T_B = 44,       // + a         L (T - T_eut) / T_eut
  T_DI2A = 48,    // 1/(2A^l) - 1/(2A^a), solids a < 3
  T_DCHAT = 54,   // chat^l - chat^a,     solids a < 3
  T_DCHAT2 = 60,  // 2 (chat^l - chat^a): the x/y-face sum of (c^l - c^a) (mu_face_t)
  T_EPSTDX16 = 66,   // eps T / (16 dx^2): the divergence factor of the anisotropic face fluxes,
                     // which phi_face returns scaled by 16 dx
  TAB = 68        // multiple of 4 doubles (32 B): rows stay aligned
};
static_assert(TAB % 4 == 0, "table row alignment");
// the (c = 0, 1) pair of phase a of a per-(phase, component) table entry
__device__ __forceinline__ double2 tab2(const double *__restrict__ tab, int base, int a) {
  return *reinterpret_cast<const double2 *>(tab + base + 2 * a);
}


// ---------------------------------------------------------------------------
// phi-sweep
// ---------------------------------------------------------------------------

// Cubic-anisotropy gradient of the pair energy e = gamma a_c^2 |q|^2,
// a_c = 1 - delta (3 - 4 Q4/|q|^4) (reading R3); g = 0 at q = 0.  Pinned:
// used inside face fluxes.  Returns g (without the 2 gamma factor folded:
// full g).
//
// g is homogeneous of degree 1; the direct formula needs |q|^-4 and Q4, which
// leave the double range for |q| < ~1e-77.  Below |q|^2 = 2^-400 (|q| <
// 1.5e-60 of the vector passed in: the sweeps pass 8 dx q at faces, 2 dx q in
// the cell update) g is returned as 0 — an absolute error under 1e-59 (DESIGN.md
// reading R30; the oracle evaluates those exactly by power-of-two scaling).
// The test is an integer compare on |q|^2's exponent and an early return, the
// round-1 exit for q = 0 (absent pairs: most pairs of a bulk cell) widened —
// measured: a rescaling path costs the anisotropic phi-sweep 6-40 % however it
// is written, a select instead of the exit 40 %.  Pair vectors that small need
// phase fractions near 1e-60, which the explicit step does not produce.
__device__ __forceinline__ double q2_of(const double q[3]) {
  return RN_FMA(q[2], q[2], RN_FMA(q[1], q[1], RN_MUL(q[0], q[0])));
}
__device__ __forceinline__ bool q2_tiny(double q2) {   // q2 < 2^-400 (incl. 0, subnormals)
  return ((__double2hiint(q2) >> 20) & 0x7ff) < 1023 - 400;
}
// d16 = 16 delta: a_c = 1 - delta (3 - 4x) is evaluated as 1 - d16 (3/16 - x/4)
// (power-of-two scalings commute with rounding: the same bits as the delta
// form, one multiplication fewer per call)
__device__ __forceinline__ void pair_grad_aniso(double g2, double d16, const double q[3], double out[3]) {
  const double q2 = q2_of(q);
  if (q2_tiny(q2)) { out[0] = out[1] = out[2] = 0.0; return; }
  double s2[3], s4 = 0.0;
#pragma unroll
  for (int d = 0; d < 3; ++d) { s2[d] = RN_MUL(q[d], q[d]); }
  s4 = RN_FMA(s2[2], s2[2], RN_FMA(s2[1], s2[1], RN_MUL(s2[0], s2[0])));   // Q4
  const double r2 = rcp_nr(q2);   // q2 >= 2^-400: normal, no IEEE special cases (measured -6 % aniso phi)
  const double r4 = RN_MUL(r2, r2);
  const double x = RN_MUL(s4, r4);                                          // Q4/|q|^4
  const double ac = RN_SUB(1.0, RN_MUL(d16, RN_FMA(-0.25, x, 0.1875)));    // a_c
  // |q|^2 d a_c/d q_d = 16 delta (q_d^3 - Q4 q_d / |q|^2) / |q|^2
#pragma unroll
  for (int d = 0; d < 3; ++d) {
    const double t = RN_MUL(RN_FMA(s2[d], q[d], -RN_MUL(RN_MUL(s4, r2), q[d])), r2);
    out[d] = RN_MUL(RN_MUL(g2, ac), RN_FMA(d16, t, RN_MUL(ac, q[d])));
  }
}

// Component d alone of pair_grad_aniso (the face flux needs only the normal
// component): the same pinned operations, so bitwise the same value.
__device__ __forceinline__ double pair_grad_aniso_d(double g2, double d16, const double q[3], int d) {
  const double q2 = q2_of(q);
  if (q2_tiny(q2)) return 0.0;
  double s2[3];
#pragma unroll
  for (int e = 0; e < 3; ++e) s2[e] = RN_MUL(q[e], q[e]);
  const double s4 = RN_FMA(s2[2], s2[2], RN_FMA(s2[1], s2[1], RN_MUL(s2[0], s2[0])));
  const double r2 = rcp_nr(q2);   // q2 >= 2^-400: normal, no IEEE special cases (measured -6 % aniso phi)
  const double r4 = RN_MUL(r2, r2);
  const double x = RN_MUL(s4, r4);
  const double ac = RN_SUB(1.0, RN_MUL(d16, RN_FMA(-0.25, x, 0.1875)));
  const double t = RN_MUL(RN_FMA(s2[d], q[d], -RN_MUL(RN_MUL(s4, r2), q[d])), r2);
  return RN_MUL(RN_MUL(g2, ac), RN_FMA(d16, t, RN_MUL(ac, q[d])));
}

// Face flux j_a (component d) of the phi-sweep between cells lo and hi = lo+e_d
// (oracle O4.5): phibar = (lo+hi)/2, normal gradient (hi-lo)/dx, tangential
// gradient = mean of the two centre gradients (anisotropic only);
// j_a = -sum_{b != a} g_ab,d(q_ab) phibar_b.  Pinned rounding.
// AN: -1 = the model from kp.aniso at run time, 0 / 1 = isotropic / anisotropic
// fixed at compile time (the tiled sweep's two kernels carry only their own code)
// DM: the cubic pairs' mask (bit p: delta_p != 0) fixed at compile time, or -1
// for kp.dmask at run time (the anisotropic sweep instantiates the solid-liquid
// case, C5's model, without the per-pair branch)
template <int AN = -1, int DM = -1>
__device__ __forceinline__ void phi_face(const KParams &kp, const double plo[NPH], const double phi_[NPH],
                                         const double glo[NPH][3], const double ghi[NPH][3], int d,
                                         double jf[NPH]) {
#pragma unroll
  for (int a = 0; a < NPH; ++a) jf[a] = 0.0;
  if (!(AN < 0 ? kp.aniso != 0 : AN == 1)) {
    // isotropic: with s = lo + hi = 2 phibar and t = hi - lo = dx grad_d phi,
    // j_a = -sum_b 2 gamma_ab (phibar_a grad_b - phibar_b grad_a) phibar_b
    //     = -sum_b [2 gamma_ab / (4 dx)] (s_a t_b - s_b t_a) s_b,
    // and s_a t_b - s_b t_a = 2 (lo_a hi_b - hi_a lo_b): a 2x2 determinant of
    // the two cells (gf2 = gamma / dx), no cancellation in t
    double s[NPH];
#pragma unroll
    for (int a = 0; a < NPH; ++a) s[a] = RN_ADD(plo[a], phi_[a]);
#pragma unroll
    for (int p = 0; p < 6; ++p) {
      const int a = pair_a(p), b = pair_b(p);
      const double G = RN_MUL(kp.gf2[p], RN_FMA(plo[a], phi_[b], -RN_MUL(phi_[a], plo[b])));
      jf[a] = RN_FMA(-G, s[b], jf[a]);
      jf[b] = RN_FMA(G, s[a], jf[b]);
    }
  } else {
    // anisotropic, on raw differences: glo / ghi are the cells' raw centre
    // differences phi(c+e) - phi(c-e) (= 2 dx grad), so with the face sums
    // s = lo + hi (= 2 phibar), the normal 4 (hi - lo) and the tangential sums
    // glo + ghi (both = 4 dx grad phi at the face) the pair vector is
    // q' = s_a G_b - s_b G_a = 8 dx q; g is homogeneous of degree 1 in q
    // (pin P21), so the returned flux is 16 dx j_a (divergence factor
    // T_EPSTDX16) — no 1/2, 1/dx or 1/(2dx) per operand
    double s[NPH], gn[NPH];
#pragma unroll
    for (int a = 0; a < NPH; ++a) {
      s[a] = RN_ADD(plo[a], phi_[a]);
      gn[a] = RN_MUL(4.0, RN_SUB(phi_[a], plo[a]));
    }
    double gf[NPH][3];
#pragma unroll
    for (int a = 0; a < NPH; ++a)
#pragma unroll
      for (int e = 0; e < 3; ++e)
        gf[a][e] = (e == d) ? gn[a] : RN_ADD(glo[a][e], ghi[a][e]);
#pragma unroll
    for (int p = 0; p < 6; ++p) {
      const int a = pair_a(p), b = pair_b(p);
      double q[3];
#pragma unroll
      for (int e = 0; e < 3; ++e) q[e] = RN_FMA(s[a], gf[b][e], -RN_MUL(s[b], gf[a][e]));
      // only the normal component g_d of the pair gradient enters the flux
      const bool cubic = DM < 0 ? ((kp.dmask >> p) & 1) != 0 : ((DM >> p) & 1) != 0;
      const double gd = !cubic ? RN_MUL(kp.g2[p], q[d]) : pair_grad_aniso_d(kp.g2[p], kp.delta16[p], q, d);
      jf[a] = RN_FMA(-gd, s[b], jf[a]);
      jf[b] = RN_FMA(gd, s[a], jf[b]);
    }
  }
}

// Raw centre difference hi - lo (2 dx times the centre gradient: the phi-sweep's
// and the anti-trapping current's gradients, which fold the 1/(2 dx) into
// their constants), pinned.
__device__ __forceinline__ double cdiff(double lo, double hi) { return RN_SUB(hi, lo); }


// Cell part of the phi update (oracle O4.1-4.11) given the cell value, its
// chemical potential, centre gradients, the face-flux divergence sum_d (j^+ -
// j^-) (before the 1/dx factor) and the plane's table row.  Both models take
// the raw centre differences phi(c+e) - phi(c-e) instead of the gradients:
// they enter the Gram matrix (isotropic) or the pair vectors (anisotropic,
// g homogeneous of degree 1) quadratically, the 1/(2dx)^2 folded into g2c.
// Split in two so the tiled sweep can do everything that does not need the
// face fluxes before its CTA barrier: phi_cell_rhs0 returns
// r0_a = eps T da/dphi_a + (T/eps) domega/dphi_a + dpsi/dphi_a (O4.2-4.4,
// 4.7-4.8), phi_cell_finish adds the divergence and does O4.9-4.11.
template <int AN = -1, int DM = -1>
__device__ __forceinline__ void phi_cell_rhs0(const KParams &kp, const double *__restrict__ tab,
                                              const double ph[NPH], const double mu[NMU],
                                              const double gc[NPH][3], double r0[NPH]);
__device__ __forceinline__ void phi_cell_finish(const KParams &kp, const double *__restrict__ tab,
                                                const double ph[NPH], const double r0[NPH],
                                                const double dsum[NPH], double out[NPH]);
__device__ __forceinline__ void phi_cell_project(const KParams &kp, const double ph[NPH], const double rhs[NPH],
                                                 double out[NPH]);
__device__ __forceinline__ void phi_cell_update_div(const KParams &kp, const double *__restrict__ tab,
                                                    const double ph[NPH], const double mu[NMU],
                                                    const double gc[NPH][3], const double dsum[NPH],
                                                    double out[NPH]) {
  double r0[NPH];
  phi_cell_rhs0(kp, tab, ph, mu, gc, r0);
  phi_cell_finish(kp, tab, ph, r0, dsum, out);
}

__device__ __forceinline__ void phi_cell_update(const KParams &kp, const double *__restrict__ tab,
                                                const double ph[NPH], const double mu[NMU],
                                                const double gc[NPH][3], const double jm[3][NPH],
                                                const double jp[3][NPH], double out[NPH]) {
  double dsum[NPH];
#pragma unroll
  for (int a = 0; a < NPH; ++a) dsum[a] = (jp[0][a] - jm[0][a]) + (jp[1][a] - jm[1][a]) + (jp[2][a] - jm[2][a]);
  phi_cell_update_div(kp, tab, ph, mu, gc, dsum, out);
}

template <int AN, int DM>
__device__ __forceinline__ void phi_cell_rhs0(const KParams &kp, const double *__restrict__ tab,
                                              const double ph[NPH], const double mu[NMU],
                                              const double gc[NPH][3], double r0[NPH]) {
  // d a / d phi_a = sum_{b != a} g_ab(q_ab) . grad phi_b   (O4.2-4)
  double dad[NPH] = {0.0, 0.0, 0.0, 0.0};
  if (!(AN < 0 ? kp.aniso != 0 : AN == 1)) {
    // isotropic g = 2 gamma q: q_ab . grad_b = phi_a |grad_b|^2 - phi_b (grad_a . grad_b),
    // so dad_a = sum_b 2 gamma_ab (phi_a G_bb - phi_b G_ab) with the Gram matrix G
    // of the centre differences (g2mc carries 2 gamma / (2 dx)^2)
    double Gd[NPH], Go[6];
#pragma unroll
    for (int a = 0; a < NPH; ++a) Gd[a] = gc[a][0] * gc[a][0] + gc[a][1] * gc[a][1] + gc[a][2] * gc[a][2];
#pragma unroll
    for (int p = 0; p < 6; ++p) {
      const int a = pair_a(p), b = pair_b(p);
      Go[p] = kp.g2c[p] * (gc[a][0] * gc[b][0] + gc[a][1] * gc[b][1] + gc[a][2] * gc[b][2]);
    }
#pragma unroll
    for (int a = 0; a < NPH; ++a) {
      double wd = 0.0, wo = 0.0;
#pragma unroll
      for (int b = 0; b < NPH; ++b) {
        if (b == a) continue;
        const int p = pair_of(a, b);
        wd += kp.g2c[p] * Gd[b];
        wo += ph[b] * Go[p];
      }
      dad[a] = ph[a] * wd - wo;
    }
  } else {
#pragma unroll
    for (int p = 0; p < 6; ++p) {
      const int a = pair_a(p), b = pair_b(p);
      double q[3], g[3];
#pragma unroll
      for (int e = 0; e < 3; ++e) q[e] = ph[a] * gc[b][e] - ph[b] * gc[a][e];
      // raw centre differences (2 dx grad): q is 2 dx too large, g (degree 1)
      // as well, dad by (2 dx)^2 — g2c carries the 1/(2 dx)^2
      if (DM < 0 ? ((kp.dmask >> p) & 1) != 0 : ((DM >> p) & 1) != 0) {
        pair_grad_aniso(kp.g2c[p], kp.delta16[p], q, g);
      } else {
#pragma unroll
        for (int e = 0; e < 3; ++e) g[e] = kp.g2c[p] * q[e];
      }
      dad[a] += g[0] * gc[b][0] + g[1] * gc[b][1] + g[2] * gc[b][2];
      dad[b] -= g[0] * gc[a][0] + g[1] * gc[a][1] + g[2] * gc[a][2];
    }
  }
  // thermodynamics of the plane: psi_a = B_a - sum_c mu_c (mu_c/(4A) + chat)
  double ps[NPH];
#pragma unroll
  for (int a = 0; a < NPH; ++a) {
    const double2 i4 = tab2(tab, T_INV4A, a), ch = tab2(tab, T_CHAT, a);
    double s = tab[T_B + a];
    s -= mu[0] * (mu[0] * i4.x + ch.x);
    s -= mu[1] * (mu[1] * i4.y + ch.y);
    ps[a] = s;
  }
  const double S = ph[0] * ph[0] + ph[1] * ph[1] + ph[2] * ph[2] + ph[3] * ph[3];
  // S in [1/4, 1] on simplex states.  The faithful reciprocal measured -0.4 % in
  // the anisotropic kernel and +0.9 % in the isotropic one (register allocation)
  const double rS = AN == 1 ? rcp_nr(S) : 1.0 / S;
  const double pbar = rS * (ph[0] * ph[0] * ps[0] + ph[1] * ph[1] * ps[1] + ph[2] * ph[2] * ps[2] +
                            ph[3] * ph[3] * ps[3]);
  const double epsT = tab[T_EPST], Teps = tab[T_TEPS];
  double pp[6];   // pair products phi_b phi_e of the triple terms
#pragma unroll
  for (int p = 0; p < 6; ++p) pp[p] = ph[pair_a(p)] * ph[pair_b(p)];
  const double rS2 = 2.0 * rS;
#pragma unroll
  for (int a = 0; a < NPH; ++a) {
    // O4.7 multi-obstacle derivative
    double om = 0.0;
#pragma unroll
    for (int b = 0; b < NPH; ++b) if (b != a) om += kp.omp[pair_of(a, b)] * ph[b];
#pragma unroll
    for (int x = 0; x < NPH; ++x) {
      if (x == a) continue;
      int b = -1, e = -1;
#pragma unroll
      for (int y = 0; y < NPH; ++y) if (y != a && y != x) { if (b < 0) b = y; else e = y; }
      om += kp.g3[x] * pp[pair_of(b, e)];
    }
    // O4.8 driving force
    const double dpsi = (ph[a] * rS2) * (ps[a] - pbar);
    r0[a] = epsT * dad[a] + Teps * om + dpsi;
  }
}

__device__ __forceinline__ void phi_cell_finish(const KParams &kp, const double *__restrict__ tab,
                                                const double ph[NPH], const double r0[NPH],
                                                const double dsum[NPH], double out[NPH]) {
  // O4.9 with the O4.6 divergence of the face fluxes (eps T / dx folded; the
  // anisotropic fluxes come scaled by 16 dx)
  const double epsTdx = tab[kp.aniso ? T_EPSTDX16 : T_EPSTDX];
  double rhs[NPH];
#pragma unroll
  for (int a = 0; a < NPH; ++a) rhs[a] = r0[a] - epsTdx * dsum[a];
  phi_cell_project(kp, ph, rhs, out);
}

// O4.9-4.11 given the right-hand side rhs_a (r0_a minus the scaled face
// divergence): Lagrange mean, Euler step, simplex projection.
__device__ __forceinline__ void phi_cell_project(const KParams &kp, const double ph[NPH], const double rhs[NPH],
                                                 double out[NPH]) {
  const double mean = 0.25 * ((rhs[0] + rhs[1]) + (rhs[2] + rhs[3]));
  double x[NPH];
#pragma unroll
  for (int a = 0; a < NPH; ++a) x[a] = ph[a] - kp.dt_taueps[a] * (rhs[a] - mean);   // O4.10 (minus sign, R1)

  // O4.11 Euclidean projection onto the simplex: sort descending (network),
  // theta = t_rho = (sum of the rho largest - 1)/rho with rho the largest j
  // such that u_j > t_j.  Since t_{j+1} - t_j = (u_{j+1} - t_j)/(j+1), t_j
  // rises while j < rho and falls after, so theta = max_j t_j: a max tree
  // instead of a chain of dependent selects (same value up to rounding ties).
  double u0 = x[0], u1 = x[1], u2 = x[2], u3 = x[3], t;
#define PF_CSWAP(p, q) if (p < q) { t = p; p = q; q = t; }
  PF_CSWAP(u0, u1) PF_CSWAP(u2, u3) PF_CSWAP(u0, u2) PF_CSWAP(u1, u3) PF_CSWAP(u1, u2)
#undef PF_CSWAP
  const double c1 = u0 - 1.0, c2 = c1 + u1, c3 = c2 + u2, c4 = c3 + u3;
  const double theta = fmax(fmax(c1, 0.5 * c2), fmax(c3 * (1.0 / 3.0), 0.25 * c4));
  // out = max(d, 0) on the integer pipe: every bit of a negative d cleared
  // (a double compare is an FP64-pipe instruction, the sweep's bottleneck:
  // measured -1.7 % phi time); -0 gives +0, a NaN keeps its sign's rule
#pragma unroll
  for (int a = 0; a < NPH; ++a) {
    const double d = x[a] - theta;
    const int hi = __double2hiint(d), lo = __double2loint(d), m = ~(hi >> 31);
    out[a] = __hiloint2double(hi & m, lo & m);
  }
}

// ---------------------------------------------------------------------------
// mu-sweep
// ---------------------------------------------------------------------------

// Per-cell quantities a mu face needs (oracle MuCellQ), pinned.
struct MuQ {
  double pn[NPH];     // phi^{n+1}
  double dp[NPH];     // phi^{n+1} - phi^n
  double gn[NPH][3];  // raw centre differences phi^{n+1}(c+e) - phi^{n+1}(c-e) (tangential parts used)
  double M[NMU];      // sum_a phi^n_a D/(2A)          (R11)
  double dcl[3][NMU]; // c^l - c^a for the solids a   (R10)
  double mu[NMU];
  const double *tab;  // the cell's plane table row
};

// c^l - c^a = mu (1/(2A^l) - 1/(2A^a)) + (chat^l - chat^a) at the plane's T
// (per-plane differences from the table; pinned).
__device__ __forceinline__ double dcl_of(const double *__restrict__ tab, int a, int c, double mu) {
  return RN_FMA(mu, tab[T_DI2A + a * 2 + c], tab[T_DCHAT + a * 2 + c]);
}
// mobility sum_a phi^n_a D/(2A) of both components (pinned)
__device__ __forceinline__ void mob2(const double *__restrict__ tab, const double po[NPH], double M[NMU]) {
  double2 m = tab2(tab, T_MC, 0);
  M[0] = RN_MUL(po[0], m.x);
  M[1] = RN_MUL(po[0], m.y);
#pragma unroll
  for (int a = 1; a < NPH; ++a) {
    m = tab2(tab, T_MC, a);
    M[0] = RN_FMA(po[a], m.x, M[0]);
    M[1] = RN_FMA(po[a], m.y, M[1]);
  }
}

__device__ __forceinline__ void mu_cell_q(const double *__restrict__ tab, const double po[NPH],
                                          const double pn[NPH], const double mu[NMU], MuQ &q) {
  q.tab = tab;
#pragma unroll
  for (int a = 0; a < NPH; ++a) { q.pn[a] = pn[a]; q.dp[a] = RN_SUB(pn[a], po[a]); }
  mob2(tab, po, q.M);
#pragma unroll
  for (int c = 0; c < NMU; ++c) {
    q.mu[c] = mu[c];
#pragma unroll
    for (int a = 0; a < 3; ++a) q.dcl[a][c] = dcl_of(tab, a, c, mu[c]);
  }
}

// (M grad mu - J_at)_c at the face (lo, hi = lo + e_d) — oracle mu_face.
// One pinned implementation for every operand source: QL / QH are accessors
// (registers: MuQAcc; shared-memory tiles and records: see pf_mu.cu) with
//   pn(a), dp(a) (a < 3), gt(a, e) (RAW centre difference of phi^{n+1},
//   phi(c+e) - phi(c-e), e != d), M(c), mu(c), dcl(a, c).
// Guards are exact-zero tests (reading R10).  The anti-trapping weight
//   (pi eps/4) phibar_a h_l / sqrt(phibar_a phibar_l) * dphi_a/dt * (n_a . n_l) * n_a,d
// is homogeneous of degree 0 in phibar and in each gradient vector, so it is
// evaluated on face SUMS s = lo + hi (= 2 phibar), sum of the dphi (= 2 dt
// dphi/dt) and gradients scaled by 4 dx (normal 4 (hi - lo), tangential the
// sum of the two raw centre differences): no 1/2, 1/dx or 1/dt per operand,
// the constants folded into pi eps / (16 dt) (the (c^l - c^a) sum carries the
// last 1/2):
//   w = (pi eps / 16 dt) s_a h_l pd (g_a . g_l) g_a,d / sqrt(s_a s_l |g_l|^2 |g_a|^4)
// — one FP64 rsqrt per solid (a guarded factorised fallback keeps it finite
// when the product leaves the normal range).  Equal to the oracle's literal
// form up to rounding.
// Diffusive part M grad mu of a face (arithmetic mean of the cell mobilities,
// reading R11), pinned: the value every face starts from.
__device__ __forceinline__ double mu_flux_diff(const KParams &kp, double Mlo, double Mhi, double mlo, double mhi) {
  // ((Mlo + Mhi) (mhi - mlo)) / (2 dx): the 1/2 of the mean folded into 1/(2dx)
  // (power-of-two factors commute with rounding: the same bits as
  // (0.5 (Mlo + Mhi)) (mhi - mlo) / dx, one multiplication fewer)
  return RN_MUL(RN_MUL(RN_ADD(Mlo, Mhi), RN_SUB(mhi, mlo)), kp.inv_2dx);
}

// DIFF = false: the anti-trapping part -J alone (Algorithm 2's mu-sweep-neighbor).
// ROLL: the three solids in a loop that is not unrolled (a third of the code
// and of the live temporaries; only for accessors whose operands are in
// shared memory — an operand array in registers indexed by a run-time solid
// would be put in local memory)
// exact-zero guards as integer tests on the bits (is_zero_bits)
#define PF_ZERO(x) is_zero_bits(x)
template <bool DIFF = true, bool ROLL = false, class QL, class QH>
__device__ __forceinline__ void mu_face_t(const KParams &kp, const QL &lo, const QH &hi, int d, double out[NMU]) {
#pragma unroll
  for (int c = 0; c < NMU; ++c) out[c] = DIFF ? mu_flux_diff(kp, lo.M(c), hi.M(c), lo.mu(c), hi.mu(c)) : 0.0;
  const double sl = RN_ADD(lo.pn(LIQ), hi.pn(LIQ));
  if (PF_ZERO(sl)) return;                  // no liquid: J = 0 (bulk solid exits here)
  // gradient components in the order (normal d, tangential d+1, d+2) — scalars,
  // never an array indexed by the run-time d (that would live in local memory)
  const int e1 = d == 2 ? 0 : d + 1, e2 = d == 0 ? 2 : d - 1;
  const double ln = RN_MUL(4.0, RN_SUB(hi.pn(LIQ), lo.pn(LIQ)));
  const double l1 = RN_ADD(lo.gt(LIQ, e1), hi.gt(LIQ, e1)), l2 = RN_ADD(lo.gt(LIQ, e2), hi.gt(LIQ, e2));
  const double gl2 = RN_FMA(l2, l2, RN_FMA(l1, l1, RN_MUL(ln, ln)));
  if (PF_ZERO(gl2)) return;                 // flat liquid: J = 0
  double S = RN_MUL(sl, sl);   // = sum_b s_b^2 with the liquid term first
  {
    double sa[3];
#pragma unroll
    for (int a = 0; a < 3; ++a) sa[a] = RN_ADD(lo.pn(a), hi.pn(a));
    S = RN_FMA(sa[2], sa[2], RN_FMA(sa[1], sa[1], RN_FMA(sa[0], sa[0], S)));
  }
  // S = sum_b s_b^2 >= (sum_b s_b)^2 / 4 = 1 on simplex states (and <= 16):
  // outside [2^-1000, 2^1000] only for inadmissible input — no J then (R31)
  if (exp_outside(S, 1000)) return;
  const double rS = rcp_nr(S);
  // (pi eps / 16 dt) h_l
  const double khl = RN_MUL(kp.pi_eps_16dt, RN_MUL(RN_MUL(sl, sl), rS));
  // x / y faces: both cells share the plane's table row, so the (c^l - c^a)
  // sum is (mu_lo + mu_hi) (1/2A^l - 1/2A^a) + 2 (chat^l - chat^a); a z face's
  // cells each use their own plane's row
  const double ms0 = RN_ADD(lo.mu(0), hi.mu(0)), ms1 = RN_ADD(lo.mu(1), hi.mu(1));
  double J0 = 0.0, J1 = 0.0;
  auto solid = [&](int a) {
    const double saa = RN_ADD(lo.pn(a), hi.pn(a));
    const double pal = RN_MUL(saa, sl);
    const double pd = RN_ADD(lo.dp(a), hi.dp(a));
    const double gn = RN_MUL(4.0, RN_SUB(hi.pn(a), lo.pn(a)));
    const double g1 = RN_ADD(lo.gt(a, e1), hi.gt(a, e1)), g2 = RN_ADD(lo.gt(a, e2), hi.gt(a, e2));
    const double ga2 = RN_FMA(g2, g2, RN_FMA(g1, g1, RN_MUL(gn, gn)));
    if (PF_ZERO(pal) || PF_ZERO(ga2) || PF_ZERO(pd)) return;
    const double dot = RN_FMA(g2, l2, RN_FMA(g1, l1, RN_MUL(gn, ln)));
    const double x = RN_MUL(RN_MUL(pal, gl2), RN_MUL(ga2, ga2));
    // x = s_a s_l |g_l|^2 |g_a|^4 below 2^-1000 needs a phase fraction of the
    // face below ~1e-60 (nonzero differences of O(1) values are >= ~1e-17),
    // where |w| <= c |pd| min(sqrt(s_a/s_l), (s_l/s_a)^1.5) < 1e-30 c |pd|:
    // the solid's term is dropped (R31; a factorised evaluation with library
    // rsqrt calls cost the interface mu-sweep 12 % for this never-taken case)
    if (exp_outside(x, 1000)) return;
    const double r = rsqrt_nr(x);
    const double w = RN_MUL(RN_MUL(RN_MUL(RN_MUL(khl, saa), pd), RN_MUL(dot, gn)), r);
    double dc0, dc1;
    if (d < 2) {
      const double *t = lo.tab();
      dc0 = RN_FMA(ms0, t[T_DI2A + a * 2], t[T_DCHAT2 + a * 2]);
      dc1 = RN_FMA(ms1, t[T_DI2A + a * 2 + 1], t[T_DCHAT2 + a * 2 + 1]);
    } else {
      dc0 = RN_ADD(lo.dcl(a, 0), hi.dcl(a, 0));
      dc1 = RN_ADD(lo.dcl(a, 1), hi.dcl(a, 1));
    }
    J0 = RN_FMA(w, dc0, J0);
    J1 = RN_FMA(w, dc1, J1);
  };
  if (ROLL) {
#pragma unroll 1
    for (int a = 0; a < 3; ++a) solid(a);
  } else {
    solid(0);
    solid(1);
    solid(2);
  }
  out[0] = RN_SUB(out[0], J0);
  out[1] = RN_SUB(out[1], J1);
}

struct MuQAcc {  // accessor over a register MuQ
  const MuQ &q;
  __device__ __forceinline__ double pn(int a) const { return q.pn[a]; }
  __device__ __forceinline__ double dp(int a) const { return q.dp[a]; }
  __device__ __forceinline__ double gt(int a, int e) const { return q.gn[a][e]; }
  __device__ __forceinline__ double M(int c) const { return q.M[c]; }
  __device__ __forceinline__ double mu(int c) const { return q.mu[c]; }
  __device__ __forceinline__ double dcl(int a, int c) const { return q.dcl[a][c]; }
  __device__ __forceinline__ const double *tab() const { return q.tab; }
};

__device__ __forceinline__ void mu_face(const KParams &kp, const MuQ &lo, const MuQ &hi, int d, double out[NMU]) {
  mu_face_t(kp, MuQAcc{lo}, MuQAcc{hi}, d, out);
}

// Cell part of the mu update (oracle O5.1-5.9) given phi^n, phi^{n+1}, mu^n of
// the cell, the divergence sum_d (f^+ - f^-) of the face values, and the table.
__device__ __forceinline__ void mu_cell_update(const KParams &kp, const double *__restrict__ tab,
                                               const double po[NPH], const double pn[NPH], const double mu[NMU],
                                               const double divf[NMU], double out[NMU]) {
  // With p = (phi^n)^2, q = (phi^{n+1})^2 (componentwise), S = sum: h^n = p/So,
  // h^{n+1} = q/Sn, chi_c = X_c/Sn with X_c = sum_a q_a/(2A_a) (O5.3), so
  //   s_c    = sum_a e_ca (q_a/Sn - p_a/So),  e_ca = mu_c/(2A_a) + chat_a  (O5.4)
  //   dcdT_c = (1/Sn) sum_a q_a (m_a - mu_c kappa_a)                      (O5.5)
  //   mu_c^{n+1} = mu_c + (dt Sn / X_c) [dcdT_c G v - s_c/dt + div_c]     (O5.9)
  // and one reciprocal R = 1/(So Sn X_0 X_1) serves 1/So, 1/Sn, 1/X_0, 1/X_1.
  double p[NPH], q[NPH];
#pragma unroll
  for (int a = 0; a < NPH; ++a) { p[a] = po[a] * po[a]; q[a] = pn[a] * pn[a]; }
  const double So = (p[0] + p[1]) + (p[2] + p[3]), Sn = (q[0] + q[1]) + (q[2] + q[3]);
  double X[NMU] = {0.0, 0.0}, A[NMU] = {0.0, 0.0}, B[NMU] = {0.0, 0.0}, D[NMU] = {0.0, 0.0};
#pragma unroll
  for (int a = 0; a < NPH; ++a) {
    const double2 i2a = tab2(tab, T_INV2A, a), ch = tab2(tab, T_CHAT, a);
    const double2 ka = tab2(tab, T_KAPPA, a);   // m_a,c: constant bank operand, no shared load
    const double e0 = mu[0] * i2a.x + ch.x, e1 = mu[1] * i2a.y + ch.y;
    X[0] += q[a] * i2a.x;
    X[1] += q[a] * i2a.y;
    A[0] += e0 * q[a];
    A[1] += e1 * q[a];
    B[0] += e0 * p[a];
    B[1] += e1 * p[a];
    D[0] += q[a] * (kp.mch[a][0] - mu[0] * ka.x);
    D[1] += q[a] * (kp.mch[a][1] - mu[1] * ka.y);
  }
  const double P = So * Sn, Q = X[0] * X[1];
  // faithful reciprocal: the latency-bound mu-sweep gains from the shorter
  // chain (measured -2 %); P Q is a product of O(1) sums, far from the
  // subnormal range rcp.approx.ftz would flush
  const double R = rcp_nr(P * Q);
  const double QR = Q * R, PR = P * R;
  const double rSn = So * QR, rSo = Sn * QR;           // 1/Sn, 1/So
  const double dtSn = kp.dt * Sn;
  const double f[NMU] = {dtSn * (PR * X[1]), dtSn * (PR * X[0])};   // dt Sn / X_c
#pragma unroll
  for (int c = 0; c < NMU; ++c) {
    const double sc = A[c] * rSn - B[c] * rSo;
    const double rest = (D[c] * rSn) * kp.Gv - sc * kp.inv_dt + divf[c] * kp.inv_dx;
    out[c] = mu[c] + f[c] * rest;
  }
}

// Algorithm 2's second half: add the anti-trapping
// divergence divj = sum_d ((-J)^+ - (-J)^-) (before 1/dx) to the mu-sweep-local
// result mu_loc, with the same chi(phi^{n+1}) as mu_cell_update.
__device__ __forceinline__ void mu_cell_add_j(const KParams &kp, const double *__restrict__ tab, const double pn[NPH],
                                              const double mu_loc[NMU], const double divj[NMU], double out[NMU]) {
  const double rSn = 1.0 / (pn[0] * pn[0] + pn[1] * pn[1] + pn[2] * pn[2] + pn[3] * pn[3]);
  double chi[NMU] = {0.0, 0.0};
#pragma unroll
  for (int a = 0; a < NPH; ++a) {
    const double hn = pn[a] * pn[a] * rSn;
    const double2 i2a = tab2(tab, T_INV2A, a);
    chi[0] += hn * i2a.x;
    chi[1] += hn * i2a.y;
  }
  const double rc = kp.dt / (chi[0] * chi[1]);
  out[0] = mu_loc[0] + (chi[1] * rc) * (divj[0] * kp.inv_dx);
  out[1] = mu_loc[1] + (chi[0] * rc) * (divj[1] * kp.inv_dx);
}

}  // namespace pf
