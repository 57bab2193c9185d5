"""oracle_np.py — the second, independent CPU coding of the oracle (NumPy).

TEST INFRASTRUCTURE ONLY (like oracle.cpp): imported by tests/ alone.  It shares
no code with oracle/oracle.cpp nor with the CUDA path; the two CPU codings guard
each other (SURVEY.md §8(c) "two independent CPU codings"; the paper's own
practice of checking every kernel version against the others).

It is written from the paper and DESIGN.md's readings, not from oracle.cpp, and
deliberately in another shape:
  * whole-array (vectorised) arithmetic over ghost-padded copies of the fields
    (periodic x/y by wrap padding, zero-gradient z by edge padding: PAPER.md:155,
    reading R13) instead of per-cell index functions;
  * the pair sums over ORDERED pairs (a, b), a != b, instead of a < b with the
    antisymmetric update;
  * g(q) written on the unit normal n = q/|q|: a_c = 1 - delta (3 - 4 sum n_d^4),
    d a_c/d q = (16 delta/|q|)(n^3 - n sum n^4) (reading R3);
  * d psi/d phi_a as sum_b psi_b d h_b/d phi_a with d h_b/d phi_a =
    2 phi_b [a == b]/S - 2 phi_b^2 phi_a/S^2 (reading R6),
    not the factorised (2 phi_a/S)(psi_a - psibar);
  * d omega/d phi_a from the pair and triple sums (reading R5).
Results agree with oracle.cpp up to rounding order (tests/test_oracle_second_coding.py,
<= 1e-13 relative max-norm).

Arrays: phi[4, nz, ny, nx], mu[2, nz, ny, nx] (x fastest); phases 0..3 = alpha,
beta, gamma, liquid; components 0, 1.  Parameters: the oracle's OrParams struct
is read as plain data.
"""
from __future__ import annotations

import math

import numpy as np

NPH, NMU, LIQ = 4, 2, 3


class _P:
    """OrParams as numpy arrays (data only)."""

    def __init__(self, p):
        self.dx, self.dt, self.eps = p.dx, p.dt, p.eps
        self.tau = np.array(p.tau[:])
        self.gamma = np.array([list(r) for r in p.gamma])
        self.gamma3 = np.array(p.gamma3[:])
        self.delta = np.array([list(r) for r in p.delta])
        self.T_eut, self.G, self.v, self.T0 = p.T_eut, p.G, p.v, p.T0
        self.A0 = np.array([list(r) for r in p.A0])
        self.A1 = np.array([list(r) for r in p.A1])
        self.c0 = np.array([list(r) for r in p.c0])
        self.m = np.array([list(r) for r in p.m])
        self.L = np.array(p.L[:])
        self.D = np.array([list(r) for r in p.D])
        self.aniso = bool(p.aniso)


def _pad(f, w):
    """Ghost layers of width w: periodic in x and y, zero-gradient (edge copy) in z."""
    f = np.pad(f, ((0, 0), (0, 0), (w, w), (w, w)), mode="wrap")
    return np.pad(f, ((0, 0), (w, w), (0, 0), (0, 0)), mode="edge")


def _cut(A, w, n, lo=(0, 0, 0), hi=(0, 0, 0)):
    """Cells [-lo_d, n_d + hi_d) of an array padded by w, axes (z, y, x)."""
    return A[(slice(None),) + tuple(slice(w - lo[t], w + n[t] + hi[t]) for t in range(3))]


def _axis(d):
    """Direction d = 0, 1, 2 (x, y, z) -> array axis of (c, z, y, x)."""
    return 3 - d


def _temperature(P, planes, n, zorig):
    """O1: T = T0 + G (z - v t) at cell-centre z = (k + zorig + 1/2) dx of each
    plane index k (ghost planes at their own z), t = n dt (
    reading R12).  Shape (len(planes), 1, 1)."""
    z = (np.asarray(planes, dtype=np.float64) + zorig + 0.5) * P.dx
    return (P.T0 + P.G * (z - P.v * (n * P.dt)))[:, None, None]


def _centre_grads(F, w, n, ext):
    """D3C7 centre gradients (phi(c+e_d) - phi(c-e_d)) / (2 dx) of an array padded
    by w, over the cells extended by ext; returns [d] -> (4, ...)."""
    out = []
    for d in range(3):
        lo, hi = [ext] * 3, [ext] * 3
        ax = 2 - d                     # index in (z, y, x)
        up = _cut(F, w, n, tuple(e - (t == ax) for t, e in enumerate(lo)), tuple(e + (t == ax) for t, e in enumerate(hi)))
        dn = _cut(F, w, n, tuple(e + (t == ax) for t, e in enumerate(lo)), tuple(e - (t == ax) for t, e in enumerate(hi)))
        out.append((up - dn) / 2.0)
    return out


def _pair_grad(P, a, b, q):
    """g_ab(q) = d e_ab / d q for e_ab = gamma_ab a_c(q)^2 |q|^2 (reading R3),
    q of shape (3, ...); g(0) = 0."""
    gam = P.gamma[a, b]
    if not P.aniso:
        return 2.0 * gam * q
    dl = P.delta[a, b]
    qn = np.sqrt(q[0] ** 2 + q[1] ** 2 + q[2] ** 2)
    safe = np.where(qn > 0, qn, 1.0)
    nv = q / safe
    s4 = nv[0] ** 4 + nv[1] ** 4 + nv[2] ** 4
    ac = 1.0 - dl * (3.0 - 4.0 * s4)
    g = 2.0 * gam * ac * (qn * 16.0 * dl * (nv ** 3 - nv * s4) + ac * q)
    return np.where(qn > 0, g, 0.0)


def _project(x):
    """Euclidean projection of each column x[:, ...] onto {sum = 1, x >= 0}
    (reading R14): the sort-and-threshold algorithm."""
    u = -np.sort(-x, axis=0)
    css = np.cumsum(u, axis=0)
    j = np.arange(1, x.shape[0] + 1, dtype=np.float64).reshape((-1,) + (1,) * (x.ndim - 1))
    t = (css - 1.0) / j
    ok = (u - t) > 0
    rho = x.shape[0] - 1 - np.argmax(ok[::-1], axis=0)       # largest j with u_j > t_j
    theta = np.take_along_axis(t, rho[None], axis=0)[0]
    return np.maximum(x - theta, 0.0)


def phi_sweep(p, phi, mu, n=0, zorig=0):
    """O4: phi^{n+1} from phi^n and mu^n (Eq. (1)-(2); the
    minus sign of reading R1, the Lagrange mean over all N phases of R2)."""
    P = _P(p)
    nz, ny, nx = phi.shape[1:]
    nn = (nz, ny, nx)
    dx = P.dx
    F = _pad(phi, 2)
    G1 = [g / dx for g in _centre_grads(F, 2, nn, 1)]      # cells extended by 1 (offset 1)
    ph = _cut(F, 2, nn)
    T = _temperature(P, np.arange(nz), n, zorig)

    # face fluxes j_a at the faces (c - e_d, c), then the divergence (O4.5-6)
    div = np.zeros_like(ph)
    for d in range(3):
        ax = 2 - d
        lo_ext = tuple(1 if t == ax else 0 for t in range(3))
        hi_ext = tuple(1 if t == ax else 0 for t in range(3))
        # lo cell = c - e_d for c in [0, n_d], hi cell = c
        plo = _cut(F, 2, nn, lo_ext, (0, 0, 0))
        phi_ = _cut(F, 2, nn, (0, 0, 0), hi_ext)
        glo = [_cut(g, 1, nn, lo_ext, (0, 0, 0)) for g in G1]
        ghi = [_cut(g, 1, nn, (0, 0, 0), hi_ext) for g in G1]
        pb = 0.5 * (plo + phi_)
        gf = []
        for e in range(3):
            if e == d:
                gf.append((phi_ - plo) / dx)
            elif P.aniso:
                gf.append(0.5 * (glo[e] + ghi[e]))
            else:
                gf.append(np.zeros_like(pb))
        gf = np.stack(gf)                                  # (3, 4, ...)
        jf = np.zeros_like(pb)
        for a in range(NPH):
            for b in range(NPH):
                if a == b:
                    continue
                q = pb[a] * gf[:, b] - pb[b] * gf[:, a]
                jf[a] -= _pair_grad(P, a, b, q)[d] * pb[b]
        A = _axis(d)
        up = [slice(None)] * 4
        dn = [slice(None)] * 4
        up[A] = slice(1, None)
        dn[A] = slice(None, -1)
        div += (jf[tuple(up)] - jf[tuple(dn)]) / dx

    # centre term d a / d phi_a = sum_{b != a} g_ab(q_ab) . grad phi_b (O4.2-4)
    gc = np.stack([_cut(g, 1, nn) for g in G1])            # (3, 4, nz, ny, nx)
    dadphi = np.zeros_like(ph)
    for a in range(NPH):
        for b in range(NPH):
            if a == b:
                continue
            q = ph[a] * gc[:, b] - ph[b] * gc[:, a]
            g = _pair_grad(P, a, b, q)
            dadphi[a] += (g * gc[:, b]).sum(axis=0)

    # obstacle derivative (O4.7)
    dom = np.zeros_like(ph)
    for a in range(NPH):
        for b in range(NPH):
            if b != a:
                dom[a] += (16.0 / math.pi ** 2) * P.gamma[a, b] * ph[b]
        for x in range(NPH):
            if x == a:
                continue
            rest = [b for b in range(NPH) if b not in (a, x)]
            dom[a] += P.gamma3[x] * ph[rest[0]] * ph[rest[1]]

    # driving force d psi / d phi_a = sum_b psi_b d h_b / d phi_a (O4.8)
    th = T - P.T_eut
    psi = np.zeros_like(ph)
    for a in range(NPH):
        for c in range(NMU):
            A_ = P.A0[a, c] + P.A1[a, c] * th
            ch = P.c0[a, c] + P.m[a, c] * th
            psi[a] -= mu[c] ** 2 / (4.0 * A_) + mu[c] * ch
        psi[a] += P.L[a] * th / P.T_eut
    S = (ph ** 2).sum(axis=0)
    dpsi = np.zeros_like(ph)
    for a in range(NPH):
        for b in range(NPH):
            dh = -2.0 * ph[b] ** 2 * ph[a] / S ** 2
            if a == b:
                dh = dh + 2.0 * ph[b] / S
            dpsi[a] += psi[b] * dh

    rhs = P.eps * T * (dadphi - div) + (T / P.eps) * dom + dpsi   # (O4.9)
    mean = rhs.mean(axis=0)
    star = ph - (P.dt / (P.tau[:, None, None, None] * P.eps)) * (rhs - mean)   # (O4.10)
    return _project(star)                                           # (O4.11)


def mu_sweep(p, phi_old, phi_new, mu, n=0, zorig=0):
    """O5: mu^{n+1} from mu^n, phi^n and phi^{n+1} (Eq. (3)-(4), PAPER.md:114-135;
    readings R8-R11, R24: M from phi^n; chi, h^{n+1}, dc/dT and the anti-trapping
    normals from phi^{n+1}; c^a from (mu^n, T^n); exact-zero guards)."""
    P = _P(p)
    nz, ny, nx = mu.shape[1:]
    nn = (nz, ny, nx)
    dx, dt = P.dx, P.dt
    E1 = (1, 1, 1)
    po = _cut(_pad(phi_old, 1), 1, nn, E1, E1)      # cells extended by 1 (offset 1)
    FN = _pad(phi_new, 2)
    pn = _cut(FN, 2, nn, E1, E1)
    m = _cut(_pad(mu, 1), 1, nn, E1, E1)
    gn = np.stack([g / dx for g in _centre_grads(FN, 2, nn, 1)])   # (3, 4, ...)
    T = _temperature(P, np.arange(-1, nz + 1), n, zorig)
    th = T - P.T_eut
    A2 = np.empty((NPH, NMU) + T.shape)              # 2 A_c^a(T) per plane
    chat = np.empty_like(A2)
    for a in range(NPH):
        for c in range(NMU):
            A2[a, c] = 2.0 * (P.A0[a, c] + P.A1[a, c] * th)
            chat[a, c] = P.c0[a, c] + P.m[a, c] * th
    conc = np.stack([np.stack([m[c] / A2[a, c] + chat[a, c] for c in range(NMU)]) for a in range(NPH)])
    Mob = np.stack([sum(po[a] * (P.D[a, c] / A2[a, c]) for a in range(NPH)) for c in range(NMU)])
    dph = pn - po

    div = np.zeros((NMU,) + nn)
    for d in range(3):
        ax = 2 - d
        A = _axis(d)
        lo_i = [slice(1, 1 + nn[t]) for t in range(3)]
        hi_i = [slice(1, 1 + nn[t]) for t in range(3)]
        lo_i[ax] = slice(0, nn[ax] + 1)                 # faces (c - e_d, c), c in [0, n_d]
        hi_i[ax] = slice(1, nn[ax] + 2)
        L = (slice(None),) + tuple(lo_i)
        H = (slice(None),) + tuple(hi_i)
        Fd = 0.5 * (Mob[L] + Mob[H]) * (m[H] - m[L]) / dx
        # anti-trapping current (Eq. (4), reading R10)
        pb = 0.5 * (pn[L] + pn[H])
        gf = np.stack([(pn[H] - pn[L]) / dx if e == d else 0.5 * (gn[e][L] + gn[e][H]) for e in range(3)])
        pdot = 0.5 * (dph[L] + dph[H]) / dt
        Sf = (pb ** 2).sum(axis=0)
        hl = pb[LIQ] ** 2 / Sf
        gl2 = (gf[:, LIQ] ** 2).sum(axis=0)
        Jd = np.zeros_like(Fd)
        with np.errstate(divide="ignore", invalid="ignore"):
            nl = gf[:, LIQ] / np.sqrt(gl2)
            for a in range(NPH):
                if a == LIQ:
                    continue
                pal = pb[a] * pb[LIQ]
                ga2 = (gf[:, a] ** 2).sum(axis=0)
                open_ = (pal != 0) & (ga2 != 0) & (gl2 != 0) & (pdot[a] != 0)
                na = gf[:, a] / np.sqrt(ga2)
                w = (math.pi * P.eps / 4.0) * (pb[a] * hl / np.sqrt(pal)) * pdot[a] * (na * nl).sum(axis=0) * na[d]
                for c in range(NMU):
                    dcv = 0.5 * ((conc[LIQ, c][L[1:]] - conc[a, c][L[1:]]) + (conc[LIQ, c][H[1:]] - conc[a, c][H[1:]]))
                    Jd[c] += np.where(open_, w * dcv, 0.0)
        FJ = Fd - Jd
        up = [slice(None)] * 4
        dn = [slice(None)] * 4
        up[A] = slice(1, None)
        dn[A] = slice(None, -1)
        div += (FJ[tuple(up)] - FJ[tuple(dn)]) / dx

    I = (slice(1, 1 + nz), slice(1, 1 + ny), slice(1, 1 + nx))
    hn = pn[(slice(None),) + I] ** 2 / (pn[(slice(None),) + I] ** 2).sum(axis=0)
    ho = po[(slice(None),) + I] ** 2 / (po[(slice(None),) + I] ** 2).sum(axis=0)
    A2i = A2[:, :, 1:1 + nz]
    mu0 = m[(slice(None),) + I]
    Tdot = -P.G * P.v
    out = np.empty_like(mu0)
    for c in range(NMU):
        chi = sum(hn[a] / A2i[a, c] for a in range(NPH))
        src = -sum(conc[a, c][I] * (hn[a] - ho[a]) for a in range(NPH)) / dt
        dcdT = sum(hn[a] * (P.m[a, c] - mu0[c] * 2.0 * P.A1[a, c] / A2i[a, c] ** 2) for a in range(NPH))
        out[c] = mu0[c] + dt / chi * (src - dcdT * Tdot + div[c])
    return out


def step(p, phi, mu, n=0, zorig=0):
    """One step of Algorithm 1: phi-sweep, then mu-sweep."""
    phi_new = phi_sweep(p, phi, mu, n, zorig)
    return phi_new, mu_sweep(p, phi, phi_new, mu, n, zorig)


def run(p, phi, mu, nsteps, n0=0, zorig=0):
    for s in range(nsteps):
        phi, mu = step(p, phi, mu, n0 + s, zorig)
    return phi, mu
