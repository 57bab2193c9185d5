"""Pins of the CPU oracle against what the paper and the mathematics fix.

Each test names its pin and checks the
oracle against something other than itself: closed forms, invariants, special
cases that reduce to a textbook problem, exhaustive enumeration, finite
differences of the energy the oracle differentiates.  CPU only.
"""
import itertools
import math

import numpy as np
import pytest

from inputs import gen
from oracle import oracle as O

PI2 = math.pi ** 2


def _params(pd, **kw):
    return O.make_params(pd, **kw)


def _binary_profile_z(nz, eps, z0, a=0, b=1):
    """Analytic binary obstacle profile: phi_a = 1/2[1 +
    sin(4 (z - z0)/(pi eps))] on |z - z0| <= pi^2 eps / 8, 0 / 1 outside."""
    z = np.arange(nz) + 0.5
    arg = 4.0 * (z - z0) / (math.pi * eps)
    prof = np.where(arg >= math.pi / 2, 1.0, np.where(arg <= -math.pi / 2, 0.0, 0.5 * (1 + np.sin(arg))))
    phi = np.zeros((4, nz, 1, 1))
    phi[b, :, 0, 0] = prof
    phi[a, :, 0, 0] = 1.0 - prof
    return phi


# --------------------------------------------------------------------------
# P1 — analytic 1D binary obstacle profile (A1, A5, A19; "sinus-shaped")
# --------------------------------------------------------------------------
def _p1_error(pd, eps):
    W = PI2 * eps / 4.0
    nz = int(round(4 * W)) // 2 * 2
    z0 = nz / 2.0
    pdd = dict(pd, eps=eps, G=0.0, v=0.0)
    p = _params(pdd, T0=pd["T_eut"])   # T = T_eut, mu = 0: no driving force
    phi = _binary_profile_z(nz, eps, z0)
    mu = np.zeros((2, nz, 1, 1))
    for _ in range(20000):
        new = O.phi_sweep(p, phi, mu)
        d = np.abs(new - phi).max()
        phi = new
        if d < 1e-13:
            break
    exact = _binary_profile_z(nz, eps, z0)
    assert phi[2].max() == 0.0 and phi[3].max() == 0.0, "ghost phases appeared"
    return np.abs(phi - exact).max()


@pytest.mark.slow
def test_p1_analytic_profile_converges_second_order(pv1):
    e8 = _p1_error(pv1, 8.0)
    e16 = _p1_error(pv1, 16.0)
    assert e8 / e16 >= 3.0, (e8, e16)
    assert e16 <= 3e-4, e16


def test_p1_equilibrium_width_is_stationary(pv1):
    # eps = 16/pi^2 gives W = 4 cells (reading R19); the discrete stationary
    # profile stays within 1e-2 of the analytic one (coarse resolution)
    e = _p1_error(pv1, 16.0 / PI2 * 2.0)  # W = 8 cells
    assert e < 1e-2


# --------------------------------------------------------------------------
# P2 — binary reduction to the textbook obstacle Allen-Cahn equation
# --------------------------------------------------------------------------
def _psi_closed(pd, a, mu, T):
    th = T - pd["T_eut"]
    s = 0.0
    for c in range(2):
        A = pd["A0"][a][c] + pd["A1"][a][c] * th
        ch = pd["c0"][a][c] + pd["m"][a][c] * th
        s += mu[c] ** 2 / (4 * A) + mu[c] * ch
    return -s + pd["L"][a] * th / pd["T_eut"]


def test_p2_binary_textbook_reduction(pv1):
    nx, ny, nz = 24, 20, 6
    x = np.arange(nx)[None, None, :]
    y = np.arange(ny)[None, :, None]
    z = np.arange(nz)[:, None, None]
    f = 0.5 + 0.3 * np.sin(2 * np.pi * x / nx) * np.cos(2 * np.pi * y / ny) + 0.05 * np.cos(np.pi * (z + 0.5) / nz)
    phi = np.zeros((4, nz, ny, nx))
    phi[0] = f
    phi[1] = 1.0 - f
    rng = np.random.default_rng(7)
    mu = 0.05 * rng.uniform(-1, 1, (2, nz, ny, nx))
    pd = dict(pv1, G=0.01, v=0.0)
    p = _params(pd, T0=pv1["T_eut"] - 0.05)
    new = O.phi_sweep(p, phi, mu)
    assert new[2].max() == 0.0 and new[3].max() == 0.0
    # textbook: phi_a^{n+1} = clamp(phi_a + dt/(2 tau eps) [2 gamma eps T Lap7 phi_a
    #            - (T/eps)(16/pi^2) gamma (1 - 2 phi_a) - (dpsi_a - dpsi_b)], 0, 1)
    eps, dt, tau, gam = pd["eps"], pd["dt"], pd["tau"][0], pd["gamma"][0][1]
    fz = np.concatenate([f[:1], f, f[-1:]], axis=0)  # zero-gradient z ghosts
    lap = (np.roll(f, 1, 2) + np.roll(f, -1, 2) + np.roll(f, 1, 1) + np.roll(f, -1, 1)
           + fz[:-2] + fz[2:] - 6 * f)
    out = np.empty_like(f)
    for k in range(nz):
        T = p.T0 + pd["G"] * ((k + 0.5) - 0.0)
        for j in range(ny):
            for i in range(nx):
                fa = f[k, j, i]
                m = mu[:, k, j, i]
                S = fa ** 2 + (1 - fa) ** 2
                dh = 2 * fa * (1 - fa) / S ** 2
                dpsi = dh * (_psi_closed(pd, 0, m, T) - _psi_closed(pd, 1, m, T))
                v = fa + dt / (2 * tau * eps) * (2 * gam * eps * T * lap[k, j, i]
                                                 - (T / eps) * (16 / PI2) * gam * (1 - 2 * fa) - dpsi)
                out[k, j, i] = min(max(v, 0.0), 1.0)
    assert np.abs(new[0] - out).max() <= 1e-14
    assert np.abs(new[1] - (1 - out)).max() <= 1e-14


# --------------------------------------------------------------------------
# P3 — Gibbs simplex: projection against exhaustive active-set enumeration
# --------------------------------------------------------------------------
def _project_enum(x):
    best, bd = None, np.inf
    for r in range(1, 5):
        for S in itertools.combinations(range(4), r):
            y = np.zeros(4)
            th = (sum(x[s] for s in S) - 1.0) / r
            for s in S:
                y[s] = x[s] - th
            if y.min() < -1e-15:
                continue
            d = np.sum((y - x) ** 2)
            if d < bd:
                best, bd = y, d
    return best


def test_p3_projection_matches_enumeration():
    rng = np.random.default_rng(3)
    for _ in range(2000):
        x = rng.normal(0.25, 0.6, 4)
        assert np.abs(O.project(x) - _project_enum(x)).max() <= 1e-15
    # examples of SPEC.md:328-330
    assert np.array_equal(O.project([0.5, 0.5, 0, 0]), [0.5, 0.5, 0, 0])
    assert np.array_equal(O.project([1.1, -0.1, 0, 0]), [1, 0, 0, 0])
    assert np.allclose(O.project([0.3] * 4), [0.25] * 4, atol=1e-16)


def test_p3_simplex_invariants_on_voronoi_run(pv1):
    cfg = gen.load_config("c1")
    spec = gen.spec_from_config(cfg, 16, 16)
    spec.layer_height = 6
    spec.n_seeds = 5
    spec.mu_noise = 1e-2
    phi, mu = gen.generate(spec, 16, 16, 16)
    p = _params(pv1, layer_height=6)
    ph, m, _ = O.run(p, phi, mu, 20)
    assert ph.min() == 0.0 or ph.min() > 0.0
    assert ph.min() >= 0.0
    assert np.abs(ph.sum(0) - 1.0).max() <= 4.5e-16
    # cells that were exact vertices with exact-vertex neighbourhoods stay bit-exact
    liq = (phi[3] == 1.0)
    liq_nb = liq.copy()
    for ax in (0, 1, 2):
        for s in (1, -1):
            liq_nb &= np.roll(liq, s, axis=ax)
    top = liq_nb[-6:]
    assert top.any() and np.all(ph[3][-6:][top] == 1.0)


# --------------------------------------------------------------------------
# P4 — solute conservation (A8, A9, A10, A13; Appendix B)
# --------------------------------------------------------------------------
def _solute(pd, p, phi, mu, zorig=0, n=0):
    nz = phi.shape[1]
    T = p.T0 + pd["G"] * ((np.arange(nz) + zorig + 0.5) - pd["v"] * n * pd["dt"])
    th = (T - pd["T_eut"])[:, None, None]
    S = (phi ** 2).sum(0)
    tot = np.zeros(2)
    for c in range(2):
        cc = 0.0
        for a in range(4):
            A = pd["A0"][a][c] + pd["A1"][a][c] * th
            ch = pd["c0"][a][c] + pd["m"][a][c] * th
            cc = cc + phi[a] ** 2 / S * (mu[c] / (2 * A) + ch)
        tot[c] = cc.sum()
    return tot


def _p4_drift(pd, nsteps=100):
    cfg = gen.load_config("c2")
    spec = gen.spec_from_config(cfg, 16, 16)
    spec.layer_height, spec.n_seeds, spec.mu_noise = 8, 6, 5e-2
    phi, mu = gen.generate(spec, 16, 16, 16)
    p = _params(pd, layer_height=9)   # undercooled front: it moves
    c0 = _solute(pd, p, phi, mu)
    ph, m, _ = O.run(p, phi, mu, nsteps)
    c1 = _solute(pd, p, ph, m, n=nsteps)
    moved = np.abs(ph - phi).max()
    return np.abs(c1 - c0).max() / np.abs(c0).max(), moved


def test_p4_conservation_v0(pv1):
    drift, moved = _p4_drift(dict(pv1, v=0.0, G=0.01))
    assert moved > 0.05
    assert drift <= 1e-13, drift


def test_p4_conservation_moving_T_with_A1_zero(pv1):
    pd = dict(pv1, v=0.5, G=0.01, A1=[[0.0, 0.0]] * 4)
    drift, _ = _p4_drift(pd)
    assert drift <= 1e-13, drift


def test_p4_control_discriminates(pv1):
    # moving T with T-dependent A is NOT conserved (the test can fail)
    drift, _ = _p4_drift(dict(pv1, v=0.5, G=0.01), nsteps=20)
    assert drift > 1e-9


# --------------------------------------------------------------------------
# P5 — Fourier decay in the pure-diffusion limit (closed form)
# --------------------------------------------------------------------------
def test_p5_fourier_decay(pv1):
    nx, ny, nz, kx, ky, kz = 16, 12, 10, 2, 1, 3
    pd = dict(pv1, G=0.0)
    p = _params(pd, T0=1.1)
    i = np.arange(nx)[None, None, :]
    j = np.arange(ny)[None, :, None]
    k = np.arange(nz)[:, None, None]
    mode = np.cos(2 * np.pi * kx * i / nx) * np.cos(2 * np.pi * ky * j / ny) * np.cos(np.pi * kz * (k + 0.5) / nz)
    phi = np.zeros((4, nz, ny, nx))
    phi[3] = 1.0
    amp = (0.3, -0.2)
    mu = np.stack([amp[0] * mode, amp[1] * mode])
    n = 100
    ph, m, _ = O.run(p, phi, mu, n)
    assert np.array_equal(ph, phi)
    for c in range(2):
        D = pd["D"][3][c]
        lam = 1 - 4 * pd["dt"] * D * (np.sin(np.pi * kx / nx) ** 2 + np.sin(np.pi * ky / ny) ** 2
                                      + np.sin(np.pi * kz / (2 * nz)) ** 2)
        expect = amp[c] * lam ** n * mode
        assert np.abs(m[c] - expect).max() / abs(amp[c] * lam ** n) <= 1e-13


# --------------------------------------------------------------------------
# P6 — permutation symmetry of identical phases (PARAMS-sym)
# --------------------------------------------------------------------------
def test_p6_permutation_symmetry(psym):
    cfg = gen.load_config("c1")
    spec = gen.spec_from_config(cfg, 12, 12)
    spec.layer_height, spec.n_seeds, spec.mu_noise = 5, 6, 1e-2
    phi, mu = gen.generate(spec, 12, 12, 12)
    p = _params(psym, layer_height=6)
    a, ma, _ = O.run(p, phi, mu, 30)
    sw = phi[[1, 0, 2, 3]]
    b, mb, _ = O.run(p, sw, mu, 30)
    assert np.abs(a[[1, 0, 2, 3]] - b).max() <= 1e-14
    assert np.abs(ma - mb).max() <= 1e-14
    assert np.abs(a - phi).max() > 1e-3


# --------------------------------------------------------------------------
# P7 — bulk fixed point (bit-exact)
# --------------------------------------------------------------------------
@pytest.mark.parametrize("phase", [0, 1, 2, 3])
def test_p7_bulk_fixed_point(pv1, phase):
    pd = dict(pv1, v=0.0)
    p = _params(pd, layer_height=3)
    phi = np.zeros((4, 6, 5, 4))
    phi[phase] = 1.0
    mu = np.zeros((2, 6, 5, 4))
    mu[0], mu[1] = 0.013, -0.021
    ph, m, _ = O.run(p, phi, mu, 5)
    assert np.array_equal(ph, phi) and np.array_equal(m, mu)


# --------------------------------------------------------------------------
# P8 — term identities (finite differences of the potentials the oracle uses)
# --------------------------------------------------------------------------
def _fd(f, x, h=1e-6):
    g = np.zeros_like(x)
    for d in range(x.size):
        e = np.zeros_like(x)
        e[d] = h
        g[d] = (f(x + e) - f(x - e)) / (2 * h)
    return g


def test_p8_thermo_identities(pv1):
    p = _params(pv1, layer_height=0)
    rng = np.random.default_rng(11)
    for a in range(4):
        for c in range(2):
            assert O.conc(p, a, c, 0.0, pv1["T_eut"]) == pv1["c0"][a][c]
        assert O.psi(p, a, [0.0, 0.0], pv1["T_eut"]) == 0.0
        for _ in range(10):
            mu = rng.uniform(-0.5, 0.5, 2)
            T = rng.uniform(0.9, 1.1)
            dps = _fd(lambda m: O.psi(p, a, m, T), mu)
            cc = np.array([O.conc(p, a, c, mu[c], T) for c in range(2)])
            assert np.abs(dps + cc).max() <= 1e-8 * max(1.0, np.abs(cc).max())
    for _ in range(20):
        ph = rng.dirichlet(np.ones(4))
        assert abs(O.interp_h(ph).sum() - 1.0) <= 4.5e-16
        mu = rng.uniform(-0.3, 0.3, 2)
        T = 0.97
        tot = lambda x: float(np.dot(O.interp_h(x), [O.psi(p, b, mu, T) for b in range(4)]))
        g = _fd(tot, ph)
        for a in range(4):
            assert abs(O.dpsi_dphi(p, ph, mu, T, a) - g[a]) <= 1e-8
        g = _fd(lambda x: O.omega(p, x), ph)
        for a in range(4):
            assert abs(O.domega(p, ph, a) - g[a]) <= 1e-8


def test_p8_omega_closed_form(pv1):
    p = _params(pv1)
    # two-phase reduction and vertex nullity
    assert O.omega(p, [1, 0, 0, 0]) == 0.0
    assert abs(O.domega(p, [0.3, 0.7, 0, 0], 0) - 16 / PI2 * 0.7) <= 1e-15
    assert abs(O.domega(p, [1, 0, 0, 0], 2) - 16 / PI2 * 1.0) <= 1e-15
    # triple term: d/dphi_a at (1/3,1/3,1/3,0): 16/pi^2 * 2/3 + gamma3 * (1/3)^2
    v = O.domega(p, [1 / 3, 1 / 3, 1 / 3, 0], 0)
    assert abs(v - (16 / PI2 * 2 / 3 + 10.0 / 9.0)) <= 1e-14


@pytest.mark.parametrize("delta", [0.0, 0.05])
def test_p8_gradient_energy_derivative(pv1, delta):
    p = _params(pv1, aniso=delta > 0, delta_sl=delta)
    rng = np.random.default_rng(5)
    for a, b in [(0, 3), (1, 2), (2, 3)]:
        for _ in range(10):
            q = rng.normal(0, 0.2, 3)
            g = O.pair_grad(p, a, b, q)
            fd = _fd(lambda x: O.pair_energy(p, a, b, x), q, h=1e-6)
            assert np.abs(g - fd).max() <= 1e-8 * max(1.0, np.abs(g).max())
    assert np.array_equal(O.pair_grad(p, 0, 3, np.zeros(3)), np.zeros(3))
    # cubic invariance of e(q) under axis permutations and sign flips
    q = np.array([0.3, -0.1, 0.2])
    e = O.pair_energy(p, 0, 3, q)
    for perm in itertools.permutations(range(3)):
        assert abs(O.pair_energy(p, 0, 3, -q[list(perm)]) - e) <= 1e-16


# --------------------------------------------------------------------------
# P10 / P11 — anti-trapping current zeros and single-face properties
# --------------------------------------------------------------------------
def _front_state(nz=16, shift=0.0, a=0):
    z = np.arange(nz) + 0.5
    W = 4.0
    d = 8.0 + shift - z
    s = np.where(d >= W / 2, 1.0, np.where(d <= -W / 2, 0.0, 0.5 * (1 + np.sin(np.pi * d / W))))
    phi = np.zeros((4, nz, 3, 3))
    phi[a] = s[:, None, None]
    phi[3] = 1.0 - phi[a]
    return phi


def test_p10_jat_zero_for_stationary_or_liquid_free(pv1):
    p = _params(pv1, layer_height=8)
    phi = _front_state()
    mu = np.full((2, 16, 3, 3), 0.01)
    for k in range(15):
        for d in range(3):
            _, J = O.mu_face(p, phi, phi, mu, 1, 1, k, d)   # phi^{n+1} = phi^n
            assert np.array_equal(J, [0.0, 0.0])
    sol = np.zeros_like(phi)
    sol[0, :8] = 1.0
    sol[1, 8:] = 1.0
    sol2 = sol.copy()
    sol2[0, 7], sol2[1, 7] = 0.6, 0.4
    for k in range(15):
        _, J = O.mu_face(p, sol, sol2, mu, 1, 1, k, 2)      # no liquid
        assert np.array_equal(J, [0.0, 0.0])


def test_p11_jat_single_face_properties(pv1):
    p = _params(pv1, layer_height=8)
    old = _front_state(shift=0.0)
    new = _front_state(shift=0.05)       # solid advances into the liquid: dphi_alpha/dt > 0
    mu = np.zeros((2, 16, 3, 3))
    def dc_face(k):  # (c^l - c^alpha) averaged over the face's two cells (own-plane T)
        out = np.zeros(2)
        for kk in (k, k + 1):
            T = p.T0 + pv1["G"] * (kk + 0.5)
            out += 0.5 * np.array([O.conc(p, 3, c, 0.0, T) - O.conc(p, 0, c, 0.0, T) for c in range(2)])
        return out
    seen = 0
    for k in range(15):
        dc = dc_face(k)
        for d in (0, 1):
            _, J = O.mu_face(p, old, new, mu, 1, 1, k, d)
            assert np.array_equal(J, [0.0, 0.0])       # tangential faces of a 1D front
        _, J = O.mu_face(p, old, new, mu, 1, 1, k, 2)
        if np.any(J != 0):
            seen += 1
            # parallel to the normal and proportional to (c^l - c^alpha), pointing
            # from the solid towards the liquid for c^l > c^alpha
            assert abs(J[0] / J[1] - dc[0] / dc[1]) <= 1e-12 * abs(dc[0] / dc[1])
            assert np.all(np.sign(J) == np.sign(dc))
    assert seen >= 2
    # magnitude at one face, Eq. (4) written out for a 1D alpha|l profile:
    k = 7
    pa = 0.5 * (new[0, k, 1, 1] + new[0, k + 1, 1, 1])
    pl = 0.5 * (new[3, k, 1, 1] + new[3, k + 1, 1, 1])
    pdot = 0.5 * ((new[0, k] - old[0, k]) + (new[0, k + 1] - old[0, k + 1]))[1, 1] / pv1["dt"]
    hl = pl ** 2 / (pa ** 2 + pl ** 2)
    # n_a . n_l = -1 and n_a,z = -1 for a solid below the liquid
    expect = math.pi * pv1["eps"] / 4 * pa * hl / math.sqrt(pa * pl) * pdot * (-1.0) * (-1.0) * dc_face(k)
    _, J = O.mu_face(p, old, new, mu, 1, 1, k, 2)
    assert np.abs(J - expect).max() <= 1e-14 * np.abs(expect).max()


# --------------------------------------------------------------------------
# P12 — undercooling sign (A1, O2)
# --------------------------------------------------------------------------
def _front_pos(phi):
    col = phi[3, :, 0, 0]
    k = int(np.argmax(col >= 0.5))
    return (k - 1) + (0.5 - col[k - 1]) / (col[k] - col[k - 1]) + 0.5


def test_p12_undercooling_sign(pv1):
    vel = []
    for dT in (0.0, 0.05, 0.1, 0.2):
        pd = dict(pv1, G=0.0, v=0.0)
        p = _params(pd, T0=pv1["T_eut"] - dT)
        phi = np.zeros((4, 32, 2, 2))
        z = np.arange(32) + 0.5
        s = np.clip(0.5 * (1 + np.sin(np.pi * np.clip((12 - z) / 4, -0.5, 0.5))), 0, 1)
        phi[0] = s[:, None, None]
        phi[3] = 1 - phi[0]
        mu = np.zeros((2, 32, 2, 2))
        z0 = _front_pos(phi)
        ph, _, _ = O.run(p, phi, mu, 300)
        vel.append(_front_pos(ph) - z0)
    assert abs(vel[0]) < 0.02
    assert vel[1] > 0 and vel[1] < vel[2] < vel[3], vel


# --------------------------------------------------------------------------
# P13 — cubic symmetry of the anisotropic step (A3)
# --------------------------------------------------------------------------
def test_p13_cubic_symmetry_anisotropic(pv1):
    cfg = gen.load_config("c5")
    spec = gen.spec_from_config(cfg, 12, 12)
    spec.layer_height, spec.n_seeds, spec.mu_noise = 6, 5, 1e-2
    phi, mu = gen.generate(spec, 12, 12, 12)
    p = _params(pv1, layer_height=7, aniso=True, delta_sl=0.05)
    a, ma, _ = O.run(p, phi, mu, 10)
    t = lambda x: np.ascontiguousarray(np.swapaxes(x, 2, 3))
    b, mb, _ = O.run(p, t(phi), t(mu), 10)
    assert np.abs(t(b) - a).max() <= 1e-14
    assert np.abs(t(mb) - ma).max() <= 1e-14
    iso = _params(pv1, layer_height=7)
    c, _, _ = O.run(iso, phi, mu, 10)
    assert np.abs(c - a).max() > 1e-6   # the anisotropy is active


# --------------------------------------------------------------------------
# sampled one-step map == whole-domain step
# --------------------------------------------------------------------------
def test_step_cells_matches_full_step(pv1):
    cfg = gen.load_config("c2")
    spec = gen.spec_from_config(cfg, 10, 9)
    spec.layer_height, spec.n_seeds = 4, 4
    phi, mu = gen.generate(spec, 10, 9, 8)
    p = _params(pv1, layer_height=4, aniso=True, delta_sl=0.05)
    ph, m = O.step(p, phi, mu, n=3, zorig=2)
    rng = np.random.default_rng(0)
    cells = np.concatenate([[0, 10 * 9 * 8 - 1], rng.integers(0, 10 * 9 * 8, 40)])
    po, mo = O.step_cells(p, phi, mu, cells, n=3, zorig=2)
    assert np.array_equal(po, ph.reshape(4, -1)[:, cells])
    assert np.array_equal(mo, m.reshape(2, -1)[:, cells])


def test_p14_roofline_arithmetic():
    # 80 GiB/s : 680 B/LUP = 126.3 MLUP/s; 4.2 MLUP/s * 1384 FLOP = 5.8 GFLOP/s
    assert round(80 * 2 ** 30 / 680 / 1e6, 1) == 126.3
    assert round(4.2e6 * 1384 / 1e9, 1) == 5.8
    assert round(5.8 / 21.6 * 100) == 27


# ---------------------------------------------------------------------------
# P15: FP32 checkpoint format (NEXT-3)
# ---------------------------------------------------------------------------
def _golden_bytes(name):
    import os
    path = os.path.join(os.path.dirname(__file__), "golden", name)
    hexs = " ".join(line.split("#", 1)[0] for line in open(path))
    return bytes.fromhex("".join(hexs.split()))


def test_p15_checkpoint_matches_hand_assembled_bytes():
    from oracle import checkpoint as CK
    phi = np.array([[1.0, 0.1], [0.0, 1 / 3], [0.0, 0.5], [0.0, 0.0625]]).reshape(4, 1, 1, 2)
    mu = np.array([[1 + 2.0 ** -24, 1 + 3 * 2.0 ** -24], [-2.0, 1e-50]]).reshape(2, 1, 1, 2)
    want = _golden_bytes("checkpoint_2x1x1.hex")
    assert len(want) == 72 + 6 * 2 * 4
    assert CK.encode(phi, mu, dx=1.0, t=0.3, step=10, z_origin=7) == want
    hdr, p32, m32 = CK.decode(want)
    assert hdr == dict(nx=2, ny=1, nz=1, n_phases=4, n_mu=2, dx=1.0, t=0.3, step=10, z_origin=7)
    # round-to-nearest-even ties and underflow, read back as exact binary32 values
    assert m32[0, 0, 0, 0] == 1.0 and m32[0, 0, 0, 1] == 1 + 2.0 ** -22 and m32[1, 0, 0, 1] == 0.0


def test_p15_checkpoint_roundtrip_is_binary32_cast_and_size(tmp_path):
    from oracle import checkpoint as CK
    rng = np.random.default_rng(5)
    phi = rng.standard_normal((4, 5, 3, 7)) * 10.0 ** rng.integers(-44, 36, (4, 5, 3, 7))
    mu = rng.standard_normal((2, 5, 3, 7))
    p = tmp_path / "c.pfcp"
    CK.write_checkpoint(p, phi, mu, dx=0.5, t=1.25, step=3, z_origin=11)
    assert p.stat().st_size == 72 + 6 * 5 * 3 * 7 * 4
    hdr, p32, m32 = CK.decode(p.read_bytes())
    assert (hdr["nx"], hdr["ny"], hdr["nz"], hdr["step"], hdr["z_origin"]) == (7, 3, 5, 3, 11)
    # each stored value is the float32 nearest to the original (ties: even); check
    # by brute force against its two float32 neighbours
    for orig, got in ((phi, p32), (mu, m32)):
        g = got.astype(np.float64)
        up = np.nextafter(got, np.float32(np.inf)).astype(np.float64)
        dn = np.nextafter(got, np.float32(-np.inf)).astype(np.float64)
        fin = np.isfinite(g) & (np.abs(orig) < 3e38)
        assert np.all(np.abs(orig - g)[fin] <= np.abs(orig - up)[fin])
        assert np.all(np.abs(orig - g)[fin] <= np.abs(orig - dn)[fin])
    # size of a 64^3 checkpoint
    assert len(CK.encode(np.zeros((4, 64, 64, 64)), np.zeros((2, 64, 64, 64)), 1.0, 0.0, 0, 0)) == 72 + 6 * 64 ** 3 * 4


def test_p15_checkpoint_rejects_bad_files():
    from oracle import checkpoint as CK
    good = _golden_bytes("checkpoint_2x1x1.hex")
    with pytest.raises(CK.CheckpointError):
        CK.decode(b"XFCP0001" + good[8:])
    with pytest.raises(CK.CheckpointError):
        CK.decode(good[:-1])
    with pytest.raises(CK.CheckpointError):
        CK.decode(good[:40])


# ---------------------------------------------------------------------------
# P16: marching cubes (NEXT-4, reading R26)
# ---------------------------------------------------------------------------
def _tri_normals(pos):
    return np.cross(pos[:, 1] - pos[:, 0], pos[:, 2] - pos[:, 0])


def _unwrap(pos, Lx, Ly):
    """Minimal-image copy of each triangle (vertex x, y are wrapped into the
    periodic box, so a triangle on the seam has vertices on both sides)."""
    pos = pos.copy()
    for ax, L in ((0, Lx), (1, Ly)):
        d = pos[:, 1:, ax] - pos[:, :1, ax]
        pos[:, 1:, ax] -= np.round(d / L) * L
    return pos


def _unpaired_directed_edges(ids, skip=lambda a, b: False):
    from collections import Counter
    E = Counter()
    for tr in ids:
        for s in range(3):
            E[(int(tr[s]), int(tr[(s + 1) % 3]))] += 1
    return [e for e in E if not skip(*e) and (E[e] != 1 or E.get((e[1], e[0]), 0) != 1)]


def test_p16_uniform_field_gives_empty_mesh():
    from oracle import mesh as MC
    for v in (0.0, 0.3, 0.5, 0.9, 1.0):
        ids, pos = MC.marching_cubes(np.full((5, 4, 6), v))
        assert ids.shape == (0, 3) and pos.shape == (0, 3, 3)


def test_p16_plane_area_and_orientation():
    from oracle import mesh as MC
    NX, NY, NZ, dx = 7, 5, 6, 0.5
    z = np.arange(NZ) + 0.5
    phi = np.broadcast_to((0.5 + 0.2 * (2.8 - z))[:, None, None], (NZ, NY, NX))   # solid below z = 2.8
    ids, pos = MC.marching_cubes(phi, dx=dx)
    assert pos[:, :, :2].min() >= 0.5 * dx and pos[:, :, :2].max() <= (max(NX, NY) - 0.5) * dx
    n = _tri_normals(_unwrap(pos, NX * dx, NY * dx))
    assert np.allclose(pos[:, :, 2], 2.8 * dx, rtol=0, atol=1e-14)
    assert abs(0.5 * np.linalg.norm(n, axis=1).sum() - NX * NY * dx * dx) < 1e-12
    assert np.all(n[:, 2] > 0) and np.allclose(n[:, :2], 0)      # out of the phase: +z


def test_p16_sphere_area_volume_euler():
    # radius 10 dx sphere -> closed, chi = 2, area / volume within 2 %
    from oracle import mesh as MC
    N, R = 32, 10.0
    z, y, x = np.meshgrid(*(np.arange(N) + 0.5,) * 3, indexing="ij")
    r = np.sqrt((x - 16.2) ** 2 + (y - 15.9) ** 2 + (z - 16.1) ** 2)
    ids, pos = MC.marching_cubes(np.clip(0.5 - 0.25 * (r - R), 0, 1))
    n = _tri_normals(pos)
    area = 0.5 * np.linalg.norm(n, axis=1).sum()
    vol = np.einsum("ij,ij->i", pos[:, 0], n).sum() / 6
    assert abs(area / (4 * math.pi * R * R) - 1) < 0.02
    assert abs(vol / (4 / 3 * math.pi * R ** 3) - 1) < 0.02      # > 0: normals point outward
    assert not _unpaired_directed_edges(ids)
    V = len(set(ids.ravel().tolist()))
    E = 3 * len(ids) // 2
    assert V - E + len(ids) == 2


@pytest.mark.parametrize("seed", range(6))
def test_p16_random_fields_watertight_and_oriented(seed):
    # every directed mesh edge meets its reverse exactly once (periodic x/y);
    # only segments inside the bottom / top sample planes stay open.  Random
    # fields hit the face-ambiguous configurations many times.
    from oracle import mesh as MC
    rng = np.random.default_rng(seed)
    NX, NY, NZ = 9, 8, 7
    phi = rng.random((NZ, NY, NX))
    ids, pos = MC.marching_cubes(phi)
    assert len(ids) > 100

    def plane_of(e):
        ax, lin = e % 3, e // 3
        k = lin // (NX * NY)
        return k if ax != 2 else -1

    def skip(a, b):
        pa, pb = plane_of(a), plane_of(b)
        return pa == pb and pa in (0, NZ - 1)

    assert not _unpaired_directed_edges(ids, skip)
    # vertices: on their edge, where the linear interpolant equals iso
    for tr, ps in zip(ids[:200], pos[:200]):
        for e, p in zip(tr, ps):
            ax, lin = e % 3, e // 3
            lo = [lin % NX, (lin // NX) % NY, lin // (NX * NY)]
            hi = list(lo)
            hi[ax] += 1
            f0 = phi[lo[2], lo[1], lo[0]]
            f1 = phi[hi[2] % NZ, hi[1] % NY, hi[0] % NX]
            t = p[ax] - (lo[ax] + 0.5)
            assert 0 <= t <= 1 and abs(f0 + t * (f1 - f0) - 0.5) < 1e-12
            for q in range(3):
                if q != ax:
                    assert p[q] == lo[q] + 0.5


def test_p16_normals_point_down_the_gradient():
    from oracle import mesh as MC
    rng = np.random.default_rng(3)
    N = 24
    z, y, x = np.meshgrid(*(np.arange(N) + 0.5,) * 3, indexing="ij")
    phi = 0.5 + 0.3 * np.sin(2 * np.pi * x / N) * np.cos(2 * np.pi * y / N) + 0.1 * np.sin(2 * np.pi * z / N + 0.3)
    ids, pos = MC.marching_cubes(phi)
    pos = _unwrap(pos, N, N)
    c = pos.mean(axis=1)
    gx = 0.3 * (2 * np.pi / N) * np.cos(2 * np.pi * c[:, 0] / N) * np.cos(2 * np.pi * c[:, 1] / N)
    gy = -0.3 * (2 * np.pi / N) * np.sin(2 * np.pi * c[:, 0] / N) * np.sin(2 * np.pi * c[:, 1] / N)
    gz = 0.1 * (2 * np.pi / N) * np.cos(2 * np.pi * c[:, 2] / N + 0.3)
    dots = np.einsum("ij,ij->i", _tri_normals(pos), np.stack([gx, gy, gz], 1))
    assert np.mean(dots < 0) > 0.99


def test_p16_cube_cases_exhaustive():
    # all 256 corner configurations: the triangle vertices are exactly the
    # crossing edges, each triangle's edges lie in the cube, counts <= 5
    from oracle import mesh as MC
    for case in range(256):
        ins = [(case >> c) & 1 == 1 for c in range(8)]
        tris = MC.cube_triangles(ins)
        cross = {e for e, (a, b, _) in enumerate(MC.EDGES) if ins[a] != ins[b]}
        used = {e for t in tris for e in t}
        assert used == cross, case
        assert len(tris) <= 5
        assert all(len(set(t)) == 3 for t in tris)
        # the cube's patch is a surface with its boundary on the cube faces:
        # a triangle side lying in a cube face is used once, any other side
        # (a fan diagonal through the interior) exactly once in each direction
        from collections import Counter
        sides = Counter((t[s], t[(s + 1) % 3]) for t in tris for s in range(3))
        for (a, b), n in sides.items():
            on_face = any(set(MC.EDGES[a][:2]) | set(MC.EDGES[b][:2]) <= set(f) for f in MC.FACES)
            assert n == 1 and (sides.get((b, a), 0) == (0 if on_face else 1)), (case, a, b)


def test_committed_flop_counts_match_oracle():
    # bench.py's roofline reads profiles/flop_counts.json (written by
    # tools/count_flops.py); it must be the oracle's own count
    import json
    import os
    from inputs import gen
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    d = json.load(open(os.path.join(root, "profiles", "flop_counts.json")))["configs"]
    pd = gen.load_params("v1")
    for name, fl in d.items():
        cfg = gen.load_config(name)
        ref = O.count_flops(O.make_params(pd, layer_height=cfg["init"]["layer_height"], aniso=cfg.get("aniso", False),
                                          delta_sl=cfg.get("delta_sl")))
        assert {k: int(v) for k, v in ref.items()} == fl, name


def test_p17_window_transparency_within_light_cone(pv1):
    # O7 / reading A16 pinned against "the same physics in a taller box": a
    # window run (the front forced past 2/3 height so it shifts) equals, bit for
    # bit, a non-windowed run of a taller domain on the planes that neither the
    # bottom ghost nor the liquid fill can reach in M steps (the stencil of one
    # step reaches 2 planes: the mu-sweep reads phi^{n+1}, which read phi^n)
    from inputs import gen
    cfg = gen.load_config("c2")
    nx, ny, nz, extra, M = 12, 12, 48, 6, 6
    spec = gen.spec_from_config(cfg, nx, ny)
    spec.layer_height, spec.n_seeds = 33.5, 4
    tall_phi, tall_mu = gen.generate(spec, nx, ny, nz + extra)
    p = O.make_params(pv1, layer_height=33.5)
    shifts = []
    wphi, wmu, zorig = O.run(p, tall_phi[:, :nz], tall_mu[:, :nz], M, window_on=True, shifts=shifts)
    tphi, tmu, _ = O.run(p, tall_phi, tall_mu, M)
    assert zorig == len(shifts) >= 1
    lo, hi = 2 * M + 1, nz - 2 * M - 1
    assert np.array_equal(wphi[:, lo:hi], tphi[:, lo + zorig:hi + zorig])
    assert np.array_equal(wmu[:, lo:hi], tmu[:, lo + zorig:hi + zorig])
    # and the shift really moved the data: without the origin offset they differ
    assert not np.array_equal(wphi[:, lo:hi], tphi[:, lo:hi])


@pytest.mark.parametrize("aniso", [False, True])
def test_p18_mirror_symmetry(pv1, aniso):
    # the step commutes with the mirrors x -> -x and y -> -y (periodic axes; the
    # cubic anisotropy is mirror-symmetric): catches a face flux or gradient
    # taken from the wrong side in one direction, which x<->y swaps (P13) miss
    cfg = gen.load_config("c5" if aniso else "c2")
    spec = gen.spec_from_config(cfg, 12, 10)
    spec.layer_height, spec.n_seeds, spec.mu_noise = 6, 5, 1e-2
    phi, mu = gen.generate(spec, 12, 10, 12)
    p = _params(pv1, layer_height=7, aniso=aniso, delta_sl=0.05 if aniso else None)
    a, ma, _ = O.run(p, phi, mu, 10)
    assert np.abs(a - phi).max() > 1e-3
    for axis in (3, 2):          # x, y
        mr = lambda x: np.ascontiguousarray(np.flip(x, axis=axis))   # i -> N-1-i
        b, mb, _ = O.run(p, mr(phi), mr(mu), 10)
        assert np.abs(mr(b) - a).max() <= 1e-14, axis
        assert np.abs(mr(mb) - ma).max() <= 1e-14, axis


# --------------------------------------------------------------------------
# P19 — the dc/dT source of Eq. (3) against the exact solution of the
# temperature-driven liquid (north_star "dT/dt source term")
# --------------------------------------------------------------------------
def _kappa_run(pd, T0, mu0, dt, t_end):
    p = O.make_params(dict(pd, dt=dt), T0=T0)
    phi = np.zeros((4, 1, 2, 2))
    phi[3] = 1.0
    mu = np.empty((2, 1, 2, 2))
    mu[0], mu[1] = mu0
    nsteps = int(round(t_end / dt))
    ph, m, _ = O.run(p, phi, mu, nsteps)
    assert np.array_equal(ph, phi)           # bulk liquid stays a vertex (P7)
    return m[:, 0, 0, 0]


@pytest.mark.parametrize("m_l", [[0.2, -0.1], [0.0, 0.0]])
def test_p19_dcdT_source_converges_to_exact_solution(pv1, m_l):
    # One uniform liquid layer (no gradients, no phase change) under a moving
    # frozen temperature: Eq. (3) reduces to chi dmu/dt = -(dc/dT) dT/dt, whose
    # exact solution conserves c = mu/(2A(T)) + c_hat(T):
    #   mu(t) = 2 A(T(t)) (c_0 - c_hat(T(t))),  T(t) = T0 + G (z - v t).
    # With m = 0 it is mu(t) = mu_0 A(T(t))/A(T_0), linear in t, and explicit
    # Euler reproduces it exactly (mu^n = K A^n => mu^{n+1} = K A^{n+1}): only
    # the kappa = 2 A1/(2A)^2 term of dc/dT drives it.  With m != 0 mu(t) is
    # quadratic in t and Euler converges at first order in dt.
    pd = dict(pv1, G=0.1, v=1.0, m=[list(r) for r in pv1["m"][:3]] + [m_l])
    T0, mu0, t_end = pv1["T_eut"] + 0.02, np.array([0.4, -0.3]), 2.0
    z = 0.5                                   # cell-centre height of plane 0

    def exact(t):
        T = T0 + pd["G"] * (z - pd["v"] * t)
        th0, th = T0 + pd["G"] * z - pd["T_eut"], T - pd["T_eut"]
        out = np.empty(2)
        for c in range(2):
            A_0 = pd["A0"][3][c] + pd["A1"][3][c] * th0
            A_t = pd["A0"][3][c] + pd["A1"][3][c] * th
            c0 = mu0[c] / (2 * A_0) + pd["c0"][3][c] + pd["m"][3][c] * th0
            out[c] = 2 * A_t * (c0 - (pd["c0"][3][c] + pd["m"][3][c] * th))
        return out

    ref = exact(t_end)
    assert np.abs(ref - mu0).max() > 1e-2     # the source moves mu by O(1e-2)
    errs = [np.abs(_kappa_run(pd, T0, mu0, dt, t_end) - ref).max() for dt in (0.02, 0.01, 0.005)]
    if m_l == [0.0, 0.0]:
        assert max(errs) <= 1e-14, errs
    else:
        assert errs[2] <= 1e-3, errs
        for e1, e2 in zip(errs, errs[1:]):
            assert 1.9 <= e1 / e2 <= 2.1, errs    # first order in dt


# --------------------------------------------------------------------------
# P20 — face gradients are exact for linear fields (D3C19 tangential averages,
# reading R4 / SURVEY.md §8(c) O4.5, O5.8): the discrete anti-trapping current
# and the anisotropic phi face flux then equal their continuous formulas at
# the face centre
# --------------------------------------------------------------------------
def _linear_phi(n, grads, base, centre):
    """phi_a = base_a + grads_a . (x - centre) on an n^3 grid (cell centres at
    integer indices), phi_l = 1 - sum of the solids."""
    k, j, i = np.meshgrid(*(np.arange(n),) * 3, indexing="ij")
    phi = np.zeros((4, n, n, n))
    for a in range(3):
        g = grads[a]
        phi[a] = base[a] + g[0] * (i - centre[0]) + g[1] * (j - centre[1]) + g[2] * (k - centre[2])
    phi[3] = 1.0 - phi[:3].sum(0)
    return phi


def test_p20_antitrapping_exact_on_linear_fields(pv1):
    n, c = 9, (4, 4, 4)
    grads = [np.array([0.010, 0.020, -0.015]), np.array([-0.012, 0.008, 0.011]), np.zeros(3)]
    base = [0.30, 0.20, 0.05]
    new = _linear_phi(n, grads, base, c)
    old = _linear_phi(n, grads, [0.30 - 0.004, 0.20 + 0.003, 0.05], c)   # d phi/dt uniform per phase
    assert new.min() > 0 and old.min() > 0
    rng = np.random.default_rng(3)
    mu = rng.uniform(-0.2, 0.2, (2, n, n, n))
    pd = dict(pv1, G=0.01, v=0.3)
    p = O.make_params(pd, layer_height=2.0)
    step_n, zorig = 4, 1
    gl = -(grads[0] + grads[1] + grads[2])           # liquid gradient
    for d in range(3):
        e = np.eye(3, dtype=int)[d]
        lo = np.array(c)
        hi = lo + e
        xf = lo + 0.5 * e                            # face centre
        ph = np.array([base[a] + grads[a] @ (xf - c) for a in range(3)])
        ph = np.append(ph, 1.0 - ph.sum())
        hl = ph[3] ** 2 / (ph ** 2).sum()
        nl = gl / np.linalg.norm(gl)
        expect = np.zeros(2)
        for a in range(2):                           # gamma has no gradient: its guard closes
            na = grads[a] / np.linalg.norm(grads[a])
            pdot = (new[a, 0, 0, 0] - old[a, 0, 0, 0]) / pd["dt"]
            w = math.pi * pd["eps"] / 4 * ph[a] * hl / math.sqrt(ph[a] * ph[3]) * pdot * (na @ nl) * na[d]
            for cc in range(2):
                dc = 0.0
                for cell in (lo, hi):
                    T = p.T0 + pd["G"] * ((cell[2] + zorig + 0.5) - pd["v"] * step_n * pd["dt"])
                    m = mu[cc, cell[2], cell[1], cell[0]]
                    dc += 0.5 * (O.conc(p, 3, cc, m, T) - O.conc(p, a, cc, m, T))
                expect[cc] += w * dc
        _, J = O.mu_face(p, old, new, mu, int(lo[0]), int(lo[1]), int(lo[2]), d, n=step_n, zorig=zorig)
        assert np.abs(J - expect).max() <= 1e-13 * np.abs(expect).max(), (d, J, expect)


def test_p20_anisotropic_phi_face_exact_on_linear_fields(pv1):
    n, c = 9, (4, 4, 4)
    grads = [np.array([0.010, 0.020, -0.015]), np.array([-0.012, 0.008, 0.011]), np.array([0.004, -0.009, 0.006])]
    base = [0.30, 0.20, 0.15]
    phi = _linear_phi(n, grads, base, c)
    p = _params(pv1, aniso=True, delta_sl=0.05)
    g4 = grads + [-(grads[0] + grads[1] + grads[2])]
    for d in range(3):
        e = np.eye(3, dtype=int)[d]
        xf = np.array(c) + 0.5 * e
        pb = np.array([base[a] + grads[a] @ (xf - c) for a in range(3)])
        pb = np.append(pb, 1.0 - pb.sum())
        expect = np.zeros(4)
        for a in range(4):
            for b in range(4):
                if a == b:
                    continue
                q = pb[a] * g4[b] - pb[b] * g4[a]
                # j_a = -sum_b g_ab,d(q_ab) phibar_b (O4.5); g from the pinned pair_grad (P8)
                expect[a] -= O.pair_grad(p, min(a, b), max(a, b), q if a < b else -q)[d] * (1 if a < b else -1) * pb[b]
        jf = O.phi_face(p, phi, c[0], c[1], c[2], d)
        assert np.abs(jf - expect).max() <= 1e-13 * np.abs(expect).max(), (d, jf, expect)


# --------------------------------------------------------------------------
# P21 — homogeneity of the cubic gradient energy (reading R3): a_c depends on
# q/|q| only, so e(s q) = s^2 e(q) and g(s q) = s g(q) for every s > 0, and g
# goes to 0 continuously as q -> 0 (no under/overflow of |q|^6)
# --------------------------------------------------------------------------
def test_p21_gradient_energy_homogeneity(pv1):
    p = _params(pv1, aniso=True, delta_sl=0.05)
    rng = np.random.default_rng(21)
    for _ in range(20):
        q = rng.normal(0, 1, 3)
        g1, e1 = O.pair_grad(p, 0, 3, q), O.pair_energy(p, 0, 3, q)
        for s in [1e-150, 1e-100, 1e-80, 1e-60, 1e-20, 3.7, 1e20, 1e60, 1e100]:
            gs = O.pair_grad(p, 0, 3, s * q)
            assert np.all(np.isfinite(gs))
            assert np.abs(gs - s * g1).max() <= 2e-15 * s * np.abs(g1).max(), s
            if 1e-150 < s < 1e150:
                es = O.pair_energy(p, 0, 3, s * q)
                assert abs(es - s * s * e1) <= 2e-15 * s * s * e1, s
        for s in [2.0 ** -300, 2.0 ** -40, 2.0 ** 50, 2.0 ** 300]:   # powers of two: bit for bit
            assert np.array_equal(O.pair_grad(p, 0, 3, s * q), s * g1)
