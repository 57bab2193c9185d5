"""ctypes binding of the CPU oracle (``oracle/oracle.cpp``).

TEST INFRASTRUCTURE ONLY: imported by tests/, ``__graft_entry__.smoke()`` and
bench.py's ``cpu_baseline`` / ``--impl reference`` legs — never by the product
package ``paper_1506_01684_b200``.  Shares no code with the CUDA path.

Arrays are numpy float64, SoA, interior cells only:
``phi[4, nz, ny, nx]``, ``mu[2, nz, ny, nx]`` (x fastest).
"""
from __future__ import annotations

import ctypes
import math
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "oracle.cpp")
_LIB = os.path.join(_HERE, "liboracle.so")
_lib = None

D = ctypes.c_double
I64 = ctypes.c_int64


class OrParams(ctypes.Structure):
    _fields_ = [("dx", D), ("dt", D), ("eps", D), ("tau", D * 4), ("gamma", (D * 4) * 4),
                ("gamma3", D * 4), ("delta", (D * 4) * 4), ("T_eut", D), ("G", D), ("v", D),
                ("T0", D), ("A0", (D * 2) * 4), ("A1", (D * 2) * 4), ("c0", (D * 2) * 4),
                ("m", (D * 2) * 4), ("L", D * 4), ("D", (D * 2) * 4),
                ("aniso", ctypes.c_int32), ("pad_", ctypes.c_int32)]


class OrDims(ctypes.Structure):
    _fields_ = [("nx", I64), ("ny", I64), ("nz", I64), ("step", I64), ("zorig", I64)]


def build(force: bool = False) -> str:
    # PF_ORACLE_LIB: a prebuilt copy (tools/oracle_mutants.py loads mutated
    # builds through it to show which pin catches each mutation)
    if os.environ.get("PF_ORACLE_LIB"):
        return os.environ["PF_ORACLE_LIB"]
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        subprocess.check_call(["g++", "-std=c++17", "-O2", "-fno-fast-math", "-ffp-contract=off",
                               "-fopenmp", "-shared", "-fPIC", "-o", _LIB, _SRC])
    return _LIB


def lib():
    global _lib
    if _lib is None:
        L = ctypes.CDLL(build())
        P, Dm, vp = ctypes.POINTER(OrParams), ctypes.POINTER(OrDims), ctypes.c_void_p
        dp = ctypes.POINTER(D)
        L.or_phi_sweep.argtypes = [P, Dm, vp, vp, vp]
        L.or_mu_sweep.argtypes = [P, Dm, vp, vp, vp, vp]
        L.or_front.argtypes = [Dm, D, vp]
        L.or_front.restype = I64
        L.or_window.argtypes = [Dm, D, D, vp, vp]
        L.or_step_cells.argtypes = [P, Dm, vp, vp, I64, vp, vp, vp]
        L.or_psi.argtypes = [P, ctypes.c_int, dp, D]
        L.or_psi.restype = D
        L.or_conc.argtypes = [P, ctypes.c_int, ctypes.c_int, D, D]
        L.or_conc.restype = D
        L.or_interp_h.argtypes = [dp, dp]
        L.or_omega.argtypes = [P, dp]
        L.or_omega.restype = D
        L.or_domega.argtypes = [P, dp, ctypes.c_int]
        L.or_domega.restype = D
        L.or_dpsi_dphi.argtypes = [P, dp, dp, D, ctypes.c_int]
        L.or_dpsi_dphi.restype = D
        L.or_pair_energy.argtypes = [P, ctypes.c_int, ctypes.c_int, dp]
        L.or_pair_energy.restype = D
        L.or_pair_grad.argtypes = [P, ctypes.c_int, ctypes.c_int, dp, dp]
        L.or_project.argtypes = [dp, dp]
        if hasattr(L, "or_phi_face"):
            L.or_phi_face.argtypes = [P, Dm, vp, I64, I64, I64, ctypes.c_int, dp]
        L.or_mu_face.argtypes = [P, Dm, vp, vp, vp, I64, I64, I64, ctypes.c_int, dp, dp]
        L.or_count_flops.argtypes = [P, ctypes.POINTER(I64)]
        _lib = L
    return _lib


def set_threads(n: int | None):
    """OpenMP threads of the oracle's z-plane loops (None: all host cores)."""
    L = lib()
    L.omp_set_num_threads.argtypes = [ctypes.c_int]
    L.omp_set_num_threads(int(n) if n else (os.cpu_count() or 1))


def make_params(pd: dict, *, layer_height: float | None = None, T0: float | None = None,
                aniso: bool = False, delta_sl: float | None = None) -> OrParams:
    """Fill OrParams from a params/*.json dict.  T0 = T_eut - G*layer_height
    (reading R12: the eutectic isotherm at the initial front) unless given."""
    p = OrParams()
    p.dx, p.dt, p.eps = pd["dx"], pd["dt"], pd["eps"]
    for a in range(4):
        p.tau[a] = pd["tau"][a]
        p.gamma3[a] = pd["gamma3"][a]
        p.L[a] = pd["L"][a]
        for b in range(4):
            p.gamma[a][b] = pd["gamma"][a][b]
            p.delta[a][b] = pd["delta"][a][b]
        for c in range(2):
            p.A0[a][c] = pd["A0"][a][c]
            p.A1[a][c] = pd["A1"][a][c]
            p.c0[a][c] = pd["c0"][a][c]
            p.m[a][c] = pd["m"][a][c]
            p.D[a][c] = pd["D"][a][c]
    p.T_eut, p.G, p.v = pd["T_eut"], pd["G"], pd["v"]
    if T0 is None:
        T0 = pd["T_eut"] - pd["G"] * (layer_height or 0.0)
    p.T0 = T0
    if delta_sl is not None:
        for a in range(3):
            p.delta[a][3] = p.delta[3][a] = delta_sl
    p.aniso = 1 if aniso else 0
    return p


def dims(nx, ny, nz, step=0, zorig=0) -> OrDims:
    return OrDims(nx, ny, nz, step, zorig)


def _c(a):
    a = np.ascontiguousarray(a, dtype=np.float64)
    return a, a.ctypes.data


def phi_sweep(p: OrParams, phi, mu, step=0, zorig=0):
    phi, pp = _c(phi)
    mu, mp = _c(mu)
    out = np.empty_like(phi)
    g = dims(phi.shape[3], phi.shape[2], phi.shape[1], step, zorig)
    lib().or_phi_sweep(ctypes.byref(p), ctypes.byref(g), pp, mp, out.ctypes.data)
    return out


def mu_sweep(p: OrParams, phi_old, phi_new, mu, step=0, zorig=0):
    phi_old, a = _c(phi_old)
    phi_new, b = _c(phi_new)
    mu, c = _c(mu)
    out = np.empty_like(mu)
    g = dims(mu.shape[3], mu.shape[2], mu.shape[1], step, zorig)
    lib().or_mu_sweep(ctypes.byref(p), ctypes.byref(g), a, b, c, out.ctypes.data)
    return out


def step(p: OrParams, phi, mu, n=0, zorig=0):
    """One time step (Algorithm 1) without the window."""
    phi_new = phi_sweep(p, phi, mu, n, zorig)
    mu_new = mu_sweep(p, phi, phi_new, mu, n, zorig)
    return phi_new, mu_new


def window(phi, mu, frac=2.0 / 3.0, front_phi_l=0.5):
    """O7 in place; returns 1 if the window shifted."""
    g = dims(phi.shape[3], phi.shape[2], phi.shape[1])
    assert phi.flags.c_contiguous and mu.flags.c_contiguous
    return lib().or_window(ctypes.byref(g), frac, front_phi_l, phi.ctypes.data, mu.ctypes.data)


def front(phi, thr=0.5):
    g = dims(phi.shape[3], phi.shape[2], phi.shape[1])
    phi, pp = _c(phi)
    return int(lib().or_front(ctypes.byref(g), thr, pp))


def run(p: OrParams, phi, mu, nsteps, n0=0, zorig=0, window_on=False, frac=2.0 / 3.0,
        front_phi_l=0.5, shifts=None):
    """nsteps of Algorithm 1 (+ O7 after each step when window_on)."""
    phi = np.array(phi, dtype=np.float64, copy=True)
    mu = np.array(mu, dtype=np.float64, copy=True)
    for s in range(nsteps):
        phi, mu = step(p, phi, mu, n0 + s, zorig)
        if window_on and window(phi, mu, frac, front_phi_l):
            zorig += 1
            if shifts is not None:
                shifts.append(n0 + s)
    return phi, mu, zorig


def step_cells(p: OrParams, phi, mu, cells, n=0, zorig=0):
    """One-step map at global linear cell indices; returns (phi[4,m], mu[2,m])."""
    phi, pp = _c(phi)
    mu, mp = _c(mu)
    cells = np.ascontiguousarray(cells, dtype=np.int64)
    m = cells.size
    po = np.empty((4, m))
    mo = np.empty((2, m))
    g = dims(phi.shape[3], phi.shape[2], phi.shape[1], n, zorig)
    lib().or_step_cells(ctypes.byref(p), ctypes.byref(g), pp, mp, m, cells.ctypes.data,
                        po.ctypes.data, mo.ctypes.data)
    return po, mo


def _dp(x):
    x = np.ascontiguousarray(x, dtype=np.float64)
    return x, x.ctypes.data_as(ctypes.POINTER(D))


def psi(p, a, mu, T):
    mu, mp = _dp(mu)
    return lib().or_psi(ctypes.byref(p), a, mp, T)


def conc(p, a, c, mu_c, T):
    return lib().or_conc(ctypes.byref(p), a, c, mu_c, T)


def interp_h(ph):
    ph, pp = _dp(ph)
    h = np.empty(4)
    lib().or_interp_h(pp, h.ctypes.data_as(ctypes.POINTER(D)))
    return h


def omega(p, ph):
    ph, pp = _dp(ph)
    return lib().or_omega(ctypes.byref(p), pp)


def domega(p, ph, a):
    ph, pp = _dp(ph)
    return lib().or_domega(ctypes.byref(p), pp, a)


def dpsi_dphi(p, ph, mu, T, a):
    ph, pp = _dp(ph)
    mu, mp = _dp(mu)
    return lib().or_dpsi_dphi(ctypes.byref(p), pp, mp, T, a)


def pair_energy(p, a, b, q):
    q, qp = _dp(q)
    return lib().or_pair_energy(ctypes.byref(p), a, b, qp)


def pair_grad(p, a, b, q):
    q, qp = _dp(q)
    g = np.empty(3)
    lib().or_pair_grad(ctypes.byref(p), a, b, qp, g.ctypes.data_as(ctypes.POINTER(D)))
    return g


def project(x):
    x, xp = _dp(x)
    o = np.empty(4)
    lib().or_project(xp, o.ctypes.data_as(ctypes.POINTER(D)))
    return o


def mu_face(p, phi_old, phi_new, mu, i, j, k, d, n=0, zorig=0):
    phi_old, a = _c(phi_old)
    phi_new, b = _c(phi_new)
    mu, c = _c(mu)
    g = dims(mu.shape[3], mu.shape[2], mu.shape[1], n, zorig)
    F = np.zeros(2)
    J = np.zeros(2)
    lib().or_mu_face(ctypes.byref(p), ctypes.byref(g), a, b, c, i, j, k, d,
                     F.ctypes.data_as(ctypes.POINTER(D)), J.ctypes.data_as(ctypes.POINTER(D)))
    return F, J


def phi_face(p, phi, i, j, k, d, n=0, zorig=0):
    """O4.5 face flux j_a between cell (i,j,k) and (i,j,k)+e_d (global indices)."""
    phi, pp = _c(phi)
    g = dims(phi.shape[3], phi.shape[2], phi.shape[1], n, zorig)
    jf = np.zeros(4)
    lib().or_phi_face(ctypes.byref(p), ctypes.byref(g), pp, i, j, k, d, jf.ctypes.data_as(ctypes.POINTER(D)))
    return jf


def count_flops(p: OrParams) -> dict:
    out = (I64 * 6)()
    lib().or_count_flops(ctypes.byref(p), out)
    return {"phi_cell": out[0], "phi_face": out[1], "mu_cell": out[2], "mu_face": out[3],
            "phi_per_lup": out[4], "mu_per_lup": out[5]}


def rel_maxnorm(x, ref):
    """Reading R21: max|x - ref| / max|ref| (absolute if max|ref| == 0)."""
    den = float(np.max(np.abs(ref))) if np.size(ref) else 0.0
    num = float(np.max(np.abs(np.asarray(x) - np.asarray(ref)))) if np.size(ref) else 0.0
    return num / den if den > 0 else num


EPS_EQ = 16.0 / math.pi ** 2
