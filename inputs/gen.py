"""Seeded synthetic initial states (the shared input generator).

Thin ctypes wrapper over ``inputs/pfgen.c``.  Holds none of the method's
arithmetic — it only lays out initial conditions (recipe in
DESIGN.md §3).  Both the oracle side (tests) and the CUDA side (via
``pf_write``) consume its output, so neither side generates the other's inputs.
"""
from __future__ import annotations

import ctypes
import json
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "pfgen.c")
_LIB = os.path.join(_HERE, "libpfgen.so")
_lib = None

KINDS = {"voronoi": 0, "lamellar": 1, "planar": 2}


class PfgenSpec(ctypes.Structure):
    _fields_ = [("kind", ctypes.c_int32), ("n_seeds", ctypes.c_int32),
                ("lam_wmin", ctypes.c_int32), ("lam_wmax", ctypes.c_int32),
                ("planar_phase", ctypes.c_int32), ("pad_", ctypes.c_int32),
                ("layer_height", ctypes.c_double), ("iface_width", ctypes.c_double),
                ("mu_noise", ctypes.c_double), ("seed", ctypes.c_uint64)]


def build(force: bool = False) -> str:
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        subprocess.check_call(["gcc", "-O2", "-fno-fast-math", "-ffp-contract=off", "-fopenmp",
                               "-shared", "-fPIC", "-o", _LIB, _SRC, "-lm"])
    return _LIB


def lib():
    global _lib
    if _lib is None:
        _lib = ctypes.CDLL(build())
        _lib.pfgen_box.restype = ctypes.c_int
        _lib.pfgen_box.argtypes = [ctypes.POINTER(PfgenSpec)] + [ctypes.c_int64] * 9 + \
            [ctypes.c_void_p, ctypes.c_void_p]
        _lib.pfgen_rng.restype = ctypes.c_uint64
        _lib.pfgen_rng.argtypes = [ctypes.c_uint64] * 3
        _lib.pfgen_u01.restype = ctypes.c_double
        _lib.pfgen_u01.argtypes = [ctypes.c_uint64] * 3
        _lib.pfgen_ramp.restype = ctypes.c_double
        _lib.pfgen_ramp.argtypes = [ctypes.c_double, ctypes.c_double]
    return _lib


def spec_from_config(cfg: dict, nx: int, ny: int, seed: int | None = None) -> PfgenSpec:
    """Build the generator spec of a configs/*.json entry for a global nx*ny base."""
    ini = cfg["init"]
    s = PfgenSpec()
    s.kind = KINDS[ini["kind"]]
    if "n_seeds" in ini:
        s.n_seeds = int(ini["n_seeds"])
    elif "seeds_per_area" in ini:
        s.n_seeds = max(1, int(round(nx * ny * float(ini["seeds_per_area"]))))
    s.lam_wmin = int(ini.get("lam_wmin", 8))
    s.lam_wmax = int(ini.get("lam_wmax", 24))
    s.planar_phase = int(ini.get("planar_phase", 0))
    s.layer_height = float(ini["layer_height"])
    s.iface_width = float(ini.get("iface_width", 4.0))
    s.mu_noise = float(ini.get("mu_noise", 0.0))
    s.seed = int(cfg.get("seed", 0) if seed is None else seed)
    return s


def generate(spec: PfgenSpec, nx: int, ny: int, nz: int, box=None):
    """Return (phi[4,bz,by,bx], mu[2,bz,by,bx]) float64 for a box of the global grid."""
    if box is None:
        box = (0, 0, 0, nx, ny, nz)
    x0, y0, z0, bx, by, bz = box
    phi = np.empty((4, bz, by, bx), dtype=np.float64)
    mu = np.empty((2, bz, by, bx), dtype=np.float64)
    rc = lib().pfgen_box(ctypes.byref(spec), nx, ny, nz, x0, y0, z0, bx, by, bz,
                         phi.ctypes.data, mu.ctypes.data)
    if rc != 0:
        raise ValueError(f"pfgen_box failed ({rc}) for box {box} of {(nx, ny, nz)}")
    return phi, mu


def load_config(name: str) -> dict:
    root = os.path.dirname(_HERE)
    with open(os.path.join(root, "configs", f"{name}.json")) as f:
        return json.load(f)


def load_params(name: str = "v1") -> dict:
    root = os.path.dirname(_HERE)
    with open(os.path.join(root, "params", f"{name}.json")) as f:
        return json.load(f)


def interface_state_torch(shape, seed: int, device="cuda"):
    """Interface-dense measurement state on the device (torch RNG, seeded):
    phi = 0.05 + U(0,1) per phase, normalised onto the simplex, so all four
    phases are present in every cell and every anti-trapping guard is open on
    every face (the no-shortcut count of PAPER.md:508-509); mu = U(-0.3, 0.3).
    Input layout only: phi[4, nz, ny, nx], mu[2, nz, ny, nx] float64."""
    import torch
    g = torch.Generator(device=device)
    g.manual_seed(int(seed) * 7919 + 17)
    phi = torch.rand((4,) + tuple(shape), generator=g, device=device, dtype=torch.float64).add_(0.05)
    phi /= phi.sum(dim=0, keepdim=True)
    mu = torch.rand((2,) + tuple(shape), generator=g, device=device, dtype=torch.float64).mul_(0.6).sub_(0.3)
    return phi, mu
