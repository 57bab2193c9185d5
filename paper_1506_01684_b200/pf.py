"""Thin ctypes binding of libpf.so (include/pf.h) — argument marshalling only.

Every step of the path runs in the CUDA kernels behind the C ABI; there is no
CPU fallback: if libpf.so is missing or no GPU is present the calls fail loudly.
Entry points keep the C names: ``pf_create``, ``pf_init``, ``pf_step``,
``pf_read`` (+ ``pf_write``, ``pf_set_time``, ``pf_set_timing``, ``pf_info``,
``pf_last_error``, ``pf_destroy``, ``pf_nccl_unique_id``), wrapped by the
``Context`` class.
"""
from __future__ import annotations

import ctypes
import math
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
# PF_LIB: an alternative build of the same library (A/B timing tools only)
LIB_PATH = os.environ.get("PF_LIB") or os.path.join(_HERE, "libpf.so")

D = ctypes.c_double
I32 = ctypes.c_int32
I64 = ctypes.c_int64

PF_OK, PF_ERR_CONFIG, PF_ERR_NUMERICAL, PF_ERR_CUDA, PF_ERR_COMM, PF_ERR_STATE, PF_ERR_ARG, PF_ERR_IO = \
    0, -1, -2, -3, -4, -5, -6, -7
STATUS_NAMES = {0: "PF_OK", -1: "PF_ERR_CONFIG", -2: "PF_ERR_NUMERICAL", -3: "PF_ERR_CUDA", -4: "PF_ERR_COMM",
                -5: "PF_ERR_STATE", -6: "PF_ERR_ARG", -7: "PF_ERR_IO"}
EXPORTS = ["pf_nccl_unique_id", "pf_halo_plan", "pf_create", "pf_init", "pf_write", "pf_set_time", "pf_step", "pf_read",
           "pf_step_io", "pf_save", "pf_load", "pf_mesh", "pf_mesh_table", "pf_set_timing", "pf_set_shortcuts", "pf_set_fusion", "pf_info", "pf_last_error",
           "pf_destroy"]


def mesh_table():
    """The marching-cubes case table libpf.so generated (pf_mesh_table; host
    only): int8[256, 16] = {ntri, then 3 cube-edge numbers per triangle}."""
    t = np.zeros((256, 16), dtype=np.int8)
    st = lib().pf_mesh_table(t.ctypes.data)
    if st != PF_OK:
        raise PfError(st, "pf_mesh_table")
    return t


class PfGrid(ctypes.Structure):
    _fields_ = [("nx", I64), ("ny", I64), ("nz", I64), ("px", I32), ("py", I32), ("pz", I32),
                ("rank", I32), ("nranks", I32), ("device", I32), ("nccl_id", ctypes.c_uint8 * 128),
                ("stream", ctypes.c_void_p)]


class PfParams(ctypes.Structure):
    _fields_ = [("dx", D), ("dt", D), ("eps", D), ("tau", D * 4), ("gamma", (D * 4) * 4), ("gamma3", D * 4),
                ("delta", (D * 4) * 4), ("T_eut", D), ("G", D), ("v", D), ("T0", D),
                ("A0", (D * 2) * 4), ("A1", (D * 2) * 4), ("c0", (D * 2) * 4), ("m", (D * 2) * 4),
                ("L", D * 4), ("D", (D * 2) * 4), ("aniso", I32), ("window", I32), ("window_frac", D),
                ("window_phi_l", D), ("nan_check_every", I32), ("variant", I32), ("init_kind", I32),
                ("init_n_seeds", I32), ("init_lam_wmin", I32), ("init_lam_wmax", I32),
                ("init_planar_phase", I32), ("shortcuts", I32), ("init_layer_height", D),
                ("init_iface_width", D), ("init_mu_noise", D), ("overlap", I32), ("graph", I32)]


class PfInfo(ctypes.Structure):
    _fields_ = [("nx_l", I64), ("ny_l", I64), ("nz_l", I64), ("x0", I64), ("y0", I64), ("z0", I64),
                ("step", I64), ("z_origin", I64), ("shifts", I64), ("last_front", I64),
                ("nblocks_local", I32), ("timing", I32), ("ms_phi", D), ("ms_mu", D), ("ms_halo", D),
                ("ms_other", D), ("launches", I64), ("phi_launches", I64), ("mu_launches", I64),
                ("ms_fused", D), ("fused_launches", I64), ("fusion", I32), ("pad_", I32)]


_lib = None


class PfError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"{STATUS_NAMES.get(status, status)}: {msg}")
        self.status = status


def lib():
    """Load libpf.so (built in-tree by __graft_entry__.build()); fail loudly."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(f"{LIB_PATH} not built: run `python -c 'import __graft_entry__ as g; g.build()'` "
                               "(the CUDA path has no CPU fallback)")
        L = ctypes.CDLL(LIB_PATH)
        vp = ctypes.c_void_p
        L.pf_nccl_unique_id.argtypes = [ctypes.POINTER(ctypes.c_uint8)]
        L.pf_halo_plan.argtypes = [ctypes.POINTER(PfGrid), I32, ctypes.POINTER(I64), ctypes.POINTER(I64)]
        L.pf_create.argtypes = [ctypes.POINTER(PfGrid), ctypes.POINTER(PfParams), ctypes.POINTER(vp)]
        L.pf_init.argtypes = [vp, ctypes.c_uint64]
        L.pf_write.argtypes = [vp, vp, vp]
        L.pf_set_time.argtypes = [vp, I64, I64]
        L.pf_step.argtypes = [vp, I64]
        L.pf_read.argtypes = [vp, vp, vp]
        L.pf_step_io.argtypes = [vp, vp, vp, vp, vp]
        L.pf_save.argtypes = [vp, ctypes.c_char_p]
        L.pf_load.argtypes = [vp, ctypes.c_char_p]
        L.pf_mesh.argtypes = [vp, I32, D, I64, vp, vp, ctypes.POINTER(I64)]
        L.pf_mesh_table.argtypes = [vp]
        L.pf_set_timing.argtypes = [vp, I32]
        L.pf_set_shortcuts.argtypes = [vp, I32]
        L.pf_set_fusion.argtypes = [vp, I32]
        L.pf_info.argtypes = [vp, ctypes.POINTER(PfInfo)]
        L.pf_last_error.argtypes = [vp]
        L.pf_last_error.restype = ctypes.c_char_p
        L.pf_destroy.argtypes = [vp]
        L.pf_destroy.restype = None
        for f in EXPORTS:
            if f not in ("pf_last_error", "pf_destroy"):
                getattr(L, f).restype = ctypes.c_int
        _lib = L
    return _lib


def make_params(pd: dict, cfg: dict | None = None, *, layer_height: float | None = None, T0: float | None = None,
                aniso: bool | None = None, delta_sl: float | None = None, window: bool | None = None,
                variant: int = 0, nan_check_every: int = 0, nx: int | None = None, ny: int | None = None,
                shortcuts: bool = False, overlap: int = 0, graph: bool = False) -> PfParams:
    """PfParams from a params/*.json dict and (optionally) a configs/*.json dict."""
    p = PfParams()
    p.dx, p.dt, p.eps = pd["dx"], pd["dt"], pd["eps"]
    for a in range(4):
        p.tau[a], p.gamma3[a], p.L[a] = pd["tau"][a], pd["gamma3"][a], pd["L"][a]
        for b in range(4):
            p.gamma[a][b] = pd["gamma"][a][b]
            p.delta[a][b] = pd["delta"][a][b]
        for c in range(2):
            p.A0[a][c], p.A1[a][c] = pd["A0"][a][c], pd["A1"][a][c]
            p.c0[a][c], p.m[a][c], p.D[a][c] = pd["c0"][a][c], pd["m"][a][c], pd["D"][a][c]
    p.T_eut, p.G, p.v = pd["T_eut"], pd["G"], pd["v"]
    ini = (cfg or {}).get("init", {})
    if layer_height is None:
        layer_height = float(ini.get("layer_height", 0.0))
    p.T0 = pd["T_eut"] - pd["G"] * layer_height if T0 is None else T0
    if aniso is None:
        aniso = bool((cfg or {}).get("aniso", False))
    if delta_sl is None and cfg is not None and cfg.get("aniso"):
        delta_sl = cfg.get("delta_sl")
    if delta_sl is not None:
        for a in range(3):
            p.delta[a][3] = p.delta[3][a] = delta_sl
    p.aniso = 1 if aniso else 0
    p.window = 1 if (window if window is not None else (cfg or {}).get("window", False)) else 0
    p.window_frac = float((cfg or {}).get("window_frac", 2.0 / 3.0))
    p.window_phi_l = float((cfg or {}).get("window_front_phi_l", 0.5))
    p.nan_check_every = nan_check_every
    p.variant = variant
    p.shortcuts = 1 if shortcuts else 0
    p.overlap = overlap
    p.graph = 1 if graph else 0
    kinds = {"voronoi": 0, "lamellar": 1, "planar": 2}
    p.init_kind = kinds[ini.get("kind", "voronoi")]
    if "n_seeds" in ini:
        p.init_n_seeds = int(ini["n_seeds"])
    elif "seeds_per_area" in ini and nx and ny:
        p.init_n_seeds = max(1, int(round(nx * ny * float(ini["seeds_per_area"]))))
    p.init_lam_wmin = int(ini.get("lam_wmin", 8))
    p.init_lam_wmax = int(ini.get("lam_wmax", 24))
    p.init_planar_phase = int(ini.get("planar_phase", 0))
    p.init_layer_height = layer_height
    p.init_iface_width = float(ini.get("iface_width", 4.0))
    p.init_mu_noise = float(ini.get("mu_noise", 0.0))
    return p


def nccl_unique_id() -> bytes:
    buf = (ctypes.c_uint8 * 128)()
    st = lib().pf_nccl_unique_id(buf)
    if st != PF_OK:
        raise PfError(st, "pf_nccl_unique_id failed")
    return bytes(buf)


def halo_plan(nx, ny, nz, px, py, pz, rank, nranks, field):
    """Host-only message plan of one ghost exchange: (send_counts, recv_counts)
    in doubles per peer rank (pf_halo_plan; no GPU needed)."""
    g = PfGrid()
    g.nx, g.ny, g.nz, g.px, g.py, g.pz, g.rank, g.nranks = nx, ny, nz, px, py, pz, rank, nranks
    snd = (I64 * nranks)()
    rcv = (I64 * nranks)()
    st = lib().pf_halo_plan(ctypes.byref(g), field, snd, rcv)
    if st != PF_OK:
        raise PfError(st, "pf_halo_plan")
    return list(snd), list(rcv)


def _ptr(x, nelem=None):
    """Raw pointer of a numpy array or a torch tensor (host or device).  Raises
    ValueError unless it is contiguous float64 and, when nelem is given, holds
    exactly nelem elements (the C ABI reads / writes that many)."""
    if isinstance(x, np.ndarray):
        if x.dtype != np.float64 or not x.flags.c_contiguous:
            raise ValueError("expected a C-contiguous float64 array")
        n, p = x.size, x.ctypes.data
    else:
        if str(getattr(x, "dtype", "")) != "torch.float64" or not x.is_contiguous():
            raise ValueError("expected a contiguous torch.float64 tensor")
        n, p = x.numel(), x.data_ptr()
    if nelem is not None and n != nelem:
        raise ValueError(f"buffer holds {n} doubles, the context's box needs {nelem}")
    return p


class Context:
    """Owns one pf_ctx (one rank's blocks on one GPU)."""

    def __init__(self, nx, ny, nz, params: PfParams, px=1, py=1, pz=1, rank=0, nranks=1, device=0,
                 nccl_id: bytes | None = None, stream: int | None = None):
        g = PfGrid()
        g.nx, g.ny, g.nz, g.px, g.py, g.pz = nx, ny, nz, px, py, pz
        g.rank, g.nranks, g.device = rank, nranks, device
        if nccl_id is not None:
            ctypes.memmove(g.nccl_id, nccl_id, 128)
        g.stream = stream
        self._c = ctypes.c_void_p()
        st = lib().pf_create(ctypes.byref(g), ctypes.byref(params), ctypes.byref(self._c))
        if st != PF_OK:
            raise PfError(st, lib().pf_last_error(None).decode())
        self.params = params
        inf = self.info()
        self.shape = (int(inf.nz_l), int(inf.ny_l), int(inf.nx_l))

    def _phi_ptr(self, x):
        return _ptr(x, 4 * self.shape[0] * self.shape[1] * self.shape[2])

    def _mu_ptr(self, x):
        return _ptr(x, 2 * self.shape[0] * self.shape[1] * self.shape[2])

    def _check(self, st):
        if st != PF_OK:
            raise PfError(st, lib().pf_last_error(self._c).decode())

    def init(self, seed: int):
        self._check(lib().pf_init(self._c, seed))

    def write(self, phi, mu):
        self._check(lib().pf_write(self._c, self._phi_ptr(phi), self._mu_ptr(mu)))

    def set_time(self, step: int, z_origin: int = 0):
        self._check(lib().pf_set_time(self._c, step, z_origin))

    def step(self, n: int = 1):
        self._check(lib().pf_step(self._c, n))

    def read(self, phi=None, mu=None):
        if phi is None:
            phi = np.empty((4,) + self.shape)
            mu = np.empty((2,) + self.shape)
        self._check(lib().pf_read(self._c, self._phi_ptr(phi), self._mu_ptr(mu)))
        return phi, mu

    def step_io(self, phi_in, mu_in, phi_out=None, mu_out=None):
        """One step from a host state to a host state (pf_step_io: upload, sweeps and
        download overlapped in z-slabs; = write + step(1) + read, bit for bit)."""
        if phi_out is None:
            phi_out = np.empty((4,) + self.shape)
            mu_out = np.empty((2,) + self.shape)
        self._check(lib().pf_step_io(self._c, self._phi_ptr(phi_in), self._mu_ptr(mu_in), self._phi_ptr(phi_out),
                                     self._mu_ptr(mu_out)))
        return phi_out, mu_out

    def save(self, path):
        """FP32 checkpoint of the current state (pf_save; collective)."""
        self._check(lib().pf_save(self._c, os.fsencode(path)))

    def load(self, path):
        """Restore a pf_save checkpoint (pf_load; collective)."""
        self._check(lib().pf_load(self._c, os.fsencode(path)))

    def mesh(self, phase: int, iso: float = 0.5):
        """Marching-cubes mesh of one phase over this rank's box (pf_mesh):
        (ids int64[T, 3], pos float64[T, 3, 3])."""
        n = I64(0)
        self._check(lib().pf_mesh(self._c, phase, iso, 0, None, None, ctypes.byref(n)))
        ids = np.empty((n.value, 3), dtype=np.int64)
        pos = np.empty((n.value, 3, 3))
        if n.value:
            self._check(lib().pf_mesh(self._c, phase, iso, n.value, ids.ctypes.data, pos.ctypes.data, ctypes.byref(n)))
        return ids, pos

    def set_timing(self, on: bool):
        self._check(lib().pf_set_timing(self._c, 1 if on else 0))

    def set_fusion(self, on: bool):
        """Fused mu(n) + phi(n+1) steps on / off for the following steps (pf_set_fusion; bitwise the same results)."""
        self._check(lib().pf_set_fusion(self._c, 1 if on else 0))

    def set_shortcuts(self, on: bool):
        """Region shortcuts on / off for the following steps (pf_set_shortcuts; bitwise the same results)."""
        self._check(lib().pf_set_shortcuts(self._c, 1 if on else 0))

    def info(self) -> PfInfo:
        o = PfInfo()
        lib().pf_info(self._c, ctypes.byref(o))
        return o

    def close(self):
        if self._c:
            lib().pf_destroy(self._c)
            self._c = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()


def mlups(cells: int, steps: int, seconds: float) -> float:
    return cells * steps / seconds / 1e6 if seconds > 0 else math.nan
