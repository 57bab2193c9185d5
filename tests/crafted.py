"""Crafted admissible states for parity tests (SURVEY.md §4 layer 3).

Input generation only (no step arithmetic of the method): every phase vector is
put on the Gibbs simplex by normalisation, mu is uniform noise.  Used by the
oracle's second-coding comparison (CPU) and the GPU parity tests alike.
"""
import numpy as np


def crafted(kind, nx, ny, nz, seed):
    """kind: 'random' (every face a multi-phase interface: all anti-trapping
    guards open), 'triple' (three solids meeting along z-lines, liquid above),
    'binary' (1D alpha|liquid front along x).  mu in [-0.3, 0.3]."""
    rng = np.random.default_rng(seed)
    mu = rng.uniform(-0.3, 0.3, (2, nz, ny, nx))
    if kind == "random":
        phi = rng.random((4, nz, ny, nx)) ** 3
        phi[rng.random((4, nz, ny, nx)) < 0.2] = 0.0
        phi[3] += 1e-3                # no empty cell
    elif kind == "triple":
        x, y = np.meshgrid(np.arange(nx) + 0.5, np.arange(ny) + 0.5)
        ang = np.arctan2(y - ny / 2, x - nx / 2)
        phi = np.zeros((4, nz, ny, nx))
        for a in range(3):
            w = np.clip(1.0 - np.abs(((ang - 2 * np.pi * a / 3 + np.pi) % (2 * np.pi)) - np.pi) / (np.pi / 1.5), 0, 1)
            phi[a] = w[None]
        z = np.arange(nz)[:, None, None] + 0.5
        s = np.clip(0.5 + (nz / 2 - z) / 4, 0, 1)
        phi[:3] *= s
        phi[3] = 1 - s + 1e-3
    elif kind == "binary":
        x = np.arange(nx) + 0.5
        r = np.clip(0.5 + (nx / 2 - x) / 4, 0, 1)
        phi = np.zeros((4, nz, ny, nx))
        phi[0] = r[None, None, :]
        phi[3] = 1 - r[None, None, :]
    else:
        raise ValueError(kind)
    phi /= phi.sum(axis=0, keepdims=True)
    return phi, mu


def random_interface(nx, ny, nz, seed, mu_amp=0.3):
    """Interface-dense admissible state for the mu-sweep measurement with every
    guard open: all four phases present in every cell,
    smooth enough in z to keep the explicit step stable."""
    rng = np.random.default_rng(seed)
    phi = 0.05 + rng.random((4, nz, ny, nx))
    phi /= phi.sum(axis=0, keepdims=True)
    mu = rng.uniform(-mu_amp, mu_amp, (2, nz, ny, nx))
    return phi, mu
