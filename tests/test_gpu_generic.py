"""GPU (CUDA path through the C ABI) versus the CPU oracle with PARAMS-generic:
every per-phase, per-pair and per-triple coefficient distinct (params/generic.json;
tau, gamma, gamma3, the full delta matrix, A0, A1, c0, m, L, D).  PARAMS-v1 is
symmetric in the solids (equal gamma, gamma3, tau, A, L; D = 0 and m = 0 in the
solids), so a kernel or runtime table that reads the wrong pair, triple, phase
or component coefficient agrees with the oracle on v1 and disagrees here.

Tolerances as in test_gpu_parity.py (reading R21): 1e-10 after one step, 1e-8
after 100.
"""
import numpy as np
import pytest

from crafted import crafted
from inputs import gen
from oracle import oracle as O

pytestmark = pytest.mark.gpu

TOL1, TOL100 = 1e-10, 1e-8


def _pf():
    from paper_1506_01684_b200 import pf
    return pf


def _prm(pd, cfg, aniso, **kw):
    # aniso: the whole per-pair delta matrix of pd (delta_sl unset)
    return _pf().make_params(pd, cfg, aniso=aniso, delta_sl=None, window=False, **kw)


def _oprm(pd, cfg, aniso):
    return O.make_params(pd, layer_height=cfg["init"]["layer_height"], aniso=aniso, delta_sl=None)


def _gpu(pd, cfg, phi, mu, nsteps, aniso, blocks=(1, 1, 1), **kw):
    pf = _pf()
    nz, ny, nx = phi.shape[1:]
    with pf.Context(nx, ny, nz, _prm(pd, cfg, aniso, **kw), *blocks) as ctx:
        ctx.write(phi, mu)
        ctx.step(nsteps)
        return ctx.read()


def _voronoi(nx, ny, nz, lh=9.0):
    cfg = gen.load_config("c2")
    cfg = dict(cfg, init=dict(cfg["init"], layer_height=lh))
    spec = gen.spec_from_config(cfg, nx, ny)
    spec.layer_height, spec.n_seeds, spec.mu_noise = lh, 9, 1e-2
    return cfg, gen.generate(spec, nx, ny, nz)


@pytest.mark.parametrize("aniso", [False, True])
def test_generic_one_step(pgen, aniso):
    cfg, (phi, mu) = _voronoi(37, 29, 23)
    g = _gpu(pgen, cfg, phi, mu, 1, aniso)
    o = O.step(_oprm(pgen, cfg, aniso), phi, mu)
    assert O.rel_maxnorm(g[0], o[0]) <= TOL1
    assert O.rel_maxnorm(g[1], o[1]) <= TOL1


@pytest.mark.parametrize("aniso", [False, True])
def test_generic_100_steps(pgen, aniso):
    cfg, (phi, mu) = _voronoi(32, 32, 32)
    g = _gpu(pgen, cfg, phi, mu, 100, aniso)
    o = O.run(_oprm(pgen, cfg, aniso), phi, mu, 100)
    assert O.rel_maxnorm(g[0], o[0]) <= TOL100
    assert O.rel_maxnorm(g[1], o[1]) <= TOL100
    assert np.abs(o[0] - phi).max() > 1e-3   # the state moved


@pytest.mark.parametrize("kind", ["random", "triple"])
@pytest.mark.parametrize("aniso", [False, True])
def test_generic_every_guard_open(pgen, kind, aniso):
    # several tiles in x and y plus ragged tails; every face carries J_at for
    # the random state, three solids meet for the triple state
    phi, mu = crafted(kind, 40, 19, 12, seed=21)
    cfg = dict(gen.load_config("c2"))
    cfg["init"] = dict(cfg["init"], layer_height=6.0)
    g = _gpu(pgen, cfg, phi, mu, 1, aniso)
    o = O.step(_oprm(pgen, cfg, aniso), phi, mu)
    assert O.rel_maxnorm(g[0], o[0]) <= TOL1
    assert O.rel_maxnorm(g[1], o[1]) <= TOL1


def test_generic_blocks_and_shortcuts_bitwise(pgen):
    # decomposition invariance (2x2x2 blocks on one GPU) and region shortcuts
    # stay bit-exact with distinct coefficients
    cfg, (phi, mu) = _voronoi(48, 40, 36, lh=14.0)
    ref = _gpu(pgen, cfg, phi, mu, 6, True)
    blk = _gpu(pgen, cfg, phi, mu, 6, True, blocks=(2, 2, 2))
    sc = _gpu(pgen, cfg, phi, mu, 6, True, shortcuts=True)
    for a, b in ((ref, blk), (ref, sc)):
        assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])
