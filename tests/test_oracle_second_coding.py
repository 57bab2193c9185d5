"""The two independent CPU codings guard each other ("two
independent CPU codings (C++ oracle and NumPy 8^3 cross-check)"; the paper's
equivalence checks across kernel versions).

oracle/oracle.cpp (scalar, per-cell index functions, a < b pair updates, the
factorised driving force) against oracle/oracle_np.py (vectorised over padded
arrays, ordered pairs, the chain-rule driving force, g on the unit normal) on
crafted 8^3 states where every term is active: random admissible states with
every anti-trapping guard open, a triple junction, a binary front, each
isotropic and cubic-anisotropic, with a moving temperature (G v != 0, A1 != 0:
the dc/dT terms), a non-zero time level and window origin.  CPU only.
"""
import numpy as np
import pytest

from crafted import crafted
from inputs import gen
from oracle import oracle as O
from oracle import oracle_np as ON

TOL1, TOLN = 1e-13, 1e-12


def _params(pd, aniso, **over):
    return O.make_params(dict(pd, **over), layer_height=3.0, aniso=aniso, delta_sl=0.05 if aniso else None)


@pytest.mark.parametrize("kind", ["random", "triple", "binary"])
@pytest.mark.parametrize("aniso", [False, True])
def test_one_step_agrees(pv1, kind, aniso):
    phi, mu = crafted(kind, 8, 8, 8, seed=5)
    p = _params(pv1, aniso, G=0.02, v=0.5)
    a = O.step(p, phi, mu, n=7, zorig=3)
    b = ON.step(p, phi, mu, n=7, zorig=3)
    assert O.rel_maxnorm(b[0], a[0]) <= TOL1
    assert O.rel_maxnorm(b[1], a[1]) <= TOL1
    assert np.abs(a[0] - phi).max() > 1e-4 and np.abs(a[1] - mu).max() > 1e-4   # both fields move


@pytest.mark.parametrize("aniso", [False, True])
def test_sweeps_separately_agree(pv1, aniso):
    # each sweep on its own inputs (the mu-sweep with a phi^{n+1} that is not
    # the phi-sweep's output: M(phi^n) vs chi(phi^{n+1}) time levels, reading R9)
    phi, mu = crafted("random", 8, 7, 6, seed=8)
    phi2, _ = crafted("random", 8, 7, 6, seed=9)
    p = _params(pv1, aniso, G=0.02, v=0.5)
    assert O.rel_maxnorm(ON.phi_sweep(p, phi, mu, 2, 1), O.phi_sweep(p, phi, mu, 2, 1)) <= TOL1
    assert O.rel_maxnorm(ON.mu_sweep(p, phi, phi2, mu, 2, 1), O.mu_sweep(p, phi, phi2, mu, 2, 1)) <= TOL1


@pytest.mark.parametrize("aniso", [False, True])
def test_trajectory_agrees(pv1, aniso):
    # a Voronoi layer with mu noise (the configs' recipe) over 20 coupled steps
    cfg = gen.load_config("c5" if aniso else "c2")
    spec = gen.spec_from_config(cfg, 12, 10)
    spec.n_seeds, spec.layer_height, spec.mu_noise = 4, 4.0, 5e-2
    phi, mu = gen.generate(spec, 12, 10, 8)
    p = _params(pv1, aniso, G=0.02, v=0.5)
    a = O.run(p, phi, mu, 20)
    b = ON.run(p, phi, mu, 20)
    assert O.rel_maxnorm(b[0], a[0]) <= TOLN
    assert O.rel_maxnorm(b[1], a[1]) <= TOLN
    assert np.abs(a[0] - phi).max() > 1e-3


@pytest.mark.parametrize("aniso", [False, True])
def test_unequal_mobilities_agree(pv1, aniso):
    # with equal tau the Lagrange mean is a uniform shift that the simplex
    # projection removes; unequal tau_a (reading R15) make the
    # mean over all N phases (reading R2) visible
    phi, mu = crafted("random", 8, 8, 8, seed=6)
    p = _params(pv1, aniso, G=0.02, v=0.5, tau=[1.0, 2.0, 0.5, 1.5])
    a = O.step(p, phi, mu, n=1, zorig=0)
    b = ON.step(p, phi, mu, n=1, zorig=0)
    assert O.rel_maxnorm(b[0], a[0]) <= TOL1
    assert O.rel_maxnorm(b[1], a[1]) <= TOL1


def _generic(pd, aniso, **over):
    # the full per-pair delta matrix of PARAMS-generic (no delta_sl override)
    return O.make_params(dict(pd, **over), layer_height=3.0, aniso=aniso, delta_sl=None)


@pytest.mark.parametrize("kind", ["random", "triple", "binary"])
@pytest.mark.parametrize("aniso", [False, True])
def test_generic_parameters_agree(pgen, kind, aniso):
    # every per-phase / per-pair / per-triple coefficient distinct (params/generic.json):
    # a transposed pair index, a triple taken from the wrong phase or a solid's
    # coefficient read for another solid changes the result in one coding only
    phi, mu = crafted(kind, 8, 8, 8, seed=11)
    p = _generic(pgen, aniso, G=0.02, v=0.5)
    a = O.step(p, phi, mu, n=4, zorig=2)
    b = ON.step(p, phi, mu, n=4, zorig=2)
    assert O.rel_maxnorm(b[0], a[0]) <= TOL1
    assert O.rel_maxnorm(b[1], a[1]) <= TOL1
    assert np.abs(a[0] - phi).max() > 1e-4 and np.abs(a[1] - mu).max() > 1e-4


def test_generic_parameters_matter(pgen, pv1):
    # the generic set is not a relabelling of v1: both codings move away from v1's result
    phi, mu = crafted("random", 8, 8, 8, seed=11)
    a = O.step(_generic(pgen, True, G=0.02, v=0.5), phi, mu, n=4, zorig=2)
    v = O.step(_params(pv1, True, G=0.02, v=0.5), phi, mu, n=4, zorig=2)
    assert np.abs(a[0] - v[0]).max() > 1e-4 and np.abs(a[1] - v[1]).max() > 1e-4


@pytest.mark.parametrize("aniso", [False, True])
def test_generic_trajectory_agrees(pgen, aniso):
    cfg = gen.load_config("c2")
    spec = gen.spec_from_config(cfg, 12, 10)
    spec.n_seeds, spec.layer_height, spec.mu_noise = 5, 4.0, 5e-2
    phi, mu = gen.generate(spec, 12, 10, 8)
    p = _generic(pgen, aniso, G=0.02, v=0.5)
    a = O.run(p, phi, mu, 20)
    b = ON.run(p, phi, mu, 20)
    assert O.rel_maxnorm(b[0], a[0]) <= TOLN
    assert O.rel_maxnorm(b[1], a[1]) <= TOLN
