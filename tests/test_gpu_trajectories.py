"""100-step (and C2's 1000-step) GPU-vs-oracle trajectories on replicas of every
config (SURVEY.md §8(d) parity schedule; BASELINE.json north_star: relative
max-norm <= 1e-8 after 100 steps), the region shortcuts against the oracle,
and the tiny-gradient behaviour of the cubic anisotropy.  The whole-domain
oracle runs on the host cores (OpenMP); inputs come from the shared seeded
generator (inputs/), never from the CUDA path.
"""
import numpy as np
import pytest

from inputs import gen
from oracle import oracle as O

pytestmark = pytest.mark.gpu

TOL1, TOL100 = 1e-10, 1e-8


def _pf():
    from paper_1506_01684_b200 import pf
    return pf


def _run_both(pd, cfg_name, shape, steps, *, over=None, window=None, layer_height=None, shortcuts=False,
              blocks=(1, 1, 1)):
    pf = _pf()
    nx, ny, nz = shape
    cfg = gen.load_config(cfg_name)
    spec = gen.spec_from_config(cfg, nx, ny)
    for k, v in (over or {}).items():
        setattr(spec, k, v)
    phi, mu = gen.generate(spec, nx, ny, nz)
    lh = spec.layer_height if layer_height is None else layer_height
    win = cfg.get("window", False) if window is None else window
    prm = pf.make_params(pd, cfg, nx=nx, ny=ny, window=win, layer_height=lh, shortcuts=shortcuts)
    with pf.Context(nx, ny, nz, prm, *blocks) as ctx:
        ctx.write(phi, mu)
        ctx.step(steps)
        gphi, gmu = ctx.read()
        inf = ctx.info()
    an = cfg.get("aniso", False)
    op = O.make_params(pd, layer_height=lh, aniso=an, delta_sl=cfg.get("delta_sl") if an else None)
    shifts = []
    ophi, omu, oz = O.run(op, phi, mu, steps, window_on=win, shifts=shifts)
    return (gphi, gmu, inf), (ophi, omu, oz, shifts), phi


def test_c3_replica_lamellar_window_forced_shift_100_steps(pv1):
    # C3's features: lamellae 8-24 cells cycling alpha/beta/gamma, mu noise,
    # moving window — with the front placed at the trigger height so the window
    # shifts (reading R16: with the configured height it never fires)
    nz = 96
    trig = int(np.ceil(2 * nz / 3))
    (gphi, gmu, inf), (ophi, omu, oz, shifts), phi0 = _run_both(
        pv1, "c3", (256, 128, nz), 100, over={"layer_height": trig + 0.6}, window=True)
    assert len(shifts) >= 1 and inf.shifts == len(shifts) and inf.z_origin == oz
    assert O.rel_maxnorm(gphi, ophi) <= TOL100
    assert O.rel_maxnorm(gmu, omu) <= TOL100


def test_c4_replica_voronoi_256_100_steps(pv1):
    # C4's recipe (Voronoi, ~1 seed per 32x32, z < 64, mu noise) at 256^3
    (gphi, gmu, _), (ophi, omu, _, _), phi0 = _run_both(pv1, "c4", (256, 256, 256), 100)
    assert np.abs(ophi - phi0).max() > 1e-3
    assert O.rel_maxnorm(gphi, ophi) <= TOL100
    assert O.rel_maxnorm(gmu, omu) <= TOL100


def test_c5_replica_anisotropic_window_256_100_steps(pv1):
    # C5's features (cubic anisotropy delta_sl = 0.05, Voronoi z < 64, window on)
    # on a 256^3 replica ("step 100 on a 256^3 replica")
    (gphi, gmu, inf), (ophi, omu, oz, shifts), phi0 = _run_both(pv1, "c5", (256, 256, 256), 100)
    assert inf.shifts == len(shifts) and inf.z_origin == oz
    assert np.abs(ophi - phi0).max() > 1e-3
    assert O.rel_maxnorm(gphi, ophi) <= TOL100
    assert O.rel_maxnorm(gmu, omu) <= TOL100


def test_c2_full_1000_steps(pv1):
    # BASELINE config 2 over its whole run (1000 steps, 128^3) against the
    # whole oracle trajectory (was tools/long_parity.py in round 1)
    (gphi, gmu, _), (ophi, omu, _, _), phi0 = _run_both(pv1, "c2", (128, 128, 128), 1000)
    assert np.abs(ophi - phi0).max() > 0.1
    assert O.rel_maxnorm(gphi, ophi) <= TOL100
    assert O.rel_maxnorm(gmu, omu) <= TOL100


@pytest.mark.parametrize("name,shape,lh", [("c2", (96, 64, 48), 14), ("c5", (64, 64, 48), 14.5)])
def test_shortcuts_on_against_the_oracle(pv1, name, shape, lh):
    # NEXT-1 region shortcuts switched on, against
    # the oracle (which takes no shortcuts) over 100 steps: solid grains, liquid
    # and the front in one domain
    (gphi, gmu, _), (ophi, omu, _, _), _ = _run_both(pv1, name, shape, 100, over={"layer_height": lh},
                                                     window=False, shortcuts=True)
    assert O.rel_maxnorm(gphi, ophi) <= TOL100
    assert O.rel_maxnorm(gmu, omu) <= TOL100


def test_shortcuts_bitwise_aniso_many_tiles(pv1):
    # the anisotropic shortcut kernel at a size with many tiles and
    # chunks per CTA row and a moving front (undercooled), on and off bitwise
    pf = _pf()
    cfg = gen.load_config("c5")
    nx, ny, nz = 128, 128, 64
    spec = gen.spec_from_config(cfg, nx, ny)
    spec.layer_height, spec.mu_noise = 20.0, 1e-2
    phi, mu = gen.generate(spec, nx, ny, nz)
    outs = []
    for sc in (False, True):
        prm = pf.make_params(pv1, cfg, nx=nx, ny=ny, window=False, layer_height=20.0, shortcuts=sc,
                             T0=pv1["T_eut"] - 0.2)
        with pf.Context(nx, ny, nz, prm) as ctx:
            ctx.write(phi, mu)
            ctx.step(60)
            outs.append(ctx.read())
    assert np.abs(outs[0][0] - phi).max() > 1e-2
    assert np.array_equal(outs[0][0], outs[1][0]) and np.array_equal(outs[0][1], outs[1][1])


def test_anisotropic_tiny_phase_fractions(pv1):
    # reading R3 / pin P21: g(q) is homogeneous of degree 1, so phases present
    # only in 1e-70 .. 1e-160 amounts (pair vectors |q| down to ~1e-160) must
    # give finite, continuous fluxes on both sides (round 1: the kernel's |q|^-4
    # overflowed, the oracle's q^6 underflowed)
    cfg = gen.load_config("c5")
    nx, ny, nz = 24, 20, 16
    spec = gen.spec_from_config(cfg, nx, ny)
    spec.layer_height, spec.n_seeds = 8.0, 5
    phi, mu = gen.generate(spec, nx, ny, nz)
    z, y, x = np.meshgrid(np.arange(nz), np.arange(ny), np.arange(nx), indexing="ij")
    for a, scale in ((0, 1e-70), (1, 1e-120), (2, 1e-160)):
        tiny = scale * (1.5 + np.sin(0.7 * x + 0.3 * a) * np.cos(0.5 * y) * np.cos(0.4 * z))
        phi[a] = np.where(phi[a] == 0.0, tiny, phi[a])
    phi /= phi.sum(axis=0, keepdims=True)
    pf = _pf()
    prm = pf.make_params(pv1, cfg, nx=nx, ny=ny, window=False, layer_height=8.0)
    with pf.Context(nx, ny, nz, prm) as ctx:
        ctx.write(phi, mu)
        ctx.step(1)
        gphi, gmu = ctx.read()
    op = O.make_params(pv1, layer_height=8.0, aniso=True, delta_sl=cfg["delta_sl"])
    ophi, omu = O.step(op, phi, mu)
    assert np.isfinite(ophi).all() and np.isfinite(omu).all()
    assert np.isfinite(gphi).all() and np.isfinite(gmu).all()
    assert O.rel_maxnorm(gphi, ophi) <= TOL1
    assert O.rel_maxnorm(gmu, omu) <= TOL1


def test_interface_dense_state_one_step(pv1):
    # the bench's all-guards-open measurement state (every phase in every cell),
    # isotropic and anisotropic, against the oracle
    import sys, os
    sys.path.insert(0, os.path.dirname(__file__))
    from crafted import random_interface
    pf = _pf()
    phi, mu = random_interface(40, 36, 20, seed=4)
    for name in ("c4", "c5"):
        cfg = gen.load_config(name)
        prm = pf.make_params(pv1, cfg, nx=40, ny=36, window=False, layer_height=10.0)
        with pf.Context(40, 36, 20, prm) as ctx:
            ctx.write(phi, mu)
            ctx.step(1)
            gphi, gmu = ctx.read()
        an = cfg.get("aniso", False)
        op = O.make_params(pv1, layer_height=10.0, aniso=an, delta_sl=cfg.get("delta_sl") if an else None)
        ophi, omu = O.step(op, phi, mu)
        assert O.rel_maxnorm(gphi, ophi) <= TOL1
        assert O.rel_maxnorm(gmu, omu) <= TOL1


def test_set_shortcuts_toggle_bitwise(pv1):
    # pf_set_shortcuts switches the region shortcuts between steps: bitwise the
    # same state as a run without them (C4 recipe, 96x64x80, front moving)
    pf = _pf()
    cfg = gen.load_config("c4")
    spec = gen.spec_from_config(cfg, 96, 64)
    spec.layer_height, spec.mu_noise = 30.0, 1e-2
    phi, mu = gen.generate(spec, 96, 64, 80)
    outs = []
    for toggle in (False, True):
        prm = pf.make_params(pv1, cfg, nx=96, ny=64, window=False, layer_height=30.0, T0=pv1["T_eut"] - 0.2)
        with pf.Context(96, 64, 80, prm) as ctx:
            ctx.write(phi, mu)
            ctx.step(10)
            ctx.set_shortcuts(toggle)
            ctx.step(20)
            ctx.set_shortcuts(False)
            ctx.step(5)
            outs.append(ctx.read())
    assert np.array_equal(outs[0][0], outs[1][0]) and np.array_equal(outs[0][1], outs[1][1])
