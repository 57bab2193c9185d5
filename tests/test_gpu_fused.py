"""Fused steps (pf_set_fusion): the mu-sweep of step n and the phi-sweep of step
n+1 in one kernel (pf_fused.cu; Algorithm 1, with the
phi-sweep reading mu at the cell only, D3C1).

Every case runs the same seeded state with fusion off and on and requires the
two trajectories to be BITWISE equal (the fused kernel evaluates every face and
cell with the pinned routines in the separate sweeps' expression order), and
anchors the fused run to the oracle at the north_star tolerances.  Covered:
isotropic and anisotropic models (the solid-liquid mask of C5 and the full
per-pair delta matrix), ragged tiles, multiple blocks on one GPU, the moving
window with forced shifts (the run is cut before each window check), the NaN
watchdog cadence, every anti-trapping guard open, and single-step calls.
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


def _gpu(prm, phi, mu, calls, fusion, blocks=(1, 1, 1), timing=False):
    """Run pf_step(n) for each n in `calls` from (phi, mu); return fields + info."""
    pf = _pf()
    nz, ny, nx = phi.shape[1:]
    with pf.Context(nx, ny, nz, prm, *blocks) as ctx:
        ctx.set_fusion(fusion)
        if timing:
            ctx.set_timing(True)
        ctx.write(phi, mu)
        for n in calls:
            ctx.step(n)
        gphi, gmu = ctx.read()
        return gphi, gmu, ctx.info()


def _voronoi(cfg_name, nx, ny, nz, lh=None, seed=None):
    cfg = gen.load_config(cfg_name)
    spec = gen.spec_from_config(cfg, nx, ny, seed=seed)
    if lh is not None:
        spec.layer_height = lh
    return cfg, spec.layer_height, gen.generate(spec, nx, ny, nz)


def _same(a, b):
    assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])


@pytest.mark.parametrize("shape", [(37, 29, 23), (64, 48, 40), (16, 8, 5)])
def test_fused_bitwise_isotropic(pv1, shape):
    pf = _pf()
    cfg, lh, (phi, mu) = _voronoi("c2", *shape, lh=min(12.0, shape[2] / 2))
    prm = pf.make_params(pv1, cfg, nx=shape[0], ny=shape[1], layer_height=lh, window=False)
    off = _gpu(prm, phi, mu, [9], False)
    on = _gpu(prm, phi, mu, [9], True, timing=True)
    _same(off, on)
    assert on[2].fusion == 1 and on[2].fused_launches == 8 and on[2].mu_launches == 1 and on[2].phi_launches == 1
    assert np.abs(on[0] - phi).max() > 1e-4   # the state moved


@pytest.mark.parametrize("model", ["c5", "all_pairs"])
def test_fused_bitwise_anisotropic(pv1, pgen, model):
    pf = _pf()
    nx, ny, nz = 40, 27, 21
    cfg, lh, (phi, mu) = _voronoi("c5", nx, ny, nz, lh=10.0)
    if model == "c5":   # delta on the solid-liquid pairs only (the compile-time mask)
        prm = pf.make_params(pv1, cfg, nx=nx, ny=ny, layer_height=lh, window=False)
    else:               # every coefficient distinct, the full delta matrix (run-time mask)
        prm = pf.make_params(pgen, gen.load_config("c2"), nx=nx, ny=ny, layer_height=lh, window=False, aniso=True,
                             delta_sl=None)
    _same(_gpu(prm, phi, mu, [8], False), _gpu(prm, phi, mu, [8], True))


@pytest.mark.parametrize("aniso", [False, True])
def test_fused_bitwise_every_guard_open(pgen, aniso):
    # every face carries the anti-trapping current (all guards open) on both
    # sweeps' inputs; several tiles in x and y with ragged tails
    pf = _pf()
    phi, mu = crafted("random", 40, 19, 12, seed=21)
    cfg = dict(gen.load_config("c2"))
    cfg["init"] = dict(cfg["init"], layer_height=6.0)
    prm = pf.make_params(pgen, cfg, nx=40, ny=19, aniso=aniso, delta_sl=None, window=False)
    _same(_gpu(prm, phi, mu, [3], False), _gpu(prm, phi, mu, [3], True))


def test_fused_bitwise_blocks_and_calls(pv1):
    # 2x2x1 blocks on one GPU, and a mix of pf_step lengths (n = 1 runs the
    # separate sweeps; every call ends on a complete time level)
    pf = _pf()
    cfg, lh, (phi, mu) = _voronoi("c2", 48, 40, 30, lh=12.0)
    prm = pf.make_params(pv1, cfg, nx=48, ny=40, layer_height=lh, window=False)
    ref = _gpu(prm, phi, mu, [10], False)
    _same(ref, _gpu(prm, phi, mu, [10], True, blocks=(2, 2, 1)))
    _same(ref, _gpu(prm, phi, mu, [1, 3, 2, 4], True))
    # fusion switched off (the third copy released) and on again mid-run
    pf = _pf()
    with pf.Context(48, 40, 30, prm) as ctx:
        ctx.write(phi, mu)
        for on, n in ((True, 3), (False, 2), (True, 5)):
            ctx.set_fusion(on)
            ctx.step(n)
        _same(ref, ctx.read())


@pytest.mark.parametrize("aniso", [False, True])
def test_fused_with_shortcuts_bitwise(pgen, aniso):
    # region shortcuts inside the fused kernel (the vote on phi^{n+1}): bulk
    # solid below, bulk liquid above, interfaces between — bitwise the plain run
    pf = _pf()
    nx, ny, nz = 64, 48, 40
    cfg, lh, (phi, mu) = _voronoi("c2", nx, ny, nz, lh=16.0)
    base = dict(nx=nx, ny=ny, layer_height=lh, window=False, aniso=aniso, delta_sl=None)
    ref = _gpu(pf.make_params(pgen, cfg, **base), phi, mu, [12], False)
    on = _gpu(pf.make_params(pgen, cfg, shortcuts=True, **base), phi, mu, [12], True, timing=True)
    assert on[2].fused_launches == 11
    _same(ref, on)


def test_fused_window_forced_shifts_and_nan_cadence(pv1):
    # the front at the trigger height: the window shifts during the run; the
    # fused run is cut before every due window check and NaN check
    pf = _pf()
    nz = 48
    trig = int(np.ceil(2 * nz / 3))
    cfg, lh, (phi, mu) = _voronoi("c3", 64, 32, nz, lh=trig + 0.6)
    prm = pf.make_params(pv1, cfg, nx=64, ny=32, layer_height=lh, window=True, nan_check_every=7)
    off = _gpu(prm, phi, mu, [40], False)
    on = _gpu(prm, phi, mu, [40], True)
    assert on[2].shifts >= 1 and on[2].shifts == off[2].shifts and on[2].z_origin == off[2].z_origin
    _same(off, on)


def test_fused_vs_oracle(pv1):
    # the fused trajectory against the oracle directly: 2 steps at the one-step
    # tolerance, 100 steps at the north_star's 1e-8
    pf = _pf()
    cfg, lh, (phi, mu) = _voronoi("c2", 37, 29, 23, lh=10.0)
    prm = pf.make_params(pv1, cfg, nx=37, ny=29, layer_height=lh, window=False)
    op = O.make_params(pv1, layer_height=lh, aniso=False)
    g2 = _gpu(prm, phi, mu, [2], True)
    o2 = O.run(op, phi, mu, 2)
    assert O.rel_maxnorm(g2[0], o2[0]) <= TOL1 and O.rel_maxnorm(g2[1], o2[1]) <= TOL1
    g = _gpu(prm, phi, mu, [100], True)
    o = O.run(op, phi, mu, 100)
    assert O.rel_maxnorm(g[0], o[0]) <= TOL100 and O.rel_maxnorm(g[1], o[1]) <= TOL100


@pytest.mark.parametrize("name,shape,steps,lh", [
    ("c3", (256, 128, 96), 100, 64.6),     # lamellar + window, front at the trigger: forced shifts
    ("c4", (256, 256, 256), 100, None),    # Voronoi, C4's recipe at 256^3
    ("c5", (256, 256, 256), 100, None),    # anisotropic (solid-liquid mask) + window
    ("c4", (512, 512, 512), 12, None),     # C4 at its bench size and launch configuration
])
def test_fused_bitwise_config_replicas(pv1, name, shape, steps, lh):
    # every config's features over a long run (or at full size): fused == separate, bit for bit
    pf = _pf()
    nx, ny, nz = shape
    cfg = gen.load_config(name)
    prm = pf.make_params(pv1, cfg, nx=nx, ny=ny, **({"layer_height": lh} if lh else {}))
    res = []
    for fusion in (False, True):
        with pf.Context(nx, ny, nz, prm) as ctx:
            ctx.set_fusion(fusion)
            if lh:   # the generator's state with the front moved up to the window trigger
                spec = gen.spec_from_config(cfg, nx, ny)
                spec.layer_height = lh
                ctx.write(*gen.generate(spec, nx, ny, nz))
            else:
                ctx.init(cfg["seed"])
            ctx.step(steps)
            inf = ctx.info()
            phi, mu = ctx.read()
            res.append((phi[:, ::3], mu[:, ::3], inf.shifts, inf.z_origin))
    (p0, m0, s0, z0), (p1, m1, s1, z1) = res
    assert s0 == s1 and z0 == z1 and (name != "c3" or s0 > 0)
    assert np.array_equal(p0, p1) and np.array_equal(m0, m1)


def test_fused_then_step_io(pv1):
    # pf_step_io after fused runs (the phi copies have rotated: its slab copy
    # lists are rebuilt for the new addresses) and fused runs after it
    pf = _pf()
    cfg, lh, (phi, mu) = _voronoi("c2", 40, 36, 64, lh=20.0)
    prm = pf.make_params(pv1, cfg, nx=40, ny=36, layer_height=lh, window=False)
    ref = _gpu(prm, phi, mu, [12], False)
    with pf.Context(40, 36, 64, prm) as ctx:
        ctx.set_fusion(True)
        ctx.write(phi, mu)
        ctx.step(4)
        ctx.step_io(*ctx.read())   # step 5 through the slab pipeline
        ctx.step(3)
        p, m = ctx.step_io(*ctx.read())   # step 9 (the rotation has moved on)
        ctx.step(3)
        _same(ref, ctx.read())
