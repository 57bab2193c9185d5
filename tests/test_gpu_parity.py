"""GPU (CUDA path through the C ABI) versus the CPU oracle.

Tolerance (BASELINE.json north_star; reading R21): relative max-norm per field
<= 1e-10 after one step, <= 1e-8 after 100 steps.  Inputs come from the shared
seeded generator (inputs/), never from the CUDA path.
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


def _state(cfg_name, nx, ny, nz, **over):
    cfg = gen.load_config(cfg_name)
    spec = gen.spec_from_config(cfg, nx, ny)
    for k, v in over.items():
        setattr(spec, k, v)
    return cfg, gen.generate(spec, nx, ny, nz)


def _gpu_run(pd, cfg, phi, mu, nsteps, variant=0, blocks=(1, 1, 1), window=None, aniso=None, delta_sl=None,
             layer_height=None, n0=0, zorig=0):
    pf = _pf()
    nz, ny, nx = phi.shape[1:]
    prm = pf.make_params(pd, cfg, variant=variant, window=window, aniso=aniso, delta_sl=delta_sl,
                         layer_height=layer_height)
    with pf.Context(nx, ny, nz, prm, *blocks) as ctx:
        ctx.write(phi, mu)
        ctx.set_time(n0, zorig)
        ctx.step(nsteps)
        out = ctx.read()
        inf = ctx.info()
        return out[0], out[1], inf


def _oracle_params(pd, cfg, aniso=None, delta_sl=None, layer_height=None):
    lh = cfg["init"]["layer_height"] if layer_height is None else layer_height
    an = cfg.get("aniso", False) if aniso is None else aniso
    ds = cfg.get("delta_sl") if delta_sl is None else delta_sl
    return O.make_params(pd, layer_height=lh, aniso=an, delta_sl=ds if an else None)


@pytest.mark.parametrize("variant", [0, 1])
def test_c1_one_step(pv1, variant):
    cfg, (phi, mu) = _state("c1", 32, 32, 32)
    gphi, gmu, _ = _gpu_run(pv1, cfg, phi, mu, 1, variant=variant)
    ophi, omu = O.step(_oracle_params(pv1, cfg), phi, mu)
    assert O.rel_maxnorm(gphi, ophi) <= TOL1
    assert O.rel_maxnorm(gmu, omu) <= TOL1


def test_c1_100_steps(pv1):
    cfg, (phi, mu) = _state("c1", 32, 32, 32)
    gphi, gmu, _ = _gpu_run(pv1, cfg, phi, mu, 100)
    ophi, omu, _ = O.run(_oracle_params(pv1, cfg), phi, mu, 100)
    assert O.rel_maxnorm(gphi, ophi) <= TOL100
    assert O.rel_maxnorm(gmu, omu) <= TOL100
    assert np.abs(ophi - phi).max() > 1e-3   # the state moved


@pytest.mark.parametrize("shape", [(37, 29, 23), (70, 9, 12), (33, 40, 5)])
def test_ragged_shapes(pv1, shape):
    nx, ny, nz = shape
    cfg, (phi, mu) = _state("c2", nx, ny, nz, layer_height=min(nz - 2, 9), n_seeds=7, mu_noise=1e-2)
    gphi, gmu, _ = _gpu_run(pv1, cfg, phi, mu, 3, layer_height=min(nz - 2, 9))
    ophi, omu, _ = O.run(_oracle_params(pv1, cfg, layer_height=min(nz - 2, 9)), phi, mu, 3)
    assert O.rel_maxnorm(gphi, ophi) <= TOL1
    assert O.rel_maxnorm(gmu, omu) <= TOL1


@pytest.mark.parametrize("shape", [(2, 2, 2), (2, 5, 3), (3, 2, 7), (2, 2, 40)])
@pytest.mark.parametrize("aniso", [False, True])
def test_minimum_sizes(pv1, shape, aniso):
    # the smallest blocks pf_create accepts (2 cells per axis): a tile is mostly
    # inactive threads, the periodic ghosts are the other interior cell, a
    # z-chunk may hold one plane
    nx, ny, nz = shape
    lh = nz / 2
    cfg, (phi, mu) = _state("c2", nx, ny, nz, layer_height=lh, mu_noise=1e-2)
    gphi, gmu, _ = _gpu_run(pv1, cfg, phi, mu, 3, aniso=aniso, delta_sl=0.05 if aniso else None, layer_height=lh)
    ophi, omu, _ = O.run(_oracle_params(pv1, cfg, aniso=aniso, delta_sl=0.05 if aniso else None, layer_height=lh),
                         phi, mu, 3)
    assert O.rel_maxnorm(gphi, ophi) <= TOL1
    assert O.rel_maxnorm(gmu, omu) <= TOL1


@pytest.mark.parametrize("variant", [0, 1])
def test_anisotropic(pv1, variant):
    cfg, (phi, mu) = _state("c5", 24, 20, 16, layer_height=8, n_seeds=6)
    gphi, gmu, _ = _gpu_run(pv1, cfg, phi, mu, 1, variant=variant, window=False, layer_height=8)
    op = _oracle_params(pv1, cfg, layer_height=8)
    ophi, omu = O.step(op, phi, mu)
    assert O.rel_maxnorm(gphi, ophi) <= TOL1
    assert O.rel_maxnorm(gmu, omu) <= TOL1
    gphi, gmu, _ = _gpu_run(pv1, cfg, phi, mu, 100, variant=variant, window=False, layer_height=8)
    ophi, omu, _ = O.run(op, phi, mu, 100)
    assert O.rel_maxnorm(gphi, ophi) <= TOL100
    assert O.rel_maxnorm(gmu, omu) <= TOL100


def test_time_level_and_origin(pv1):
    # T(z, t) depends on the step index and the window origin (reading R12)
    cfg, (phi, mu) = _state("c2", 16, 16, 16, layer_height=6, n_seeds=5)
    pd = dict(pv1, v=2.0, G=0.01)
    gphi, gmu, _ = _gpu_run(pd, cfg, phi, mu, 2, layer_height=6, n0=37, zorig=5)
    ophi, omu, _ = O.run(_oracle_params(pd, cfg, layer_height=6), phi, mu, 2, n0=37, zorig=5)
    assert O.rel_maxnorm(gphi, ophi) <= TOL1
    assert O.rel_maxnorm(gmu, omu) <= TOL1


def test_moving_window_forced_shift(pv1):
    # front initialised just below 2/3 of the height so that the window fires
    # (reading R16: with the configs as written it never does)
    nz = 24
    cfg, (phi, mu) = _state("c3", 16, 16, nz, layer_height=16.95)
    pd = dict(pv1, G=0.0)
    op = O.make_params(pd, T0=pv1["T_eut"] - 0.5)   # strongly undercooled: the front advances
    shifts = []
    ophi, omu, oz = O.run(op, phi, mu, 120, window_on=True, shifts=shifts)
    assert len(shifts) >= 2   # one at once, one after the front advanced
    pf = _pf()
    prm = pf.make_params(pd, cfg, window=True, T0=pv1["T_eut"] - 0.5)
    with pf.Context(16, 16, nz, prm) as ctx:
        ctx.write(phi, mu)
        ctx.step(120)
        gphi, gmu = ctx.read()
        inf = ctx.info()
    assert inf.z_origin == oz and inf.shifts == len(shifts)
    assert O.rel_maxnorm(gphi, ophi) <= TOL100
    assert O.rel_maxnorm(gmu, omu) <= TOL100


@pytest.mark.parametrize("blocks", [(2, 1, 1), (1, 2, 1), (1, 1, 2), (2, 2, 1), (2, 2, 2)])
def test_decomposition_bitwise(pv1, blocks):
    # P9: any block decomposition equals the single block bit for bit
    cfg, (phi, mu) = _state("c2", 32, 24, 20, layer_height=9, n_seeds=8)
    a = _gpu_run(pv1, cfg, phi, mu, 7, layer_height=9)
    b = _gpu_run(pv1, cfg, phi, mu, 7, blocks=blocks, layer_height=9)
    assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])


def test_decomposition_bitwise_aniso_window(pv1):
    cfg, (phi, mu) = _state("c5", 16, 16, 24, layer_height=16.95, n_seeds=4)
    pd = dict(pv1, G=0.0)
    pf = _pf()
    outs = []
    for blocks in [(1, 1, 1), (2, 2, 2)]:
        prm = pf.make_params(pd, cfg, window=True, T0=pv1["T_eut"] - 0.5, layer_height=16.95)
        with pf.Context(16, 16, 24, prm, *blocks) as ctx:
            ctx.write(phi, mu)
            ctx.step(120)
            outs.append(ctx.read() + (ctx.info().shifts,))
    assert outs[0][2] >= 1 and outs[0][2] == outs[1][2]
    assert np.array_equal(outs[0][0], outs[1][0]) and np.array_equal(outs[0][1], outs[1][1])


def test_conservation_gpu(pv1):
    # P4 on the CUDA path: flux-form divergence with pinned face rounding
    cfg, (phi, mu) = _state("c2", 16, 16, 16, layer_height=8, n_seeds=6, mu_noise=5e-2)
    pd = dict(pv1, v=0.0, G=0.01)
    gphi, gmu, _ = _gpu_run(pd, cfg, phi, mu, 100, layer_height=9)
    import sys, os
    sys.path.insert(0, os.path.dirname(__file__))
    from test_oracle_pins import _solute
    p = O.make_params(pd, layer_height=9)
    c0, c1 = _solute(pd, p, phi, mu), _solute(pd, p, gphi, gmu, n=100)
    assert np.abs(c1 - c0).max() / np.abs(c0).max() <= 1e-13


def test_pf_init_matches_generator(pv1):
    pf = _pf()
    for name, shape in [("c1", (32, 32, 32)), ("c3", (64, 32, 48))]:
        cfg = gen.load_config(name)
        nx, ny, nz = shape
        prm = pf.make_params(pv1, cfg, nx=nx, ny=ny)
        spec = gen.spec_from_config(cfg, nx, ny)
        phi, mu = gen.generate(spec, nx, ny, nz)
        with pf.Context(nx, ny, nz, prm, 2, 1, 2) as ctx:
            ctx.init(cfg["seed"])
            gphi, gmu = ctx.read()
        assert np.abs(gphi - phi).max() <= 1e-15
        assert np.array_equal(gmu, mu)


def test_abi_errors(pv1):
    pf = _pf()
    cfg = gen.load_config("c1")
    prm = pf.make_params(pv1, cfg)
    with pytest.raises(pf.PfError) as e:
        pf.Context(30, 32, 32, prm, 4, 1, 1)
    assert e.value.status == pf.PF_ERR_CONFIG and "axis x" in str(e.value)
    with pf.Context(16, 16, 16, prm) as ctx:
        with pytest.raises(pf.PfError) as e:
            ctx.step(1)
        assert e.value.status == pf.PF_ERR_STATE
    prm = pf.make_params(pv1, cfg, nan_check_every=1)
    spec = gen.spec_from_config(cfg, 16, 16)
    phi, mu = gen.generate(spec, 16, 16, 16)
    with pf.Context(16, 16, 16, prm) as ctx:
        ctx.write(phi, mu)
        p2, m2 = ctx.read()
        assert np.array_equal(p2, phi) and np.array_equal(m2, mu)   # read round-trips write
        mu2 = mu.copy()
        mu2[1, 5, 6, 7] = np.nan
        ctx.write(phi, mu2)
        with pytest.raises(pf.PfError) as e:
            ctx.step(3)
        assert e.value.status == pf.PF_ERR_NUMERICAL and "step 1" in str(e.value)
        with pytest.raises(pf.PfError) as e:
            ctx.step(1)
        assert e.value.status == pf.PF_ERR_STATE


def test_device_pointer_read(pv1):
    import torch
    pf = _pf()
    cfg, (phi, mu) = _state("c1", 16, 16, 16, layer_height=6)
    prm = pf.make_params(pv1, cfg)
    with pf.Context(16, 16, 16, prm) as ctx:
        ctx.write(torch.from_numpy(phi).cuda(), torch.from_numpy(mu).cuda())
        ctx.step(2)
        tp = torch.empty((4, 16, 16, 16), dtype=torch.float64, device="cuda")
        tm = torch.empty((2, 16, 16, 16), dtype=torch.float64, device="cuda")
        ctx.read(tp, tm)
        hp, hm = ctx.read()
    assert np.array_equal(tp.cpu().numpy(), hp) and np.array_equal(tm.cpu().numpy(), hm)


# ---------------------------------------------------------------------------
# full-size configurations: whole-domain oracle where it finishes in seconds,
# sampled one-step map at the sizes bench.py runs
# ---------------------------------------------------------------------------
def _sample_cells(nx, ny, nz, m, seed=0):
    rng = np.random.default_rng(seed)
    pts = [(0, 0, 0), (nx - 1, ny - 1, nz - 1), (0, ny - 1, nz // 2), (nx - 1, 0, 0), (nx // 2, ny // 2, nz - 1)]
    cells = [(k * ny + j) * nx + i for i, j, k in pts]
    cells += list(rng.integers(0, nx * ny * nz, m))
    return np.array(cells, dtype=np.int64)


def test_c5_full_size_1024_sampled(pv1):
    # C5 at its one-GPU size (1024^3, anisotropic, moving window) in bench.py's
    # launch configuration: the state from pf_init (the generator's recipe on the
    # device, <= 1e-15 from the host generator), one step, the result read into
    # device memory and sampled; the oracle steps the same cells of a z-slab the
    # host generator builds around the front, with the slab's origin as window
    # origin (T(z) of the global planes) — cells >= 3 planes from the slab's ends
    # see no difference from the whole domain (the step's reach is 2 planes)
    import torch
    pf = _pf()
    cfg = gen.load_config("c5")
    n = 1024
    lh = int(cfg["init"]["layer_height"])
    z0, nzs = lh - 11, 22
    prm = pf.make_params(pv1, cfg, nx=n, ny=n)
    rng = np.random.default_rng(5)
    loc = np.stack([rng.integers(0, n, 4000), rng.integers(0, n, 4000), rng.integers(3, nzs - 3, 4000)])
    cells = (loc[2] + z0) * n * n + loc[1] * n + loc[0]
    with pf.Context(n, n, n, prm) as ctx:
        ctx.init(cfg["seed"])
        ctx.step(1)
        assert ctx.info().shifts == 0
        tp = torch.empty((4, n, n, n), dtype=torch.float64, device="cuda")
        tm = torch.empty((2, n, n, n), dtype=torch.float64, device="cuda")
        ctx.read(tp, tm)
    idx = torch.from_numpy(cells).cuda()
    gp = tp.reshape(4, -1)[:, idx].cpu().numpy()
    gm = tm.reshape(2, -1)[:, idx].cpu().numpy()
    del tp, tm
    torch.cuda.empty_cache()
    spec = gen.spec_from_config(cfg, n, n)
    phi, mu = gen.generate(spec, n, n, n, box=(0, 0, z0, n, n, nzs))
    op = _oracle_params(pv1, cfg)   # T0 from the global layer height; zorig = z0 places the planes
    lc = loc[2] * n * n + loc[1] * n + loc[0]
    po, mo = O.step_cells(op, phi, mu, lc, n=0, zorig=z0)
    assert O.rel_maxnorm(gp, po) <= TOL1
    assert O.rel_maxnorm(gm, mo) <= TOL1
    assert np.abs(po - phi.reshape(4, -1)[:, lc]).max() > 1e-6   # the sample sees the front move


def test_c2_full_one_step(pv1):
    cfg, (phi, mu) = _state("c2", 128, 128, 128)
    gphi, gmu, _ = _gpu_run(pv1, cfg, phi, mu, 1)
    ophi, omu = O.step(_oracle_params(pv1, cfg), phi, mu)
    assert O.rel_maxnorm(gphi, ophi) <= TOL1
    assert O.rel_maxnorm(gmu, omu) <= TOL1


@pytest.mark.parametrize("name,shape", [("c4", (512, 512, 512)), ("c3", (256, 256, 1024)), ("c5", (1024, 1024, 256))])
def test_full_size_sampled_one_step(pv1, name, shape):
    nx, ny, nz = shape
    cfg, (phi, mu) = _state(name, nx, ny, nz)
    gphi, gmu, _ = _gpu_run(pv1, cfg, phi, mu, 1)
    cells = _sample_cells(nx, ny, nz, 3000)
    # bias the sample towards the front band where all terms are active
    lh = int(cfg["init"]["layer_height"])
    rng = np.random.default_rng(1)
    band = rng.integers(0, nx * ny, 3000) + (lh - 3 + rng.integers(0, 6, 3000)) * nx * ny
    cells = np.concatenate([cells, band]).astype(np.int64)
    po, mo = O.step_cells(_oracle_params(pv1, cfg), phi, mu, cells)
    gp = gphi.reshape(4, -1)[:, cells]
    gm = gmu.reshape(2, -1)[:, cells]
    assert O.rel_maxnorm(gp, po) <= TOL1
    assert O.rel_maxnorm(gm, mo) <= TOL1


# ---------------------------------------------------------------------------
# NEXT-1 region shortcuts: bitwise identical to the full update
# ---------------------------------------------------------------------------
@pytest.mark.parametrize("name,shape", [("c4", (512, 512, 512)), ("c5", (1024, 1024, 256))])
def test_full_size_shortcuts_bitwise(pv1, name, shape):
    # the region-shortcut kernels at the bench sizes (the skip-faces path over
    # whole liquid / solid tiles) bitwise against the plain kernels, 3 steps
    nx, ny, nz = shape
    cfg, (phi, mu) = _state(name, nx, ny, nz)
    a = _run_variant(pv1, cfg, phi, mu, 3, False, nx=nx, ny=ny)
    b = _run_variant(pv1, cfg, phi, mu, 3, True, nx=nx, ny=ny)
    assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])


def _run_variant(pd, cfg, phi, mu, nsteps, shortcuts, blocks=(1, 1, 1), **kw):
    pf = _pf()
    nz, ny, nx = phi.shape[1:]
    prm = pf.make_params(pd, cfg, shortcuts=shortcuts, **kw)
    with pf.Context(nx, ny, nz, prm, *blocks) as ctx:
        ctx.write(phi, mu)
        ctx.step(nsteps)
        return ctx.read()


@pytest.mark.parametrize("name,shape,steps", [("c1", (32, 32, 32), 100), ("c2", (48, 40, 36), 30)])
def test_shortcuts_bitwise(pv1, name, shape, steps):
    nx, ny, nz = shape
    cfg, (phi, mu) = _state(name, nx, ny, nz, layer_height=min(nz // 3, 12))
    lh = min(nz // 3, 12)
    a = _run_variant(pv1, cfg, phi, mu, steps, False, layer_height=lh)
    b = _run_variant(pv1, cfg, phi, mu, steps, True, layer_height=lh)
    assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])


def test_shortcuts_bitwise_aniso_window_blocks(pv1):
    cfg, (phi, mu) = _state("c5", 16, 16, 24, layer_height=16.95, n_seeds=4)
    pd = dict(pv1, G=0.0)
    kw = dict(window=True, T0=pv1["T_eut"] - 0.5, layer_height=16.95)
    a = _run_variant(pd, cfg, phi, mu, 120, False, **kw)
    b = _run_variant(pd, cfg, phi, mu, 120, True, blocks=(2, 2, 2), **kw)
    assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])


def test_c2_full_100_steps(pv1):
    # BASELINE config 2 at full size against the whole oracle trajectory
    cfg, (phi, mu) = _state("c2", 128, 128, 128)
    gphi, gmu, _ = _gpu_run(pv1, cfg, phi, mu, 100)
    ophi, omu, _ = O.run(_oracle_params(pv1, cfg), phi, mu, 100)
    assert O.rel_maxnorm(gphi, ophi) <= TOL100
    assert O.rel_maxnorm(gmu, omu) <= TOL100


@pytest.mark.parametrize("name,shape,steps", [("c2", (128, 128, 128), 1000), ("c4", (512, 512, 512), 500),
                                              ("c3", (256, 256, 1024), 2000), ("c5", (1024, 1024, 256), 200)])
def test_full_size_one_step_map_at_run_end(pv1, name, shape, steps):
    # each config's full size and step count (BASELINE.json), in the bench's
    # launch configuration: the GPU's last step from its own step-(n-1) state,
    # against the oracle's one-step map on sampled cells (front band + random)
    pf = _pf()
    nx, ny, nz = shape
    cfg, (phi, mu) = _state(name, nx, ny, nz)
    prm = pf.make_params(pv1, cfg, nx=nx, ny=ny)
    with pf.Context(nx, ny, nz, prm) as ctx:
        ctx.write(phi, mu)
        ctx.step(steps - 1)
        inf = ctx.info()
        sphi, smu = ctx.read()
        ctx.step(1)
        gphi, gmu = ctx.read()
    assert np.abs(sphi - phi).max() > 1e-3        # the state evolved
    cells = _sample_cells(nx, ny, nz, 3000)
    lh = int(cfg["init"]["layer_height"])
    rng = np.random.default_rng(2)
    band = rng.integers(0, nx * ny, 3000) + (lh - 3 + rng.integers(0, 6, 3000)) * nx * ny
    cells = np.concatenate([cells, band]).astype(np.int64)
    po, mo = O.step_cells(_oracle_params(pv1, cfg), sphi, smu, cells, n=int(inf.step), zorig=int(inf.z_origin))
    assert O.rel_maxnorm(gphi.reshape(4, -1)[:, cells], po) <= TOL1
    assert O.rel_maxnorm(gmu.reshape(2, -1)[:, cells], mo) <= TOL1


def _crafted(kind, nx, ny, nz, seed):
    from crafted import crafted
    return crafted(kind, nx, ny, nz, seed)


@pytest.mark.parametrize("kind", ["random", "triple", "binary"])
@pytest.mark.parametrize("aniso", [False, True])
def test_crafted_states_one_step(pv1, kind, aniso):
    nx, ny, nz = 21, 18, 14
    cfg = gen.load_config("c5" if aniso else "c2")
    phi, mu = _crafted(kind, nx, ny, nz, seed=11)
    gphi, gmu, _ = _gpu_run(pv1, cfg, phi, mu, 1, window=False, layer_height=7, blocks=(1, 1, 1))
    ophi, omu = O.step(_oracle_params(pv1, cfg, layer_height=7), phi, mu)
    assert O.rel_maxnorm(gphi, ophi) <= 1e-12
    assert O.rel_maxnorm(gmu, omu) <= 1e-12
    # the same state split over blocks: bitwise
    bphi, bmu, _ = _gpu_run(pv1, cfg, phi, mu, 1, window=False, layer_height=7, blocks=(1, 2, 2))
    assert np.array_equal(bphi, gphi) and np.array_equal(bmu, gmu)
