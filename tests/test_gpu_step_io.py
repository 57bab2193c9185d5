"""pf_step_io: one step from a host state to a host state with the upload, the
sweeps and the download overlapped in z-slabs.  It must equal pf_write +
pf_step(1) + pf_read bit for bit — the returned state and the state it leaves
on the device — on the slab pipeline (single block: ragged last slab, one-slab
and many-slab grids, anisotropic, in place) and on the paths that fall back to
the plain calls (several blocks, moving window, Algorithm 2's split)."""
import numpy as np
import pytest

from inputs import gen

pytestmark = pytest.mark.gpu


def _pf():
    from paper_1506_01684_b200 import pf
    return pf


def _state(cfg_name, nx, ny, nz):
    cfg = gen.load_config(cfg_name)
    return cfg, gen.generate(gen.spec_from_config(cfg, nx, ny), nx, ny, nz)


def _pair(pd, cfg, phi, mu, blocks=(1, 1, 1), more=3, **kw):
    """(step_io result, plain result, states after `more` further pf_steps)"""
    pf = _pf()
    nz, ny, nx = phi.shape[1:]
    prm = pf.make_params(pd, cfg, **kw)
    with pf.Context(nx, ny, nz, prm, *blocks) as a, pf.Context(nx, ny, nz, prm, *blocks) as b:
        ra = a.step_io(phi, mu)
        b.write(phi, mu)
        b.step(1)
        rb = b.read()
        assert a.info().step == b.info().step == 1
        a.step(more)
        b.step(more)
        return ra, rb, a.read(), b.read()


def _equal(x, y):
    return np.array_equal(x[0], y[0]) and np.array_equal(x[1], y[1])


@pytest.mark.parametrize("shape", [(32, 24, 20), (64, 48, 130), (128, 128, 128), (40, 32, 8)])
def test_step_io_bitwise(pv1, shape):
    cfg, (phi, mu) = _state("c2", *shape)
    ra, rb, sa, sb = _pair(pv1, cfg, phi, mu, layer_height=shape[2] * 0.45, window=False)
    assert _equal(ra, rb) and _equal(sa, sb)
    assert not np.array_equal(ra[0], phi)   # the step moved the state


def test_step_io_anisotropic(pv1):
    cfg, (phi, mu) = _state("c5", 48, 40, 72)
    ra, rb, sa, sb = _pair(pv1, cfg, phi, mu, layer_height=30.5, window=False)
    assert _equal(ra, rb) and _equal(sa, sb)


def test_step_io_in_place_trajectory(pv1):
    # the same host arrays in and out, three steps: the trajectory of pf_step(3)
    pf = _pf()
    cfg, (phi, mu) = _state("c2", 64, 64, 96)
    prm = pf.make_params(pv1, cfg, layer_height=40.0, window=False)
    hphi, hmu = phi.copy(), mu.copy()
    with pf.Context(64, 64, 96, prm) as a, pf.Context(64, 64, 96, prm) as b:
        for _ in range(3):
            a.step_io(hphi, hmu, hphi, hmu)
        b.write(phi, mu)
        b.step(3)
        ref = b.read()
        assert a.info().step == 3
    assert _equal((hphi, hmu), ref)


def test_step_io_window_shifts(pv1):
    # moving window with shifts during the run (front above 2/3 of the height):
    # the streamed step re-reads the state a shift changed after its download
    pf = _pf()
    cfg, (phi, mu) = _state("c5", 24, 24, 24)
    prm = pf.make_params(pv1, cfg, layer_height=17.5, window=True)
    ha, ma, hb, mb = phi.copy(), mu.copy(), phi.copy(), mu.copy()
    with pf.Context(24, 24, 24, prm) as a, pf.Context(24, 24, 24, prm) as b:
        for _ in range(6):
            a.step_io(ha, ma, ha, ma)
            b.write(hb, mb)
            b.step(1)
            b.read(hb, mb)
            assert _equal((ha, ma), (hb, mb))
        assert a.info().shifts == b.info().shifts > 0
        assert a.info().z_origin == b.info().z_origin


@pytest.mark.parametrize("kw", [dict(blocks=(2, 1, 1)), dict(blocks=(1, 1, 2)), dict(window=True),
                                dict(overlap=2)])
def test_step_io_fallback_paths(pv1, kw):
    cfg, (phi, mu) = _state("c2", 32, 32, 40)
    blocks = kw.pop("blocks", (1, 1, 1))
    kw.setdefault("window", False)
    ra, rb, sa, sb = _pair(pv1, cfg, phi, mu, blocks=blocks, layer_height=20.5, **kw)
    assert _equal(ra, rb) and _equal(sa, sb)


def test_step_io_pinned_torch_buffers(pv1):
    import torch
    pf = _pf()
    cfg, (phi, mu) = _state("c2", 64, 32, 48)
    prm = pf.make_params(pv1, cfg, layer_height=20.5, window=False)
    tphi = torch.from_numpy(phi).pin_memory()
    tmu = torch.from_numpy(mu).pin_memory()
    with pf.Context(64, 32, 48, prm) as a, pf.Context(64, 32, 48, prm) as b:
        a.step_io(tphi, tmu, tphi, tmu)
        b.write(phi, mu)
        b.step(1)
        ref = b.read()
    assert _equal((tphi.numpy(), tmu.numpy()), ref)


def test_step_io_null_pointer(pv1):
    pf = _pf()
    cfg, (phi, mu) = _state("c2", 16, 16, 16)
    prm = pf.make_params(pv1, cfg, layer_height=8.5, window=False)
    with pf.Context(16, 16, 16, prm) as a:
        with pytest.raises(pf.PfError) as e:
            a._check(pf.lib().pf_step_io(a._c, None, None, None, None))
        assert e.value.status == pf.PF_ERR_ARG
