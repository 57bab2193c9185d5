"""GPU marching cubes (pf_mesh, NEXT-4, reading R26) against
the oracle's plain sweep (oracle/mesh.py) on the GPU state read back through
the C ABI.  Ids are integers (bit-exact); vertex positions are IEEE-rounded
the same way on both sides (bit-exact); the order is the serial (k, j, i)
sweep order on both sides, so the arrays are compared as they are."""
import numpy as np
import pytest

from inputs import gen
from oracle import mesh as MC

pytestmark = pytest.mark.gpu


def _pf():
    from paper_1506_01684_b200 import pf
    return pf


def _run(nx, ny, nz, steps, blocks=(1, 1, 1), zorig=0, cfg_name="c1", seed_state=None):
    pf = _pf()
    cfg = gen.load_config(cfg_name)
    spec = gen.spec_from_config(cfg, nx, ny)
    spec.layer_height = nz / 2
    phi, mu = gen.generate(spec, nx, ny, nz)
    prm = pf.make_params(gen.load_params("v1"), cfg, layer_height=nz / 2, window=False)
    ctx = pf.Context(nx, ny, nz, prm, *blocks)
    ctx.write(phi, mu)
    ctx.set_time(0, zorig)
    ctx.step(steps)
    return ctx


def _check(ctx, phase, iso=0.5, zorig=0, dx=1.0):
    gphi, _ = ctx.read()
    ids, pos = ctx.mesh(phase, iso)
    rids, rpos = MC.marching_cubes(gphi[phase], iso=iso, dx=dx, z_origin=zorig)
    assert ids.shape == rids.shape
    assert np.array_equal(ids, rids)
    assert np.array_equal(pos, rpos)        # bit-exact: same IEEE operations
    return len(ids)


@pytest.mark.parametrize("phase", range(4))
def test_mesh_matches_oracle_every_phase(phase):
    with _run(32, 32, 24, 5) as ctx:
        n = _check(ctx, phase)
        assert n > 100


def test_mesh_ragged_sizes_and_iso():
    # rows longer than a warp and not a multiple of 32; iso off 1/2
    with _run(45, 13, 11, 3) as ctx:
        for a in (0, 3):
            for iso in (0.5, 0.2, 0.83):
                _check(ctx, a, iso)


def test_mesh_decomposition_and_window_origin():
    # 2x2x2 blocks on one GPU (corners read from block ghosts) and a window
    # origin: identical to the single-block sweep
    with _run(24, 20, 16, 4, blocks=(2, 2, 2), zorig=7) as ctx:
        for a in range(4):
            _check(ctx, a, zorig=7)


def test_mesh_empty_and_cap():
    pf = _pf()
    with _run(32, 32, 16, 2) as ctx:
        # a phase with no interface in the box: pure-liquid top cannot produce
        # triangles for iso above every value
        ids, pos = ctx.mesh(0, iso=1.5)
        assert ids.shape == (0, 3) and pos.shape == (0, 3, 3)
        full_ids, full_pos = ctx.mesh(3)
        # cap: the first `cap` triangles of the full list, total reported
        import ctypes
        cap = len(full_ids) // 3
        ids = np.zeros((cap, 3), dtype=np.int64)
        pos = np.zeros((cap, 3, 3))
        n = ctypes.c_int64(0)
        st = pf.lib().pf_mesh(ctx._c, 3, 0.5, cap, ids.ctypes.data, pos.ctypes.data, ctypes.byref(n))
        assert st == pf.PF_OK and n.value == len(full_ids)
        assert np.array_equal(ids, full_ids[:cap]) and np.array_equal(pos, full_pos[:cap])
        with pytest.raises(pf.PfError):
            ctx.mesh(4)


def test_mesh_device_output():
    import torch
    pf = _pf()
    with _run(32, 32, 16, 2) as ctx:
        ref_ids, ref_pos = ctx.mesh(1)
        import ctypes
        n = len(ref_ids)
        ids = torch.zeros((n, 3), dtype=torch.int64, device="cuda")
        pos = torch.zeros((n, 3, 3), dtype=torch.float64, device="cuda")
        m = ctypes.c_int64(0)
        st = pf.lib().pf_mesh(ctx._c, 1, 0.5, n, ids.data_ptr(), pos.data_ptr(), ctypes.byref(m))
        assert st == pf.PF_OK and m.value == n
        assert np.array_equal(ids.cpu().numpy(), ref_ids) and np.array_equal(pos.cpu().numpy(), ref_pos)
