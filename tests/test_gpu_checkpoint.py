"""FP32 checkpoint / restart on the CUDA path (NEXT-3; PAPER.md:239-245,
format SPEC.md:462-466) against the oracle's plain encoder (oracle/checkpoint.py).

Byte work, so bit-exact: pf_save's file equals the oracle encoding of the
state pf_read returns; pf_load reproduces the exact binary64 widening of the
stored binary32 values; a resumed run equals, bit for bit, the same run
restarted from the binary32-cast state, and stays within the 100-step parity
tolerance of the oracle run from that state.
"""
import numpy as np
import pytest

from inputs import gen
from oracle import checkpoint as CK
from oracle import oracle as O

pytestmark = pytest.mark.gpu

TOL100 = 1e-8


def _pf():
    from paper_1506_01684_b200 import pf
    return pf


def _state(cfg_name, nx, ny, nz, **over):
    cfg = gen.load_config(cfg_name)
    spec = gen.spec_from_config(cfg, nx, ny)
    for k, v in over.items():
        setattr(spec, k, v)
    return cfg, gen.generate(spec, nx, ny, nz)


@pytest.mark.parametrize("blocks", [(1, 1, 1), (2, 2, 2), (1, 3, 2)])
def test_save_matches_oracle_encoding(pv1, tmp_path, blocks):
    pf = _pf()
    nx, ny, nz = 40, 24, 20
    cfg, (phi, mu) = _state("c2", nx, ny, nz, layer_height=9, n_seeds=8, mu_noise=1e-2)
    prm = pf.make_params(pv1, cfg, layer_height=9)
    path = tmp_path / "s.pfcp"
    with pf.Context(nx, ny, nz, prm, *blocks) as ctx:
        ctx.write(phi, mu)
        ctx.set_time(3, 2)
        ctx.step(5)
        gphi, gmu = ctx.read()
        ctx.save(path)
        ctx.step(1)                    # the context stays usable after a save
    want = CK.encode(gphi, gmu, pv1["dx"], 8 * pv1["dt"], 8, 2)
    assert path.read_bytes() == want


@pytest.mark.parametrize("blocks", [(1, 1, 1), (2, 1, 2)])
def test_load_oracle_file(pv1, tmp_path, blocks):
    pf = _pf()
    nx, ny, nz = 24, 16, 12
    cfg, (phi, mu) = _state("c2", nx, ny, nz, layer_height=6, n_seeds=5, mu_noise=1e-2)
    path = tmp_path / "o.pfcp"
    CK.write_checkpoint(path, phi, mu, pv1["dx"], 123 * pv1["dt"], 123, 45)
    _, p32, m32 = CK.read_checkpoint(path)
    prm = pf.make_params(pv1, cfg, layer_height=6)
    with pf.Context(nx, ny, nz, prm, *blocks) as ctx:
        ctx.load(path)
        gphi, gmu = ctx.read()
        inf = ctx.info()
    assert inf.step == 123 and inf.z_origin == 45
    assert np.array_equal(gphi, p32.astype(np.float64)) and np.array_equal(gmu, m32.astype(np.float64))


def test_resume_equivalence_with_window(pv1, tmp_path):
    # run 60 steps, checkpoint, resume in a fresh context (other decomposition)
    # for 60 more; the window fires in both halves (same setup as the forced
    # shift test)
    pf = _pf()
    nx, ny, nz = 16, 16, 24
    cfg, (phi, mu) = _state("c3", nx, ny, nz, layer_height=16.95)
    pd = dict(pv1, G=0.0)
    prm = pf.make_params(pd, cfg, window=True, T0=pv1["T_eut"] - 0.5)
    path = tmp_path / "w.pfcp"
    with pf.Context(nx, ny, nz, prm) as a:
        a.write(phi, mu)
        a.step(60)
        a.save(path)
        mid = a.read()
        ia = a.info()
    assert ia.shifts >= 1
    with pf.Context(nx, ny, nz, prm, 2, 1, 2) as b:
        b.load(path)
        b.step(60)
        rphi, rmu = b.read()
        ib = b.info()
    # the same continuation from the binary32-cast state, written directly
    cphi = mid[0].astype(np.float32).astype(np.float64)
    cmu = mid[1].astype(np.float32).astype(np.float64)
    with pf.Context(nx, ny, nz, prm) as c:
        c.write(cphi, cmu)
        c.set_time(60, ia.z_origin)
        c.step(60)
        sphi, smu = c.read()
        ic = c.info()
    assert ib.step == ic.step == 120 and ib.z_origin == ic.z_origin
    assert np.array_equal(rphi, sphi) and np.array_equal(rmu, smu)
    # and the oracle from the cast state agrees within the parity tolerance
    op = O.make_params(pd, T0=pv1["T_eut"] - 0.5)
    ophi, omu, oz = O.run(op, cphi, cmu, 60, n0=60, zorig=ia.z_origin, window_on=True)
    assert oz == ib.z_origin
    assert O.rel_maxnorm(rphi, ophi) <= TOL100 and O.rel_maxnorm(rmu, omu) <= TOL100


def test_multichunk_roundtrip(pv1, tmp_path):
    # 128 x 128 x 600: more than one 32 MB conversion chunk per component
    pf = _pf()
    nx, ny, nz = 128, 128, 600
    cfg = gen.load_config("c3")
    prm = pf.make_params(pv1, cfg, nx=nx, ny=ny)
    path = tmp_path / "m.pfcp"
    with pf.Context(nx, ny, nz, prm) as ctx:
        ctx.init(cfg["seed"])
        ctx.step(2)
        gphi, gmu = ctx.read()
        ctx.save(path)
        ctx.load(path)
        lphi, lmu = ctx.read()
    assert path.stat().st_size == 72 + 6 * nx * ny * nz * 4
    hdr, p32, m32 = CK.read_checkpoint(path)
    assert hdr["step"] == 2 and hdr["nz"] == nz
    assert np.array_equal(p32, gphi.astype(np.float32)) and np.array_equal(m32, gmu.astype(np.float32))
    assert np.array_equal(lphi, p32.astype(np.float64)) and np.array_equal(lmu, m32.astype(np.float64))


def test_load_errors_leave_context_usable(pv1, tmp_path):
    pf = _pf()
    nx, ny, nz = 16, 16, 16
    cfg, (phi, mu) = _state("c1", nx, ny, nz, layer_height=6)
    prm = pf.make_params(pv1, cfg)
    good = CK.encode(phi, mu, pv1["dx"], 0.0, 0, 0)
    bad = {
        "magic": b"XFCP0001" + good[8:],
        "trunc": good[:-4],
        "dims": CK.encode(phi[:, :, :, :8], mu[:, :, :, :8], pv1["dx"], 0.0, 0, 0),
        "dx": CK.encode(phi, mu, 2 * pv1["dx"], 0.0, 0, 0),
    }
    with pf.Context(nx, ny, nz, prm) as ctx:
        ctx.write(phi, mu)
        for name, data in bad.items():
            p = tmp_path / f"{name}.pfcp"
            p.write_bytes(data)
            with pytest.raises(pf.PfError) as e:
                ctx.load(p)
            assert e.value.status == pf.PF_ERR_IO, name
        with pytest.raises(pf.PfError) as e:
            ctx.load(tmp_path / "missing.pfcp")
        assert e.value.status == pf.PF_ERR_IO
        with pytest.raises(pf.PfError) as e:
            ctx.save(tmp_path / "no_such_dir" / "x.pfcp")
        assert e.value.status == pf.PF_ERR_IO
        # state untouched, context still steps
        p2, m2 = ctx.read()
        assert np.array_equal(p2, phi) and np.array_equal(m2, mu)
        ctx.step(1)
