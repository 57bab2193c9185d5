"""CPU-side checks of the C-ABI library: it loads without a GPU and exports
every symbol include/pf.h declares (no compute calls here)."""
import ctypes
import os
import re

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    src = open(os.path.join(ROOT, "include", "pf.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(pf_[a-z_]+)\s*\(", src)))


def test_library_builds_and_exports_all_declared_symbols():
    from paper_1506_01684_b200 import build, pf
    build.build()
    lib = ctypes.CDLL(pf.LIB_PATH)
    names = _declared()
    assert "pf_create" in names and "pf_step" in names and "pf_read" in names and "pf_init" in names
    for n in names:
        assert hasattr(lib, n), n
    assert set(names) == set(pf.EXPORTS)


def test_struct_sizes_match_header():
    # the ctypes mirrors must match the C layout (compiled probe)
    import subprocess
    import tempfile
    from paper_1506_01684_b200 import pf
    code = '#include <stdio.h>\n#include "pf.h"\nint main(){printf("%zu %zu %zu\\n", sizeof(pf_grid),' \
           ' sizeof(pf_params), sizeof(pf_info_t));return 0;}\n'
    with tempfile.TemporaryDirectory() as d:
        c = os.path.join(d, "p.c")
        open(c, "w").write(code)
        exe = os.path.join(d, "p")
        subprocess.check_call(["gcc", "-I", os.path.join(ROOT, "include"), "-o", exe, c])
        out = subprocess.check_output([exe]).decode().split()
    assert [int(x) for x in out] == [ctypes.sizeof(pf.PfGrid), ctypes.sizeof(pf.PfParams), ctypes.sizeof(pf.PfInfo)]


def test_create_without_gpu_fails_loudly():
    import torch
    if torch.cuda.is_available():
        return
    from paper_1506_01684_b200 import pf
    from inputs import gen
    prm = pf.make_params(gen.load_params("v1"), gen.load_config("c1"))
    try:
        pf.Context(8, 8, 8, prm)
    except pf.PfError as e:
        assert e.status in (pf.PF_ERR_CUDA,)
    else:
        raise AssertionError("pf_create succeeded without a GPU")


def test_mesh_case_table_matches_oracle():
    # host logic of the CUDA path (pf_mesh_table, generated in C++ from reading
    # R26) against the oracle's own case construction, all 256 cases
    from paper_1506_01684_b200 import pf
    from oracle import mesh as MC
    t = pf.mesh_table()
    for case in range(256):
        ref = [tuple(tr) for tr in MC.cube_triangles([(case >> c) & 1 == 1 for c in range(8)])]
        got = [tuple(int(x) for x in t[case, 1 + 3 * i:4 + 3 * i]) for i in range(t[case, 0])]
        assert got == ref, case


def test_create_validates_before_the_device():
    # empty, degenerate and inconsistent configurations are rejected by
    # pf_create's validation (PF_ERR_CONFIG, message in pf_last_error) before
    # any device is touched, so this runs without a GPU
    import pytest
    from paper_1506_01684_b200 import pf
    from inputs import gen
    cfg = gen.load_config("c1")
    good = dict(nx=16, ny=16, nz=16, blocks=(1, 1, 1))
    cases = [(dict(nx=0), "axis x: non-positive"), (dict(nz=-4), "axis z: non-positive"),
             (dict(ny=1), "axis y: blocks must be >= 2"), (dict(nx=16, blocks=(16, 1, 1)), "axis x: blocks must be >= 2"),
             (dict(nz=15, blocks=(1, 1, 2)), "axis z: 15 cells not divisible")]
    for over, msg in cases:
        a = dict(good, **over)
        prm = pf.make_params(gen.load_params("v1"), cfg)
        with pytest.raises(pf.PfError) as e:
            pf.Context(a["nx"], a["ny"], a["nz"], prm, *a["blocks"])
        assert e.value.status == pf.PF_ERR_CONFIG and msg in str(e.value), (over, str(e.value))
    prm = pf.make_params(gen.load_params("v1"), cfg)
    prm.gamma[0][1] = 0.5 * prm.gamma[0][1]   # not symmetric any more
    with pytest.raises(pf.PfError) as e:
        pf.Context(16, 16, 16, prm)
    assert e.value.status == pf.PF_ERR_CONFIG and "not symmetric" in str(e.value)


def test_create_rejects_unstable_dt_and_nonpositive_A():
    # the explicit-Euler bound (reading R29) and
    # A(T) > 0 over the initial window (reading R7) — before the device
    import pytest
    from paper_1506_01684_b200 import pf
    from inputs import gen
    cfg = gen.load_config("c1")
    pd = gen.load_params("v1")
    # PARAMS-v1: D_mu = 1 * 1.0/0.5 = 2, D_phi = 2 * 1 * T_max / 1 ~ 2: bound ~ 1/12
    for dt, ok in [(0.03, True), (0.08, True), (0.09, False), (0.5, False)]:
        prm = pf.make_params(dict(pd, dt=dt), cfg)
        if ok:
            try:
                pf.Context(8, 8, 8, prm)
            except pf.PfError as e:   # no GPU here: validation passed, the device step failed
                assert e.status == pf.PF_ERR_CUDA, str(e)
        else:
            with pytest.raises(pf.PfError) as e:
                pf.Context(8, 8, 8, prm)
            assert e.value.status == pf.PF_ERR_CONFIG and "explicit-Euler bound" in str(e.value), str(e.value)
    prm = pf.make_params(dict(pd, G=0.5), cfg)        # T over the window reaches A^l(T) <= 0
    with pytest.raises(pf.PfError) as e:
        pf.Context(8, 8, 8, prm)
    assert e.value.status == pf.PF_ERR_CONFIG and "<= 0" in str(e.value), str(e.value)


def test_generic_params_pass_validation():
    # params/generic.json (distinct coefficients, tests/test_gpu_generic.py) is
    # inside the explicit-Euler bound and keeps A(T) > 0: pf_create's
    # validation accepts it, isotropic and with the full anisotropy matrix
    from paper_1506_01684_b200 import pf
    from inputs import gen
    cfg = gen.load_config("c2")
    for aniso in (False, True):
        prm = pf.make_params(gen.load_params("generic"), cfg, aniso=aniso)
        try:
            pf.Context(40, 19, 12, prm).close()
        except pf.PfError as e:   # no GPU here: validation passed, the device step failed
            assert e.status == pf.PF_ERR_CUDA, str(e)
