"""The multi-rank data path (pack -> NCCL send/recv -> unpack halos, the
window allreduce, collective checkpoints, per-rank meshes) with 2, 4 and 8
ranks as threads of one process on the one GPU of this environment, over an
in-process NCCL stand-in (tests/fakenccl/nccl_fake.cu, linked into a test copy
of libpf instead of libnccl).  Every rank's state must equal, bit for bit,
the same global problem run as one context (SURVEY.md §8(e) / pin P9)."""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
FAKE = os.path.join(ROOT, "build", "libpf_fakenccl.so")


@pytest.fixture(scope="module")
def fakelib():
    from paper_1506_01684_b200 import build as B
    srcs = [os.path.join(B.CSRC, f) for f in B.SOURCES + B.HEADERS] + [os.path.join(ROOT, "tests", "fakenccl",
                                                                                      "nccl_fake.cu")]
    if not os.path.exists(FAKE) or any(os.path.getmtime(s) > os.path.getmtime(FAKE) for s in srcs):
        B.build(out=FAKE, extra_sources=[srcs[-1]], nccl=False)
    return FAKE


def _run(lib, **spec):
    env = dict(os.environ, PF_LIB=lib)
    p = subprocess.run([sys.executable, os.path.join(ROOT, "tests", "fakenccl", "run_ranks.py"), json.dumps(spec)],
                       env=env, capture_output=True, text=True, timeout=900)
    assert p.returncode == 0, p.stderr[-3000:]
    out = json.loads(p.stdout.strip().splitlines()[-1])
    assert not out["errors"] and not any(out["alive"]), out
    return out


@pytest.mark.parametrize("blocks", [(2, 1, 1), (2, 2, 1), (2, 2, 2), (1, 2, 2)])
def test_ranks_bitwise_equal_single_context(fakelib, blocks):
    out = _run(fakelib, grid=[32, 24, 20], blocks=list(blocks), steps=12, layer_height=9.5)
    assert out["equal_phi"] and out["equal_mu"] and out["moved"] > 1e-3


@pytest.mark.parametrize("overlap", [1, 2, 3])
def test_ranks_overlap_modes(fakelib, overlap):
    out = _run(fakelib, grid=[32, 24, 20], blocks=[2, 2, 2], steps=8, overlap=overlap, layer_height=9.5)
    assert out["equal_phi"] and out["equal_mu"]


@pytest.mark.parametrize("blocks", [(2, 1, 1), (2, 2, 2)])
def test_ranks_fused_bitwise_equal_single_context(fakelib, blocks):
    # every rank with fused steps (both ghost exchanges after each fused kernel,
    # over the NCCL stand-in) against one context with the separate sweeps
    out = _run(fakelib, grid=[32, 24, 20], blocks=list(blocks), steps=12, layer_height=9.5, fusion=True)
    assert out["equal_phi"] and out["equal_mu"] and out["moved"] > 1e-3


def test_ranks_fused_window_aniso(fakelib):
    out = _run(fakelib, grid=[24, 24, 24], blocks=[2, 2, 2], steps=30, window=True, config="c5",
               layer_height=17.5, aniso=True, fusion=True)
    assert out["equal_phi"] and out["equal_mu"]
    assert out["ref_shifts"] > 0 and out["shifts"] == [out["ref_shifts"]] * 8


def test_ranks_step_io(fakelib):
    out = _run(fakelib, grid=[32, 24, 20], blocks=[2, 1, 2], steps=6, step_io=True, layer_height=9.5)
    assert out["equal_phi"] and out["equal_mu"]


def test_ranks_window_aniso(fakelib):
    # forced window shifts through the allreduce(max) of the front, D3C19 halos
    out = _run(fakelib, grid=[24, 24, 24], blocks=[2, 2, 2], steps=30, window=True, config="c5",
               layer_height=17.5, aniso=True)
    assert out["equal_phi"] and out["equal_mu"]
    assert out["ref_shifts"] > 0 and out["shifts"] == [out["ref_shifts"]] * 8


def test_ranks_checkpoint_and_mesh(fakelib):
    out = _run(fakelib, grid=[32, 24, 20], blocks=[2, 1, 2], steps=10, checkpoint=True, mesh=True,
               layer_height=9.5)
    assert out["equal_phi"] and out["equal_mu"]
    assert out["checkpoint_equal"] and out["mesh_equal"]


def test_ranks_interior_shell_mode(fakelib):
    # overlap mode 4 with blocks large enough to have interior mu tiles (3 x 3
    # tiles of 32 x 8 per block): the phi halo beside the interior mu-sweep
    out = _run(fakelib, grid=[192, 48, 24], blocks=[2, 2, 2], steps=6, overlap=4, layer_height=11.5)
    assert out["equal_phi"] and out["equal_mu"]
