"""Index-slip mutants of the CUDA path's coefficient tables, against the GPU
parity tests with PARAMS-v1 and with PARAMS-generic (tests/test_gpu_generic.py).

Each mutant is one plausible index slip in the runtime's kernel constants
(pf_runtime.cu: KParams / TabParams), compiled to a scratch libpf build.  The
point: PARAMS-v1 is symmetric in the solids, so most of these slips pass its
parity tests; every one of them must fail a PARAMS-generic test.

usage: python tools/gpu_index_mutants.py --build          (here: nvcc, build/mut/*.so)
       python tools/gpu_index_mutants.py --run [--out F]  (GPU box: PF_LIB per mutant, pytest)
"""
import argparse
import os
import re
import shutil
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
SRC = "pf_runtime.cu"

MUTANTS = [
    ("triple coefficient gamma3 of the next triple",
     "kp.g3[a] = p->gamma3[a];", "kp.g3[a] = p->gamma3[(a + 1) & 3];"),
    ("pair gamma_ab read as gamma_a,l (gradient energy, faces, obstacle)",
     "kp.g2[q] = 2.0 * p->gamma[pair_a(q)][pair_b(q)];", "kp.g2[q] = 2.0 * p->gamma[pair_a(q)][3];"),
    ("relaxation time tau of phase 0 for every phase",
     "kp.dt_taueps[a] = p->dt / (p->tau[a] * p->eps);", "kp.dt_taueps[a] = p->dt / (p->tau[0] * p->eps);"),
    ("anisotropy delta_ab read as delta_a,l",
     "kp.delta16[q] = p->aniso ? 16.0 * p->delta[pair_a(q)][pair_b(q)] : 0.0;",
     "kp.delta16[q] = p->aniso ? 16.0 * p->delta[pair_a(q)][3] : 0.0;"),
    ("diffusivity of component 0 for both components",
     "tp.D[a][q] = p->D[a][q];", "tp.D[a][q] = p->D[a][0];"),
    ("A1 of component 0 for both components",
     "tp.A0[a][q] = p->A0[a][q]; tp.A1[a][q] = p->A1[a][q];", "tp.A0[a][q] = p->A0[a][q]; tp.A1[a][q] = p->A1[a][0];"),
]

TESTS_V1 = ["tests/test_gpu_parity.py::test_c1_one_step", "tests/test_gpu_parity.py::test_c1_100_steps",
            "tests/test_gpu_parity.py::test_ragged_shapes", "tests/test_gpu_trajectories.py::test_interface_dense_state_one_step"]
TESTS_GENERIC = ["tests/test_gpu_generic.py"]


def lib_of(i):
    return os.path.join(ROOT, "build", "mut", f"libpf_m{i}.so")


def build():
    from paper_1506_01684_b200 import build as B
    src = os.path.join(ROOT, "paper_1506_01684_b200", "csrc")
    for i, (name, old, new) in enumerate(MUTANTS):
        d = os.path.join(ROOT, "build", "mut", f"m{i}", "csrc")
        os.makedirs(d, exist_ok=True)
        inc = os.path.join(ROOT, "build", "mut", "include")   # csrc/../../include (pf_runtime.cu)
        if not os.path.exists(inc):
            os.symlink(os.path.join(ROOT, "include"), inc)
        for f in B.SOURCES + B.HEADERS:
            shutil.copy(os.path.join(src, f), os.path.join(d, f))
        text = open(os.path.join(src, SRC)).read()
        assert text.count(old) == 1, name
        open(os.path.join(d, SRC), "w").write(text.replace(old, new))
        B.build(out=lib_of(i), csrc=d)
        print("built", lib_of(i), name, flush=True)


def run(out):
    rows = []
    for i, (name, _, _) in enumerate(MUTANTS):
        res = []
        for tests in (TESTS_V1, TESTS_GENERIC):
            r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-m", "gpu", "-p", "no:cacheprovider", *tests],
                               cwd=ROOT, env=dict(os.environ, PF_LIB=lib_of(i)), capture_output=True, text=True)
            nf = re.search(r"(\d+) failed", r.stdout)
            np_ = re.search(r"(\d+) passed", r.stdout)
            res.append((int(nf.group(1)) if nf else 0, int(np_.group(1)) if np_ else 0))
        rows.append((name, res))
        print(name, res, flush=True)
    with open(out, "w") as f:
        f.write("# Index-slip mutants of the CUDA path's coefficient tables (round 2)\n\n")
        f.write("`python tools/gpu_index_mutants.py --build` here, `--run` on a B200: each row is one slip in\n"
                "`pf_runtime.cu`'s kernel constants, built as a scratch libpf and run (PF_LIB) against the PARAMS-v1\n"
                "GPU parity tests (" + ", ".join(t.split("::")[-1] for t in TESTS_V1) + ") and\n"
                "`tests/test_gpu_generic.py` (PARAMS-generic: every coefficient distinct).\n\n")
        f.write("| mutant | v1 tests failed / passed | generic tests failed / passed |\n|---|---|---|\n")
        for name, ((f1, p1), (f2, p2)) in rows:
            f.write(f"| {name} | {f1} / {p1} | {'**' if f2 == 0 else ''}{f2}{'**' if f2 == 0 else ''} / {p2} |\n")
        f.write(f"\n{sum(1 for _, r in rows if r[1][0] > 0)} of {len(rows)} mutants fail a generic test; "
                f"{sum(1 for _, r in rows if r[0][0] > 0)} of {len(rows)} fail a v1 test.\n")
    print("->", out)


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--build", action="store_true")
    ap.add_argument("--run", action="store_true")
    ap.add_argument("--out", default=os.path.join(ROOT, "gpurun_out", "gpu_index_mutants.md"))
    a = ap.parse_args()
    if a.build:
        build()
    if a.run:
        run(a.out)
