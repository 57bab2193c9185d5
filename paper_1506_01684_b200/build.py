"""Build libpf.so (sm_100a) in-tree with nvcc.  Called by __graft_entry__.build()."""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libpf.so")
SOURCES = ["pf_runtime.cu", "pf_kernels.cu", "pf_phi.cu", "pf_mu.cu", "pf_fused.cu", "pf_mesh.cu"]
HEADERS = ["pf_dev.cuh", "pf_kernels.cuh", "pf_tile.cuh"]


def _nccl_dirs():
    import importlib.util
    spec = importlib.util.find_spec("nvidia")
    roots = list(spec.submodule_search_locations) if spec else []
    for r in roots:
        inc, lib = os.path.join(r, "nccl", "include"), os.path.join(r, "nccl", "lib")
        if os.path.exists(os.path.join(inc, "nccl.h")):
            return inc, lib
    return "/usr/include", "/usr/lib/x86_64-linux-gnu"


def needs_build() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = [os.path.join(CSRC, f) for f in SOURCES + HEADERS]
    deps.append(os.path.join(os.path.dirname(HERE), "include", "pf.h"))
    return any(os.path.getmtime(d) > t for d in deps)


def build(force: bool = False, verbose: bool = False, out: str | None = None, defines=(),
          csrc: str | None = None, extra_sources=(), nccl: bool = True, extra_flags=()) -> str:
    """Compile libpf.so; `out`/`defines`/`csrc` build an alternative copy for A/B timing (tools/);
    `extra_sources` + nccl=False link a test stand-in instead of libnccl (tests/fakenccl)."""
    if out is None and not force and not needs_build():
        return LIB
    src = csrc or CSRC
    inc, libdir = _nccl_dirs()
    os.makedirs(os.path.dirname(os.path.abspath(out or LIB)), exist_ok=True)   # build/ is not in git
    cmd = ["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
           "-Xcompiler", "-fPIC", "-shared", "-Xptxas", "-v" if verbose else "-O3",
           "-I", inc, "-I", os.path.join(os.path.dirname(HERE), "include"),
           *[f"-D{d}" for d in defines], *extra_flags,
           "-o", out or LIB] + [os.path.join(src, f) for f in SOURCES] + list(extra_sources) + \
          (["-L", libdir, "-l:libnccl.so.2", "-Xlinker", "-rpath=" + libdir] if nccl else [])
    subprocess.check_call(cmd)
    return out or LIB


if __name__ == "__main__":
    build(force=True, verbose="-v" in sys.argv)
    print(LIB)
