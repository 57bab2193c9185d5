"""Build alternative libpf.so copies for A/B timing (tools/ab_lib.py on the GPU box).

usage: ab_build.py NAME [REV] [-DFOO ...]
  NAME  output build/libpf_NAME.so
  REV   git revision to take csrc/ from (default: the working tree)
"""
import os, subprocess, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_1506_01684_b200 import build as B

name, rest = sys.argv[1], sys.argv[2:]
defs = [a[2:] for a in rest if a.startswith("-D")]
flags = [a[2:] for a in rest if a.startswith("-F")]          # -F<nvcc flag>, e.g. -F-Xptxas=-foo
revs = [a for a in rest if not a.startswith("-D") and not a.startswith("-F")]
src = None
if revs:
    base = os.path.join(ROOT, "build", "ab")
    src = os.path.join(base, name, "csrc")   # ../../include -> build/ab/include
    os.makedirs(src, exist_ok=True)
    inc = os.path.join(base, "include")
    if not os.path.exists(inc):
        os.symlink(os.path.join(ROOT, "include"), inc)
    for f in B.SOURCES + B.HEADERS:
        blob = subprocess.run(["git", "show", f"{revs[0]}:paper_1506_01684_b200/csrc/{f}"], cwd=ROOT,
                              capture_output=True, check=True).stdout
        open(os.path.join(src, f), "wb").write(blob)
out = os.path.join(ROOT, "build", f"libpf_{name}.so")
B.build(out=out, defines=defs, csrc=src, extra_flags=flags)
print(out)
