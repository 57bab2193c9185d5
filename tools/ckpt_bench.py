"""FP32 checkpoint throughput (NEXT-3): pf_save / pf_load of
the C4 state at 512^3 (24 B per cell: 3.2 GB) to a file under $CKPT_DIR
(default /tmp), three repetitions each, plus a restart check (the loaded state
equals the binary32 cast of the saved one: tests/test_gpu_checkpoint.py covers
it bitwise, here only the timing).  Prints one JSON line."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from inputs import gen  # noqa: E402
from paper_1506_01684_b200 import pf  # noqa: E402

n = int(os.environ.get("N", 512))
d = os.environ.get("CKPT_DIR", "/tmp")
path = os.path.join(d, f"pf_ckpt_{os.getpid()}.bin")
cfg = gen.load_config("c4")
prm = pf.make_params(gen.load_params("v1"), cfg, nx=n, ny=n)
out = {"cells": n ** 3, "bytes": 72 + 24 * n ** 3, "dir": d}
with pf.Context(n, n, n, prm) as ctx:
    ctx.init(cfg["seed"])
    ctx.step(2)
    for op in ("save", "load"):
        ts = []
        for _ in range(3):
            t0 = time.perf_counter()
            (ctx.save if op == "save" else ctx.load)(path)
            ts.append(time.perf_counter() - t0)
        ts.sort()
        out[f"{op}_s"] = [round(t, 3) for t in ts]
        out[f"{op}_gbs_median"] = round(out["bytes"] / ts[1] / 1e9, 2)
os.remove(path)
print(json.dumps(out))
