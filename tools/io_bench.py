"""pf_write / pf_read throughput at 512^3 (6 x 1 GiB of state): pinned host
buffers (PCIe + layout kernels) and device buffers (layout kernels only)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
from inputs import gen  # noqa: E402
from paper_1506_01684_b200 import pf  # noqa: E402

n = int(os.environ.get("N", 512))
cfg = gen.load_config("c4")
prm = pf.make_params(gen.load_params("v1"), cfg, nx=n, ny=n)
with pf.Context(n, n, n, prm) as ctx:
    ctx.init(cfg["seed"])
    nbytes = 6 * n ** 3 * 8
    for where in ("pinned host", "device"):
        kw = dict(dtype=torch.float64, pin_memory=True) if where == "pinned host" else dict(dtype=torch.float64,
                                                                                            device="cuda")
        phi = torch.empty((4, n, n, n), **kw)
        mu = torch.empty((2, n, n, n), **kw)
        ctx.read(phi, mu)
        for op in ("read", "write"):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            for _ in range(3):
                (ctx.read if op == "read" else ctx.write)(phi, mu)
            torch.cuda.synchronize()
            dt = (time.perf_counter() - t0) / 3
            print(f"pf_{op} {where}: {dt * 1e3:.1f} ms, {nbytes / dt / 1e9:.1f} GB/s")
        del phi, mu
