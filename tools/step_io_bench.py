"""pf_step_io vs pf_write + pf_step(1) + pf_read at the C4 size (pinned host
buffers, in place): the e2e path of bench.py."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from inputs import gen
from paper_1506_01684_b200 import pf

n = int(sys.argv[1]) if len(sys.argv) > 1 else 512
cfg, pd = gen.load_config("c4"), gen.load_params("v1")
prm = pf.make_params(pd, cfg, nx=n, ny=n, window=False)
with pf.Context(n, n, n, prm) as ctx:
    ctx.init(cfg["seed"])
    hphi = torch.empty((4, n, n, n), dtype=torch.float64, pin_memory=True)
    hmu = torch.empty((2, n, n, n), dtype=torch.float64, pin_memory=True)
    ctx.read(hphi, hmu)
    for name, fn in (("write+step+read", lambda: (ctx.write(hphi, hmu), ctx.step(1), ctx.read(hphi, hmu))),
                     ("step_io", lambda: ctx.step_io(hphi, hmu, hphi, hmu))):
        fn()
        ts = []
        for _ in range(3):
            t0 = time.perf_counter()
            fn()
            ts.append(time.perf_counter() - t0)
        t = min(ts)
        print(f"{name:16s} {1e3 * t:8.1f} ms/step  {n ** 3 / t / 1e6:8.1f} MLUP/s  "
              f"{2 * 48 * n ** 3 / t / 1e9:6.1f} GB/s over PCIe (both directions)")
