"""Step time with CUDA-graph replay vs kernels launched one by one
(pf_params.graph), for the small configs where launch overhead matters
(C1 32^3, C2 128^3) and the bench workload (C4 512^3).  Markdown table."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
from inputs import gen  # noqa: E402
from paper_1506_01684_b200 import pf  # noqa: E402

rows = ["| config | cells | eager ms/step | graph ms/step | gain |", "|---|---|---|---|---|"]
pd = gen.load_params("v1")
for name, n, steps in (("c1", 32, 400), ("c2", 128, 200), ("c4", 512, 20)):
    cfg = gen.load_config(name)
    t = {}
    for ng in (True, False):
        prm = pf.make_params(pd, cfg, nx=n, ny=n, graph=not ng, window=False)
        s = torch.cuda.Stream()
        with pf.Context(n, n, n, prm, stream=s.cuda_stream) as ctx:
            ctx.init(cfg["seed"])
            ctx.step(5)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(s)
            ctx.step(steps)
            e1.record(s)
            torch.cuda.synchronize()
            t[ng] = e0.elapsed_time(e1) / steps
    rows.append(f"| {name} | {n}^3 | {t[True]:.4f} | {t[False]:.4f} | {t[True] / t[False]:.2f}x |")
print("# CUDA-graph replay vs eager launches, one B200 (tools/graph_gain.py)\n")
print("\n".join(rows))
