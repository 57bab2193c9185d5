"""Scenario benchmarks: per-sweep time on
blocks that are all interface (C4 front), all solid (Voronoi grains with grain
boundaries, no liquid) or all liquid, with and without region shortcuts
(NEXT-1).  Prints a markdown table; 256^3 blocks by default (N env); ANISO=1: the
C5 model (cubic anisotropy on the solid-liquid pairs)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from inputs import gen
from paper_1506_01684_b200 import pf

n = int(os.environ.get("N", 256))
pd = gen.load_params("v1")
aniso = os.environ.get("ANISO") == "1"
cfg = gen.load_config("c5" if aniso else "c4")
spec = gen.spec_from_config(cfg, n, n)
scen = {}
spec.layer_height = n / 2
scen["interface (front at mid-height)"] = gen.generate(spec, n, n, n)
spec.layer_height = 2 * n
scen["solid (grains, no liquid)"] = gen.generate(spec, n, n, n)
phi = np.zeros((4, n, n, n))
phi[3] = 1.0
rng = np.random.default_rng(0)
scen["liquid"] = (phi, 1e-3 * rng.uniform(-1, 1, (2, n, n, n)))
rows = ["| scenario | shortcuts | phi ms | mu ms | phi MLUP/s | mu MLUP/s | step MLUP/s |", "|---|---|---|---|---|---|---|"]
for name, (phi, mu) in scen.items():
    for sc in (False, True):
        prm = pf.make_params(pd, cfg, layer_height=n / 2, shortcuts=sc)
        s = torch.cuda.Stream()
        with pf.Context(n, n, n, prm, stream=s.cuda_stream) as ctx:
            ctx.write(phi, mu)
            ctx.step(3)
            ctx.set_timing(True)
            ctx.step(10)
            inf = ctx.info()
            tp, tm = inf.ms_phi / inf.phi_launches, inf.ms_mu / inf.mu_launches
        cells = n ** 3
        rows.append(f"| {name} | {'on' if sc else 'off'} | {tp:.3f} | {tm:.3f} | {cells / tp / 1e3:.0f} | "
                    f"{cells / tm / 1e3:.0f} | {cells / (tp + tm) / 1e3:.0f} |")
print(f"# Scenario benchmarks, {n}^3 block, one B200 (tools/scenarios.py)\n")
print("\n".join(rows))
