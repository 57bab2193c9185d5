"""Run a few steps of the bench workload (C4, 512^3) for ncu captures."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import argparse
from inputs import gen
from paper_1506_01684_b200 import pf

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=512)
ap.add_argument("--steps", type=int, default=2)
ap.add_argument("--aniso", action="store_true")
ap.add_argument("--variant", type=int, default=0)
ap.add_argument("--interface", action="store_true", help="all-guards-open state (bench mu_interface)")
ap.add_argument("--fusion", action="store_true", help="fused mu(n) + phi(n+1) kernel (pf_set_fusion)")
a = ap.parse_args()
cfg = gen.load_config("c5" if a.aniso else "c4")
pd = gen.load_params("v1")
prm = pf.make_params(pd, cfg, nx=a.n, ny=a.n, variant=a.variant, window=False)
with pf.Context(a.n, a.n, a.n, prm) as ctx:
    ctx.set_fusion(a.fusion)
    if a.interface:
        phi, mu = gen.interface_state_torch(ctx.shape, seed=cfg["seed"], device="cuda")
        for _ in range(a.steps):
            ctx.write(phi, mu)
            ctx.step(3 if a.fusion else 1)
    else:
        ctx.init(cfg["seed"])
        ctx.step(a.steps)
    print("ok", ctx.info().launches)
