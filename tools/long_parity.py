"""Long-trajectory parity (evidence beyond the 100-step test): C2 at full size
(128^3), GPU vs the CPU oracle over the whole trajectory, relative max-norm
every `every` steps.  Prints a markdown table.  ~3 min of oracle time."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from inputs import gen  # noqa: E402
from oracle import oracle as O  # noqa: E402
from paper_1506_01684_b200 import pf  # noqa: E402

steps = int(os.environ.get("STEPS", 1000))
every = int(os.environ.get("EVERY", 100))
n = 128
cfg = gen.load_config("c2")
pd = gen.load_params("v1")
spec = gen.spec_from_config(cfg, n, n)
phi, mu = gen.generate(spec, n, n, n)
op = O.make_params(pd, layer_height=cfg["init"]["layer_height"])
prm = pf.make_params(pd, cfg)
rows = ["| step | rel max-norm phi | rel max-norm mu | max abs change phi vs step 0 |", "|---|---|---|---|"]
t0 = time.time()
with pf.Context(n, n, n, prm) as ctx:
    ctx.write(phi, mu)
    ophi, omu = phi, mu
    for s in range(every, steps + 1, every):
        ctx.step(every)
        gphi, gmu = ctx.read()
        ophi, omu, _ = O.run(op, ophi, omu, every, n0=s - every)
        rows.append(f"| {s} | {O.rel_maxnorm(gphi, ophi):.2e} | {O.rel_maxnorm(gmu, omu):.2e} | "
                    f"{abs(gphi - phi).max():.3f} |")
print(f"# Long-trajectory parity, C2 128^3, {steps} steps (tools/long_parity.py, {time.time() - t0:.0f} s)\n")
print("\n".join(rows))
