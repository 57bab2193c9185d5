"""Four-way communication-hiding ablation (NEXT-2):
pf_params.overlap = 1 none, 0 mu only (default), 2 phi only (Algorithm 2
split), 3 both, 4 both without Algorithm 2's second pass (mu-sweep interior
tiles beside the phi halo, the shell after it), on the C4 workload (512^3) as one block and as 2x2x2 blocks on
one GPU (halos are then real device copies).  Step time from CUDA events on
the context's stream; prints a markdown table."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from inputs import gen
from paper_1506_01684_b200 import pf

n = int(os.environ.get("N", 512))
cfg = gen.load_config("c4")
pd = gen.load_params("v1")
names = {1: "none", 0: "mu only (default)", 2: "phi only (Algorithm 2 split)", 3: "both (Algorithm 2)",
         4: "both (mu interior / shell split)"}
rows = ["| blocks | overlap | step ms | phi ms | mu ms (local+neighbor) | halo ms (not hidden) | MLUP/s |",
        "|---|---|---|---|---|---|---|"]
for blocks in ((1, 1, 1), (2, 2, 2)):
    for ov in (1, 0, 2, 3, 4):
        prm = pf.make_params(pd, cfg, nx=n, ny=n, overlap=ov)
        s = torch.cuda.Stream()
        with pf.Context(n, n, n, prm, *blocks, stream=s.cuda_stream) as ctx:
            ctx.init(cfg["seed"])
            ctx.step(3)
            steps = 20
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(s)
            ctx.step(steps)
            e1.record(s)
            torch.cuda.synchronize()
            ms = e0.elapsed_time(e1) / steps
            ctx.set_timing(True)
            ctx.step(steps)
            inf = ctx.info()
            rows.append(f"| {'x'.join(map(str, blocks))} | {ov}: {names[ov]} | {ms:.3f} | {inf.ms_phi / steps:.3f} | "
                        f"{inf.ms_mu / steps:.3f} | {inf.ms_halo / steps:.3f} | {n ** 3 / ms / 1e3:.0f} |")
print(f"# Communication-hiding ablation, {n}^3 (C4), one B200 (tools/overlap_ablation.py)\n")
print("\n".join(rows))
