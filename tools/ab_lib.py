"""Time the C4 step with an alternative libpf build (timing experiments only)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1506_01684_b200.pf as pfm
if len(sys.argv) > 1:
    pfm.LIB_PATH = sys.argv[1]
import torch
from inputs import gen
cfg = gen.load_config("c4"); pd = gen.load_params("v1"); n = 512
prm = pfm.make_params(pd, cfg, nx=n, ny=n)
s = torch.cuda.Stream()
with pfm.Context(n, n, n, prm, stream=s.cuda_stream) as ctx:
    ctx.init(cfg["seed"]); ctx.step(3); ctx.set_timing(True); ctx.step(20)
    inf = ctx.info()
    print(sys.argv[1:] or "default", "phi", round(inf.ms_phi / inf.phi_launches, 3), "mu", round(inf.ms_mu / inf.mu_launches, 3))
