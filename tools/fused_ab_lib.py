"""Time the fused step with one libpf build (PF_LIB; timing experiments only):
C4 512^3, or C5's anisotropic model on a 512^3 block with ANISO=1."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1506_01684_b200.pf as pfm
import torch
from inputs import gen
aniso = os.environ.get("ANISO") == "1"
cfg = gen.load_config("c5" if aniso else "c4"); pd = gen.load_params("v1"); n = 512
prm = pfm.make_params(pd, cfg, nx=n, ny=n, window=False, shortcuts=os.environ.get("SHORTCUTS") == "1")
s = torch.cuda.Stream()
with pfm.Context(n, n, n, prm, stream=s.cuda_stream) as ctx:
    ctx.set_fusion(os.environ.get("FUSION", "1") == "1")
    ctx.init(cfg["seed"]); ctx.step(3)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize(); e0.record(s); ctx.step(20); e1.record(s); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 20
    ctx.set_timing(True); ctx.step(20)
    inf = ctx.info()
    print(os.environ.get("PF_LIB", "default"), "aniso" if aniso else "iso", "sc" + os.environ.get("SHORTCUTS", "0"), "step", round(ms, 3),
          "fused", round(inf.ms_fused / max(1, inf.fused_launches), 3),
          "phi", round(inf.ms_phi / max(1, inf.phi_launches), 3), "mu", round(inf.ms_mu / max(1, inf.mu_launches), 3))
