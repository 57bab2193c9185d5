"""Time the step with one libpf build (PF_LIB; timing experiments only).
Workload: C4 512^3 (isotropic), or C5's anisotropic model on a 512^3 block with ANISO=1."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1506_01684_b200.pf as pfm
import torch
from inputs import gen
aniso = os.environ.get("ANISO") == "1"
cfg = gen.load_config("c5" if aniso else "c4"); pd = gen.load_params("v1"); n = 512
prm = pfm.make_params(pd, cfg, nx=n, ny=n, window=False, variant=int(os.environ.get("VARIANT", 0)),
                      shortcuts=os.environ.get("SHORTCUTS") == "1")
s = torch.cuda.Stream()
with pfm.Context(n, n, n, prm, stream=s.cuda_stream) as ctx:
    ctx.init(cfg["seed"]); ctx.step(3); ctx.set_timing(True); ctx.step(20)
    inf = ctx.info()
    print(os.environ.get("PF_LIB", "default"), "v" + os.environ.get("VARIANT", "0"), "sc" + os.environ.get("SHORTCUTS", "0"), "aniso" if aniso else "iso", "phi", round(inf.ms_phi / inf.phi_launches, 3),
          "mu", round(inf.ms_mu / inf.mu_launches, 3), "halo", round(inf.ms_halo / 20, 3))
