"""A/B timing of kernel variants on the bench workload (C4 512^3) in one process."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from inputs import gen
from paper_1506_01684_b200 import pf

cfg = gen.load_config("c4")
pd = gen.load_params("v1")
n = int(os.environ.get("N", 512))
variants = [int(v) for v in sys.argv[1:]] or [0, 2]
res = {}
for rep in range(2):
    for v in variants:
        prm = pf.make_params(pd, cfg, nx=n, ny=n, variant=v)
        s = torch.cuda.Stream()
        with pf.Context(n, n, n, prm, stream=s.cuda_stream) as ctx:
            ctx.init(cfg["seed"])
            ctx.step(3)
            ctx.set_timing(True)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(s); ctx.step(20); e1.record(s); torch.cuda.synchronize()
            inf = ctx.info()
            res[(rep, v)] = dict(step=e0.elapsed_time(e1) / 20, phi=inf.ms_phi / inf.phi_launches,
                                 mu=inf.ms_mu / inf.mu_launches, halo=inf.ms_halo / 20)
for k, r in res.items():
    print(k, {kk: round(vv, 3) for kk, vv in r.items()})
