"""A/B of the fused mu(n) + phi(n+1) kernel against the separate sweeps on one
config (default C4 512^3): ms per step with fusion off / on, per-kernel device
times (pf_set_timing), and a bitwise comparison of the two end states.

    python tools/fused_ab.py [--config c4] [--steps 20] [--grid NX NY NZ]
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c4")
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--grid", type=int, nargs=3)
    ap.add_argument("--shortcuts", action="store_true")
    a = ap.parse_args()
    import numpy as np
    import torch
    from inputs import gen
    from paper_1506_01684_b200 import pf
    cfg = gen.load_config(a.config)
    NX, NY, NZ = a.grid or (cfg["nx"], cfg["ny"], cfg["nz"])
    prm = pf.make_params(gen.load_params("v1"), cfg, nx=NX, ny=NY, shortcuts=a.shortcuts)
    stream = torch.cuda.Stream()
    out = {"config": a.config, "grid": [NX, NY, NZ], "steps": a.steps}
    states = {}
    for fusion in (False, True, False, True):
        with pf.Context(NX, NY, NZ, prm, stream=stream.cuda_stream) as ctx:
            ctx.set_fusion(fusion)
            ctx.init(cfg["seed"])
            ctx.step(3)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            ctx.step(a.steps)
            e1.record(stream)
            torch.cuda.synchronize()
            ms = e0.elapsed_time(e1) / a.steps
            ctx.set_timing(True)
            ctx.step(a.steps)
            inf = ctx.info()
            k = "fused" if fusion else "plain"
            out[k] = {"ms_per_step": round(ms, 4), "mlups": round(NX * NY * NZ / ms / 1e3, 1),
                      "ms_phi": round(inf.ms_phi / max(1, inf.phi_launches), 4),
                      "ms_mu": round(inf.ms_mu / max(1, inf.mu_launches), 4),
                      "ms_fused": round(inf.ms_fused / max(1, inf.fused_launches), 4),
                      "ms_halo_per_step": round(inf.ms_halo / a.steps, 4),
                      "ms_other_per_step": round(inf.ms_other / a.steps, 4)}
            if k not in states:
                phi, mu = ctx.read()
                states[k] = (phi[:, ::7], mu[:, ::7])
    out["bitwise_equal"] = bool(np.array_equal(states["plain"][0], states["fused"][0]) and
                                np.array_equal(states["plain"][1], states["fused"][1]))
    print(json.dumps(out))


if __name__ == "__main__":
    main()
