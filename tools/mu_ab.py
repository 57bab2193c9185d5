"""Per-sweep times of a libpf build (PF_LIB selects an A/B copy from
tools/ab_build.py) on the C4 state and on the all-guards-open interface state
(the bench's mu_interface measurement): CUDA-event times (pf_set_timing),
median of the repetitions; --variants picks pf_params.variant (0 tiled, 1 naive).

usage: [PF_LIB=build/libpf_X.so] python tools/mu_ab.py [--n 512] [--reps 5] [--variants 0] [--aniso]"""
import argparse
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from inputs import gen  # noqa: E402
from paper_1506_01684_b200 import pf  # noqa: E402


def sweep_ms(ctx, state=None, steps=5):
    ph, mu = [], []
    for _ in range(steps):
        if state is not None:
            ctx.write(*state)
        ctx.set_timing(True)
        ctx.step(1)
        inf = ctx.info()
        ph.append(inf.ms_phi / max(1, inf.phi_launches))
        mu.append(inf.ms_mu / max(1, inf.mu_launches))
    ctx.set_timing(False)
    return statistics.median(ph), statistics.median(mu)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=512)
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--variants", type=int, nargs="+", default=[0])
    ap.add_argument("--tag", default=os.environ.get("PF_LIB", "default"))
    ap.add_argument("--aniso", action="store_true")
    a = ap.parse_args()
    cfg = gen.load_config("c5" if a.aniso else "c4")
    pd = gen.load_params("v1")
    out = {}
    for v in a.variants:
        prm = pf.make_params(pd, cfg, nx=a.n, ny=a.n, variant=v, window=False)
        with pf.Context(a.n, a.n, a.n, prm) as ctx:
            ctx.init(cfg["seed"])
            ctx.step(3)
            c4 = sweep_ms(ctx, steps=a.reps)
            st = gen.interface_state_torch(ctx.shape, seed=cfg["seed"], device="cuda")
            sweep_ms(ctx, st, steps=1)
            itf = sweep_ms(ctx, st, steps=a.reps)
            del st
        out[v] = {"c4_phi_ms": c4[0], "c4_mu_ms": c4[1], "iface_phi_ms": itf[0], "iface_mu_ms": itf[1]}
        print(json.dumps({"lib": a.tag, "variant": v, **{k: round(x, 4) for k, x in out[v].items()}}), flush=True)


if __name__ == "__main__":
    main()
