"""Write profiles/flop_counts.json: the algorithmic FLOP/LUP of each config's
sweeps, counted by the oracle's own source (oracle.count_flops: + - x / sqrt
count 1, each face charged once, per-plane T-only values free, every term
evaluated — PAPER.md:508-509).  bench.py reads this file for its roofline, so
the benchmark itself never executes oracle code outside its cpu_baseline leg.

usage: python tools/count_flops.py"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from inputs import gen  # noqa: E402
from oracle import oracle as O  # noqa: E402

out = {"source": "tools/count_flops.py -> oracle.count_flops (oracle/oracle.cpp, or_count_flops)", "configs": {}}
pd = gen.load_params("v1")
for name in ("c1", "c2", "c3", "c4", "c5"):
    cfg = gen.load_config(name)
    fl = O.count_flops(O.make_params(pd, layer_height=cfg["init"]["layer_height"], aniso=cfg.get("aniso", False),
                                     delta_sl=cfg.get("delta_sl")))
    out["configs"][name] = {k: int(v) for k, v in fl.items()}
path = os.path.join(ROOT, "profiles", "flop_counts.json")
json.dump(out, open(path, "w"), indent=1)
print(json.dumps(out["configs"]))
