"""The CPU oracle timed on the GPU box's host cores (SURVEY.md
§8(d) "oracle timed beside it"): C1 and C2 100-step runs, C4 at full size,
the C5 slab, each on all cores and on one core, full step and the mu-sweep
alone (the paper's 4.2 MLUP/s/core is its SIMD mu-kernel on one SuperMUC
core).  Median of 3 timed repetitions after warm-up steps.
The oracle is run as it stands (not tuned for this).

usage: python tools/cpu_baseline.py [--out gpurun_out/cpu_baseline.json] [--quick]
(the committed copy is profiles/r02_cpu_baseline.json)
"""
import argparse
import json
import os
import platform
import statistics
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from inputs import gen  # noqa: E402
from oracle import oracle as O  # noqa: E402


def state(name, box=None):
    cfg = gen.load_config(name)
    spec = gen.spec_from_config(cfg, cfg["nx"], cfg["ny"])
    b = box or (0, 0, 0, cfg["nx"], cfg["ny"], cfg["nz"])
    phi, mu = gen.generate(spec, cfg["nx"], cfg["ny"], cfg["nz"], box=b)
    lh = cfg["init"]["layer_height"] - b[2]
    p = O.make_params(gen.load_params("v1"), layer_height=lh, aniso=cfg.get("aniso", False),
                      delta_sl=cfg.get("delta_sl"))
    return p, phi, mu


def timed(fn, reps, warm):
    for _ in range(warm):
        fn()
    ts = []
    for _ in range(reps):
        t0 = time.perf_counter()
        fn()
        ts.append(time.perf_counter() - t0)
    return statistics.median(ts), ts


def case(label, name, steps, threads, reps, warm, sweep="step", box=None):
    p, phi, mu = state(name, box)
    cells = phi.shape[1] * phi.shape[2] * phi.shape[3]
    O.set_threads(threads)
    if sweep == "mu":
        phi1 = O.phi_sweep(p, phi, mu)
        fn = lambda: [O.mu_sweep(p, phi, phi1, mu) for _ in range(steps)]   # noqa: E731
    elif sweep == "phi":
        fn = lambda: [O.phi_sweep(p, phi, mu) for _ in range(steps)]   # noqa: E731
    else:
        fn = lambda: O.run(p, phi, mu, steps)   # noqa: E731
    med, ts = timed(fn, reps, warm)
    O.set_threads(None)
    v = cells * steps / med / 1e6
    r = {"case": label, "config": name, "cells": cells, "steps": steps, "threads": threads, "sweep": sweep,
         "reps_s": [round(t, 3) for t in ts], "median_s": round(med, 3), "mlups": round(v, 4),
         "mlups_per_core": round(v / threads, 4), "box": list(box) if box else None}
    print(json.dumps(r), flush=True)
    return r


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=os.path.join(ROOT, "gpurun_out", "cpu_baseline.json"))
    ap.add_argument("--quick", action="store_true")
    a = ap.parse_args()
    nc = os.cpu_count() or 1
    R = 1 if a.quick else 3
    rows = [
        case("C1 full, 100 steps, all cores", "c1", 100, nc, R, 1),
        case("C1 full, 100 steps, one core", "c1", 100, 1, R, 1),
        case("C2 full, 100 steps, all cores", "c2", 100, nc, R, 0),
        case("C2 full, 10 steps, one core", "c2", 10, 1, R, 0),
        case("C2 mu-sweep alone, 10 sweeps, all cores", "c2", 10, nc, R, 1, sweep="mu"),
        case("C2 mu-sweep alone, 2 sweeps, one core", "c2", 2, 1, R, 1, sweep="mu"),
        case("C2 phi-sweep alone, 10 sweeps, all cores", "c2", 10, nc, R, 1, sweep="phi"),
        case("C2 phi-sweep alone, 2 sweeps, one core", "c2", 2, 1, R, 1, sweep="phi"),
        case("C4 512^3, 10 steps, all cores", "c4", 10, nc, 1, 0),
        case("C5 slab 1024x1024x256 (the per-GPU share at 4 GPUs), 1 step, all cores", "c5", 1, nc, 1, 0,
             box=(0, 0, 0, 1024, 1024, 256)),
        case("C5 slab 256x256x16 at the front, 1 step, one core", "c5", 1, 1, 1, 0, box=(0, 0, 56, 256, 256, 16)),
    ]
    try:
        ram = os.sysconf("SC_PAGE_SIZE") * os.sysconf("SC_PHYS_PAGES") / 1e9
    except (ValueError, OSError):
        ram = 0
    if ram >= 160 and not a.quick:   # the whole 1024^3 state and its successor in host memory (~110 GB)
        rows.append(case("C5 1024^3, 1 step, all cores", "c5", 1, nc, 1, 0))
    cpu = None
    try:
        for ln in open("/proc/cpuinfo"):
            if ln.startswith("model name"):
                cpu = ln.split(":", 1)[1].strip()
                break
    except OSError:
        pass
    try:
        mem_gb = os.sysconf("SC_PAGE_SIZE") * os.sysconf("SC_PHYS_PAGES") / 1e9
    except (ValueError, OSError):
        mem_gb = None
    out = {"host": platform.node(), "cpu": cpu, "nproc": nc, "host_ram_gb": mem_gb,
           "oracle": "oracle/oracle.cpp, g++ -O2 -fno-fast-math -ffp-contract=off -fopenmp (OpenMP over z-planes)",
           "paper_context": "4.2 MLUP/s per SuperMUC Sandy Bridge core, SIMD mu-kernel only (PAPER.md:526)",
           "rows": rows}
    json.dump(out, open(a.out, "w"), indent=1)
    print(a.out)


if __name__ == "__main__":
    main()
