#!/usr/bin/env python
"""Benchmark of the explicit phase-field time step (BASELINE.json metric:
MLUP/s of phi+mu cell updates at 1/2/4/8 B200, % of the FP64/HBM roofline).

Workload: configs/c4.json — weak scaling, 512^3 cells per GPU, blocks
1x1x1 / 2x1x1 / 2x2x1 / 2x2x2, seeded Voronoi solid layer,
PARAMS-v1, synthetic data.  One "step" = one pass of the whole hot path
(table, phi-sweep, phi halo, mu-sweep, mu halo, swap).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl reference]

N > 1 runs one rank per GPU over NCCL: under torch.distributed.run (the
driver's launch; WORLD_SIZE must equal N), or — started as a plain process —
bench.py re-launches itself under torch.distributed.run with N ranks.  Rank 0
prints one JSON line.  --impl reference times the CPU oracle (the only
reference implementation of this tier) on host cores.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CONFIG = "c4"
# Algorithmic work per LUP: FLOPs counted from the oracle
# (oracle.count_flops, isotropic), compulsory FP64 bytes.
BYTES_PHI, BYTES_MU = 80, 96
BYTES_FUSED = 128   # fused mu(n) + phi(n+1): read phi^n, phi^{n+1}, mu^n; write mu^{n+1}, phi^{n+2}
PEAK_FP64_DERIVED = 148 * 64 * 2 * 1.965e9 / 1e12   # TFLOP/s: SMs x FP64 FMA/clk x 2 x max clock
# SURVEY.md §8(d)'s counted FLOP/LUP (a scratch op count of O4/O5 made during
# the survey), reported beside the oracle's own count
FLOP_SURVEY = {"phi_iso": 522, "phi_aniso": 1422, "mu": 638}
FLOP_METHOD = ("oracle/oracle.cpp or_count_flops: + - x / sqrt = 1 each, every face charged once, per-plane "
               "(T-only) values free, no shortcuts and every anti-trapping guard open (PAPER.md:508-509); "
               "de-duplicated: S and psi-bar once per cell, only the normal component g_d of a pair gradient "
               "at a face, the liquid normal once per face")


def _env_int(k, d):
    try:
        return int(os.environ.get(k, d))
    except ValueError:
        return d


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""
    FIELDS = ["clocks.sm", "clocks.max.sm", "clocks_event_reasons.hw_slowdown",
              "clocks_event_reasons.hw_thermal_slowdown", "clocks_event_reasons.sw_thermal_slowdown",
              "clocks_event_reasons.sw_power_cap"]
    NAMES = [None, None, "hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]

    def __init__(self, device: int):
        self.device = device
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), "--query-gpu=" + ",".join(self.FIELDS),
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except (FileNotFoundError, OSError):
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        sm, mx, reasons = [], [], set()
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) != len(self.FIELDS):
                continue
            try:
                sm.append(float(parts[0]))
                mx.append(float(parts[1]))
            except ValueError:
                continue
            for name, val in zip(self.NAMES, parts):
                if name and val.lower().startswith("active"):
                    reasons.add(name)
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(sm)}


def cpu_model():
    try:
        for ln in open("/proc/cpuinfo"):
            if ln.startswith("model name"):
                return ln.split(":", 1)[1].strip()
    except OSError:
        pass
    return None


def load_cfg(name):
    return json.load(open(os.path.join(ROOT, "configs", f"{name}.json")))


def workload(name: str, world: int, grid=None):
    """Global grid, block grid and per-rank cells of a config at `world` ranks:
    weak scaling (per-GPU block, C4) or strong scaling (fixed global grid, C5);
    `grid` overrides the global grid (e.g. C5's 1024x1024x256 slab, reading A22)."""
    from paper_1506_01684_b200 import dist as pdist
    cfg = load_cfg(name)
    if grid:
        cfg = dict(cfg, nx=grid[0], ny=grid[1], nz=grid[2], per_gpu=False)
        return cfg, tuple(grid), pdist.decomposition(world, name), grid[0] * grid[1] * grid[2] // world, "strong"
    if cfg.get("per_gpu"):
        (NX, NY, NZ), blocks = pdist.weak_grid(world, per=cfg["nx"], config=name)
        scaling = "weak"
    else:
        NX, NY, NZ = cfg["nx"], cfg["ny"], cfg["nz"]
        blocks = pdist.decomposition(world, name)
        scaling = "strong"
    return cfg, (NX, NY, NZ), blocks, NX * NY * NZ // world, scaling


def flops_per_lup(name):
    """Algorithmic FLOP/LUP of the config's sweeps, as counted from the oracle's
    source by tools/count_flops.py (committed in profiles/flop_counts.json)."""
    d = json.load(open(os.path.join(ROOT, "profiles", "flop_counts.json")))
    return d["configs"][name]


def cpu_oracle_sample(name: str, steps: int, nz_slab: int = 16, threads: int | None = None, sweep: str = "step",
                      nxy: int = 512):
    """Time the CPU oracle (as it stands) on a bounded sample of the workload:
    an nxy x nxy x nz_slab slab of one GPU's block around the solid-liquid front
    of the config's initial state, stepped as its own domain (uniform per-cell
    work: the oracle takes no shortcuts).  sweep = "step" (phi + mu) or "mu"
    (the mu-sweep alone, the paper's per-core figure is mu-only).
    threads = OpenMP threads (None: all host cores).
    Returns (MLUP/s, threads, sample text)."""
    from inputs import gen
    from oracle import oracle as O
    cfg = load_cfg(name)
    pd = gen.load_params("v1")
    lh = cfg["init"]["layer_height"]
    nx, ny = min(cfg["nx"], nxy), min(cfg["ny"], nxy)
    spec = gen.spec_from_config(cfg, cfg["nx"], cfg["ny"])
    nz_slab = min(nz_slab, cfg["nz"])
    z0 = max(0, min(int(lh) - nz_slab // 2, cfg["nz"] - nz_slab))
    phi, mu = gen.generate(spec, cfg["nx"], cfg["ny"], cfg["nz"], box=(0, 0, z0, nx, ny, nz_slab))
    p = O.make_params(pd, layer_height=lh - z0, aniso=cfg.get("aniso", False), delta_sl=cfg.get("delta_sl"))
    cores = int(threads) if threads else (os.cpu_count() or 1)
    O.set_threads(cores)
    if sweep == "mu":
        phi1 = O.phi_sweep(p, phi, mu, 0, 0)
    t0 = time.perf_counter()
    for s in range(steps):
        if sweep == "mu":
            mu = O.mu_sweep(p, phi, phi1, mu, 0, 0)
        else:
            phi, mu = O.step(p, phi, mu, s, 0)
    dt = time.perf_counter() - t0
    O.set_threads(None)
    cells = nx * ny * nz_slab
    what = "mu-sweep(s)" if sweep == "mu" else "oracle step(s)"
    return cells * steps / dt / 1e6, cores, \
        f"{steps} {what} of the {nx}x{ny}x{nz_slab} slab z in [{z0},{z0 + nz_slab}) of the " \
        f"{cfg['name']} state on {cores} thread(s) ({cells * steps} LUP, {dt:.1f} s)"


def cpu_baseline(name: str, steps: int, aniso: bool):
    """The oracle on the box's host cores:
    all cores and one core, full step and mu-sweep alone; MLUP/s and per core."""
    nzs = 16 if aniso else 64
    v, cores, sample = cpu_oracle_sample(name, steps, nz_slab=nzs)
    v1, _, s1 = cpu_oracle_sample(name, 1, nz_slab=16, threads=1, nxy=256)
    vm, _, sm = cpu_oracle_sample(name, max(1, steps // 2), nz_slab=nzs, sweep="mu")
    vm1, _, sm1 = cpu_oracle_sample(name, 1, nz_slab=16, threads=1, sweep="mu", nxy=256)
    return {"value": round(v, 3), "unit": "MLUP/s", "cores": cores, "per_core": round(v / cores, 3),
            "cpu": cpu_model(), "kind": "oracle", "sample": sample,
            "single_core": {"value": round(v1, 3), "sample": s1},
            "mu_sweep": {"all_cores": round(vm, 3), "per_core": round(vm / cores, 3), "single_core": round(vm1, 3),
                         "samples": [sm, sm1]},
            "more": "profiles/r02_cpu_baseline.json (tools/cpu_baseline.py: C1 and C2 100-step runs, "
                    "median of 3 after warm-up)"}


def describe(cfg, grid, blocks, scaling):
    NX, NY, NZ = grid
    px, py, pz = blocks
    kind = "anisotropic (cubic, delta_sl = %g)" % cfg["delta_sl"] if cfg.get("aniso") else "isotropic"
    per = f"{cfg['nx']}^3 cells per GPU (weak scaling)" if scaling == "weak" else \
        f"{NX}x{NY}x{NZ} cells total (strong scaling)"
    return (f"{cfg['name']}: {per}, FP64, N=4 phases, K=3 components, periodic x/y, zero-flux z, "
            f"{cfg['init']['kind']} solid layer z<{cfg['init']['layer_height']}, mu noise "
            f"{cfg['init'].get('mu_noise', 0)}, {kind}" + (", moving window" if cfg.get("window") else ""))


def run_reference(args):
    rank = _env_int("RANK", 0)
    if rank != 0:
        return 0
    steps, warm = args.steps, args.warmup
    world = _env_int("WORLD_SIZE", 1)
    cfg, grid, blocks, cells_local, scaling = workload(args.config, world, args.grid)
    # each step: one oracle step over a bounded sample of the workload
    if warm:
        cpu_oracle_sample(args.config, 1, nz_slab=16)
    v, cores, sample = cpu_oracle_sample(args.config, steps, nz_slab=16)
    line = {"impl": "reference", "metric": "MLUP/s", "value": round(v, 3), "unit": "MLUP/s",
            "n_gpus": world, "steps": steps, "warmup": warm, "higher_is_better": True,
            "scaling": scaling, "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": describe(cfg, grid, blocks, scaling) + " — CPU oracle on a bounded slab sample",
                       "global_cells": cells_local * world},
            "cpu_baseline": {"value": round(v, 3), "unit": "MLUP/s", "cores": cores, "kind": "oracle",
                             "sample": sample},
            "e2e": {"value": round(v, 3), "unit": "MLUP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


def run_gpu(args):
    import torch
    import torch.distributed as dist
    from paper_1506_01684_b200 import pf
    from paper_1506_01684_b200 import dist as pdist

    rank, world, local = pdist.env_rank()
    if world > 1:
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    else:
        torch.cuda.set_device(0)
    cfg, (NX, NY, NZ), (px, py, pz), cells_local, scaling = workload(args.config, world, args.grid)
    from inputs import gen
    pd = gen.load_params("v1")
    prm = pf.make_params(pd, cfg, nx=NX, ny=NY, nan_check_every=0, graph=args.graph)
    nid = pdist.share_from_rank0(pf.nccl_unique_id) if world > 1 else None
    stream = torch.cuda.Stream()
    ctx = pf.Context(NX, NY, NZ, prm, px, py, pz, rank=rank if world > 1 else 0, nranks=world,
                     device=local if world > 1 else 0, nccl_id=nid, stream=stream.cuda_stream)
    ctx.init(cfg["seed"])
    shape = ctx.shape

    def barrier():
        if world > 1:
            dist.barrier()

    def max_over_ranks(x):
        return pdist.max_over_ranks(x, device="cuda")

    # warm-up
    ctx.step(args.warmup)
    torch.cuda.synchronize()
    # timed region: the production path (kernels launched one by one: measured as
    # fast as a CUDA-graph replay, tools/graph_gain.py, and keeps the mu halo
    # beside the next phi-sweep)
    clocks = ClockSampler(local if world > 1 else 0)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    # per-sweep device times for the roofline, live inside the timed region:
    # CUDA events around each sweep on the launching stream (pf_set_timing;
    # a graph replay has no per-sweep events, so --graph times them after)
    ctx.set_timing(not args.graph)
    l0 = ctx.info().launches
    # args.reps windows of exactly args.steps steps, each bracketed by a barrier
    # and a synchronize; the median window is reported
    windows = []
    clocks.start()
    for _ in range(max(1, args.reps)):
        ctx.set_timing(not args.graph)   # resets the per-sweep accumulators
        barrier()
        torch.cuda.synchronize()
        e0.record(stream)
        ctx.step(args.steps)
        e1.record(stream)
        torch.cuda.synchronize()
        barrier()
        inf = ctx.info()
        windows.append((max_over_ranks(e0.elapsed_time(e1)), inf.ms_phi / max(1, inf.phi_launches),
                        inf.ms_mu / max(1, inf.mu_launches)))
    clk = clocks.stop()
    launches = int(ctx.info().launches - l0) // max(1, args.reps)
    order = sorted(range(len(windows)), key=lambda i: windows[i][0])
    ms, ms_phi, ms_mu = windows[order[len(order) // 2]]
    # the same windows' length with the region shortcuts on (NEXT-1; bitwise the
    # same results, pf_set_shortcuts): reported beside the headline, which keeps
    # them off so that its FLOP count per cell is exact
    sc = None
    if not args.graph and not args.no_shortcuts:
        ctx.set_shortcuts(True)
        ctx.set_timing(True)
        barrier()
        torch.cuda.synchronize()
        e0.record(stream)
        ctx.step(args.steps)
        e1.record(stream)
        torch.cuda.synchronize()
        barrier()
        inf = ctx.info()
        sc_ms = max_over_ranks(e0.elapsed_time(e1))
        sc = {"value": round(cells_local * world * args.steps / (sc_ms / 1e3) / 1e6, 2),
              "ms_per_step": round(sc_ms / args.steps, 4),
              "phi_ms": round(inf.ms_phi / max(1, inf.phi_launches), 4),
              "mu_ms": round(inf.ms_mu / max(1, inf.mu_launches), 4),
              "what": "region shortcuts on (pf_set_shortcuts): bitwise-identical results; the headline keeps them "
                      "off for the exact FLOP count"}
        ctx.set_shortcuts(False)
        ctx.set_timing(False)
    # the same windows' length with fused steps (pf_set_fusion: the mu-sweep of
    # step n and the phi-sweep of step n+1 as one kernel, 128 B/LUP instead of
    # 176; bitwise the same results), beside the headline, which keeps the two
    # sweeps so that each has its own roofline line
    fu = None
    if not args.graph and not args.no_fused:
        try:
            ctx.set_fusion(True)
        except RuntimeError as ex:   # no room for the third phi copy
            fu = {"value": None, "what": f"not run: {ex}"}
        if fu is None:
            ctx.set_timing(True)
            barrier()
            torch.cuda.synchronize()
            e0.record(stream)
            ctx.step(args.steps)
            e1.record(stream)
            torch.cuda.synchronize()
            barrier()
            inf = ctx.info()
            fu_ms = max_over_ranks(e0.elapsed_time(e1))
            fk = inf.ms_fused / max(1, inf.fused_launches)
            # and with the region shortcuts on inside the fused kernel (bitwise the same)
            ctx.set_shortcuts(True)
            ctx.set_timing(True)
            barrier()
            torch.cuda.synchronize()
            e0.record(stream)
            ctx.step(args.steps)
            e1.record(stream)
            torch.cuda.synchronize()
            barrier()
            inf2 = ctx.info()
            fs_ms = max_over_ranks(e0.elapsed_time(e1))
            ctx.set_shortcuts(False)
            fu = {"value": round(cells_local * world * args.steps / (fu_ms / 1e3) / 1e6, 2),
                  "ms_per_step": round(fu_ms / args.steps, 4), "fused_ms": round(fk, 4),
                  "fused_launches": int(inf.fused_launches),
                  "phi_ms": round(inf.ms_phi / max(1, inf.phi_launches), 4),
                  "mu_ms": round(inf.ms_mu / max(1, inf.mu_launches), 4),
                  "fused_bytes_per_lup": BYTES_FUSED,
                  "fused_gbs": round(BYTES_FUSED * cells_local / (fk / 1e3) / 1e9, 1),
                  "with_shortcuts": {"value": round(cells_local * world * args.steps / (fs_ms / 1e3) / 1e6, 2),
                                     "ms_per_step": round(fs_ms / args.steps, 4),
                                     "fused_ms": round(inf2.ms_fused / max(1, inf2.fused_launches), 4)},
                  "what": "fused steps on (pf_set_fusion): pf_step(steps) = phi-sweep, steps-1 fused mu(n)+phi(n+1) "
                          "kernels, mu-sweep; bitwise-identical results; the headline keeps the separate sweeps"}
            ctx.set_fusion(False)
        ctx.set_timing(False)
    if args.graph:
        ctx.set_timing(True)
        ctx.step(min(args.steps, 10))
        inf = ctx.info()
        ms_phi = inf.ms_phi / max(1, inf.phi_launches)
        ms_mu = inf.ms_mu / max(1, inf.mu_launches)
    ctx.set_timing(False)
    value = cells_local * world * args.steps / (ms / 1e3) / 1e6

    # end-to-end through the C ABI with host buffers: each step uploads the
    # state from pinned host memory, advances one step and reads it back —
    # pf_step_io, which overlaps the upload, the sweeps and the download in
    # z-slabs (= pf_write + pf_step(1) + pf_read, bit for bit)
    e2e = e2e_job = None
    state_bytes = cells_local * 6 * 8
    e2e_steps = min(args.steps, args.e2e_steps)
    if e2e_steps > 0:
        hphi = torch.empty((4,) + shape, dtype=torch.float64, pin_memory=True)
        hmu = torch.empty((2,) + shape, dtype=torch.float64, pin_memory=True)
        ctx.read(hphi, hmu)
        ctx.step_io(hphi, hmu, hphi, hmu)   # untimed: the slab pipeline's one-time setup (copy lists, streams)
        barrier()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(e2e_steps):
            ctx.step_io(hphi, hmu, hphi, hmu)
        barrier()
        e2e_s = max_over_ranks(time.perf_counter() - t0)
        e2e = cells_local * world * e2e_steps / e2e_s / 1e6
        # whole-job variant: the state uploaded once, the timed steps, read back once
        barrier()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        ctx.write(hphi, hmu)
        ctx.step(args.steps)
        ctx.read(hphi, hmu)
        barrier()
        job_s = max_over_ranks(time.perf_counter() - t0)
        e2e_job = cells_local * world * args.steps / job_s / 1e6
        del hphi, hmu

    # the no-shortcut, interface-dense measurement ("without
    # the shortcut optimizations ... the total number of executed floating point
    # operations per cell can be determined exactly"; the interface scenario,
    # PAPER.md:424-427): a state with all four phases in every cell (every
    # anti-trapping guard open on every face) written with pf_write, one timed
    # step per repetition from that state
    iface = None
    if not args.no_interface:
        from inputs import gen as _gen
        dphi, dmu = _gen.interface_state_torch(shape, seed=cfg["seed"], device="cuda")
        reps = []
        for _ in range(5):
            ctx.write(dphi, dmu)
            ctx.set_timing(True)
            ctx.step(1)
            inf = ctx.info()
            reps.append((inf.ms_phi / max(1, inf.phi_launches), inf.ms_mu / max(1, inf.mu_launches)))
        ctx.set_timing(False)
        # the fused kernel from the same state (pf_step(2): phi-sweep, one fused
        # mu(0) + phi(1) kernel, mu-sweep), where its FLOP count is exact too
        freps = []
        if not args.no_fused and not args.graph:
            try:
                ctx.set_fusion(True)
                for _ in range(3):
                    ctx.write(dphi, dmu)
                    ctx.set_timing(True)
                    ctx.step(2)
                    inf = ctx.info()
                    if inf.fused_launches:   # (with the window on, a due front check cuts the run)
                        freps.append(inf.ms_fused / inf.fused_launches)
                ctx.set_timing(False)
                ctx.set_fusion(False)
            except RuntimeError:   # no room for the third phi copy next to the interface state
                freps = []
        del dphi, dmu
        torch.cuda.empty_cache()
        iface = {"phi_ms": max_over_ranks(float(np.median([r[0] for r in reps]))),
                 "mu_ms": max_over_ranks(float(np.median([r[1] for r in reps])))}
        if freps:
            iface["fused_ms"] = max_over_ranks(float(np.median(freps)))

    if rank == 0:
        fl = flops_per_lup(args.config)
        peaks = {}
        try:
            peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
        except (OSError, ValueError):
            pass
        hbm = float(peaks.get("hbm_gbs", 6650.0))
        aniso = bool(cfg.get("aniso"))
        f_svy = {"phi": FLOP_SURVEY["phi_aniso" if aniso else "phi_iso"], "mu": FLOP_SURVEY["mu"]}
        sweeps = {
            "phi": {"ms": ms_phi, "flop": fl["phi_per_lup"], "bytes": BYTES_PHI},
            "mu": {"ms": ms_mu, "flop": fl["mu_per_lup"], "bytes": BYTES_MU},
        }
        for k, s in sweeps.items():
            s["tflops"] = s["flop"] * cells_local / (s["ms"] / 1e3) / 1e12
            s["gbs"] = s["bytes"] * cells_local / (s["ms"] / 1e3) / 1e9
            s["frac_fp64"] = s["tflops"] / PEAK_FP64_DERIVED
            s["frac_hbm"] = s["gbs"] / hbm
            s["flop_survey"] = f_svy[k]
            s["frac_fp64_survey"] = f_svy[k] * cells_local / (s["ms"] / 1e3) / 1e12 / PEAK_FP64_DERIVED
        if iface:
            for k in ("phi", "mu"):
                t = iface[f"{k}_ms"] / 1e3
                iface[f"{k}_frac_fp64"] = sweeps[k]["flop"] * cells_local / t / 1e12 / PEAK_FP64_DERIVED
                iface[f"{k}_frac_hbm"] = sweeps[k]["bytes"] * cells_local / t / 1e9 / hbm
                iface[f"{k}_frac_fp64_survey"] = f_svy[k] * cells_local / t / 1e12 / PEAK_FP64_DERIVED
            if "fused_ms" in iface:   # mu(n) + phi(n+1): both sweeps' algorithmic FLOPs and 128 B per LUP
                t = iface["fused_ms"] / 1e3
                iface["fused_frac_fp64"] = (sweeps["phi"]["flop"] + sweeps["mu"]["flop"]) * cells_local / t / 1e12 / \
                    PEAK_FP64_DERIVED
                iface["fused_frac_hbm"] = BYTES_FUSED * cells_local / t / 1e9 / hbm
            iface["state"] = ("inputs/gen.py interface_state_torch: phi = 0.05 + U(0,1) per phase, normalised "
                              "(all four phases in every cell), mu = U(-0.3, 0.3); one step from it per repetition, "
                              "median of 5")
        dom = max(sweeps, key=lambda k: sweeps[k]["ms"])
        d = sweeps[dom]
        traffic = None
        try:
            prof = json.load(open(os.path.join(ROOT, "profiles", "ncu_summary.json")))
            if prof.get("config", "c4") == args.config:
                traffic = prof.get("dram_bytes_per_launch", {}).get(dom)
        except (OSError, ValueError):
            pass
        cpu = {"value": None, "unit": "MLUP/s", "cores": None, "kind": "oracle", "sample": "skipped"}
        if world == 1 and not args.no_cpu:
            cpu = cpu_baseline(args.config, args.cpu_steps, bool(cfg.get("aniso")))
        line = {
            "metric": "MLUP/s", "value": round(value, 2), "unit": "MLUP/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms / args.steps, 4),
            "reps": {"n": len(windows), "ms_per_step": [round(w[0] / args.steps, 4) for w in windows],
                     "reported": "median window"},
            "higher_is_better": True, "scaling": scaling, "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded initial state, PARAMS-v1)",
            "config": {"workload": describe(cfg, (NX, NY, NZ), (px, py, pz), scaling),
                       "global_cells": cells_local * world, "grid": [NX, NY, NZ], "blocks": [px, py, pz],
                       "parallelism": f"block{px}x{py}x{pz}",
                       "l2": f"inputs larger than L2 ({cells_local * 96 / 1e9:.1f} GB of fields per GPU vs 126 MB L2)"},
            "roofline": {"bound": "alu", "kernel": f"{dom}-sweep", "achieved": round(d["tflops"], 3),
                         "peak": round(PEAK_FP64_DERIVED, 2), "unit": "TFLOP/s",
                         "frac": round(d["frac_fp64"], 4), "traffic": traffic,
                         "flop_per_lup": d["flop"], "flop_method": FLOP_METHOD,
                         "frac_at_survey_flop": round(d["frac_fp64_survey"], 4),
                         "peak_source": "derived: 148 SMs x 64 FP64 FMA/clk x 2 x 1.965 GHz (DESIGN.md §6); "
                                        "measured DFMA loop 34.2 TFLOP/s",
                         "sweeps": {k: {kk: (round(vv, 4) if isinstance(vv, float) else vv)
                                        for kk, vv in s.items()} for k, s in sweeps.items()},
                         "note": "flop = algorithmic FLOP/LUP (flop_method); flop_survey = SURVEY.md §8(d)'s count. "
                                 "On the C4 state the mu-sweep's exact-zero anti-trapping guards skip most of its "
                                 "FP64 work (bulk planes), so there mu is judged by frac_hbm (96 B/LUP) and by "
                                 "mu_interface, the all-guards-open state",
                         "mu_interface_ms": round(iface["mu_ms"], 4) if iface else None,
                         "interface": {k: (round(v, 4) if isinstance(v, float) else v) for k, v in iface.items()}
                         if iface else None,
                         "hbm_peak_gbs": hbm},
            "cpu_baseline": cpu,
            "paper_context": {"mlups_per_core": 4.2, "what": "mu-kernel only (no phi), one SuperMUC Sandy Bridge "
                              "core, SIMD-optimised, Ag-Al-Cu parameters (PAPER.md:526); the paper prints no GPU "
                              "or full-step number", "unit": "MLUP/s/core"},
            "e2e": {"value": round(e2e, 2) if e2e else None, "unit": "MLUP/s",
                    "h2d_bytes_per_step": state_bytes if e2e else 0,
                    "d2h_bytes_per_step": state_bytes if e2e else 0, "steps": e2e_steps,
                    "what": "pf_step_io(pinned host state in, pinned host state out) per step: upload, step and download "
                            "overlapped in z-slabs (single block per GPU; else pf_write + pf_step(1) + pf_read)",
                    "job": {"value": round(e2e_job, 2) if e2e_job else None, "steps": args.steps,
                            "what": "pf_write(pinned host state) once + pf_step(steps) + pf_read(pinned host) once"}},
            "shortcuts": sc,
            "fused": fu,
            "gpu_launches": launches,
            "clocks": clk,
        }
        print(json.dumps(line), flush=True)
    ctx.close()
    if world > 1:
        dist.destroy_process_group()
    return 0


def relaunch_distributed(n: int) -> int:
    """Started as a plain process with --gpus N > 1: run the same command as N
    ranks under torch.distributed.run (one per GPU, rendezvous on 127.0.0.1)."""
    import socket
    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        port = so.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__)] + sys.argv[1:]
    print(f"bench.py: --gpus {n} without a launcher: {' '.join(cmd)}", file=sys.stderr, flush=True)
    return subprocess.call(cmd)


def check_world(args) -> int | None:
    """--gpus N against the launcher's WORLD_SIZE: re-launch when there is no
    launcher, refuse a mismatch (a run must not label one GPU's number as N's).
    Returns an exit code to stop with, or None to go on."""
    ws = os.environ.get("WORLD_SIZE")
    if ws is None:
        if args.gpus > 1:
            if args.impl == "ours":
                import torch
                have = torch.cuda.device_count()
                if have < args.gpus:
                    print(f"bench.py: --gpus {args.gpus} but {have} GPU(s) visible", file=sys.stderr)
                    return 2
            return relaunch_distributed(args.gpus)
        return None
    if int(ws) != args.gpus:
        print(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={ws}: refusing to run", file=sys.stderr)
        return 2
    return None


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--e2e-steps", type=int, default=2)
    ap.add_argument("--cpu-steps", type=int, default=8)
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--reps", type=int, default=3, help="timed windows of --steps steps each; the median is reported")
    ap.add_argument("--no-interface", action="store_true", help="skip the all-guards-open sweep measurement")
    ap.add_argument("--no-shortcuts", action="store_true", help="skip the region-shortcut window")
    ap.add_argument("--no-fused", action="store_true", help="skip the fused-step window")
    ap.add_argument("--graph", action="store_true", help="replay each step as a CUDA graph (single rank)")
    ap.add_argument("--grid", type=int, nargs=3, metavar=("NX", "NY", "NZ"),
                    help="global grid overriding the config's (its physics and init recipe kept)")
    ap.add_argument("--config", default=CONFIG, choices=["c1", "c2", "c3", "c4", "c5"],
                    help="c4: weak scaling 512^3 per GPU (default, the headline); c5: strong scaling 1024^3, "
                         "anisotropic; c1-c3: the single-GPU parity configs")
    args = ap.parse_args()
    if args.gpus < 1:
        ap.error("--gpus must be >= 1")
    rc = check_world(args)
    if rc is not None:
        return rc
    if args.warmup < 3 and args.impl == "ours":
        print("warning: fewer than 3 warm-up steps", file=sys.stderr)
    if args.impl == "reference":
        return run_reference(args)
    return run_gpu(args)


if __name__ == "__main__":
    sys.exit(main())
