"""bench.py's output contract: one JSON line per run with the keys the driver
reads (metric/value/unit, timing, config.workload, roofline, cpu_baseline,
e2e, gpu_launches, clocks), for the GPU arm and the reference (CPU oracle) arm."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BASE_KEYS = {"metric", "value", "unit", "n_gpus", "steps", "warmup", "higher_is_better", "scaling", "vs_baseline",
             "dtype", "data", "config", "e2e"}


def _bench(*args, env=None, timeout=900, rc=0, drop=()):
    e = dict(os.environ, **(env or {}))
    for k in drop:
        e.pop(k, None)
    p = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], cwd=ROOT, capture_output=True,
                       text=True, timeout=timeout, env=e)
    assert p.returncode == rc, p.stderr[-3000:]
    if rc:
        return p.stderr
    lines = [ln for ln in p.stdout.splitlines() if ln.strip()]
    return lines


def test_reference_arm_line():
    lines = _bench("--impl", "reference", "--steps", "1", "--warmup", "0", "--config", "c1")
    assert len(lines) == 1
    line = json.loads(lines[0])
    assert BASE_KEYS <= set(line) and line["impl"] == "reference"
    assert line["metric"] == "MLUP/s" and line["unit"] == "MLUP/s" and line["higher_is_better"] is True
    assert line["value"] > 0 and line["dtype"] == "f64"
    assert "workload" in line["config"]
    cb = line["cpu_baseline"]
    assert cb["kind"] == "oracle" and cb["cores"] >= 1 and cb["value"] == line["value"] and cb["sample"]
    assert line["e2e"] == {"value": line["value"], "unit": "MLUP/s", "h2d_bytes_per_step": 0,
                           "d2h_bytes_per_step": 0}


def test_reference_arm_other_ranks_silent():
    assert _bench("--impl", "reference", "--gpus", "2", "--steps", "1", "--warmup", "0", "--config", "c1",
                  env={"RANK": "1", "WORLD_SIZE": "2"}) == []


def test_gpus_flag_must_match_the_launcher():
    # a launcher's WORLD_SIZE that differs from --gpus is refused (a 1-rank
    # number must never be labelled as N GPUs')
    err = _bench("--impl", "reference", "--gpus", "1", "--steps", "1", "--warmup", "0", "--config", "c1",
                 env={"RANK": "0", "WORLD_SIZE": "2"}, rc=2)
    assert "WORLD_SIZE=2" in err
    err = _bench("--impl", "reference", "--gpus", "4", "--steps", "1", "--warmup", "0", "--config", "c1",
                 env={"RANK": "0", "WORLD_SIZE": "2"}, rc=2)
    assert "--gpus 4" in err


def test_gpus_flag_self_launches_ranks():
    # started as a plain process, --gpus 2 re-launches bench.py under
    # torch.distributed.run with 2 ranks (127.0.0.1 rendezvous); rank 0 prints
    # the one line, rank 1 is silent
    lines = _bench("--impl", "reference", "--gpus", "2", "--steps", "1", "--warmup", "0", "--config", "c1",
                   drop=("RANK", "WORLD_SIZE", "LOCAL_RANK", "MASTER_ADDR", "MASTER_PORT"), timeout=300)
    js = [json.loads(ln) for ln in lines if ln.startswith("{")]
    assert len(js) == 1 and js[0]["n_gpus"] == 2 and js[0]["impl"] == "reference"


@pytest.mark.gpu
def test_gpu_arm_line():
    lines = _bench("--steps", "3", "--warmup", "3", "--config", "c2", "--e2e-steps", "1", "--cpu-steps", "1")
    assert len(lines) == 1
    line = json.loads(lines[0])
    assert BASE_KEYS <= set(line) and line.get("impl", "ours") != "reference"
    assert line["n_gpus"] == 1 and line["steps"] == 3 and line["warmup"] == 3 and line["value"] > 0
    assert abs(line["value"] - 128 ** 3 / (line["ms_per_step"] * 1e3)) <= 1e-3 * line["value"]
    rf = line["roofline"]
    assert rf["bound"] in ("alu", "hbm", "tensor") and 0 < rf["frac"] <= 1.0
    assert abs(rf["frac"] - rf["achieved"] / rf["peak"]) < 1e-3
    assert set(rf["sweeps"]) == {"phi", "mu"}
    assert rf["flop_per_lup"] == rf["sweeps"][rf["kernel"].split("-")[0]]["flop"] and rf["flop_method"]
    assert rf["mu_interface_ms"] > 0 and rf["interface"]["phi_ms"] > 0
    assert line["reps"]["n"] == 3 and len(line["reps"]["ms_per_step"]) == 3
    assert sorted(line["reps"]["ms_per_step"])[1] == line["ms_per_step"]
    cb = line["cpu_baseline"]
    assert cb["kind"] == "oracle" and cb["cores"] >= 1 and cb["value"] > 0
    assert cb["single_core"]["value"] > 0 and cb["mu_sweep"]["per_core"] > 0
    e2e = line["e2e"]
    # the step's inputs (phi, mu: 48 B/cell) up and its result down, every step
    assert e2e["h2d_bytes_per_step"] == 48 * 128 ** 3 and e2e["d2h_bytes_per_step"] == 48 * 128 ** 3
    assert 0 < e2e["value"] < line["value"]
    assert line["gpu_launches"] >= 4 * line["steps"]
    fu = line["fused"]
    assert fu["value"] > 0 and fu["fused_launches"] == line["steps"] - 1 and fu["fused_ms"] > 0
    assert {"sm_mhz", "sm_max_mhz", "reasons"} <= set(line["clocks"])
