"""Process-group plumbing for multi-GPU runs (one process per GPU).

torch.distributed only bootstraps: it broadcasts the ncclUniqueId that libpf's
own NCCL communicator uses for the halo exchange, and reduces timings (max over
ranks).  The data path itself (halo send/recv, window allreduce) runs inside
libpf.so.  Works with the gloo backend on CPU (tests) and nccl on GPUs (bench).
"""
from __future__ import annotations

import json
import os

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

# block grids for 1/2/4/8 GPUs
DECOMP = {1: (1, 1, 1), 2: (2, 1, 1), 4: (2, 2, 1), 8: (2, 2, 2)}


def env_rank():
    return (int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)),
            int(os.environ.get("LOCAL_RANK", 0)))


def decomposition(n: int, config: str = "c4"):
    """(px, py, pz) for n ranks from configs/<config>.json (fallback DECOMP)."""
    try:
        cfg = json.load(open(os.path.join(ROOT, "configs", f"{config}.json")))
        return tuple(cfg["decomp"][str(n)])
    except (OSError, KeyError):
        if n in DECOMP:
            return DECOMP[n]
        raise ValueError(f"no block decomposition for {n} ranks")


def weak_grid(n: int, per: int = 512, config: str = "c4"):
    """Global grid of a weak-scaling run: per^3 cells per rank."""
    px, py, pz = decomposition(n, config)
    return (per * px, per * py, per * pz), (px, py, pz)


def block_of_rank(rank: int, blocks):
    """Block coordinates of `rank` (rank = ix + px*(iy + py*iz), include/pf.h)."""
    px, py, _ = blocks
    return rank % px, (rank // px) % py, rank // (px * py)


def share_from_rank0(make, group=None):
    """Value produced by make() on rank 0, broadcast to every rank."""
    import torch.distributed as dist
    obj = [make() if dist.get_rank() == 0 else None]
    dist.broadcast_object_list(obj, src=0, group=group)
    return obj[0]


def max_over_ranks(x: float, device=None) -> float:
    import torch
    import torch.distributed as dist
    if not dist.is_initialized() or dist.get_world_size() == 1:
        return float(x)
    t = torch.tensor([float(x)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())
