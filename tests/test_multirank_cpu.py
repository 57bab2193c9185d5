"""Multi-rank host logic on CPU (gloo, world size 2 and 8): the halo message
plan every rank derives independently must match pairwise (what rank a sends
to b is exactly what b expects from a), the bootstrap broadcast and the
max-over-ranks timing reduction of bench.py."""
import os
import socket

import pytest
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    import sys
    sys.path.insert(0, ROOT)
    import torch
    import torch.distributed as dist
    from paper_1506_01684_b200 import dist as pdist, pf
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        (NX, NY, NZ), blocks = pdist.weak_grid(world, per=64)
        out = {}
        for field in (0, 1):
            snd, rcv = pf.halo_plan(NX, NY, NZ, *blocks, rank, world, field)
            t = torch.tensor([snd, rcv], dtype=torch.int64)
            allt = [torch.zeros_like(t) for _ in range(world)]
            dist.all_gather(allt, t)
            out[field] = [a.tolist() for a in allt]
        nid = pdist.share_from_rank0(lambda: bytes(range(128)))
        mx = pdist.max_over_ranks(float(rank) * 1.5 + 1.0)
        q.put((rank, out, nid == bytes(range(128)), mx, blocks))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2])
def test_gloo_plan_symmetry_and_bootstrap(world):
    from paper_1506_01684_b200 import build
    build.build()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    res.sort()
    for rank, out, id_ok, mx, blocks in res:
        assert id_ok
        assert mx == (world - 1) * 1.5 + 1.0
        for field in (0, 1):
            allt = out[field]
            for a in range(world):
                for b in range(world):
                    assert allt[a][0][b] == allt[b][1][a]   # a->b send == b<-a recv
            ncomp = 4 if field == 0 else 2
            # 2x1x1 of 64^3 blocks, periodic x: both x faces, the 8 x-edges and the
            # 8 corners come from the peer
            assert allt[0][1][1] == ncomp * (2 * 64 * 64 + 8 * 64 + 8)


def test_plan_8_ranks_in_process():
    """2x2x2 blocks: every pair's send/recv counts agree; totals equal the ghost
    region sizes not served locally (z walls are local clamps)."""
    from paper_1506_01684_b200 import dist as pdist, pf
    (NX, NY, NZ), blocks = pdist.weak_grid(8, per=32)
    for field, ncomp in ((0, 4), (1, 2)):
        plans = [pf.halo_plan(NX, NY, NZ, *blocks, r, 8, field) for r in range(8)]
        for a in range(8):
            for b in range(8):
                assert plans[a][0][b] == plans[b][1][a]
            assert plans[a][0][a] == 0 and plans[a][1][a] == 0
        n = 32
        for r in range(8):
            bx, by, bz = pdist.block_of_rank(r, blocks)
            # faces: x and y from peers (2 each), one z face from the z peer, the
            # other z face is a wall (local clamp)
            faces = 4 * n * n + n * n
            # edges: 4 xy-edges (peers), 4 xz/yz edges toward the z peer, the 4
            # toward the wall come from the x/y peers (clamped) -> all remote
            edges = 4 * n + 8 * n
            corners = 8          # every corner has dx != 0: an x peer
            assert sum(plans[r][1]) == ncomp * (faces + edges + corners), (r, bx, by, bz)


def test_plan_single_rank_has_no_messages():
    from paper_1506_01684_b200 import pf
    snd, rcv = pf.halo_plan(64, 64, 64, 2, 2, 2, 0, 1, 0)
    assert snd == [0] and rcv == [0]
    with pytest.raises(pf.PfError):
        pf.halo_plan(65, 64, 64, 2, 1, 1, 0, 2, 0)
