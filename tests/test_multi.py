"""Multi-process partitioning on CPU (gloo, world_size 2): frames and row bands
cover the work exactly once, band halos cover every row the border mapping
reaches, and the timing reduction is a max over ranks."""
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
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_1811_02168_b200 import shard
    res = {}
    res["frames"] = shard.frame_range(64, rank, world)
    bands = {}
    for H, theta in ((16384, 10.0), (37, 5.0), (5, 3.0)):
        for border in (0, 1, 2):
            b = shard.band_for_rank(H, rank, world, theta, border)
            bands[(H, theta, border)] = (b.out_row0, b.out_rows, b.src_row0, b.src_rows)
    res["bands"] = bands
    res["max"] = shard.max_over_ranks(10.0 * (rank + 1))
    gathered = [None] * world
    dist.all_gather_object(gathered, res)
    dist.barrier()
    dist.destroy_process_group()
    if rank == 0:
        q.put(gathered)


def py_reach(H, y0, n, r, border):
    rows = set()
    for y in range(y0 - r, y0 + n + r):
        if 0 <= y < H:
            rows.add(y)
        elif border == 1:
            rows.add(0 if y < 0 else H - 1)
        elif border == 0:
            m = y % (2 * H)
            rows.add(m if m < H else 2 * H - 1 - m)
    return rows


def test_partitions_gloo_world2():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    gathered = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    frames = [g["frames"] for g in gathered]
    covered = [f for a, b in frames for f in range(a, b)]
    assert sorted(covered) == list(range(64))
    for key in gathered[0]["bands"]:
        H, theta, border = key
        r = int(-(-3 * theta // 1))
        rows = []
        for g in gathered:
            y0, n, s0, sn = g["bands"][key]
            rows += list(range(y0, y0 + n))
            need = py_reach(H, y0, n, r, border)
            assert need <= set(range(s0, s0 + sn))
        assert sorted(rows) == list(range(H))
    assert all(g["max"] == 20.0 for g in gathered)
