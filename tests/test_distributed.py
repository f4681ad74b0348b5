"""Multi-process host logic of the sharded sweep on CPU (gloo, world size 2).

On GPUs each rank runs points p = rank (mod W) on its own device and the summaries are
all-gathered over NCCL (api.run_distributed).  Here the device part is replaced by
summaries each rank fabricates for exactly the points it owns; everything else -- shard
assignment, fixed-slot padding, the all-gather, dropping padding, import into the C-ABI
handle, and summary-backed quantile queries for points run elsewhere -- is the real code."""
import os
import socket

import numpy as np
import pytest


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def fake_summaries(points):
    import paper_2503_08415_b200 as P
    a = np.zeros(len(points), P.SUMMARY_DTYPE)
    a["version"] = 1
    a["point"] = points
    a["n_requests"] = 1000
    a["n_finished"] = 1000 - (np.asarray(points) % 3)
    for m in range(5):
        for q in range(5):
            a["stat"][:, m, q] = np.asarray(points) * 1.0 + m * 0.1 + q * 0.01
    return a


def _worker(rank, world, port, out_q):
    import torch.distributed as dist

    import sweep_inputs as si
    import paper_2503_08415_b200 as P
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        sw = P.Sweep(si.c2())
        b, e, s = P.shard_range(sw.num_points, rank, world)
        mine = list(range(b, e, s))
        allv = P.gather_summaries(fake_summaries(mine), sw.num_points)
        sw.import_summaries(allv)
        ok = list(allv["point"]) == list(range(sw.num_points))
        for p in range(sw.num_points):
            g = sw.summary(p)
            ok &= int(g["point"]) == p and int(g["n_finished"]) == 1000 - p % 3
            q = sw.latency_quantiles(p, "e2e", [5000, 9000, 9900, 10000])
            ok &= np.allclose(q, [p + 0.2, p + 0.21, p + 0.22, p + 0.23])
        try:
            sw.latency_quantiles(0, "e2e", [2500])
            ok = False
        except P.TokensimError as e:
            ok &= e.status == -4  # E_STATE: only summary-backed quantiles off-rank
        out_q.put((rank, bool(ok), len(mine)))
    finally:
        dist.destroy_process_group()


def test_shard_gather_import_gloo_world2():
    import torch.multiprocessing as mp
    from paper_2503_08415_b200 import build
    build.build()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=180) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    assert sorted(r[0] for r in res) == [0, 1]
    assert all(r[1] for r in res), res
    assert sum(r[2] for r in res) == 128 and all(r[2] == 64 for r in res)


def _worker_idle(rank, world, port, out_q):
    """More ranks than points: the idle rank joins the all-gather with an empty slot."""
    import torch.distributed as dist

    import sweep_inputs as si
    import paper_2503_08415_b200 as P
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        cfg = si.subset(si.c2(), rates=[0], seeds=[0, 1])
        sw = P.Sweep(cfg)
        b, e, s = P.shard_range(sw.num_points, rank, world)
        mine = list(range(b, e, s))
        allv = P.gather_summaries(fake_summaries(mine), sw.num_points)
        sw.import_summaries(allv)
        ok = list(allv["point"]) == [0, 1]
        out_q.put((rank, bool(ok), len(mine)))
    finally:
        dist.destroy_process_group()


def test_more_ranks_than_points_gloo_world3():
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker_idle, args=(r, 3, port, q)) for r in range(3)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=180) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    assert [r[2] for r in res] == [1, 1, 0] and all(r[1] for r in res), res
