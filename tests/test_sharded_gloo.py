"""Multi-process (world_size 2, gloo, CPU) test of the sharded objective plumbing:
the nnz-balanced row split covers every row once, and broadcast + all-reduce of
the shard partials reproduces the whole-problem f and grad f (oracle).  The
per-shard partial is injected (oracle) because there is no GPU here; on B200 it
is asaga_partial_obj_grad (tests/test_gpu_parity.py checks the shard sums)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import datagen
import oracle
from paper_1606_04809_b200.sharded import ShardedObjective, row_block, shard_rows


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        p = datagen.make("c3", n_rows=3000)
        lo, hi = shard_rows(p.indptr, world, rank)
        ip, ix, dt, yy = row_block(p.indptr, p.indices, p.data, p.y, lo, hi)
        shard = datagen.Problem("shard", hi - lo, p.d, ip, ix, dt, yy, 1.0)

        def partial(x, out):
            xn = x.numpy()
            ns = shard.n
            out[p.d] = ns * oracle.objective(shard, shard.y, 0.0, xn)
            out[: p.d] = torch.from_numpy(ns * oracle.full_grad(shard, shard.y, 0.0, xn))

        obj = ShardedObjective(p.n, p.d, p.lam, partial=partial)
        x = torch.from_numpy(np.random.default_rng(rank).standard_normal(p.d))  # rank 0's wins
        f, g = obj(x)
        q.put((rank, lo, hi, float(f), g.numpy()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2])
def test_sharded_objective_gloo(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for pr in procs:
        pr.start()
    res = [q.get(timeout=300) for _ in range(world)]
    for pr in procs:
        pr.join(timeout=60)
        assert pr.exitcode == 0
    res.sort()
    p = datagen.make("c3", n_rows=3000)
    # the blocks tile [0, n) and are balanced by nnz
    assert res[0][1] == 0 and res[-1][2] == p.n
    for a, b in zip(res[:-1], res[1:]):
        assert a[2] == b[1]
    nnzs = [p.indptr[r[2]] - p.indptr[r[1]] for r in res]
    assert max(nnzs) - min(nnzs) <= p.row_lengths().max()
    x0 = np.random.default_rng(0).standard_normal(p.d)
    f_ref = oracle.objective(p, p.y, p.lam, x0)
    g_ref = oracle.full_grad(p, p.y, p.lam, x0)
    for _, _, _, f, g in res:
        assert f == pytest.approx(f_ref, rel=1e-12)
        assert np.linalg.norm(g - g_ref) <= 1e-12 * np.linalg.norm(g_ref)


def test_shard_rows_edge_cases():
    indptr = np.array([0, 5, 5 + 1, 5 + 2, 5 + 3])  # one heavy row then light ones
    blocks = [shard_rows(indptr, 3, r) for r in range(3)]
    assert blocks[0][0] == 0 and blocks[-1][1] == 4
    assert all(a[1] == b[0] for a, b in zip(blocks[:-1], blocks[1:]))
    assert shard_rows(indptr, 1, 0) == (0, 4)
    # more ranks than rows: empty blocks allowed, still a tiling
    bl = [shard_rows(np.array([0, 1, 2]), 4, r) for r in range(4)]
    assert bl[0][0] == 0 and bl[-1][1] == 2 and all(x[0] <= x[1] for x in bl)


def _sweep_worker(rank, world, port, q):
    import bench

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        p = datagen.make("c1")
        lam = bench.sweep_lambda(p, world, rank)
        local_ms = 100.0 * (rank + 1)  # rank 1 is the slower one
        value, ms = bench.job_rate(local_ms, world, p.n, 4, torch.device("cpu"))
        q.put((rank, bench.default_workload(world), lam, value, ms))
    finally:
        dist.destroy_process_group()


def test_bench_sweep_rank_logic_gloo():
    """bench.py --gpus N (BASELINE config 5): each rank gets its own lambda = 10^-(r+1)/n, the
    default workload is c3's shape, and the job's rate is all ranks' updates over the MAX of
    the ranks' timed totals (world size 2, gloo)."""
    import bench

    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_sweep_worker, args=(r, world, port, q)) for r in range(world)]
    for pr in procs:
        pr.start()
    res = sorted(q.get(timeout=300) for _ in range(world))
    for pr in procs:
        pr.join(timeout=60)
        assert pr.exitcode == 0
    p = datagen.make("c1")
    assert [r[1] for r in res] == ["c3", "c3"] and bench.default_workload(1) == "c4"
    assert res[0][2] == pytest.approx(0.1 / p.n, rel=1e-15) and res[1][2] == pytest.approx(0.01 / p.n, rel=1e-15)
    assert bench.sweep_lambda(p, 1, 0) == p.lam
    for _, _, _, value, ms in res:  # every rank sees the max (200 ms) and the aggregate rate
        assert ms == 200.0
        assert value == pytest.approx(world * p.n * 4 / 0.2, rel=1e-15)
