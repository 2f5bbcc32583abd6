"""Row-sharded objective / full gradient over torch.distributed.

The ASAGA update loop does not shard (replicas only); the evaluation pass A9 does:
each rank owns a contiguous block of rows balanced by nnz, computes

    out[0:d] = sum_{i in shard} sigma_i(x) a_i,   out[d] = sum_{i in shard} log(1+exp(-b_i a_i.x))

with ``asaga_partial_obj_grad`` (its shard context's kernels), and one all-reduce of
the (d+1)-vector (NCCL over NVLink on B200) gives every rank

    f = out[d]/n + lambda/2 ||x||^2,     grad f = out[0:d]/n + lambda x

(Section 4.1).  x is broadcast from rank 0 first so all ranks evaluate
the same point.  ``partial`` can be injected (the CPU gloo tests do); the default
is the CUDA path and there is no fallback.
"""
from __future__ import annotations

import numpy as np


def shard_rows(indptr: np.ndarray, world: int, rank: int) -> tuple[int, int]:
    """Contiguous row block [lo, hi) of `rank`, boundaries where the cumulative nnz
    crosses k * nnz / world (every row in exactly one block)."""
    indptr = np.asarray(indptr, dtype=np.int64)
    n = indptr.shape[0] - 1
    nnz = int(indptr[-1])
    cuts = [0]
    for k in range(1, world):
        cuts.append(int(np.searchsorted(indptr, k * nnz / world, side="left")))
    cuts.append(n)
    cuts = np.maximum.accumulate(np.clip(cuts, 0, n))
    return int(cuts[rank]), int(cuts[rank + 1])


def row_block(indptr, indices, data, y, lo: int, hi: int):
    """CSR arrays of rows [lo, hi) with a rebased indptr (numpy, host)."""
    a, b = int(indptr[lo]), int(indptr[hi])
    ip = np.asarray(indptr[lo:hi + 1], dtype=np.int64) - a
    return ip, np.asarray(indices[a:b]), np.asarray(data[a:b]), np.asarray(y[lo:hi])


class ShardedObjective:
    """f and grad f of the whole problem from row shards, one all-reduce per call."""

    def __init__(self, n_total: int, d: int, lam: float, partial=None, shard_ctx=None,
                 group=None, device=None):
        import torch

        self.n, self.d, self.lam = int(n_total), int(d), float(lam)
        self.group = group
        self.device = device if device is not None else torch.device("cpu")
        if partial is None:
            if shard_ctx is None:
                raise ValueError("need the shard's Asaga context (CUDA) or an explicit partial")
            # on torch's current stream: ordered after the broadcast / copy of x and
            # before the all-reduce of out (the context's own stream is not).  torch's
            # default stream has handle 0, which the C-ABI reads as "the context's stream",
            # so it is passed as cudaStreamLegacy (0x1).
            def partial(x, out):
                h = torch.cuda.current_stream(self.device).cuda_stream
                shard_ctx.partial_obj_grad(x, out, stream=h if h != 0 else 1)
        self.partial = partial
        self.out = torch.zeros(self.d + 1, dtype=torch.float64, device=self.device)

    def __call__(self, x):
        """x: float64 tensor of d on self.device (rank 0's value is used).  Returns (f, grad)
        as tensors on self.device (f 0-dimensional): no host round trip.  Everything is
        ordered on torch's current stream -- the broadcast, the partial (launched on that
        stream) and the all-reduce (NCCL is stream-ordered) -- so nothing synchronises the
        host; read f with float(f) when it is needed there."""
        import torch
        import torch.distributed as dist

        x = x.to(self.device, dtype=torch.float64).contiguous()
        if dist.is_initialized():
            dist.broadcast(x, src=0, group=self.group)
        self.partial(x, self.out)
        if dist.is_initialized():
            dist.all_reduce(self.out, op=dist.ReduceOp.SUM, group=self.group)
        f = self.out[self.d] / self.n + 0.5 * self.lam * torch.dot(x, x)
        g = self.out[: self.d] / self.n + self.lam * x
        return f, g
