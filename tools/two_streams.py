"""Experiment: two independent bench steps in flight (two contexts, two streams) on one GPU.

Each context runs the bench step (asaga_reload_device_async + one epoch + objective) on its
own stream over the same borrowed device matrix; steps alternate between the contexts, so two
independent problems' kernels can overlap.  Prints the aggregate updates/s against one stream.

    python tools/two_streams.py [--workload c4] [--steps 10]
"""
import argparse
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402
import datagen  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="c4")
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--contexts", type=int, default=2)
    args = ap.parse_args()
    import torch
    from paper_1606_04809_b200 import Asaga

    p = datagen.make(args.workload)
    op = bench.OPERATING_POINT[args.workload]
    dev = torch.device("cuda", 0)
    t = lambda a: torch.from_numpy(a).to(dev)
    A = (t(p.indptr), t(p.indices), t(p.data), t(p.y))
    res = {}
    for nctx in sorted({1, args.contexts}):
        ctxs = []
        for _ in range(nctx):
            a = Asaga(*A, p.d, p.lam, 1.0, concurrency=op["W"], **bench.asaga_options(op))
            a.set_gamma(op["gscale"] / (3.0 * a.stats()["L"]))
            ctxs.append(a)
        streams = [torch.cuda.ExternalStream(a.stream, device=dev) for a in ctxs]
        fs = [torch.zeros(1, dtype=torch.float64, device=dev) for _ in ctxs]

        def step(k):
            a = ctxs[k % nctx]
            a.reload_async(*A)
            a.run_async(p.n, datagen.SAMPLE_SEED)
            a.objective_device(fs[k % nctx])

        for k in range(2 * nctx):
            step(k)
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        for s in streams:  # every context's stream starts after e0
            s.wait_event(e0)
        for k in range(args.steps):
            step(k)
        for s in streams:
            ev = torch.cuda.Event()
            ev.record(s)
            torch.cuda.current_stream().wait_event(ev)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1)
        res[nctx] = {"updates_per_s": p.n * args.steps / (ms / 1e3), "ms_per_step": ms / args.steps,
                     "f": [float(f) for f in fs]}
        for a in ctxs:
            a.close()
    print(json.dumps({"workload": p.name, "steps": args.steps, "results": res}))


if __name__ == "__main__":
    main()
