"""bench.py -- ASAGA hot path on B200: updates/s of one full step of the path.

A "step" = one pass of every SURVEY.md section 8(a) row over one batch of
synthetic input, all through the C-ABI (libasaga.so):
    A0+A1  asaga_reload_device  (validate, fold labels, n_v / D / L)     2 kernels
    A2-A8  asaga_run_async(n)   (one epoch = n ASAGA updates)           1 kernel
    A9     asaga_objective_device (f at the new iterate)                3 kernels
value = n updates / step time (device time, CUDA events on the context's
stream, max over ranks).  L2 is flushed (a 512 MiB write) between steps,
outside the timed events.  N > 1 ranks run independent lambda-sweep
instances (lambda_r = 10^-r / n): weak scaling, no collective on
the data path.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--workload c2]
                    [--concurrency 0] [--impl ours|reference]
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

import datagen  # noqa: E402

# Algorithmic bytes per update, labels folded:
#   HBM   : row (4 B index + 8 B value) * s + indptr pair 16 B + alpha_i RMW 16 B
#   L2    : one 32-byte {x, abar, D} sector gather per entry + 2 REDs per entry
def hbm_bytes_per_update(mean_s: float) -> float:
    return 12.0 * mean_s + 16.0 + 16.0


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--workload", default="c2", choices=["c1", "c2", "c3", "c4"])
    ap.add_argument("--concurrency", type=int, default=0, help="samples in flight (0 = auto)")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=15.0)
    return ap.parse_args()


def dist_setup(args):
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled every 200 ms during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu: int):
        self.gpu = gpu
        self.rows = []
        self._stop = threading.Event()
        self._t = threading.Thread(target=self._run, daemon=True)

    def _run(self):
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.Q}",
                                      "--format=csv,noheader,nounits"], capture_output=True,
                                     text=True, timeout=5).stdout.strip()
                if out:
                    self.rows.append([c.strip() for c in out.split(",")])
            except Exception:
                pass
            self._stop.wait(0.2)

    def __enter__(self):
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._t.join(timeout=10)

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[j] for r in self.rows for j in range(4)
                          if len(r) > 3 + j and r[3 + j].lower() == "active"})
        return {"sm_mhz": float(np.median(sm)) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(self.rows)}


def peaks():
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))), "measured"
    except Exception:
        return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0}, "fallback"


def ncu_traffic(workload: str):
    """dram bytes per launch of the update kernel from the committed ncu capture, if any."""
    try:
        t = json.load(open(os.path.join(ROOT, "profiles", "traffic.json")))
        return t.get(workload)
    except Exception:
        return None


def cpu_baseline(p, gamma, seconds: float):
    """The oracle (sequential fp64 Sparse SAGA, 1 host thread) on a bounded sample."""
    import oracle

    st = oracle.State(p.n, p.d)
    D = oracle.reweight(p.n, oracle.column_counts(p))
    probe = min(p.n, 20_000)
    t0 = time.perf_counter()
    oracle.sparse_saga(p, p.y, p.lam, gamma, datagen.SAMPLE_SEED, probe, st, D)
    dt = time.perf_counter() - t0
    T = max(probe, int(probe * seconds / max(dt, 1e-6)))
    t0 = time.perf_counter()
    oracle.sparse_saga(p, p.y, p.lam, gamma, datagen.SAMPLE_SEED, T, st, D)
    dt = time.perf_counter() - t0
    return {"value": T / dt, "unit": "updates/s", "cores": 1, "kind": "oracle",
            "sample": f"{T} sequential updates (t={probe}..{probe + T - 1}) of {p.name} from x=0 "
                      f"after a {probe}-update probe; {dt:.1f} s on 1 host thread ({os.cpu_count()} cores on host)"}


def run_reference(args, world, rank):
    """--impl reference: the oracle as it stands, on the host cores, rank 0 only."""
    if rank != 0:
        return
    import oracle

    p = datagen.make(args.workload)
    gamma = 1.0 / (3.0 * oracle.lipschitz(p, p.lam))
    st = oracle.State(p.n, p.d)
    D = oracle.reweight(p.n, oracle.column_counts(p))
    per_step = max(1000, min(p.n, 2_000_000 // max(args.steps + args.warmup, 1)))
    for _ in range(args.warmup):
        oracle.sparse_saga(p, p.y, p.lam, gamma, datagen.SAMPLE_SEED, per_step, st, D)
    t0 = time.perf_counter()
    for _ in range(args.steps):
        oracle.sparse_saga(p, p.y, p.lam, gamma, datagen.SAMPLE_SEED, per_step, st, D)
    dt = time.perf_counter() - t0
    v = per_step * args.steps / dt
    sample = f"{args.steps} steps x {per_step} sequential updates of {p.name} (bounded sample of an epoch of n={p.n})"
    print(json.dumps({
        "impl": "reference", "metric": "ASAGA updates/s", "value": v, "unit": "updates/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": dt / args.steps * 1e3, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": p.name, "n": p.n, "d": p.d, "nnz": p.nnz},
        "cpu_baseline": {"value": v, "unit": "updates/s", "cores": 1, "kind": "oracle",
                         "sample": sample},
        "e2e": {"value": v, "unit": "updates/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }))


def main():
    args = parse()
    world, rank, local = dist_setup(args)
    if args.impl == "reference":
        run_reference(args, world, rank)
        return
    import torch
    import torch.distributed as dist

    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    from paper_1606_04809_b200 import Asaga

    p = datagen.make(args.workload)
    lam = p.lam * (10.0 ** (-rank))  # rank 0: lambda = 1/n (the BASELINE config)
    # L = max ||a_i||^2/4 + lambda; rows are unit-norm (reading R7) -> gamma = 1/(3L)
    dev = torch.device("cuda", local)
    t = lambda a: torch.from_numpy(a).to(dev)
    indptr, indices, data, y = t(p.indptr), t(p.indices), t(p.data), t(p.y)
    a = Asaga(indptr, indices, data, y, p.d, lam, 1.0, concurrency=args.concurrency, device=local)
    gamma = 1.0 / (3.0 * a.stats()["L"])
    a.set_gamma(gamma)
    stream = torch.cuda.ExternalStream(a.stream, device=dev)
    flush = torch.empty(512 << 20, dtype=torch.uint8, device=dev)
    f_dev = torch.zeros(1, dtype=torch.float64, device=dev)
    seed = datagen.SAMPLE_SEED
    ev = lambda: torch.cuda.Event(enable_timing=True)

    def step(evs):
        evs[0].record(stream)
        a.reload(indptr, indices, data, y)  # A0 + A1
        evs[1].record(stream)
        a.run_async(p.n, seed)  # A2..A8, one epoch
        evs[2].record(stream)
        a.objective_device(f_dev)  # A9
        evs[3].record(stream)

    with torch.cuda.stream(stream):
        for _ in range(args.warmup):
            step([ev() for _ in range(4)])
            flush.zero_()
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        all_evs = []
        with ClockSampler(local) as clk:
            for _ in range(args.steps):
                evs = [ev() for _ in range(4)]
                step(evs)
                all_evs.append(evs)
                flush.zero_()
            torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
    step_ms = [e[0].elapsed_time(e[3]) for e in all_evs]
    upd_ms = [e[1].elapsed_time(e[2]) for e in all_evs]
    ing_ms = [e[0].elapsed_time(e[1]) for e in all_evs]
    obj_ms = [e[2].elapsed_time(e[3]) for e in all_evs]
    total_ms = float(sum(step_ms))
    f_final = float(f_dev.item())
    tmax = torch.tensor([total_ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(tmax, op=dist.ReduceOp.MAX)
    total_ms_max = float(tmax.item())
    value = world * p.n * args.steps / (total_ms_max / 1e3)

    # ---- e2e: the same step through the host-buffer C-ABI path (pinned host inputs,
    # H2D copies and the D2H read of f inside the timed region)
    hp = [torch.from_numpy(arr).pin_memory() for arr in (p.indptr, p.indices, p.data, p.y)]
    h2d = sum(x.numel() * x.element_size() for x in hp)
    e2e_ms = []
    for k in range(args.warmup + args.steps):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        a.reload(*hp)  # H2D + A0 + A1
        a.run_async(p.n, seed)
        f_host = a.objective()  # A9 + D2H of f (blocking)
        dt = (time.perf_counter() - t0) * 1e3
        if k >= args.warmup:
            e2e_ms.append(dt)
        flush.zero_()
    e2e_t = torch.tensor([sum(e2e_ms)], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(e2e_t, op=dist.ReduceOp.MAX)
    e2e_value = world * p.n * args.steps / (float(e2e_t.item()) / 1e3)

    if rank == 0:
        st = a.stats()
        pk, pk_kind = peaks()
        mean_s = p.nnz / p.n
        bytes_launch = hbm_bytes_per_update(mean_s) * p.n
        upd_avg_s = float(np.mean(upd_ms)) / 1e3
        achieved = bytes_launch / upd_avg_s / 1e9
        out = {
            "metric": "ASAGA updates/s (one step = ingest + 1 epoch of updates + objective)",
            "value": value, "unit": "updates/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": total_ms_max / args.steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic",
            "config": {"workload": p.name, "n": p.n, "d": p.d, "nnz": p.nnz,
                       "samples_in_flight": st["concurrency"], "lanes_per_sample": st["lanes_per_sample"],
                       "gamma": gamma, "lambda": "10^-rank / n", "l2_flush": "512 MiB write between steps",
                       "parallelism": f"{world} independent lambda-sweep instances" if world > 1 else "1 GPU"},
            "breakdown_ms": {"ingest_A0_A1": float(np.mean(ing_ms)), "updates_A2_A8": float(np.mean(upd_ms)),
                             "objective_A9": float(np.mean(obj_ms))},
            "update_kernel_updates_per_s": p.n / upd_avg_s,
            "f_after_step": f_final,
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": pk["hbm_gbs"], "unit": "GB/s",
                         "frac": achieved / pk["hbm_gbs"], "traffic": ncu_traffic(p.name),
                         "kernel": "asaga_update_kernel",
                         "bytes_per_update": hbm_bytes_per_update(mean_s), "peak_source": pk_kind},
            "e2e": {"value": e2e_value, "unit": "updates/s", "h2d_bytes_per_step": h2d,
                    "d2h_bytes_per_step": 8, "f_host": f_host},
            "gpu_launches": 6 * args.steps,
            "clocks": clk.summary(),
        }
        if not args.no_cpu_baseline:
            out["cpu_baseline"] = cpu_baseline(p, gamma, args.cpu_seconds)
        print(json.dumps(out))
    a.close()
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
