"""bench.py -- the ASAGA hot path on B200, through the C-ABI (libasaga.so).

A "step" = one pass of every SURVEY.md section 8(a) row over one batch of
synthetic input:
    A0+A1  asaga_reload_device_async  validate (read-only), n_v / D / L (non-blocking;
                                      the validation is read back by A9's call)
    A2-A8  asaga_run_async(n)      one epoch = n ASAGA updates (c2: the combine kernel,
                                   c3/c4: the plain kernel with the hot split)   1 kernel
    A9     asaga_objective_device  f at the new iterate                   1 kernel
value = n updates / step time (CUDA events on the context's stream, summed
over the K timed steps, max over ranks).  512 MiB is written and read back
between steps, outside the timed events (a cold, clean L2 at every step).  The update kernel runs at the
workload's convergent operating point (samples in flight W, step gamma =
scale / (3L)) chosen from the sweeps in profiles/ (DESIGN.md "Operating
point"); the line also reports time-to-1e-6 from x = 0 at that point.

Workload: at N = 1 the default is c4, BASELINE.json's largest single-GPU configuration
(URL-like, n = 2,396,130, d = 3,231,961).  N > 1 ranks run BASELINE config 5: c3's shape as
independent lambda-sweep instances, lambda_r = 10^-(r+1) / n on rank r: weak
scaling, no collective on the data path.  `--workload` overrides either.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--workload c4]
                    [--concurrency W] [--gamma-scale s] [--impl ours|reference]
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

# The same metric string in both arms (ours and --impl reference), so the driver can pair them.
METRIC = "ASAGA updates/s"
STEP = "one step = ingest A0-A1 + one epoch of n updates A2-A8 + objective A9"


def default_workload(world: int) -> str:
    """c4 at one GPU (BASELINE's largest single-GPU config); config 5 (c3 sweep) for N > 1."""
    return "c4" if world <= 1 else "c3"


def sweep_lambda(p, world: int, rank: int) -> float:
    """lambda of this rank: 1/n at N = 1 (configs 1-4); config 5's 10^-(r+1)/n for N > 1."""
    return p.lam if world <= 1 else p.lam * 10.0 ** (-(rank + 1))


def cpu_model() -> str:
    try:
        for ln in open("/proc/cpuinfo"):
            if ln.startswith("model name"):
                return ln.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


class pinned_core:
    """Pin the calling thread (the oracle runs in it, through ctypes) to one host core for the
    CPU baseline (`taskset -c 0`), restoring the previous affinity after."""

    def __init__(self):
        self.core = None
        self.prev = None

    def __enter__(self):
        try:
            self.prev = os.sched_getaffinity(0)
            self.core = min(self.prev)
            os.sched_setaffinity(0, {self.core})
        except (AttributeError, OSError):
            self.core = None
        return self

    def __exit__(self, *a):
        if self.prev is not None:
            try:
                os.sched_setaffinity(0, self.prev)
            except OSError:
                pass

# Convergent operating points (W samples in flight, gamma scale vs 1/(3L), bulk-scatter
# feature frequency) from tools/sweep.py on B200 (profiles/r01_operating_point.md):
# the fastest time-to-1e-6 whose epoch count stays within 1.5x the oracle's.
OPERATING_POINT = {
    # c1 (n = 1000): 64 in flight = 6.4 % of n (Thm 2 asks tau < n/10) at half the step:
    # 11-13 epochs in one-epoch launches (W = 16, gamma 1/(3L): 12-14 at a third of the rate)
    "c1": dict(W=64, gscale=0.5, bulk=0.0, split=0.0, repl=0, comb=0.0, unpaired=1),
    # c2: every feature combined per thread block (asaga_combine_kernel), 40 workers per SM
    # (W = 6808, 46 per SM, is 7 % faster but sits at the edge: one round-end test run saw
    # all three streams miss 1e-6 in 15 one-epoch launches; 5920 gives 11 epochs with margin)
    # (last session: with the final build's 1.3 us communication pass, W = 6512 reaches 1e-6 in
    # 10 epochs in every stream, 3.76e9 /s; 6808: 11 epochs, 3.85e9, gamma window 0.04 only;
    # profiles/r02_update_kernel.md section 22)
    "c2": dict(W=6512, gscale=0.04, bulk=0.0, split=0.0, repl=0, comb=1e-300),
    # c3 / c4: plain kernel, paired scatter (the x and abar adds of one entry in one reduction
    # instruction: one L2 request per {x, abar} sector), rows staged by 1-D TMA bulk copies;
    # no hot split (with pairing the popular pair's line takes a load and one merged request
    # per update).  c1 keeps the unpaired scatter (6 % faster there).  Round-2 sweeps in
    # profiles/r02_update_kernel.md section 10: c3 1.72e8 -> 1.76e8 at the same W; c4 at
    # W = 480 (15 epochs in every stream) 1.59e8 -> 1.79e8.
    # c3: the record layout ({x, abar, D, .} per coordinate: one 256-bit gather and one paired
    # request per entry, no per-entry D stream, no expand pass) at W = 352: 1.87e8 in 12 epochs
    # (the default layout: 1.76e8 at W = 384, 12 epochs; section 11 of the same file)
    "c3": dict(W=352, gscale=0.3, bulk=0.0, split=0.0, repl=0, comb=0.0, rowcp=0, rec=1),
    # c4: D_c gathered per entry from the d-vector with the coordinate gather (d_gather: no
    # per-entry D stream, no expand pass per reload -- 1.07 ms of the step) at W = 480: 1.78e8
    # in 15 epochs (W = 544 does not converge); with the D stream the kernel reaches 1.82e8 but
    # the step pays the expand pass (sections 15 and 18 of the same file)
    "c4": dict(W=480, gscale=0.25, bulk=0.0, split=0.0, repl=0, comb=0.0, rowcp=0, dgather=1),
}


def asaga_options(op):
    """Asaga keyword options of an operating point."""
    return dict(bulk_scatter_min_freq=op["bulk"], hot_split_min_freq=op["split"],
                smem_replica_refresh=op["repl"], combine_min_freq=op["comb"],
                l2_persist_state=bool(op.get("persist", False)),
                row_copy_elementwise=bool(op.get("rowcp", 0)),
                scatter_unpaired=bool(op.get("unpaired", 0)),
                record_layout=bool(op.get("rec", 0)), d_gather=bool(op.get("dgather", 0)))


def hbm_bytes_per_update(mean_s: float) -> float:
    """Algorithmic HBM bytes of one update: the row
    (int32 index + fp64 folded value) * s, the indptr pair, the alpha_i read-modify-write.
    (D_v is a d-vector the method keeps resident; the plain kernel's per-entry copy of it is
    an implementation choice, not algorithmic traffic -- it shows up in `traffic`.)"""
    return 12.0 * mean_s + 16.0 + 16.0


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--workload", default=None, choices=["c1", "c2", "c3", "c4"],
                    help="default: c4 at N = 1, c3 (config 5 sweep) at N > 1")
    ap.add_argument("--concurrency", type=int, default=None, help="samples in flight")
    ap.add_argument("--gamma-scale", type=float, default=None)
    ap.add_argument("--l2-persist", type=int, default=None, help="override l2_persist_state (0/1)")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-ttt", action="store_true", help="skip the time-to-1e-6 run")
    ap.add_argument("--cpu-seconds", type=float, default=15.0)
    return ap.parse_args()


class ClockSampler:
    """SM clocks / clock-event (throttle) reasons sampled every 5 ms during the timed region,
    in process through NVML (what nvidia-smi reads): no fork of this large CUDA process while
    the timed steps are being enqueued (spawning nvidia-smi there stalled the enqueueing
    thread and starved the GPU: c2's ingest phase read 57 instead of 44 us).  Falls back to
    one background `nvidia-smi -lms 200` started before the timed region."""

    def __init__(self, gpu: int):
        self.gpu = gpu
        self.rows = []
        self._stop = threading.Event()
        self._t = None
        self._proc = None
        self._nv = None
        try:
            import pynvml as nv

            nv.nvmlInit()
            h = None
            try:
                import torch

                pr = torch.cuda.get_device_properties(gpu)
                bus = "%08x:%02x:%02x.0" % (pr.pci_domain_id, pr.pci_bus_id, pr.pci_device_id)
                h = nv.nvmlDeviceGetHandleByPciBusId_v2(bus)
            except Exception:
                h = nv.nvmlDeviceGetHandleByIndex(gpu)
            self._nv, self._h = nv, h
            self._t = threading.Thread(target=self._run_nvml, daemon=True)
        except Exception:
            self._nv = None

    def _run_nvml(self):
        nv, h = self._nv, self._h
        bits = [("hw_slowdown", nv.nvmlClocksEventReasonHwSlowdown),
                ("hw_thermal_slowdown", nv.nvmlClocksEventReasonHwThermalSlowdown),
                ("sw_thermal_slowdown", nv.nvmlClocksEventReasonSwThermalSlowdown),
                ("sw_power_cap", nv.nvmlClocksEventReasonSwPowerCap)]
        while True:
            try:
                sm = nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM)
                mx = nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM)
                rs = nv.nvmlDeviceGetCurrentClocksEventReasons(h)
                self.rows.append([str(sm), str(mx), ""] + ["Active" if rs & b else "Not Active" for _, b in bits])
            except Exception:
                pass
            if self._stop.wait(0.005):
                break

    def __enter__(self):
        if self._t is not None:
            self._t.start()
        else:
            self._proc = subprocess.Popen(["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.Q}",
                                           "--format=csv,noheader,nounits", "-lms", "200"],
                                          stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self._t is not None:
            self._t.join(timeout=10)
        if self._proc is not None:
            self._proc.terminate()  # this Popen's own PID
            try:
                out = self._proc.communicate(timeout=5)[0]
            except Exception:
                out = ""
            self.rows += [[c.strip() for c in ln.split(",")] for ln in out.splitlines() if ln.strip()]

    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        fl = lambda v: float(v) if v.replace(".", "", 1).isdigit() else None
        sm = [fl(r[0]) for r in self.rows if fl(r[0]) is not None]
        mx = [fl(r[1]) for r in self.rows if fl(r[1]) is not None]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[j] for r in self.rows for j in range(4)
                          if len(r) > 3 + j and r[3 + j].lower() == "active"})
        return {"sm_mhz": float(np.median(sm)) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(self.rows)}


def load_json(*parts):
    try:
        return json.load(open(os.path.join(ROOT, *parts)))
    except Exception:
        return None


def peaks():
    pk = load_json("MEASURED_PEAKS.json")
    if pk:
        return pk, "measured (MEASURED_PEAKS.json)"
    return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0}, "fallback (B200_PROFILING.md)"


def cpu_baseline(p, lam, gamma, seconds: float):
    """The oracle (sequential fp64 Sparse SAGA, 1 host thread pinned to one core) on a bounded
    sample, plus its time to 1e-6: the oracle's epoch count from the golden file (written by
    scripts/compute_fstar.py, f checked every n/10 updates) x n / the rate measured here --
    extrapolated, not run to the end (SURVEY 8(d) allows it for the large configs)."""
    import oracle

    st = oracle.State(p.n, p.d)
    D = oracle.reweight(p.n, oracle.column_counts(p))
    probe = min(p.n, 20_000)
    with pinned_core() as pin:
        t0 = time.perf_counter()
        oracle.sparse_saga(p, p.y, lam, gamma, datagen.SAMPLE_SEED, probe, st, D)
        dt = time.perf_counter() - t0
        T = max(probe, int(probe * seconds / max(dt, 1e-6)))
        t0 = time.perf_counter()
        oracle.sparse_saga(p, p.y, lam, gamma, datagen.SAMPLE_SEED, T, st, D)
        dt = time.perf_counter() - t0
    rate = T / dt
    out = {"value": rate, "unit": "updates/s", "cores": 1, "kind": "oracle",
           "cpu_model": cpu_model(), "host_threads": os.cpu_count(), "pinned_core": pin.core,
           "sample": f"{T} sequential updates (t={probe}..{probe + T - 1}) of {p.name} from x=0 "
                     f"after a {probe}-update probe, gamma=1/(3L); {dt:.1f} s on 1 host thread "
                     f"(pinned to core {pin.core}) of {os.cpu_count()}"}
    gold = load_json("tests", "golden", f"fstar_{p.name}.json")
    if gold is not None and gold.get("sha256") == p.sha256() and lam == p.lam:
        ep = gold["oracle_epochs_to_1e-6"]
        out["time_to_1e-6"] = {"epochs": ep, "seconds": ep * p.n / rate,
                               "how": "extrapolated: the oracle's epochs to 1e-6 (golden file, f every "
                                      "n/10 updates) x n / the updates/s measured here"}
    return out


def run_reference(args, rank):
    """--impl reference: the oracle as it stands, on the host cores, rank 0 only."""
    if rank != 0:
        return
    import oracle

    world = int(os.environ.get("WORLD_SIZE", "1"))
    p = datagen.make(args.workload or default_workload(world))
    lam = sweep_lambda(p, world, 0)
    gamma = 1.0 / (3.0 * oracle.lipschitz(p, lam))
    st = oracle.State(p.n, p.d)
    D = oracle.reweight(p.n, oracle.column_counts(p))
    per_step = max(1000, min(p.n, 3_000_000 // max(args.steps + args.warmup, 1)))
    with pinned_core() as pin:
        for _ in range(args.warmup):
            oracle.sparse_saga(p, p.y, lam, gamma, datagen.SAMPLE_SEED, per_step, st, D)
        t0 = time.perf_counter()
        for _ in range(args.steps):
            oracle.sparse_saga(p, p.y, lam, gamma, datagen.SAMPLE_SEED, per_step, st, D)
        dt = time.perf_counter() - t0
    v = per_step * args.steps / dt
    sample = (f"{args.steps} steps x {per_step} sequential updates of {p.name} "
              f"(a bounded sample of the n={p.n}-update epoch), 1 host thread (pinned to core "
              f"{pin.core}) of {os.cpu_count()} ({cpu_model()}); the oracle is the reference arm "
              f"(the paper's Scala code is not available)")
    print(json.dumps({
        "impl": "reference", "metric": METRIC, "value": v, "unit": "updates/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": dt / args.steps * 1e3, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": p.name, "n": p.n, "d": p.d, "nnz": p.nnz, "lambda": lam,
                   "step": f"{per_step} oracle updates (a bounded sample of {STEP})"},
        "cpu_baseline": {"value": v, "unit": "updates/s", "cores": 1, "kind": "oracle",
                         "cpu_model": cpu_model(), "pinned_core": pin.core, "sample": sample},
        "e2e": {"value": v, "unit": "updates/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }))


def job_rate(local_ms: float, world: int, n: int, steps: int, device) -> tuple[float, float]:
    """Whole-job throughput: every rank ran `steps` steps of n updates; the job's time is the
    MAX over ranks of their timed totals (all-reduce MAX when world > 1).  Returns
    (updates/s of all ranks together, the max total in ms)."""
    import torch
    import torch.distributed as dist

    t = torch.tensor([float(local_ms)], dtype=torch.float64, device=device)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms = float(t.item())
    return world * n * steps / (ms / 1e3), ms


def time_to_target(a, p, stream, seed, tol=1e-6, max_epochs=30):
    """From x = 0: epochs and update-kernel seconds until f - f* <= tol, in the launch regime
    `value` is measured in -- one launch per epoch, f checked after each (evaluation
    excluded) -- against the oracle's epoch count at the same whole-epoch cadence (its
    0.1-epoch count from the golden file, rounded up).  f* from the oracle's golden file."""
    import math

    import torch

    gold = load_json("tests", "golden", f"fstar_{p.name}.json")
    if gold is None or gold.get("sha256") != p.sha256():
        return None
    fstar = gold["f_star"]
    oracle_ep = math.ceil(gold["oracle_epochs_to_1e-6"] - 1e-9)
    ms = 0.0
    a.set_state(np.zeros(p.d), np.zeros(p.n), np.zeros(p.d), 0)
    f = float("nan")
    for j in range(1, max_epochs + 1):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        a.run_async(p.n, seed)
        e1.record(stream)
        f = a.objective()
        ms += e0.elapsed_time(e1)
        if f - fstar <= tol:
            return {"epochs": j, "seconds": ms / 1e3, "tol": tol, "f_star": fstar,
                    "launch": "one epoch per launch, f checked between launches",
                    "oracle_epochs": oracle_ep, "oracle_epochs_tenths": gold["oracle_epochs_to_1e-6"],
                    "within_1p5x_oracle_epochs": j <= 1.5 * oracle_ep}
        if not np.isfinite(f):
            break
    return {"epochs": None, "seconds": None, "tol": tol, "f_star": fstar, "last_subopt": f - fstar,
            "oracle_epochs": oracle_ep}


def main():
    args = parse()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        run_reference(args, rank)
        return
    import torch
    import torch.distributed as dist

    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    from paper_1606_04809_b200 import Asaga

    workload = args.workload or default_workload(world)
    p = datagen.make(workload)
    op = dict(OPERATING_POINT[workload])
    if args.l2_persist is not None:
        op["persist"] = bool(args.l2_persist)
    W = args.concurrency if args.concurrency is not None else op["W"]
    gscale = args.gamma_scale if args.gamma_scale is not None else op["gscale"]
    bulk = op["bulk"]
    lam = sweep_lambda(p, world, rank)
    dev = torch.device("cuda", local)
    t = lambda arr: torch.from_numpy(arr).to(dev)
    indptr, indices, data, y = t(p.indptr), t(p.indices), t(p.data), t(p.y)
    a = Asaga(indptr, indices, data, y, p.d, lam, 1.0, concurrency=W, device=local, **asaga_options(op))
    L = a.stats()["L"]
    gamma = gscale / (3.0 * L)
    a.set_gamma(gamma)
    stream = torch.cuda.ExternalStream(a.stream, device=dev)
    flush = torch.empty(512 << 20, dtype=torch.uint8, device=dev)
    flush_sink = torch.zeros(1, dtype=torch.int64, device=dev)

    def l2_flush():
        """Between steps, outside the timed events: write a buffer 4x the L2 (evicts the
        step's data), then read it back so the lines left in L2 are clean -- the next step
        starts cold without paying to write back the flush's own dirty lines."""
        flush.zero_()
        torch.sum(flush.view(torch.int64), dim=0, keepdim=True, out=flush_sink)
    f_dev = torch.zeros(1, dtype=torch.float64, device=dev)
    seed = datagen.SAMPLE_SEED
    ev = lambda: torch.cuda.Event(enable_timing=True)

    def step(evs):
        evs[0].record(stream)
        a.reload_async(indptr, indices, data, y)  # A0 + A1 (validated at the objective below)
        evs[1].record(stream)
        a.run_async(p.n, seed)  # A2..A8, one epoch
        evs[2].record(stream)
        a.objective_device(f_dev)  # A9
        evs[3].record(stream)

    with torch.cuda.stream(stream):
        for _ in range(args.warmup):
            step([ev() for _ in range(4)])
            l2_flush()
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
                l2_flush()
            torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
    st_timed = a.stats()  # of the last timed step's update launch (combine_passes)
    step_ms = [e[0].elapsed_time(e[3]) for e in all_evs]
    upd_ms = [e[1].elapsed_time(e[2]) for e in all_evs]
    ing_ms = [e[0].elapsed_time(e[1]) for e in all_evs]
    obj_ms = [e[2].elapsed_time(e[3]) for e in all_evs]
    f_final = float(f_dev.item())
    value, total_ms_max = job_rate(float(sum(step_ms)), world, p.n, args.steps, dev)

    # ---- e2e: the same step through the host-buffer C-ABI path (pinned host inputs; every
    # step's H2D copy and the D2H read of its f inside the timed region).  Pipelined as a
    # user would run it: asaga_reload_async copies step k+1's matrix on the context's copy
    # stream into its second device buffer while step k computes; f of step k is read on
    # the host while step k+1 is in flight.
    hp = [torch.from_numpy(arr).pin_memory() for arr in (p.indptr, p.indices, p.data, p.y)]
    h2d = sum(x.numel() * x.element_size() for x in hp)
    f_pin = torch.zeros(2, dtype=torch.float64).pin_memory()
    f_devs = torch.zeros(2, dtype=torch.float64, device=dev)

    def e2e_run(k_steps):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        done = []
        f_last = None
        side = torch.cuda.current_stream(dev)  # torch's stream: the D2H of f (pinned memory
        # is recorded on it, never on the context's stream, which dies with the context)
        for k in range(k_steps):
            a.reload_async(*hp)  # H2D (copy stream) + A0 + A1
            a.run_async(p.n, seed)
            a.objective_device(f_devs[k % 2:k % 2 + 1])
            ready = torch.cuda.Event()
            ready.record(stream)
            side.wait_event(ready)
            f_pin[k % 2:k % 2 + 1].copy_(f_devs[k % 2:k % 2 + 1], non_blocking=True)  # D2H of f
            e = torch.cuda.Event()
            e.record(side)
            done.append(e)
            with torch.cuda.stream(stream):
                l2_flush()  # (on the compute stream, which has slack while the copies bind)
            if k >= 1:
                done[k - 1].synchronize()
                f_last = float(f_pin[(k - 1) % 2])
        done[-1].synchronize()
        f_last = float(f_pin[(k_steps - 1) % 2])
        return (time.perf_counter() - t0) * 1e3, f_last

    e2e_run(args.warmup)
    e2e_total, f_host = e2e_run(args.steps)
    a.stats()  # a blocking call: the last asynchronous reload's validation
    e2e_value, _ = job_rate(e2e_total, world, p.n, args.steps, dev)

    ttt = None
    if rank == 0 and not args.no_ttt and lam == p.lam:  # f* is known for lambda = 1/n
        # three runs with three sample streams (the paper averages 3 runs; SURVEY P14:
        # judged on the mean, the worst reported)
        a.reload(indptr, indices, data, y)
        runs = [time_to_target(a, p, stream, seed + r) for r in range(3)]
        if all(r is not None for r in runs):
            ep = [r["epochs"] for r in runs]
            sec = [r["seconds"] for r in runs]
            ttt = dict(runs[0])
            ttt["runs"] = [{"epochs": e, "seconds": s} for e, s in zip(ep, sec)]
            if all(e is not None for e in ep):
                ttt["epochs"] = float(np.mean(ep))
                ttt["seconds"] = float(np.mean(sec))
                ttt["worst_epochs"] = float(max(ep))
                ttt["worst_seconds"] = float(max(sec))
                ttt["within_1p5x_oracle_epochs"] = ttt["epochs"] <= 1.5 * ttt["oracle_epochs"]
                ttt["worst_within_1p5x_oracle_epochs"] = max(ep) <= 1.5 * ttt["oracle_epochs"]
            else:
                ttt["epochs"] = ttt["seconds"] = None
                ttt["within_1p5x_oracle_epochs"] = False

    # the max-throughput tau -- the update kernel alone at more samples in
    # flight than the convergent point (one-epoch launches, no flush), and whether that
    # point still meets the 1.5x budget (one sample stream)
    maxtp = None
    if rank == 0 and not args.no_ttt:
        scan = []
        for mult in (1, 2, 4, 8):
            try:
                a.set_concurrency(W * mult)
            except Exception:
                break
            a.reload(indptr, indices, data, y)
            a.run(p.n, seed)  # warm
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            a.run_async(p.n, seed)
            e1.record(stream)
            torch.cuda.synchronize()
            scan.append({"samples_in_flight": a.stats()["concurrency"],
                         "updates_per_s": p.n / (e0.elapsed_time(e1) / 1e3)})
        best = max(scan, key=lambda r: r["updates_per_s"])
        maxtp = {"scan": scan, "samples_in_flight": best["samples_in_flight"],
                 "updates_per_s": best["updates_per_s"], "gamma": gamma}
        if lam == p.lam:
            a.set_concurrency(best["samples_in_flight"])
            r = time_to_target(a, p, stream, seed)
            if r is not None:
                maxtp["epochs_to_1e-6"] = r["epochs"]
                maxtp["within_1p5x_oracle_epochs"] = (r["epochs"] is not None
                                                     and r["epochs"] <= 1.5 * r["oracle_epochs"])
        a.set_concurrency(W)

    if rank == 0:
        st = a.stats()
        pk, pk_kind = peaks()
        mean_s = p.nnz / p.n
        bpu = hbm_bytes_per_update(mean_s)
        upd_avg_s = float(np.mean(upd_ms)) / 1e3
        ups = p.n / upd_avg_s
        achieved = bpu * p.n / upd_avg_s / 1e9
        # the ceiling of the hottest feature's line for THIS configuration's per-update
        # operations on it (tools/microbench, profiles/microbench_b200.json)
        mb = load_json("profiles", "microbench_b200.json") or {}
        bp = mb.get("bulk_pair") or {}
        hot_achieved = ups
        if op["comb"] > 0 and st_timed["combine_passes"] > 0:
            # combining: the hot line takes one pair load + two REDs per block per pass,
            # not per update; achieved = those line operations per second
            hot = (mb.get("hot_pair") or {}).get("k10", {}).get("updates_per_s_per_pair")
            hot_ops = (f"one pair load + two REDs per thread block per communication pass "
                       f"({st_timed['combine_passes'] / p.n:.4f} per update, {st_timed['combine_blocks']} blocks, "
                       f"pass {upd_ms[-1] * 1e3 * st_timed['combine_blocks'] / st_timed['combine_passes']:.2f} us)")
            hot_achieved = st_timed["combine_passes"] / (upd_ms[-1] / 1e3)
        elif bulk > 0 and op["repl"] > 0:
            hot, hot_ops = bp.get("hot_k10_bulk_only_per_s_per_pair"), "one 16-B bulk reduction (reads from the SMEM replica) per update"
        elif bulk > 0:
            hot, hot_ops = bp.get("hot_k10_updates_per_s_per_pair"), "pair load + one 16-B bulk reduction per update"
        elif op["split"] == 0 and not op.get("unpaired", 0):
            # paired scatter: the popular pair's line takes one 16-B load and ONE request
            # carrying both adds per update (tools/red_pairing.cu)
            rp = load_json("profiles", "microbench_red_pairing.json") or {}
            hot, hot_ops = (rp.get("hot_k10_paired_updates_per_s_per_pair"),
                            "pair load + one paired reduction (x and abar adds of one sector in one instruction) per update")
        elif op["split"] > 0:
            hot, hot_ops = (mb.get("hot_line") or {}).get("ld_red_k10", {}).get("per_line"), "load + RED (x, abar split) per update"
        else:
            hot, hot_ops = (mb.get("hot_pair") or {}).get("k10", {}).get("updates_per_s_per_pair"), "pair load + two REDs per update"
        out = {
            "metric": METRIC,
            "value": value, "unit": "updates/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": total_ms_max / args.steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (datagen recipe, DESIGN.md 'Input recipe')",
            "config": {"workload": p.name, "n": p.n, "d": p.d, "nnz": p.nnz, "step": STEP,
                       "samples_in_flight": st["concurrency"], "lanes_per_sample": st["lanes_per_sample"],
                       "gamma": gamma, "gamma_scale_vs_1_over_3L": gscale,
                       "lambda": lam if world == 1 else "10^-(rank+1) / n (BASELINE config 5)",
                       "bulk_scatter_min_freq": bulk, "hot_split_min_freq": op["split"],
                       "smem_replica_refresh": op["repl"], "combine_min_freq": op["comb"],
                       "combine_hot_features": st["combine_hot"],
                       "l2_flush": "512 MiB write + read-back between steps (outside the timed events): every step starts with a cold, clean L2",
                       "parallelism": f"{world} independent lambda-sweep instances" if world > 1 else "1 GPU"},
            "breakdown_ms": {"ingest_A0_A1": float(np.mean(ing_ms)), "updates_A2_A8": float(np.mean(upd_ms)),
                             "objective_A9": float(np.mean(obj_ms))},
            "update_kernel_updates_per_s": ups,
            "time_to_1e-6": ttt,
            "max_throughput_point": maxtp,
            "f_after_step": f_final,
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": pk["hbm_gbs"], "unit": "GB/s",
                         "frac": achieved / pk["hbm_gbs"], "traffic": None,
                         "kernel": "asaga_combine_kernel" if op["comb"] > 0 else "asaga_update_kernel",
                         "bytes_per_update": bpu,
                         "peak_source": pk_kind},
            "roofline_hot_line": {
                "bound": f"L2 service of the hottest feature's line: {hot_ops}",
                "achieved": hot_achieved, "peak": hot, "unit": "hot-line operation sets/s",
                "frac": (hot_achieved / hot) if hot else None,
                "peak_source": "measured by tools/microbench on B200 (profiles/microbench_b200.json)"},
            "e2e": {"value": e2e_value, "unit": "updates/s", "h2d_bytes_per_step": h2d,
                    "d2h_bytes_per_step": 8, "f_host": f_host,
                    "how": "asaga_reload_async from pinned host arrays (copy stream, two device "
                           "buffers: step k+1's H2D overlaps step k), run, objective, D2H of f; "
                           "wall clock over the K steps, L2 flushed between steps"},
            # ours per step: ingest_init (not for d <= 1024: the ingest initialises itself),
            # ingest (for d <= 4096 its last block also runs the profile and the report; else
            # profile + report kernels, and A9's dense copy of x), update, margin (its last
            # block finishes f), + expand_d unless every feature is combined, the record layout
            # carries D or the kernel gathers it (d_gather), + hot_flag and
            # hot_slot when combining with d > 4096 (CUB's scan kernels are library)
            "gpu_launches": (4 - (1 if p.d <= 1024 else 0) + (0 if p.d <= 4096 else 3)
                             + (0 if (op["comb"] > 0 and st_timed["combine_hot"] == p.d) or st_timed["record_layout"]
                                or op.get("dgather", 0) else 1)
                             + (2 if op["comb"] > 0 and p.d > 4096 else 0)) * args.steps,
            "clocks": clk.summary(),
        }
        if op["comb"] == 0 and mb.get("gather_latency_cycles"):
            # W / L_min with L_min the sum of the measured floors of one
            # sample's dependent chain -- the gather round trip of its ceil(s/G) chunks
            # (tools/microbench, 32 lanes x k independent 16-B L2 loads; +150 cycles per chunk
            # past 4), the reduce + sigma phase (clock64, profiles/r01_update_kernel.md), and
            # the issue of its 2 s REDs (1.29 cycles per lane, B300_MICROARCH REDG spread)
            G = st["lanes_per_sample"]
            chunks = max(1, int(np.ceil(mean_s / G)))
            gl = mb["gather_latency_cycles"]
            gather = gl[f"chunks{min(chunks, 4)}"] + 150.0 * max(0, chunks - 4)
            reduce_sigma, red_issue = 500.0, 2.0 * mean_s * 1.29
            L_cyc = gather + reduce_sigma + red_issue
            mhz = clk.summary().get("sm_mhz") or 1965.0
            peak_lat = st["concurrency"] / (L_cyc / (mhz * 1e6))
            out["roofline_latency"] = {
                "bound": "per-sample dependent chain at the convergent number in flight (W / L_min)",
                "achieved": ups, "peak": peak_lat, "unit": "updates/s", "frac": ups / peak_lat,
                "L_min_cycles": {"gather_round_trip": gather, "reduce_sigma": reduce_sigma,
                                 "red_issue": red_issue, "total": L_cyc, "sm_mhz": mhz},
                "samples_in_flight": st["concurrency"],
                "source": "tools/microbench (profiles/microbench_b200.json), clock64 phases (profiles/r01_update_kernel.md)"}
        ceil = (load_json("profiles", "r02_ceilings.json") or {}).get(p.name)
        if maxtp is not None and op["comb"] == 0:
            # the update kernel against the saturated rate of its own access pattern: the best
            # rate over the samples in flight scanned in THIS run (max_throughput_point); the
            # profiling build's hot-operations-only rate is the context (r02_update_kernel.md)
            peak_sat = max(r["updates_per_s"] for r in maxtp["scan"])
            out["roofline_in_situ"] = {
                "bound": "L2 service of the kernel's own access pattern (popular x lines + cold traffic): "
                         "the best rate at any number in flight, this run",
                "achieved": ups, "peak": peak_sat, "unit": "updates/s", "frac": ups / peak_sat,
                "peak_at_samples_in_flight": max(maxtp["scan"], key=lambda r: r["updates_per_s"])["samples_in_flight"],
                "hot_ops_only_vs_full_timing_build": (ceil or {}).get("hot_only_max", 0) / ceil["full_max_any_W"]
                if ceil else None,
                "source": "max_throughput_point.scan (this run); profiles/r02_ceilings.json (profiling build)"}
        tr = load_json("profiles", "traffic.json") or {}
        if p.name in tr:
            # ncu cannot run inside the timed bench: the DRAM bytes of one launch of the same
            # kernel at the same operating point, from the committed ncu capture
            out["roofline"]["traffic"] = tr[p.name]
            out["roofline"]["traffic_source"] = ("stored: dram__bytes_read.sum + dram__bytes_write.sum of one "
                                                 "update launch (one epoch) from an ncu --set full capture "
                                                 "(profiles/traffic.json), not measured in this run")
        if not args.no_cpu_baseline and world == 1:  # (the contract: rank 0 at N = 1 only)
            out["cpu_baseline"] = cpu_baseline(p, lam, 1.0 / (3.0 * L), args.cpu_seconds)
        print(json.dumps(out))
    a.close()
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
