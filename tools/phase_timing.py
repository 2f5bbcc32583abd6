"""Per-phase cycle breakdown of the update kernel (clock64-instrumented build).

    python tools/phase_timing.py c3 --conc 64,512
Phases per sample (group leaders): row wait | gathers+dot | reduce+exp | scatter issue | tail.
"""
import argparse
import ctypes
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("cfg")
    ap.add_argument("--conc", default="64,512")
    ap.add_argument("--gscale", type=float, default=0.25)
    ap.add_argument("--atomic", type=int, default=1)
    ap.add_argument("--lanes", type=int, default=0)
    ap.add_argument("--bulk", type=float, default=0.0, help="bulk_scatter_min_freq")
    ap.add_argument("--split", type=float, default=0.0, help="hot_split_min_freq")
    ap.add_argument("--repl", type=int, default=0, help="smem_replica_refresh")
    ap.add_argument("--pipe", type=float, default=0.0, help="pipe_late_min_freq")
    ap.add_argument("--merge", type=int, default=0, help="pipe_merge_ns")
    ap.add_argument("--dgather", action="store_true", help="d_gather")
    ap.add_argument("--record", action="store_true", help="record_layout")
    args = ap.parse_args()
    import importlib.util

    spec = importlib.util.spec_from_file_location(
        "_asaga_build", os.path.join(ROOT, "paper_1606_04809_b200", "_build.py"))
    _build = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(_build)
    os.environ["ASAGA_LIB"] = _build.build(timing=True)  # before the package loads its .so
    import torch

    import datagen
    from paper_1606_04809_b200 import Asaga, asaga

    lib = asaga.lib()
    lib.asaga_debug_timing.restype = ctypes.c_int
    lib.asaga_debug_timing.argtypes = [ctypes.POINTER(ctypes.c_ulonglong)]
    p = datagen.make(args.cfg)
    dev = torch.device("cuda", 0)
    t = lambda a: torch.from_numpy(a).to(dev)
    a = Asaga(t(p.indptr), t(p.indices), t(p.data), t(p.y), p.d, p.lam, 1.0,
              atomic=bool(args.atomic), lanes_per_sample=args.lanes,
              bulk_scatter_min_freq=args.bulk,
              hot_split_min_freq=args.split,
              smem_replica_refresh=args.repl, pipe_late_min_freq=args.pipe,
              pipe_merge_ns=args.merge, d_gather=args.dgather, record_layout=args.record)
    a.set_gamma(args.gscale / (3.0 * a.stats()["L"]))
    buf = (ctypes.c_ulonglong * 9)()
    names = ["row_wait", "gather_dot", "reduce_exp", "scatter", "tail", "-", "s_wait_read", "s_compute",
             "s_fence"]
    if args.pipe > 0:  # asaga_pipe_kernel's phases (asaga_pipe.cuh)
        names = ["hot_gather_issue", "cold_scatter_prev", "wait_copy", "dot_wait", "reduce_sigma", "-",
                 "hot_scatter", "merge_dstore_cold_gather", "wait_dload"]
    for W in [int(c) for c in args.conc.split(",")]:
        a.set_concurrency(W)
        a.run(p.n, 1)
        lib.asaga_debug_timing(buf)
        a.run(p.n, 1)
        lib.asaga_debug_timing(buf)
        it = max(buf[5], 1)
        st = a.stats()
        cyc = [buf[k] / it for k in range(9)]
        # plain kernel: phases 6-8 split the scatter phase [3] (their sum is <= it: marks inside
        # it); pipelined kernel: every phase but [5] (the iteration count) is disjoint
        total = sum(c for k, c in enumerate(cyc) if k != 5) if args.pipe > 0 else sum(cyc[:5])
        print(f"{args.cfg} G={st['lanes_per_sample']} bulk={args.bulk} split={args.split} repl={args.repl} "
              f"pipe={args.pipe} W={st['concurrency']} "
              f"upd/s={p.n / st['last_run_ms'] * 1e3:.4g} cycles/sample total={total:.0f}: "
              + " ".join(f"{n}={c:.0f}" for n, c in zip(names, cyc) if n != "-"))


if __name__ == "__main__":
    main()
