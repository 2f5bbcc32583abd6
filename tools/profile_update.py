"""Drive the update kernel for ncu: one warm-up launch, then one measured launch.

    ncu --set full -k regex:asaga_(update|combine) -s 1 -c 1 python tools/profile_update.py c3 --conc 512
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import datagen  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("cfg")
    ap.add_argument("--conc", type=int, default=0)
    ap.add_argument("--gscale", type=float, default=0.25)
    ap.add_argument("--updates", type=int, default=0, help="default: one epoch")
    ap.add_argument("--bulk", type=float, default=0.0, help="bulk_scatter_min_freq")
    ap.add_argument("--split", type=float, default=0.0, help="hot_split_min_freq")
    ap.add_argument("--repl", type=int, default=0, help="smem_replica_refresh")
    ap.add_argument("--comb", type=float, default=0.0, help="combine_min_freq")
    ap.add_argument("--pipe", type=float, default=0.0, help="pipe_late_min_freq")
    ap.add_argument("--rowcp", action="store_true", help="row_copy_elementwise")
    ap.add_argument("--unpaired", action="store_true", help="scatter_unpaired")
    ap.add_argument("--record", action="store_true", help="record_layout")
    ap.add_argument("--dgather", action="store_true", help="d_gather")
    args = ap.parse_args()
    import torch
    from paper_1606_04809_b200 import Asaga

    p = datagen.make(args.cfg)
    dev = torch.device("cuda", 0)
    t = lambda a: torch.from_numpy(a).to(dev)
    a = Asaga(t(p.indptr), t(p.indices), t(p.data), t(p.y), p.d, p.lam, 1.0, concurrency=args.conc,
              bulk_scatter_min_freq=args.bulk,
              hot_split_min_freq=args.split,
              smem_replica_refresh=args.repl, combine_min_freq=args.comb,
              pipe_late_min_freq=args.pipe, row_copy_elementwise=args.rowcp,
              scatter_unpaired=args.unpaired, record_layout=args.record, d_gather=args.dgather)
    a.set_gamma(args.gscale / (3.0 * a.stats()["L"]))
    T = args.updates or p.n
    a.run(T, datagen.SAMPLE_SEED)  # warm-up launch
    a.run(T, datagen.SAMPLE_SEED)  # profiled launch
    st = a.stats()
    print(f"{args.cfg} W={st['concurrency']} updates={T} ms={st['last_run_ms']:.3f} "
          f"upd/s={T / st['last_run_ms'] * 1e3:.4g}")


if __name__ == "__main__":
    main()
