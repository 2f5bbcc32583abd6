"""NEXT-1: overlap tau-hat vs samples in flight on the GPU (the paper's App. D
"Overlap" figure, measured the same way: a sparse global counter
advanced every 100 iterations).  Prints one JSON object per W.

    python tools/overlap.py c3 --conc 1,16,64,256,1024 --gscale 0.35
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import datagen  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("cfg")
    ap.add_argument("--conc", default="1,16,64,256,1024,4096")
    ap.add_argument("--gscale", type=float, default=0.25)
    ap.add_argument("--epochs", type=float, default=2.0)
    ap.add_argument("--every", type=int, default=8)
    ap.add_argument("--bulk", type=float, default=0.0)
    ap.add_argument("--split", type=float, default=0.0, help="hot_split_min_freq")
    ap.add_argument("--repl", type=int, default=0, help="smem_replica_refresh")
    args = ap.parse_args()
    import torch
    from paper_1606_04809_b200 import Asaga

    p = datagen.make(args.cfg)
    dev = torch.device("cuda", 0)
    t = lambda a: torch.from_numpy(a).to(dev)
    A = (t(p.indptr), t(p.indices), t(p.data), t(p.y))
    for W in [int(c) for c in args.conc.split(",")]:
        a = Asaga(*A, p.d, p.lam, 1.0, concurrency=W, measure_overlap=args.every,
                  bulk_scatter_min_freq=args.bulk,
              hot_split_min_freq=args.split,
              smem_replica_refresh=args.repl)
        a.set_gamma(args.gscale / (3.0 * a.stats()["L"]))
        T = int(args.epochs * p.n)
        a.run(T, datagen.SAMPLE_SEED)
        st = a.stats()
        print(json.dumps({"cfg": args.cfg, "W": st["concurrency"], "overlap_mean": st["overlap_mean"],
                          "overlap_max": st["overlap_max"], "samples": st["overlap_samples"],
                          "updates_per_s": T / st["last_run_ms"] * 1e3}), flush=True)
        a.close()


if __name__ == "__main__":
    main()
