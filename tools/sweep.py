"""Operating-point sweep on the GPU: samples in flight (concurrency) x step-size scale.

For each (W, gamma scale) runs ASAGA from x = 0 with f evaluated every n/10
updates (reading R12, evaluation time excluded) until f - f* <= 1e-6 or the
epoch budget ends; reports epochs-to-1e-6, update-kernel updates/s and the
time-to-1e-6 (sum of update-kernel event times).  f* comes from the committed
oracle file tests/golden/fstar_<cfg>.json (written by scripts/compute_fstar.py).

    python tools/sweep.py c3 --conc 64,256,1024 --scales 1,0.5,0.25 --epochs 40
"""
import argparse
import itertools
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import datagen  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("cfg")
    ap.add_argument("--conc", default="64,128,256,512,1024,2048,4096,0")
    ap.add_argument("--scales", default="1,0.5,0.25,0.125")
    ap.add_argument("--epochs", type=float, default=40)
    ap.add_argument("--tol", type=float, default=1e-6)
    ap.add_argument("--out", default=None)
    ap.add_argument("--bulk", type=float, default=0.0, help="bulk_scatter_min_freq")
    ap.add_argument("--split", type=float, default=0.0, help="hot_split_min_freq")
    ap.add_argument("--repl", type=int, default=0, help="smem_replica_refresh")
    ap.add_argument("--comb", type=float, default=0.0, help="combine_min_freq")
    ap.add_argument("--cluster", type=int, default=0, help="combine_cluster")
    ap.add_argument("--lanes", type=int, default=0, help="lanes_per_sample")
    ap.add_argument("--wt", action="store_true", help="combine_write_through")
    ap.add_argument("--maxblocks", type=int, default=0, help="combine_max_blocks")
    ap.add_argument("--persist", action="store_true", help="l2_persist_state")
    ap.add_argument("--pipe", type=float, default=0.0, help="pipe_late_min_freq (pipelined kernel)")
    ap.add_argument("--merge", type=int, default=0, help="pipe_merge_ns")
    ap.add_argument("--rowcp", action="store_true", help="row_copy_elementwise")
    ap.add_argument("--overlap", type=int, default=0, help="measure_overlap (App. D counter every k-th sample)")
    ap.add_argument("--record", action="store_true", help="record_layout (D from the coordinate record)")
    ap.add_argument("--unpaired", action="store_true", help="scatter_unpaired (one reduction instruction per word)")
    ap.add_argument("--dgather", action="store_true", help="d_gather (D_c gathered per entry, no D stream)")
    ap.add_argument("--launch", type=float, default=0.1,
                    help="epochs per asaga_run launch (f checked between launches): 0.1, or 1 as bench.py's value")
    ap.add_argument("--seeds", type=int, default=1, help="sample streams per point (seed, seed+1, ...)")
    args = ap.parse_args()
    import torch
    from paper_1606_04809_b200 import Asaga

    gold = json.load(open(os.path.join(ROOT, "tests", "golden", f"fstar_{args.cfg}.json")))
    p = datagen.make(args.cfg)
    assert p.sha256() == gold["sha256"], "generated data differs from the f* file"
    fstar = gold["f_star"]
    dev = torch.device("cuda", 0)
    t = lambda a: torch.from_numpy(a).to(dev)
    A = (t(p.indptr), t(p.indices), t(p.data), t(p.y))
    base = Asaga(*A, p.d, p.lam, 1.0, bulk_scatter_min_freq=args.bulk,
              hot_split_min_freq=args.split,
              smem_replica_refresh=args.repl, combine_min_freq=args.comb,
              combine_cluster=args.cluster, lanes_per_sample=args.lanes,
              combine_write_through=args.wt, combine_max_blocks=args.maxblocks,
              l2_persist_state=args.persist, pipe_late_min_freq=args.pipe,
              pipe_merge_ns=args.merge, row_copy_elementwise=args.rowcp, record_layout=args.record,
              scatter_unpaired=args.unpaired, d_gather=args.dgather, measure_overlap=args.overlap)
    gamma0 = 1.0 / (3.0 * base.stats()["L"])
    results = []
    grid = itertools.product([int(c) for c in args.conc.split(",")],
                             [float(s) for s in args.scales.split(",")], range(args.seeds))
    for W, sc, sd in grid:
        if True:
            a = base
            a.reload(*A)
            a.set_concurrency(W)
            a.set_gamma(gamma0 * sc)
            stream = torch.cuda.ExternalStream(a.stream, device=dev)
            step = p.n // 10 if args.launch < 1 else p.n * int(args.launch)
            per = step / p.n
            upd_ms = 0.0
            ep = None
            fs = []
            a.set_state(np.zeros(p.d), np.zeros(p.n), np.zeros(p.d), 0)
            for j in range(1, int(args.epochs / per) + 1):
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(stream)
                a.run_async(step, datagen.SAMPLE_SEED + sd)
                e1.record(stream)
                f = a.objective()
                last_ms = e0.elapsed_time(e1)
                upd_ms += last_ms
                fs.append(f - fstar)
                if not np.isfinite(f) or f - fstar > 10:
                    ep = "diverged"
                    break
                if f - fstar <= args.tol:
                    ep = round(j * per, 6)
                    break
            st = a.stats()
            r = {"cfg": args.cfg, "W": st["concurrency"], "comb_H": st["combine_hot"], "cluster": st["combine_cluster"],
                 "blocks": st["combine_blocks"], "rec": st["record_layout"], "lanes": st["lanes_per_sample"], "gamma_scale": sc, "pipe": args.pipe, "unpaired": args.unpaired, "dgather": args.dgather, "merge": args.merge, "split": args.split, "seed_offset": sd, "launch_epochs": per, "epochs_to_tol": ep,
                 "updates_per_s": len(fs) * step / (upd_ms / 1e3), "time_to_tol_s": upd_ms / 1e3 if isinstance(ep, float) else None,
                 "oracle_epochs": gold["oracle_epochs_to_1e-6"], "subopt_last": fs[-1]}
            r["subopt"] = [float("%.3g" % f) for f in fs]
            if args.overlap:
                r["overlap_mean"], r["overlap_max"] = st["overlap_mean"], st["overlap_max"]
            if st["combine_passes"]:
                r["comm_pass_us"] = last_ms * 1e3 * st["combine_blocks"] / st["combine_passes"]
            results.append(r)
            print(json.dumps(r), flush=True)
    if args.out:
        json.dump(results, open(args.out, "w"), indent=1)


if __name__ == "__main__":
    main()
