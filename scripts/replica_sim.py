"""NEXT-3 decided by simulation: multi-GPU ASAGA with periodic exchange.

The oracle's replicated model (oracle.replica_saga; Section 5: "limiting
communications can be interpreted as artificially increasing the delay"): N replicas of
(x, abar), update t on replica t mod N, each replica's own updates visible to it at once,
every copy synchronised every E = N * K global updates (K = updates per replica between
exchanges).  From x = 0, f checked every n/10 updates (reading R12) against the golden f*,
epochs to f - f* <= 1e-6 at gamma = 1/(3L); the 1.5x budget is against the oracle's own
epochs (tests/golden/fstar_<cfg>.json).  Calls only oracle/ (test infrastructure; this is an
offline study script, not the product path).

    python scripts/replica_sim.py --cfg c2,c3 --N 2,4,8 --K 1,64,1024,8192 --jobs 8 [--gscale 1,0.3]
(appends to profiles/r02_replica_sim.jsonl)
"""
import argparse
import itertools
import json
import multiprocessing as mp
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def run_one(args):
    cfg, N, K, max_epochs, gscale = args
    import datagen
    import oracle

    gold = json.load(open(os.path.join(ROOT, "tests", "golden", f"fstar_{cfg}.json")))
    p = datagen.make(cfg)
    assert p.sha256() == gold["sha256"]
    g = gscale / (3.0 * oracle.lipschitz(p, p.lam))
    D = oracle.reweight(p.n, oracle.column_counts(p))
    st = oracle.State(p.n, p.d)
    step = p.n // 10
    E = N * K
    ep = None
    t0 = time.time()
    for j in range(1, 10 * max_epochs + 1):
        # whole exchange windows only straddle checkpoints when E > step: the model exchanges
        # at the end of every call too, so calls of `step` updates add exchanges; use calls
        # that are a multiple of E when E divides n/10, else accept the extra exchange
        oracle.replica_saga(p, p.y, p.lam, g, datagen.SAMPLE_SEED, step, N, E, st, D)
        f = oracle.objective(p, p.y, p.lam, st.x)
        if f - gold["f_star"] <= 1e-6:
            ep = j / 10
            break
        if not np.isfinite(f):
            break
    return {"cfg": cfg, "N": N, "K": K, "E": E, "gamma_scale": gscale, "epochs_to_1e-6": ep,
            "oracle_epochs": gold["oracle_epochs_to_1e-6"],
            "within_1p5x": ep is not None and ep <= 1.5 * gold["oracle_epochs_to_1e-6"],
            "extra_exchange_per_check": E > step, "seconds": time.time() - t0}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--cfg", default="c2,c3")
    ap.add_argument("--N", default="2,4,8")
    ap.add_argument("--K", default="1,64,1024,16384")
    ap.add_argument("--max-epochs", type=int, default=30)
    ap.add_argument("--jobs", type=int, default=os.cpu_count())
    ap.add_argument("--gscale", default="1", help="gamma scales vs 1/(3L) (the GPU operating points: "
                                                   "c2 0.04, c3 0.3, c4 0.25)")
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "r02_replica_sim.jsonl"))
    a = ap.parse_args()
    grid = [(c, int(n), int(k), a.max_epochs, float(gs)) for c, n, k, gs in
            itertools.product(a.cfg.split(","), a.N.split(","), a.K.split(","), a.gscale.split(","))]
    with mp.get_context("spawn").Pool(a.jobs) as pool, open(a.out, "a") as f:
        for r in pool.imap_unordered(run_one, grid):
            print(json.dumps(r), flush=True)
            f.write(json.dumps(r) + "\n")


if __name__ == "__main__":
    main()
