"""Time A0-A1 (asaga_reload_device_async: ingest + column pass + expand) on full-size data.

Each repetition: write+read 512 MiB (cold L2, outside the events), then one asynchronous
device reload bracketed by CUDA events on the context's stream.  Prints one JSON line per
configuration: mean / min ms and the matrix bytes streamed / mean time.  ASAGA_LIB selects
a measurement build (e.g. the blocking rows loop, -DASAGA_INGEST_ROWS_BLOCKING).

    python tools/ingest_time.py c4 --reps 10
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
    ap.add_argument("--reps", type=int, default=10)
    ap.add_argument("--split", type=float, default=0.3)
    args = ap.parse_args()
    import torch
    from paper_1606_04809_b200 import Asaga

    p = datagen.make(args.cfg)
    dev = torch.device("cuda", 0)
    A = tuple(torch.from_numpy(a).to(dev) for a in (p.indptr, p.indices, p.data, p.y))
    a = Asaga(*A, p.d, p.lam, 1.0, hot_split_min_freq=args.split)
    stream = torch.cuda.ExternalStream(a.stream, device=dev)
    flush = torch.empty(512 << 20, dtype=torch.uint8, device=dev)
    ts = []
    for r in range(args.reps + 2):
        flush.fill_(r & 255)
        flush.sum()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        a.reload_async(*A)
        e1.record(stream)
        a.objective()  # a blocking call resolves the reload's validation
        torch.cuda.synchronize()
        if r >= 2:
            ts.append(e0.elapsed_time(e1))
    nbytes = p.indices.nbytes + p.data.nbytes + p.indptr.nbytes + p.y.nbytes
    mean = sum(ts) / len(ts)
    print(json.dumps({"cfg": args.cfg, "lib": os.path.basename(os.environ.get("ASAGA_LIB", "libasaga.so")),
                      "mean_ms": mean, "min_ms": min(ts), "matrix_bytes": nbytes,
                      "matrix_GBps_at_mean": nbytes / mean / 1e6}), flush=True)
    a.close()


if __name__ == "__main__":
    main()
