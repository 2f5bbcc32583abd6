"""Summarise an ncu --set full report's source page: top stalled SASS lines with
their dominant stall reasons (used to write profiles/*.md).

    python tools/ncu_stalls.py gpurun_out/prof.ncu-rep [--top 15] [--context 0]
"""
import csv
import io
import subprocess
import sys


def main():
    path = sys.argv[1]
    top = int(sys.argv[sys.argv.index("--top") + 1]) if "--top" in sys.argv else 15
    ctx = int(sys.argv[sys.argv.index("--context") + 1]) if "--context" in sys.argv else 0
    out = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv", "--print-source=sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, data = rows[1], rows[2:]
    isrc = hdr.index("Source")
    iall = hdr.index("Warp Stall Sampling (All Samples)")
    reasons = [(j, h) for j, h in enumerate(hdr) if h.startswith("stall_") and "(Not Issued)" not in h]
    num = lambda v: float(v) if v.replace(".", "", 1).isdigit() else 0.0
    tot = sum(num(r[iall]) for r in data) or 1.0
    agg = {}
    for r in data:
        for j, h in reasons:
            agg[h] = agg.get(h, 0.0) + num(r[j])
    print("kernel-wide stall samples:", ", ".join(f"{h[6:]} {v / tot * 100:.1f}%"
                                               for h, v in sorted(agg.items(), key=lambda x: -x[1])[:8]))
    order = sorted(range(len(data)), key=lambda j: -num(data[j][iall]))[:top]
    for j in order:
        r = data[j]
        rs = sorted(((num(r[k]), h[6:]) for k, h in reasons), reverse=True)[:2]
        print(f"{num(r[iall]) / tot * 100:5.1f}%  {r[0][-5:]}  {r[isrc].strip()[:70]:70s}  "
              + " ".join(f"{h}={v / max(num(r[iall]), 1) * 100:.0f}%" for v, h in rs if v > 0))
        for k in range(max(0, j - ctx), j):
            print(f"            {data[k][0][-5:]}  {data[k][isrc].strip()[:70]}")


if __name__ == "__main__":
    main()
