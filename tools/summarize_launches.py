"""Summarise an ncu `--metrics gpu__time_duration.sum --csv` launch list: time per kernel and share.

Usage: python tools/summarize_launches.py launches.csv [--last-step-only]
ncu times are cold-cache and serialised: compare SHARES with the live CUDA-event profile of bench.py.
"""
import csv
import re
import sys
from collections import defaultdict


def main(path):
    rows = []
    with open(path) as fh:
        lines = [l for l in fh if l.startswith('"')]
    rd = csv.reader(lines)
    hdr = next(rd)
    ik = hdr.index("Kernel Name")
    iv = hdr.index("Metric Value")
    iu = hdr.index("Metric Unit")
    for r in rd:
        try:
            v = float(r[iv].replace(",", ""))
        except ValueError:
            continue
        unit = r[iu]
        scale = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3,
                 "msecond": 1e3, "s": 1e6, "second": 1e6}.get(unit, 1.0)
        name = re.sub(r"\(.*", "", r[ik]).replace("void ", "").strip()
        rows.append((name, v * scale))
    agg = defaultdict(lambda: [0, 0.0])
    for n, us in rows:
        agg[n][0] += 1
        agg[n][1] += us
    tot = sum(a[1] for a in agg.values())
    print(f"{'kernel':50s} {'launches':>9s} {'total_ms':>10s} {'share':>7s} {'avg_us':>9s}")
    for n, (c, us) in sorted(agg.items(), key=lambda x: -x[1][1]):
        print(f"{n[:50]:50s} {c:9d} {us / 1e3:10.2f} {us / tot:7.3f} {us / c:9.1f}")
    print(f"{'TOTAL':50s} {len(rows):9d} {tot / 1e3:10.2f}")


if __name__ == "__main__":
    main(sys.argv[1])
