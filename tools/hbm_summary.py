"""Summarise the HBM-bound kernels' ncu metric lists (tools/gpu_ncu_r2.sh): per kernel launches,
average duration, DRAM bytes per launch, achieved GB/s (DRAM bytes / duration) against the measured
HBM copy bandwidth, and the ncu DRAM-throughput percentage.  python tools/hbm_summary.py CSV..."""
import csv
import collections
import json
import os
import sys

PEAK = 6554.6  # GB/s, MEASURED_PEAKS.json hbm_gbs (copy test)
try:
    PEAK = json.load(open(os.path.join(os.path.dirname(__file__), "..", "MEASURED_PEAKS.json")))["hbm_gbs"]
except Exception:
    pass


def load(path):
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hi]
    ki, ii, mi, vi, ui = (h.index("Kernel Name"), h.index("ID"), h.index("Metric Name"),
                          h.index("Metric Value"), h.index("Metric Unit"))
    launches = collections.defaultdict(dict)
    for r in rows[hi + 1:]:
        if len(r) <= vi:
            continue
        v = float(r[vi].replace(",", ""))
        unit = r[ui]
        if unit in ("Kbyte", "KB"):
            v *= 1e3
        elif unit in ("Mbyte", "MB"):
            v *= 1e6
        elif unit in ("Gbyte", "GB"):
            v *= 1e9
        elif unit == "usecond":
            v *= 1e3
        elif unit == "msecond":
            v *= 1e6
        launches[(r[ii], r[ki].split("(")[0].replace("void ", ""))][r[mi]] = v
    return launches


def main():
    out = {}
    for path in sys.argv[1:]:
        agg = collections.defaultdict(lambda: [0, 0.0, 0.0, 0.0])
        for (_, name), m in load(path).items():
            a = agg[name]
            a[0] += 1
            a[1] += m.get("gpu__time_duration.sum", 0.0)  # ns
            a[2] += m.get("dram__bytes_read.sum", 0.0) + m.get("dram__bytes_write.sum", 0.0)
            a[3] += m.get("dram__throughput.avg.pct_of_peak_sustained_elapsed", 0.0)
        print(f"== {os.path.basename(path)}")
        print(f"{'kernel':28s} {'launches':>8s} {'avg us':>9s} {'MB/launch':>10s} {'GB/s':>8s} "
              f"{'frac':>6s} {'ncu dram%':>9s}")
        for name, (n, t, b, p) in sorted(agg.items(), key=lambda x: -x[1][1]):
            gbs = b / t if t else 0.0
            print(f"{name[:28]:28s} {n:8d} {t / n / 1e3:9.1f} {b / n / 1e6:10.2f} {gbs:8.0f} "
                  f"{gbs / PEAK:6.3f} {p / n:9.1f}")
            out[f"{os.path.basename(path)}:{name}"] = {
                "launches": n, "avg_us": t / n / 1e3, "dram_MB_per_launch": b / n / 1e6,
                "achieved_GBps": gbs, "peak_GBps": PEAK, "frac": gbs / PEAK,
                "ncu_dram_pct": p / n}
    if os.environ.get("HBM_JSON"):
        json.dump(out, open(os.environ["HBM_JSON"], "w"), indent=1)


if __name__ == "__main__":
    main()
