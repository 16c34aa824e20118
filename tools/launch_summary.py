"""Sum ncu launch-list times per kernel name: python tools/launch_summary.py launches.csv"""
import collections
import csv
import sys

rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
hdr = rows[0]
ik, iv = hdr.index("Kernel Name"), hdr.index("Metric Value")
tot = collections.defaultdict(float)
cnt = collections.Counter()
for r in rows[1:]:
    if r[hdr.index("Metric Name")] != "gpu__time_duration.sum":
        continue
    name = r[ik].split("(")[0]
    tot[name] += float(r[iv].replace(",", "")) / 1e3
    cnt[name] += 1
T = sum(tot.values())
for k, v in sorted(tot.items(), key=lambda x: -x[1]):
    print(f"{v:10.1f} us {100 * v / T:5.1f}% {cnt[k]:5d} x {v / cnt[k]:8.1f} us  {k}")
print(f"{T:10.1f} us total")
