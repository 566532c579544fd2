"""Per-kernel share of an ncu launch list (--metrics gpu__time_duration.sum --csv).
Usage: launch_shares.py launches.csv"""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hi = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
h = rows[hi]
ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
SCALE = {"ns": 1e-6, "nsecond": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0}
tot, n = collections.defaultdict(float), collections.Counter()
for r in rows[hi + 1:]:
    if len(r) <= vi:
        continue
    name = r[ki].split("(")[0].replace("void ", "")
    tot[name] += float(r[vi].replace(",", "")) * SCALE[r[ui]]
    n[name] += 1
T = sum(tot.values())
for k, v in sorted(tot.items(), key=lambda x: -x[1]):
    print(f"{k:32s} {n[k]:5d} launches {v:10.3f} ms {v / T * 100:5.1f}%")
print(f"total {T:.3f} ms, {sum(n.values())} launches")
