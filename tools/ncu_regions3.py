"""Instruction and stall-sample shares of k_sweep by source region, from
`ncu -i rep --page source --csv --print-source cuda,sass` output.  Regions
are found in the current csrc/k_sweep.cu: one per __device__ / __global__
function, and sweep_unit split at its pass markers.
Usage: ncu_regions3.py src.csv [N top lines]"""
import collections
import csv
import os
import re
import sys

SRC = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                   "paper_2408_14050_b200", "csrc", "k_sweep.cu")
lines = open(SRC).read().split("\n")
marks = []
for i, l in enumerate(lines, 1):
    m = re.match(r"^(?:template <[^>]*>\s*)?__(?:device|global)__.*?\b(\w+)\(", l)
    if m and not l.rstrip().endswith(";"):
        marks.append((i, m.group(1)))
    for key, name in (("// ------------------------------------------------ pass 1", "sweep_unit: pass 1"),
                      ("// ------------------------------------------------ pass 2", "sweep_unit: pass 2 words"),
                      ("// warm-up: far filter of +b only", "sweep_unit: pass 2 warm-up"),
                      ("// tails for the pairs reaching below the block", "sweep_unit: pass 2 block masks"),
                      ("            if (__any_sync(FULL, (sP | sN) != 0u)) {", "sweep_unit: survivors + stores")):
        if l.strip().startswith(key.strip()):
            marks.append((i, name))
marks.sort()


def region(ln):
    name = "header"
    for i, n in marks:
        if i <= ln:
            name = n
    return name


rows = list(csv.reader(open(sys.argv[1])))
cur, res = None, []
for r in rows:
    if r and r[0] == "File Path":
        cur = r[1].split("/")[-1]
    if len(r) > 8 and r[0].isdigit() and r[2] == "-":
        res.append((cur, int(r[0]), int(r[7]), int(r[4]), r[1][:90]))
te = sum(x[2] for x in res) or 1
ts = sum(x[3] for x in res) or 1
agg, smp = collections.Counter(), collections.Counter()
for f, l, e, s, src in res:
    k = region(l) if f == "k_sweep.cu" else f
    agg[k] += e
    smp[k] += s
print(f"total warp instructions {te}, stall samples {ts}")
for k, v in agg.most_common():
    print(f"{k:36s} {v / te * 100:5.1f}% instr {smp[k] / ts * 100:5.1f}% samples")
n = int(sys.argv[2]) if len(sys.argv) > 2 else 30
print("--- top lines by instructions")
for f, l, e, s, src in sorted(res, key=lambda x: -x[2])[:n]:
    print(f"{e / te * 100:5.1f}% {s / ts * 100:5.1f}% {f}:{l} {src}")
