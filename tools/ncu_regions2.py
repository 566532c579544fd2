"""Executed warp instructions and stall samples of an ncu report summed over
named line ranges of one source file.  Usage: ncu_regions2.py rep file a-b:name ..."""
import csv
import io
import subprocess
import sys

rep, fname = sys.argv[1], sys.argv[2]
ranges = []
for spec in sys.argv[3:]:
    ab, name = spec.split(":")
    a, b = ab.split("-")
    ranges.append((int(a), int(b), name))
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
cur = None
acc = {n: [0, 0] for _, _, n in ranges}
other = [0, 0]
tot = [0, 0]
for r in rows:
    if r and r[0] == "File Path":
        cur = r[1].split("/")[-1]
    if len(r) > 8 and r[0].isdigit() and r[2] == "-":
        try:
            s, e, ln = int(r[4]), int(r[7]), int(r[0])
        except ValueError:
            continue
        tot[0] += s; tot[1] += e
        if cur != fname:
            other[0] += s; other[1] += e
            continue
        for a, b, n in ranges:
            if a <= ln <= b:
                acc[n][0] += s; acc[n][1] += e
                break
        else:
            other[0] += s; other[1] += e
print(f"total samples {tot[0]}, executed {tot[1]}")
for n, (s, e) in acc.items():
    print(f"{n:20s} exec {e:12d} ({100 * e / max(1, tot[1]):5.1f}%)  samples {100 * s / max(1, tot[0]):5.1f}%")
print(f"{'other':20s} exec {other[1]:12d} ({100 * other[1] / max(1, tot[1]):5.1f}%)  samples {100 * other[0] / max(1, tot[0]):5.1f}%")
