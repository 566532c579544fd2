"""Summarise an ncu report by source line: stall samples and executed
instructions per line (needs -lineinfo).  Usage: ncu_lines.py report.ncu-rep [N]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
res, cur = [], None
for r in rows:
    if r and r[0] == "File Path":
        cur = r[1].split("/")[-1]
    if len(r) > 8 and r[0].isdigit() and r[2] == "-":
        try:
            res.append((int(r[4]), int(r[7]), cur, int(r[0]), r[1][:100]))
        except ValueError:
            pass
ts = sum(x[0] for x in res) or 1
te = sum(x[1] for x in res) or 1
print(f"total stall samples {ts}, executed warp instructions {te}")
print("-- by samples")
for s, e, f, l, src in sorted(res, reverse=True)[:n]:
    print(f"{s / ts * 100:5.1f}% {e / te * 100:5.1f}%  {f}:{l}  {src}")
print("-- by executed")
for s, e, f, l, src in sorted(res, key=lambda x: -x[1])[:n]:
    print(f"{s / ts * 100:5.1f}% {e / te * 100:5.1f}%  {f}:{l}  {src}")
