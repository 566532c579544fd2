"""Source lines of an ncu report ranked by one stall reason's samples
(default stall_long_sb), with the SASS instructions that took them.
Usage: ncu_stall_lines.py report.ncu-rep [stall_column] [N]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
col = sys.argv[2] if len(sys.argv) > 2 else "stall_long_sb"
n = int(sys.argv[3]) if len(sys.argv) > 3 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
hdr, cur, res, sass = None, None, [], []
for r in csv.reader(io.StringIO(out)):
    if r and r[0] == "File Path":
        cur = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        ci = hdr.index(col)
        continue
    if hdr and len(r) > ci and r[0].isdigit():
        try:
            v = int(r[ci])
        except ValueError:
            continue
        if r[2] == "-":
            res.append((v, cur, int(r[0]), r[1].strip()[:100]))
        else:
            sass.append((v, cur, int(r[0]), r[3].strip()[:60]))
tot = sum(x[0] for x in res) or 1
print(f"{col}: {tot} samples")
for v, f, l, s in sorted(res, reverse=True)[:n]:
    print(f"{v / tot * 100:5.1f}%  {f}:{l}  {s}")
