"""Group an ncu source report's executed instructions / stall samples into
regions delimited by '// ---' markers or function starts in the sources."""
import csv, io, re, subprocess, sys
from collections import defaultdict
rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
res, cur, path = [], None, {}
for r in rows:
    if r and r[0] == "File Path":
        cur = r[1]
    if len(r) > 8 and r[0].isdigit() and r[2] == "-":
        try:
            res.append((cur, int(r[0]), int(r[4]), int(r[7])))
        except ValueError:
            pass
marks = {}
for f in set(x[0] for x in res):
    try:
        src = open(f).read().split("\n")
    except OSError:
        continue
    m = []
    for i, line in enumerate(src, 1):
        if re.search(r"//\s*-{3,}|__global__|__device__ __forceinline__|^template|// [a-e]\. ", line):
            m.append((i, line.strip()[:60]))
    marks[f] = m
def region(f, l):
    best = (0, f.split("/")[-1])
    for i, name in marks.get(f, []):
        if i <= l:
            best = (i, name)
    return f.split("/")[-1] + ":" + str(best[0]) + " " + best[1]
ts = sum(x[2] for x in res) or 1
te = sum(x[3] for x in res) or 1
g = defaultdict(lambda: [0, 0])
for f, l, s, e in res:
    k = region(f, l)
    g[k][0] += s
    g[k][1] += e
for k, (s, e) in sorted(g.items(), key=lambda kv: -kv[1][1]):
    print(f"exec {e / te * 100:5.1f}%  stall {s / ts * 100:5.1f}%  {k}")
