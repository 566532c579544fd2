"""Write profiles/ncu_traffic.json from `ncu --set full` captures of one
25-frame chunk: DRAM bytes (read + write) of k_line + k_hard, the kernels of
bench.py's "line" scope (k_cand + k_line + k_hard).
Usage: make_traffic.py [--frames N] rep1.ncu-rep rep2.ncu-rep ..."""
import csv
import io
import json
import os
import subprocess
import sys

UNITS = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}


def dram(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h, u, v = rows[0], rows[1], rows[2]
    tot = 0.0
    for k in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
        i = h.index(k)
        tot += float(v[i].replace(",", "")) * UNITS[u[i]]
    return tot, v[h.index("Kernel Name")] if "Kernel Name" in h else "?"


args = sys.argv[1:]
frames = 207                                 # first chunk at the default 2 GiB
if args and args[0] == "--frames":
    frames = int(args[1])
    args = args[2:]
parts = [dram(r) for r in args]
H, W, V = 1080, 1920, 8
res = {"kernel": "line", "bytes_per_launch": sum(p[0] for p in parts),
       "alg_bytes_per_launch": frames * H * W * (4 + V),
       "parts": {p[1][:60]: p[0] for p in parts},
       "source": f"ncu --set full --clock-control none, one {frames}-frame C5 chunk (bench --steps 2 --warmup 3)"}
root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
with open(os.path.join(root, "profiles", "ncu_traffic.json"), "w") as f:
    json.dump(res, f, indent=1)
print(json.dumps(res))
