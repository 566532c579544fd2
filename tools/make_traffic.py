"""Write profiles/ncu_traffic.json from `ncu --set full` captures of one
frame chunk: DRAM bytes (read + write) of the dominant kernel of bench.py's
roofline ("line" = k_sweep), with the other kernels of the chunk listed
beside it (k_words, k_hard).
Usage: make_traffic.py --frames N sweep.ncu-rep [words.ncu-rep hard.ncu-rep ...]"""
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
frames = 128
if args and args[0] == "--frames":
    frames = int(args[1])
    args = args[2:]
parts = [dram(r) for r in args]
H, W, V = 1080, 1920, 8
alg = frames * H * W * (4 + V)
res = {"kernel": "line", "bytes_per_launch": parts[0][0], "alg_bytes_per_launch": alg,
       "ratio": parts[0][0] / alg,
       "parts": {p[1][:60]: p[0] for p in parts},
       "source": f"ncu --set full --clock-control none, one {frames}-frame C5 chunk "
                 f"(bench --steps 2 --warmup 3, main step only)"}
root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
with open(os.path.join(root, "profiles", "ncu_traffic.json"), "w") as f:
    json.dump(res, f, indent=1)
print(json.dumps(res))
