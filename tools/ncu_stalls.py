"""Per-kernel warp-stall breakdown (pc sampling) of an ncu report."""
import csv
import subprocess
import sys

out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
h = rows[0]
for r in rows[2:]:
    name = r[h.index("Kernel Name")][:40]
    vals = []
    for i, k in enumerate(h):
        if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("not_issued"):
            try:
                vals.append((float(r[i]), k.replace("smsp__pcsamp_warps_issue_stalled_", "")))
            except ValueError:
                pass
    tot = sum(v for v, _ in vals) or 1
    print(name, " ".join(f"{k}={100 * v / tot:.0f}%" for v, k in sorted(vals, reverse=True)[:9]))
