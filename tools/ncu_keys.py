"""Key metrics of ncu reports (one launch each): time, DRAM bytes, IPC,
warps active, issue active, top stall reasons.  Usage: ncu_keys.py rep..."""
import csv
import io
import subprocess
import sys

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "sm__inst_executed.avg.per_cycle_active", "smsp__inst_executed.sum",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "launch__registers_per_thread", "launch__grid_size", "launch__block_size"]
for rep in sys.argv[1:]:
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h, u, v = rows[0], rows[1], rows[2]
    print(f"== {rep}: {v[h.index('Kernel Name')][:70]}")
    for k in KEYS:
        if k in h:
            print(f"   {k} = {v[h.index(k)]} {u[h.index(k)]}")
    st = []
    for i, k in enumerate(h):
        if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("not_issued"):
            try:
                st.append((float(v[i].replace(",", "")), k.replace("smsp__pcsamp_warps_issue_stalled_", "")))
            except ValueError:
                pass
    tot = sum(x for x, _ in st) or 1
    print("   stalls: " + ", ".join(f"{n} {x / tot * 100:.0f}%" for x, n in sorted(st, reverse=True)[:6]))
