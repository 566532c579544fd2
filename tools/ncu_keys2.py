"""Key metrics + top source lines of an ncu report (raw + source pages)."""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
keys = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "smsp__inst_executed.sum",
        "sm__inst_executed.avg.per_cycle_active", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "launch__occupancy_limit_shared_mem", "launch__occupancy_limit_registers", "launch__grid_size",
        "lts__t_bytes.sum", "l1tex__t_bytes.sum", "launch__shared_mem_per_block_dynamic"]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, units = rows[0], rows[1]
for r in rows[2:]:
    name = r[hdr.index("Kernel Name")]
    print("==", name[:80])
    for k in keys:
        if k in hdr:
            print(f"   {k} = {r[hdr.index(k)]} {units[hdr.index(k)]}")
    st = [(h, r[i]) for i, h in enumerate(hdr) if h.startswith("smsp__average_warp_latency_issue_stalled") or h.startswith("smsp__pcsamp_warps_issue_stalled")]
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda"], capture_output=True, text=True).stdout
if src:
    rs = list(csv.reader(io.StringIO(src)))
    h = rs[0]
    def col(name):
        for i, x in enumerate(h):
            if x == name:
                return i
        return None
    ie = col("Instructions Executed") or col("Warp Instructions Executed")
    isamp = col("Warp Stall Sampling (All Samples)")
    isrc = col("Source")
    iline = col("#") or col("Line")
    data = []
    for r in rs[1:]:
        try:
            data.append((float(r[ie] or 0), float(r[isamp] or 0) if isamp is not None else 0.0, r[iline], r[isrc][:110]))
        except (ValueError, IndexError, TypeError):
            pass
    tot_e = sum(d[0] for d in data) or 1
    tot_s = sum(d[1] for d in data) or 1
    print(f"total executed {tot_e:.0f}, samples {tot_s:.0f}")
    print("-- by executed")
    for d in sorted(data, key=lambda d: -d[0])[:int(sys.argv[2]) if len(sys.argv) > 2 else 40]:
        print(f"{100 * d[0] / tot_e:5.1f}% {100 * d[1] / tot_s:5.1f}%  L{d[2]}  {d[3]}")
    print("-- by samples")
    for d in sorted(data, key=lambda d: -d[1])[:25]:
        print(f"{100 * d[0] / tot_e:5.1f}% {100 * d[1] / tot_s:5.1f}%  L{d[2]}  {d[3]}")
