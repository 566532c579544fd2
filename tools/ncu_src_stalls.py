"""Per-source-line stall breakdown from `ncu -i rep --page source --csv
--print-source cuda,sass` output: the lines with the most long-scoreboard,
wait, short-scoreboard and no-instruction samples.  Usage: ncu_src_stalls.py src.csv [N]"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
n = int(sys.argv[2]) if len(sys.argv) > 2 else 12
hdr = next(r for r in rows if r and r[0] == "Line No")
col = {h: i for i, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h}
cur, res = None, []
for r in rows:
    if r and r[0] == "File Path":
        cur = r[1].split("/")[-1]
    if len(r) > 40 and r[0].isdigit() and r[2] == "-":
        res.append((cur, int(r[0]), r[1][:80], {k: int(r[i] or 0) for k, i in col.items()}))
tot = {k: sum(x[3][k] for x in res) for k in col}
allt = sum(tot.values())
print("totals:", ", ".join(f"{k[6:]} {v / allt * 100:.1f}%" for k, v in sorted(tot.items(), key=lambda kv: -kv[1]) if v))
for k in ["stall_long_sb", "stall_wait", "stall_short_sb", "stall_no_inst", "stall_branch_resolving", "stall_lg"]:
    print(f"-- {k} ({tot[k] / allt * 100:.1f}% of all samples)")
    for f, l, src, d in sorted(res, key=lambda x: -x[3][k])[:n]:
        if d[k]:
            print(f"  {d[k] / allt * 100:5.2f}%  {f}:{l}  {src}")
