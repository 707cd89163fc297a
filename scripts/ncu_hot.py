"""Print the hottest SASS lines (warp-stall samples) of one kernel in an ncu report.

usage: python scripts/ncu_hot.py REP LAUNCH_INDEX [TOP]
"""
import csv, io, subprocess, sys

rep, idx = sys.argv[1], int(sys.argv[2])
top = int(sys.argv[3]) if len(sys.argv) > 3 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass",
                      "-s", str(idx), "-c", "1"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
print(rows[0][1][:150])
h, rows = rows[1], [r for r in rows[2:] if len(r) > 5]
iS = h.index("Warp Stall Sampling (All Samples)")
iE = h.index("Instructions Executed")
num = lambda s: int(s) if s.strip().isdigit() else 0
tot = sum(num(r[iS]) for r in rows)
te = sum(num(r[iE]) for r in rows)
print(f"stall samples {tot}, warp instructions {te}, sass lines {len(rows)}")
order = sorted(range(len(rows)), key=lambda i: -num(rows[i][iS]))[:top]
for i in sorted(order):
    r = rows[i]
    print(f"{i:5d} {num(r[iS]):6d} {num(r[iE]):8d}  {r[1].strip()[:100]}")
