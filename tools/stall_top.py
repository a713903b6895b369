"""Top SASS instructions by stall samples of one kernel in an ncu report, with stall reasons
and a few preceding instructions.  usage: python tools/stall_top.py rep.ncu-rep [N]"""
import csv
import subprocess
import sys

rep = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 10
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
r = list(csv.reader(out.splitlines()))
h = r[1]
rows = r[2:]
si = h.index("Warp Stall Sampling (All Samples)")
ie = h.index("Instructions Executed")
cols = [c for c in h if c.startswith("stall_") and "Not Issued" not in c]
tot = sum(int(x[si] or 0) for x in rows)
print("samples", tot, "instructions", sum(int(x[ie] or 0) for x in rows))
idx = {x[0]: i for i, x in enumerate(rows)}
for x in sorted(rows, key=lambda x: -int(x[si] or 0))[:n]:
    i = idx[x[0]]
    rs = {c[6:]: x[h.index(c)] for c in cols if x[h.index(c)] not in ("0", "")}
    print(x[0][-5:], x[1].strip()[:50], x[si], rs)
    for y in rows[max(0, i - 3):i]:
        print("      ", y[0][-5:], y[1].strip()[:60], y[ie])
