"""Aggregate warp-stall reasons (pc sampling) of the kernels in an ncu report.
usage: python tools/stall_reasons.py rep.ncu-rep"""
import csv
import subprocess
import sys

out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "raw", "--csv"], capture_output=True, text=True).stdout
r = list(csv.reader(out.splitlines()))
h = r[0]
for row in r[2:]:
    name = row[h.index("Kernel Name")]
    st = {}
    for k, x in zip(h, row):
        if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("not_issued"):
            try:
                v = float(x.replace(",", ""))
            except ValueError:
                continue
            if v > 0:
                st[k[len("smsp__pcsamp_warps_issue_stalled_"):]] = v
    tot = sum(st.values())
    print(name[:60], "samples", int(tot))
    for k, v in sorted(st.items(), key=lambda t: -t[1])[:10]:
        print(f"   {k:28s} {v / tot * 100:5.1f}%")
