"""Per-source-line SASS instruction counts of one kernel: joins an ncu report's per-instruction
"Instructions Executed" (source page, SASS view) with the line table nvdisasm reads from the
library's cubin (-lineinfo build).  The cubin must be the one the report was captured from.

    python tools/sass_lines.py <report.ncu-rep> <kernel-substring> [--per N] [--top K] [--ops]

--per N divides every count by N/32 (N = points or symbols per launch) to print warp
instructions per unit of work; --ops adds the opcode mix of the kernel.
"""
from __future__ import annotations

import argparse
import collections
import csv
import os
import re
import subprocess
import sys
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = os.path.join(ROOT, "paper_2010_03144_b200", "lib", "libftlz_b200.so")


def sass_table(func_sub: str):
    d = tempfile.mkdtemp()
    subprocess.run(["cuobjdump", "-xelf", "all", LIB], cwd=d, capture_output=True, check=True)
    cub = [f for f in os.listdir(d) if f.endswith(".cubin")][0]
    txt = subprocess.run(["nvdisasm", "-g", "-c", os.path.join(d, cub)], capture_output=True, text=True).stdout
    out, cur, line, name = {}, None, None, None
    for ln in txt.splitlines():
        m = re.match(r"^\.text\.(\S+):", ln)
        if m:
            name = m.group(1)
            cur = out.setdefault(name, {}) if func_sub in name else None
            continue
        if cur is None:
            continue
        m = re.match(r'\s*//## File "(.*)", line (\d+)', ln)
        if m:
            line = f"{os.path.basename(m.group(1))}:{m.group(2)}"
            continue
        m = re.match(r"\s*/\*([0-9a-f]{4,})\*/\s+(.*?);", ln)
        if m:
            cur[int(m.group(1), 16)] = (line, m.group(2).strip())
    return out


def ncu_counts(rep: str, kname: str):
    txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass",
                          "--kernel-name", kname], capture_output=True, text=True).stdout
    rows = list(csv.reader(txt.splitlines()))
    hdr = next(i for i, r in enumerate(rows) if r and r[0] == "Address")
    h = rows[hdr]
    ie, ss = h.index("Instructions Executed"), h.index("Warp Stall Sampling (All Samples)")
    res, seen = [], set()
    for r in rows[hdr + 1:]:
        if len(r) < len(h) or not r[0].startswith("0x"):
            if res:
                break   # first launch only
            continue
        a = int(r[0], 16)
        if a in seen:
            break
        seen.add(a)
        num = lambda x: int(x) if x.isdigit() else 0
        res.append((a, r[1].strip(), num(r[ie]), num(r[ss])))
    return res


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("rep")
    ap.add_argument("kernel")
    ap.add_argument("--per", type=float, default=0)
    ap.add_argument("--top", type=int, default=40)
    ap.add_argument("--ops", action="store_true")
    ap.add_argument("--dump", default=None, help="file:line[-line] -> print its SASS with counts")
    a = ap.parse_args()
    counts = ncu_counts(a.rep, a.kernel)
    base = counts[0][0]
    tabs = sass_table(a.kernel)
    # choose the function whose opcode sequence matches the report
    best, bscore = None, -1
    for name, t in tabs.items():
        sc = sum(1 for (addr, op, _, _) in counts[:200] if addr - base in t and t[addr - base][1].split()[0] == op.split()[0])
        if sc > bscore:
            best, bscore = name, sc
    t = tabs[best]
    scale = a.per / 32.0 if a.per else 1.0
    per_line, per_line_st, ops = collections.Counter(), collections.Counter(), collections.Counter()
    tot = st = 0
    for addr, op, n, s in counts:
        line = t.get(addr - base, ("?", op))[0] or "?"
        per_line[line] += n
        per_line_st[line] += s
        ops[op.split()[0].split(".")[0] if not op.startswith("@") else op.split()[1].split(".")[0]] += n
        tot += n
        st += s
    print(f"{best}: {tot} warp instructions" + (f" = {tot / scale:.1f} per unit" if a.per else "") +
          f", {st} stall samples (match {bscore}/200)")
    for line, n in per_line.most_common(a.top):
        print(f"  {line:28s} {n / scale:10.2f} {100.0 * n / tot:5.1f}%  stall {100.0 * per_line_st[line] / max(1, st):5.1f}%")
    if a.dump:
        f, rng = a.dump.split(":")
        lo, hi = (int(x) for x in (rng.split("-") if "-" in rng else (rng, rng)))
        for addr, op, n, st in counts:
            line = t.get(addr - base, ("?", op))[0] or "?"
            if line.startswith(f + ":") and lo <= int(line.split(":")[1]) <= hi:
                print(f"  {addr - base:6x} {line:22s} {n / scale:8.3f}  {t.get(addr - base, (0, op))[1]}")
    if a.ops:
        print("opcode mix:")
        for op, n in ops.most_common(30):
            print(f"  {op:10s} {n / scale:10.2f} {100.0 * n / tot:5.1f}%")


if __name__ == "__main__":
    sys.exit(main())
