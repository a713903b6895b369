"""Summarise an ncu report: key metrics + top stalled SASS lines + opcode mix."""
import csv, subprocess, sys
from collections import Counter
rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True, text=True).stdout
r = list(csv.reader(out.splitlines()))
h = r[0]
want = {'Duration', 'DRAM Throughput', 'Achieved Occupancy', 'Theoretical Occupancy', 'Registers Per Thread',
        'Compute (SM) Throughput', 'Executed Ipc Active', 'Warp Cycles Per Issued Instruction', 'Grid Size', 'Block Size',
        'Issue Slots Busy', 'L1/TEX Hit Rate', 'Mem Busy', 'Max Bandwidth', 'L2 Hit Rate'}
seen = set()
for row in r[1:]:
    d = dict(zip(h, row))
    k = (d['Kernel Name'][:30], d['Metric Name'])
    if d['Metric Name'] in want and k not in seen:
        seen.add(k)
        print(k[0], d['Metric Name'], d['Metric Value'], d['Metric Unit'])
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
h = rows[1]
data, seen = [], set()
for r in rows[2:]:
    if len(r) == len(h) and r[0] not in seen:
        seen.add(r[0]); data.append(r)
ie = h.index('Instructions Executed'); ss = h.index('Warp Stall Sampling (All Samples)')
num = lambda x: int(x) if x.isdigit() else 0
tot = sum(num(r[ie]) for r in data); ts = sum(num(r[ss]) for r in data)
print('warp inst', tot, 'stall samples', ts)
c, cs = Counter(), Counter()
for r in data:
    t = r[1].strip().split()
    if not t: continue
    op = (t[1] if t[0].startswith('@') else t[0]).split('.')[0]
    c[op] += num(r[ie]); cs[op] += num(r[ss])
print('opcode mix (share of warp instructions / of stall samples):')
print('  ' + ', '.join(f'{op} {100*v/tot:.1f}%/{100*cs[op]/max(ts,1):.1f}%' for op, v in c.most_common(18)))
for r in sorted(data, key=lambda r: -num(r[ss]))[:top]:
    print(f'{num(r[ss]):7d} {num(r[ie]):10d}  {r[1].strip()[:95]}')
# basic-block groups: consecutive SASS lines with equal execution counts
groups, cur = [], None
for r in data:
    n, s = num(r[ie]), num(r[ss])
    if cur and cur[0] == n:
        cur[1] += 1; cur[2] += s
    else:
        cur = [n, 1, s, r[0]]; groups.append(cur)
agg = Counter(); aggs = Counter(); first = {}
for n, k, s, addr in groups:
    agg[n] += n * k; aggs[n] += s; first.setdefault(n, addr)
print('execution-count groups (count x instrs, share of instrs / stalls):')
for n, v in agg.most_common(8):
    print(f'  {n:9d} x {v // max(n,1):5d} = {100*v/tot:5.1f}% / {100*aggs[n]/max(ts,1):5.1f}%  first@{first[n]}')
