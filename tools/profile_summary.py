"""Summarise a tools/profile_round.sh capture into profiles/ (tracked):

    python tools/profile_summary.py <tag>

  profiles/<tag>_launches.csv   the ncu launch list (gpu__time_duration.sum per launch)
  profiles/<tag>_kernels.json   per kernel of the --set full capture: duration, DRAM bytes,
                                achieved DRAM GB/s, bank conflicts, divergence, occupancy, IPC
  profiles/<tag>_summary.txt    human-readable version + launch-list shares of the step
"""

import csv
import io
import json
import os
import shutil
import subprocess
import sys
from collections import defaultdict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
tag = sys.argv[1] if len(sys.argv) > 1 else "r1"
src = os.path.join(ROOT, "gpurun_out")
dst = os.path.join(ROOT, "profiles")
os.makedirs(dst, exist_ok=True)

METRICS = {
    "gpu__time_duration.sum": "duration",
    "dram__bytes_read.sum": "dram_read",
    "dram__bytes_write.sum": "dram_write",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed": "dram_pct_of_peak",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum": "smem_ld_bank_conflicts",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_st.sum": "smem_st_bank_conflicts",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_atom.sum": "smem_atom_bank_conflicts",
    "smsp__sass_average_branch_targets_threads_uniform.pct": "branch_uniform_pct",
    "smsp__thread_inst_executed_per_inst_executed.ratio": "threads_per_inst",
    "sm__warps_active.avg.pct_of_peak_sustained_active": "achieved_occupancy_pct",
    "sm__inst_executed.avg.per_cycle_active": "ipc",
    "launch__registers_per_thread": "registers",
    "launch__grid_size": "grid",
    "launch__block_size": "block",
    "smsp__inst_executed.sum": "warp_instructions",
}
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-9, "us": 1e-6, "usecond": 1e-6,
         "ms": 1e-3, "msecond": 1e-3, "nsecond": 1e-9, "s": 1.0, "second": 1.0}


def short(name):
    n = name.split("(")[0]
    return n.split("::")[-1]


def num(v):
    try:
        return float(v.replace(",", ""))
    except ValueError:
        return None


# ---- launch list
lcsv = os.path.join(src, f"{tag}_launches.csv")
shares = {}
if os.path.exists(lcsv):
    shutil.copy(lcsv, os.path.join(dst, f"{tag}_launches.csv"))
    txt = open(lcsv).read()
    txt = txt[txt.index('"ID"'):] if '"ID"' in txt else txt
    rows = list(csv.DictReader(io.StringIO(txt)))
    tot = defaultdict(float)
    cnt = defaultdict(int)
    for r in rows:
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        v = num(r["Metric Value"]) * SCALE.get(r["Metric Unit"], 1.0)
        k = short(r["Kernel Name"])
        tot[k] += v
        cnt[k] += 1
    all_t = sum(tot.values())
    shares = {k: {"total_ms": 1e3 * v, "launches": cnt[k], "share": v / all_t} for k, v in tot.items()}

# ---- full capture
rep = os.path.join(src, f"{tag}_full.ncu-rep")
kern = {}
if os.path.exists(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(out.splitlines()))
    head, units = r[0], r[1]
    for row in r[2:]:
        d = dict(zip(head, row))
        k = short(d.get("Kernel Name", "?"))
        e = {}
        for m, key in METRICS.items():
            if m in head:
                i = head.index(m)
                v = num(row[i])
                if v is not None and units[i] in SCALE:
                    v *= SCALE[units[i]]
                e[key] = v
        if e.get("dram_read") is not None and e.get("dram_write") is not None:
            e["dram_bytes"] = e["dram_read"] + e["dram_write"]
            if e.get("duration"):
                e["dram_gbs"] = e["dram_bytes"] / e["duration"] / 1e9
        kern[k] = e

res = {"tag": tag, "source": f"ncu --set full --clock-control none (one launch per kernel, c3 workload, "
                             f"after 3 warm-up steps); launch list: gpu__time_duration.sum",
       "kernels": kern, "launch_shares": shares}
json.dump(res, open(os.path.join(dst, f"{tag}_kernels.json"), "w"), indent=1, sort_keys=True)
with open(os.path.join(dst, f"{tag}_summary.txt"), "w") as f:
    f.write(f"# {tag}: ncu summary (c3 512^3 lognormal, rel eb 1e-3, FtConfig())\n\n")
    f.write("kernel                 dur_us   dram_MB  dram_GB/s  occ%   IPC  thr/inst  unif_br%  smem_ld_conf\n")
    for k, e in sorted(kern.items(), key=lambda kv: -(kv[1].get("duration") or 0)):
        f.write(f"{k:20s} {1e6 * (e.get('duration') or 0):8.1f} {(e.get('dram_bytes') or 0) / 1e6:9.1f} "
                f"{e.get('dram_gbs') or 0:10.1f} {e.get('achieved_occupancy_pct') or 0:5.1f} "
                f"{e.get('ipc') or 0:5.2f} {e.get('threads_per_inst') or 0:9.2f} "
                f"{e.get('branch_uniform_pct') or 0:9.1f} {e.get('smem_ld_bank_conflicts') or 0:13.0f}\n")
    f.write("\nlaunch list (all launches of the bench command, cold-cache, serialised): share of GPU time\n")
    for k, v in sorted(shares.items(), key=lambda kv: -kv[1]["total_ms"]):
        f.write(f"  {k:28s} {v['launches']:4d} launches {v['total_ms']:9.3f} ms  {100 * v['share']:5.1f}%\n")
print(open(os.path.join(dst, f"{tag}_summary.txt")).read())
