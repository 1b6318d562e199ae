"""Print the key ncu --set full details of the kernels in a report (dev tool).

    python scripts/ncu_details.py <report.ncu-rep> [name-regex]
"""
import csv
import io
import re
import subprocess
import sys

KEYS = ["Duration", "DRAM Throughput", "Memory Throughput", "Issue Slots Busy", "Achieved Occupancy",
        "Theoretical Occupancy", "Registers Per Thread", "Block Limit Registers", "Block Limit Shared Mem",
        "Dynamic Shared Memory Per Block", "Grid Size", "Block Size", "Waves Per SM", "L2 Hit Rate",
        "L1/TEX Hit Rate", "Executed Instructions", "Eligible Warps Per Scheduler", "Active Warps Per Scheduler"]
rep = sys.argv[1]
pat = re.compile(sys.argv[2]) if len(sys.argv) > 2 else None
txt = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(txt)))
h = rows[0]
ix = {k: i for i, k in enumerate(h)}
cur = None
for r in rows[1:]:
    name = r[ix["Kernel Name"]]
    if pat and not pat.search(name):
        continue
    key = (r[ix["ID"]], name)
    if key != cur:
        cur = key
        print("==", r[ix["ID"]], re.sub(r"\(aimx::HotDev.*", "", name)[:110])
    m = r[ix["Metric Name"]]
    if m in KEYS:
        print(f"   {m:32s} {r[ix['Metric Value']]} {r[ix['Metric Unit']]}")
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rr = list(csv.reader(io.StringIO(raw)))
hh = rr[0]
stall = [i for i, k in enumerate(hh) if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("not_issued")]
for r in rr[2:]:
    name = r[hh.index("Kernel Name")]
    if pat and not pat.search(name):
        continue
    vals = sorted(((float(r[i].replace(",", "") or 0), hh[i].replace("smsp__pcsamp_warps_issue_stalled_", ""))
                   for i in stall), reverse=True)[:6]
    print("stalls", r[hh.index("ID")], re.sub(r"\(aimx::HotDev.*", "", name)[:60], [(n, int(v)) for v, n in vals])
