"""Opcode mix and stall samples per opcode from an ncu report (dev tool).

    python scripts/ncu_sass_mix.py <report.ncu-rep> <kernel-regex> [top]
"""
import collections
import csv
import io
import re
import subprocess
import sys

rep, pat = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 25
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass", "-k", "regex:" + pat],
                     capture_output=True, text=True).stdout
blocks = re.split(r'(?m)^"Kernel Name",', txt)
for b in blocks[1:]:
    lines = b.splitlines()
    name = lines[0][:100]
    rows = list(csv.reader(io.StringIO("\n".join(lines[1:]))))
    h = rows[0]
    ix = {k: i for i, k in enumerate(h)}
    op, st = collections.Counter(), collections.Counter()
    for r in rows[1:]:
        if len(r) < len(h):
            continue
        s = r[ix["Source"]].strip().split()
        if not s:
            continue
        o = s[1] if s[0].startswith("@") else s[0]
        o = o.split(".")[0]
        op[o] += int(r[ix["Instructions Executed"]] or 0)
        st[o] += int(r[ix["Warp Stall Sampling (All Samples)"]] or 0)
    tot = sum(op.values()) or 1
    print("==", name, "total", tot)
    for k, v in op.most_common(top):
        print(f"  {k:10s} {v:12d} {v / tot:6.3f}  stall {st[k]}")
