"""Summarise ncu outputs into profiles/ (tracked).

    python scripts/ncu_summary.py launches <launches.csv> <out.md>
    python scripts/ncu_summary.py full <report.ncu-rep> <out.md> [--json traffic.json --key cfg2_c64]
"""
import csv
import io
import json
import re
import subprocess
import sys
from collections import defaultdict

METRICS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
           "dram__throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_sector_hit_rate.pct",
           "l1tex__t_sector_hit_rate.pct", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
           "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
           "launch__grid_size", "launch__block_size", "smsp__inst_executed.sum",
           "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active"]


def short(name):
    name = re.sub(r"\(aimx::HotDev.*", "", name)
    name = name.replace("void aimx::(anonymous namespace)::", "").replace("void aimx::<unnamed>::", "")
    return name[:70]


SETUP = ("k_chan_nonzero", "k_take", "k_static_near", "k_precorrect", "k_weights", "k_rwg_sides", "k_lam_to", "k_pack_c", "k_ent_w",
         "k_aim_fill", "k_lin_entries", "k_sample_static", "k_d2f", "k_self", "k_diag")


def launches(path, out, hot=False):
    txt = open(path).read()
    start = txt.find('"ID"')
    rows = list(csv.reader(io.StringIO(txt[start:])))
    hdr = rows[0]
    ix = {h: i for i, h in enumerate(hdr)}
    per = defaultdict(lambda: [0, 0.0])
    unit = None
    for r in rows[1:]:
        if len(r) < len(hdr) or r[ix["Metric Name"]] != "gpu__time_duration.sum":
            continue
        unit = r[ix["Metric Unit"]]
        v = float(r[ix["Metric Value"]].replace(",", ""))
        k = short(r[ix["Kernel Name"]])
        if hot and (not ("k_" in k) or any(x in k for x in SETUP)):
            continue
        per[k][0] += 1
        per[k][1] += v
    tot = sum(v[1] for v in per.values())
    with open(out, "w") as f:
        f.write(f"# ncu launch list summary ({path})\n\n")
        f.write("`ncu --metrics gpu__time_duration.sum --clock-control none` over the whole command"
                + (" -- the library's hot-path kernels only (setup kernels excluded)" if hot else "") + "\n")
        f.write("(cold-cache, serialised: compare SHARES, not absolute times).\n\n")
        f.write(f"| kernel | launches | total ({unit}) | share |\n|---|---|---|---|\n")
        for k, (n, v) in sorted(per.items(), key=lambda kv: -kv[1][1]):
            f.write(f"| `{k}` | {n} | {v:.1f} | {100 * v / tot:.1f}% |\n")
        f.write(f"\nTotal launches: {sum(v[0] for v in per.values())}\n")


def full(path, out, jpath=None, key=None):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    ix = {h: i for i, h in enumerate(hdr)}
    recs = []
    for r in rows[2:]:
        d = {"kernel": short(r[ix["Kernel Name"]])}
        for m in METRICS:
            if m in ix:
                d[m] = r[ix[m]]
                d[m + "@unit"] = units[ix[m]]
        recs.append(d)
    with open(out, "w") as f:
        f.write(f"# ncu --set full summary ({path})\n\n")
        cols = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
                "dram__throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_sector_hit_rate.pct",
                "sm__throughput.avg.pct_of_peak_sustained_elapsed",
                "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread"]
        f.write("| kernel | " + " | ".join(c.split(".")[0].replace("__", ".") + " (" + (recs[0].get(c + "@unit", "") if recs else "") + ")" for c in cols) + " |\n")
        f.write("|---" * (len(cols) + 1) + "|\n")
        for d in recs:
            f.write(f"| `{d['kernel']}` | " + " | ".join(str(d.get(c, "")) for c in cols) + " |\n")
    if jpath:
        try:
            j = json.load(open(jpath))
        except FileNotFoundError:
            j = {}
        ent = {}   # per stage: the sum over its kernels (proj_xfft = gather + x forward)
        j[key] = ent
        for d in recs:
            def num(m):
                v = float(str(d.get(m, "0")).replace(",", ""))
                u = d.get(m + "@unit", "byte")
                return v * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u, 1)
            stage = stage_of(d["kernel"])
            if stage:
                ent[stage] = ent.get(stage, 0.0) + num("dram__bytes_read.sum") + num("dram__bytes_write.sum")
        json.dump(j, open(jpath, "w"), indent=1)


def stage_of(k):
    for pat, st in (("k_interp_near", "interp_near"), ("k_zconv", "zconv"), ("k_yzconv", "zconv"),
                    ("k_yconv_plane", "zconv"), ("k_gather_b", "proj_xfft"), ("k_xfwd", "proj_xfft"),
                    ("k_yfwd", "yfwd"), ("k_yinv", "yinv"), ("k_xinv", "xinv")):
        if pat in k:
            return st
    return None


if __name__ == "__main__":
    if sys.argv[1] == "launches":
        launches(sys.argv[2], sys.argv[3], hot="--hot" in sys.argv)
    else:
        jp = key = None
        if "--json" in sys.argv:
            jp = sys.argv[sys.argv.index("--json") + 1]
            key = sys.argv[sys.argv.index("--key") + 1]
        full(sys.argv[2], sys.argv[3], jp, key)
