"""Key metrics and the stall ranking of each kernel in an `ncu --page raw --csv` export (dev tool).

    python scripts/ncu_raw_brief.py gpurun_out/<tag>_raw.csv
"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
h = rows[0]
keys = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "dram__bytes_read.sum.per_second", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "lts__t_sector_hit_rate.pct",
        "launch__registers_per_thread", "launch__grid_size", "smsp__inst_executed.sum",
        "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
        "lts__t_sectors.sum", "lts__t_sectors.avg.pct_of_peak_sustained_elapsed"]
for r in rows[2:]:
    d = dict(zip(h, r))
    print("==", d.get("Kernel Name", "")[:90])
    for k in keys:
        if k in d:
            print(f"  {k} = {d[k]} {rows[1][h.index(k)]}")
    st = [(k, float(d[k].replace(",", ""))) for k in h
          if "smsp__average_warps_issue_stalled" in k and k.endswith("_per_issue_active.ratio") and "not_issued" not in k]
    print("  stalls (warps per issue):", ", ".join(f"{k.split('stalled_')[1].split('_per')[0]} {v:.2f}"
                                                     for k, v in sorted(st, key=lambda x: -x[1])[:8]))
