#!/bin/bash
# The secondary measurements quoted in DESIGN.md, written to gpurun_out/ (copied to profiles/).
set -u
mkdir -p gpurun_out
timeout 600 python scripts/kop_probe.py 3 > gpurun_out/r1_kop_probe.json 2>/dev/null
timeout 900 python scripts/pmchwt_probe.py > gpurun_out/r1_pmchwt_probe.json 2>/dev/null
timeout 600 python scripts/multi_probe.py > gpurun_out/r1_multi_probe.jsonl 2>/dev/null
timeout 900 python scripts/aim_probe.py > gpurun_out/r1_aim_probe.jsonl 2>/dev/null
timeout 600 python scripts/cufft_compare.py > gpurun_out/r1_cufft_compare.jsonl 2>/dev/null
timeout 600 python scripts/graph_probe.py > gpurun_out/r1_graph_probe.jsonl 2>/dev/null
timeout 600 python scripts/e2e_probe.py > gpurun_out/r1_e2e_probe.json 2>/dev/null
timeout 1200 python scripts/prof_table_probe.py --nf 100 > gpurun_out/r1_prof_table.jsonl 2>/dev/null
echo done > gpurun_out/r1_probes.done
