#!/bin/bash
# Per-kernel device times (ncu gpu__time_duration, serialised) of one sweep of
# config $CFG with $NF points, for A/B comparisons; TAG names the output.
set -u
mkdir -p gpurun_out
python -m paper_2009_02281_b200.build > /dev/null 2>&1 || exit 1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/kt_${TAG:-x}.csv \
  python scripts/ncu_target.py --cfg ${CFG:-5} --nf ${NF:-32} > gpurun_out/kt_${TAG:-x}.log 2>&1
python scripts/ncu_summary.py launches gpurun_out/kt_${TAG:-x}.csv gpurun_out/kt_${TAG:-x}.md --hot
