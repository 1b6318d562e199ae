#!/bin/bash
# ncu --set full of one kernel (regex $1) in scripts/ncu_target.py (args $2...)
set -u
mkdir -p gpurun_out
K=$1; shift
OUT=${NCU_OUT:-gpurun_out/prof}
timeout 300 python scripts/ncu_target.py "$@" > gpurun_out/ncu_plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:$K -c ${NCU_COUNT:-2} -f -o $OUT python scripts/ncu_target.py "$@" > gpurun_out/ncu_run.log 2>&1
echo "rc=$?" >> gpurun_out/ncu_run.log
