#!/bin/bash
TAG=xb bash scripts/kernel_times.sh
AIMX_NO_XFWD_B=1 TAG=xg bash scripts/kernel_times.sh
for v in 0 1; do
  if [ $v = 1 ]; then export AIMX_NO_XFWD_B=1; fi
  timeout 600 python bench.py --steps 10 --no-cpu-baseline --no-secondary > gpurun_out/exp_xfwd$v.json 2>/dev/null
done
unset AIMX_NO_XFWD_B
AIMX_NEAR_SMGROUP=1 timeout 600 python bench.py --steps 10 --no-cpu-baseline --no-secondary > gpurun_out/exp_smgroup.json 2>/dev/null
AIMX_NEAR_SMGROUP=1 TAG=smg bash scripts/kernel_times.sh
