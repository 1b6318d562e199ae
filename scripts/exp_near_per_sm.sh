#!/bin/bash
# cfg5 sweep with fewer S4+S5 CTAs per SM (room for the next batch's grid kernels)
mkdir -p gpurun_out
for n in 5 4 3 2; do
  AIMX_NEAR_PER_SM=$n timeout 600 python bench.py --steps 10 --no-cpu-baseline --no-secondary > gpurun_out/exp_ps$n.json 2>/dev/null
done
