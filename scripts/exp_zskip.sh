#!/bin/bash
mkdir -p gpurun_out
for m in 0 1 9 11 15; do
  AIMX_ZSKIP_MASK=$m timeout 600 python bench.py --steps 10 --no-cpu-baseline --no-secondary > gpurun_out/exp_z$m.json 2>/dev/null
done
