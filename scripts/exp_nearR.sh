#!/bin/bash
mkdir -p gpurun_out
for r in 16 8; do
  AIMX_NEAR_R=$r timeout 600 python bench.py --steps 10 --no-cpu-baseline --no-secondary > gpurun_out/exp_R$r.json 2>/dev/null
done
