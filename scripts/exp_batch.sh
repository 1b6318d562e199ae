#!/bin/bash
# cfg5 sweep rate at 8 / 16 / 32 batch slots (AIMX_BATCH)
mkdir -p gpurun_out
for b in 16 8 32; do
  AIMX_BATCH=$b timeout 600 python bench.py --steps 10 --no-cpu-baseline --no-secondary > gpurun_out/exp_batch_$b.json 2>/dev/null
done
AIMX_NO_OVERLAP=1 timeout 600 python bench.py --steps 10 --no-cpu-baseline --no-secondary > gpurun_out/exp_nooverlap.json 2>/dev/null
