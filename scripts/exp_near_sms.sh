#!/bin/bash
# cfg5 sweep rate with the S4+S5 kernel's CTAs spread over fewer SMs
mkdir -p gpurun_out
for n in 148 128 112 96; do
  AIMX_NEAR_SMS=$n timeout 600 python bench.py --steps 10 --no-cpu-baseline --no-secondary > gpurun_out/exp_sms_$n.json 2>/dev/null
done
