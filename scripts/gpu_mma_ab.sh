#!/bin/bash
# Tensor-core S4+S5 (AIMX_NEAR_MMA=1) vs the FMA kernel: parity + bench A/B.
set -u
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_near_mma.py -x -q > gpurun_out/pytest_mma.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_mma.log
AIMX_NEAR_MMA=1 timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench_mma.json 2> gpurun_out/bench_mma.err
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench_fma.json 2> gpurun_out/bench_fma.err
if [ -n "${NCU_MMA:-}" ]; then
  AIMX_NEAR_MMA=1 K=k_interp_near_mma ARGS="--cfg 5 --nf 32" TAG=mma bash scripts/gpu_stalls.sh
fi
