#!/bin/bash
# Tensor-core S4+S5: HMMA rate probe, parity, bench A/B against the FMA kernel.
set -u
mkdir -p gpurun_out
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/hmma_rate scripts/tc/hmma_rate.cu && timeout 120 /tmp/hmma_rate > gpurun_out/hmma_rate.log 2>&1
timeout 900 python -m pytest tests/test_gpu_near_mma.py -x -q > gpurun_out/pytest_mma.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_mma.log
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench_mma.json 2> gpurun_out/bench_mma.err
AIMX_NEAR_FMA=1 timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench_fma.json 2> gpurun_out/bench_fma.err
timeout 1200 python -m pytest tests -m gpu -x -q ${PYTEST_K:-} > gpurun_out/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.log
