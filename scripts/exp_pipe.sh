#!/bin/bash
TAG=pipe bash scripts/kernel_times.sh
timeout 600 python bench.py --steps 10 --no-cpu-baseline --no-secondary > gpurun_out/exp_pipe5.json 2>/dev/null
timeout 600 python bench.py --config 2 --steps 10 --no-cpu-baseline --no-secondary > gpurun_out/exp_pipe2.json 2>/dev/null
timeout 1500 python -m pytest tests/test_gpu_fullsize.py tests/test_gpu_parity.py -m gpu -x -q > gpurun_out/exp_pipe_pytest.log 2>&1
