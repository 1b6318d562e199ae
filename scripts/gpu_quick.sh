#!/bin/bash
# Parity tests + bench + probe (no ncu).
set -u
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?" >> gpurun_out/bench.err
timeout 600 python scripts/perf_probe.py --configs ${PROBE_CFGS:-2,3,5} --iters 30 > gpurun_out/probe.jsonl 2> gpurun_out/probe.err
