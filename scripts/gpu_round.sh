#!/bin/bash
# One GPU session: parity tests, smoke, bench, launch list (each step only after the previous exits 0).
set -u
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt 2>&1
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?" >> gpurun_out/bench.err
timeout 600 python scripts/perf_probe.py --configs 1,2,3,5 --iters 30 > gpurun_out/probe.jsonl 2> gpurun_out/probe.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_bench.log 2>&1; echo "ncu rc=$?" >> gpurun_out/ncu_bench.log
NCU_COUNT=2 NCU_OUT=gpurun_out/prof_dom bash scripts/gpu_ncu.sh "k_interp_near" --cfg 2 --nf 25
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_sweep.csv python scripts/ncu_target.py --cfg 2 --nf 100 > gpurun_out/ncu_sweep.log 2>&1; echo "ncu sweep rc=$?" >> gpurun_out/ncu_sweep.log
