#!/bin/bash
# Final session of round 2: the whole -m gpu suite, smoke, the default bench
# (scripts/gpu_final.sh), then the ncu evidence of the single-column S4+S5
# kernel (--set full, cfg5) and the launch list of one cfg5 bench step.
set -u
TAG=s5 bash scripts/gpu_final.sh
K=k_interp_near1 ARGS="--cfg 5 --nf 1" TAG=n1c bash scripts/gpu_stalls.sh
python scripts/ncu_raw_brief.py gpurun_out/n1c_raw.csv > gpurun_out/n1c_brief.txt 2>&1
PARTS=launches TAG=r2h bash scripts/gpu_profiles_final.sh
tail -3 gpurun_out/s5_pytest.log; tail -2 gpurun_out/s5_smoke.log; tail -2 gpurun_out/s5_bench.err; head -c 600 gpurun_out/s5_bench.json
