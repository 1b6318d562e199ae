#!/bin/bash
# Last session of round 2: whole -m gpu suite, smoke, default bench, then the
# --set full capture of the warp-private single-column S4+S5 kernel (cfg5).
set -u
TAG=s6 bash scripts/gpu_final.sh
K=k_interp_near1w ARGS="--cfg 5 --nf 1" TAG=n1w bash scripts/gpu_stalls.sh
python scripts/ncu_raw_brief.py gpurun_out/n1w_raw.csv > gpurun_out/n1w_brief.txt 2>&1
tail -3 gpurun_out/s6_pytest.log; tail -2 gpurun_out/s6_smoke.log; tail -2 gpurun_out/s6_bench.err; cat gpurun_out/n1w_brief.txt
