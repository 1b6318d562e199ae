mkdir -p gpurun_out
for W in 1 2 3 4 8; do
AIMX_NEAR_WAVES=$W timeout 300 python bench.py --no-cpu-baseline --steps 10 > gpurun_out/exp_W$W.json 2>&1
AIMX_NEAR_WAVES=$W timeout 300 python scripts/perf_probe.py --configs 3 --iters 20 > gpurun_out/exp_W${W}_c3.jsonl 2>&1
done
