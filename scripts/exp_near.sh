for c in 2 4 6 8; do
AIMX_NEAR_CTAS_PER_SM=$c timeout 300 python scripts/perf_probe.py --configs 2,3 --precs c64 --iters 20 > gpurun_out/exp_C${c}.jsonl 2>&1
AIMX_NEAR_CTAS_PER_SM=$c timeout 300 python bench.py --no-cpu-baseline --steps 5 > gpurun_out/exp_bench_C${c}.json 2>&1
done
