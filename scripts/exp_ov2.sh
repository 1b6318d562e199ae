mkdir -p gpurun_out
for W in 0.6 0.8 1 ; do
AIMX_NEAR_WAVES=$W timeout 300 python bench.py --no-cpu-baseline --steps 10 > gpurun_out/ovw_$W.json 2>&1
done
for W in 0.6 0.8; do
AIMX_NEAR_WAVES=$W timeout 300 python scripts/perf_probe.py --configs 3 --iters 20 > gpurun_out/ovw_${W}_c3.jsonl 2>&1
done
