mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "row_group" > gpurun_out/exp_rg.log 2>&1; echo rc=$? >> gpurun_out/exp_rg.log
for R in 8 16; do
AIMX_NEAR_R=$R timeout 300 python bench.py --no-cpu-baseline --steps 10 > gpurun_out/exp_R$R.json 2>&1
AIMX_NEAR_R=$R timeout 300 python scripts/perf_probe.py --configs 3 --iters 20 > gpurun_out/exp_R${R}_c3.jsonl 2>&1
done
