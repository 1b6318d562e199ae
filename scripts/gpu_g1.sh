set -u
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/g1_smi.txt
timeout 600 python bench.py --config 5 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/g1_b5.json 2> gpurun_out/g1_b5.err
timeout 600 python bench.py --config 3 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/g1_b3.json 2> gpurun_out/g1_b3.err
timeout 600 python scripts/perf_probe.py --configs 3,5 --precs c64 --iters 30 > gpurun_out/g1_probe.jsonl 2> gpurun_out/g1_probe.err
