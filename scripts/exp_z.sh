mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py tests/test_gpu_slab.py -x -q > gpurun_out/pytest_z.log 2>&1; echo rc=$? >> gpurun_out/pytest_z.log
timeout 300 python scripts/perf_probe.py --configs 3,5 --iters 20 > gpurun_out/probe_z.jsonl 2>&1
