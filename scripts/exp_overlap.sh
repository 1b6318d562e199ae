mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_linear.py tests/test_gpu_fullsize.py -x -q -k "sweep or overlap or batch or linear" > gpurun_out/pytest_ov.log 2>&1; echo rc=$? >> gpurun_out/pytest_ov.log
for k in 1 2; do
timeout 300 python bench.py --no-cpu-baseline --steps 10 > gpurun_out/ov_on$k.json 2>&1
AIMX_NO_OVERLAP=1 timeout 300 python bench.py --no-cpu-baseline --steps 10 > gpurun_out/ov_off$k.json 2>&1
done
