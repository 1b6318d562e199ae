for m in 0 1 2; do
AIMX_DEBUG_NEAR=$m timeout 300 python bench.py --no-cpu-baseline --steps 5 > gpurun_out/exp_dbg$m.json 2>&1
done
