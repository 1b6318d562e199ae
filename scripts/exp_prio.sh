mkdir -p gpurun_out
for k in 1 2; do
for P in "0 0" "0 1" "-1 0" "-1 1" "0 -1"; do
set -- $P
AIMX_PRIO_S2=$1 AIMX_PRIO_S3=$2 timeout 300 python bench.py --no-cpu-baseline --steps 20 > "gpurun_out/prio_${1}_${2}_$k.json" 2>&1
done
done
