#!/bin/bash
# ncu --set full of kernel regex $K in scripts/ncu_target.py $ARGS; keeps only
# text extracts (details, raw metrics, per-line source with stall samples).
set -u
mkdir -p gpurun_out
T=${TAG:-st}
python -m paper_2009_02281_b200.build > /dev/null 2>&1 || exit 1
timeout 300 python scripts/ncu_target.py ${ARGS} > gpurun_out/${T}_plain.log 2>&1 || { echo "plain run failed"; exit 1; }
timeout 900 ncu --set full --clock-control none --import-source on -k regex:${K} -c 1 -f -o /tmp/${T} python scripts/ncu_target.py ${ARGS} > gpurun_out/${T}_ncu.log 2>&1
echo "ncu rc=$?" >> gpurun_out/${T}_ncu.log
ncu -i /tmp/${T}.ncu-rep --page details --csv > gpurun_out/${T}_details.csv 2>&1
ncu -i /tmp/${T}.ncu-rep --page raw --csv > gpurun_out/${T}_raw.csv 2>&1
ncu -i /tmp/${T}.ncu-rep --page source --csv --print-source sass > gpurun_out/${T}_sass.csv 2>&1
ls -la gpurun_out/${T}_* >> gpurun_out/${T}_ncu.log
