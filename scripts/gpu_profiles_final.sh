#!/bin/bash
# Final ncu evidence for profiles/ (one GPU; each capture runs after the same
# command exited 0 without ncu).  Reports stay on the box; only the text
# summaries (ncu_summary.py) and raw-metric CSVs come back.
#   launches: gpu__time_duration of every launch of one cfg5 bench step (64
#             points, two 32-column batches) -> ${T}_launches_cfg5.md
#   cfg5:     --set full of every hot kernel of one cfg5 batch (32 columns)
#   cfg3:     --set full of the cfg3 y and TMA z passes (8 columns)
set -u
mkdir -p gpurun_out
T=${TAG:-fin}
P=${PARTS:-launches cfg5 cfg3}
python -m paper_2009_02281_b200.build > /dev/null 2>&1 || exit 1
if [[ " $P " == *" launches "* ]]; then
timeout 300 python scripts/ncu_target.py --cfg 5 --nf 64 > gpurun_out/${T}_plain5.log 2>&1 || exit 2
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${T}_launches_cfg5.csv \
  python scripts/ncu_target.py --cfg 5 --nf 64 > gpurun_out/${T}_launches_cfg5.log 2>&1
python scripts/ncu_summary.py launches gpurun_out/${T}_launches_cfg5.csv gpurun_out/${T}_launches_cfg5.md --hot >> gpurun_out/${T}_launches_cfg5.log 2>&1
fi
if [[ " $P " == *" cfg5 "* ]]; then
timeout 300 python scripts/ncu_target.py --cfg 5 --nf 32 > gpurun_out/${T}_plain5b.log 2>&1 || exit 3
timeout 1500 ncu --set full --clock-control none --import-source on \
  -k regex:"k_interleave|k_gather_b|k_xfwd|k_yconv_plane|k_xinv_b|k_interp_near" -c 6 -f -o /tmp/${T}_cfg5 \
  python scripts/ncu_target.py --cfg 5 --nf 32 > gpurun_out/${T}_full5.log 2>&1
python scripts/ncu_summary.py full /tmp/${T}_cfg5.ncu-rep gpurun_out/${T}_ncu_cfg5_batch32.md --json gpurun_out/${T}_traffic.json --key cfg5_c64 >> gpurun_out/${T}_full5.log 2>&1
ncu -i /tmp/${T}_cfg5.ncu-rep --page raw --csv > gpurun_out/${T}_cfg5_raw.csv 2>/dev/null
fi
if [[ " $P " == *" cfg3 "* ]]; then
timeout 300 python scripts/ncu_target.py --cfg 3 --nf 8 > gpurun_out/${T}_plain3.log 2>&1 || exit 4
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"k_zconv_tma|k_yfwd|k_yinv|k_xinv|k_gather_b|k_xfwd|k_interp_near" -c 7 -f -o /tmp/${T}_cfg3 \
  python scripts/ncu_target.py --cfg 3 --nf 8 > gpurun_out/${T}_full3.log 2>&1
python scripts/ncu_summary.py full /tmp/${T}_cfg3.ncu-rep gpurun_out/${T}_ncu_cfg3_batch8.md --json gpurun_out/${T}_traffic.json --key cfg3_c64 >> gpurun_out/${T}_full3.log 2>&1
ncu -i /tmp/${T}_cfg3.ncu-rep --page raw --csv > gpurun_out/${T}_cfg3_raw.csv 2>/dev/null
fi
echo done
