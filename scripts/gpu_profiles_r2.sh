#!/bin/bash
# Round-2 ncu evidence (one GPU; each capture after the same command ran
# clean without ncu).  PART=launches: the launch list of one cfg5 bench step;
# PART=cfg5: --set full of every hot kernel of one cfg5 device batch (32
# columns); PART=cfg3: the cfg3 y and TMA z passes.  One report per gpurun
# call (the call returns at most 64 MiB).  Summaries go to profiles/.
set -u
mkdir -p gpurun_out
python -m paper_2009_02281_b200.build > /dev/null 2>&1 || exit 1
case "${PART:-launches}" in
  launches)
    timeout 300 python scripts/ncu_target.py --cfg 5 --nf 64 > gpurun_out/r2_plain5.log 2>&1 || exit 2
    timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2_launches_cfg5.csv \
      python scripts/ncu_target.py --cfg 5 --nf 64 > gpurun_out/r2_launches_cfg5.log 2>&1 ;;
  cfg5)
    timeout 300 python scripts/ncu_target.py --cfg 5 --nf 32 > gpurun_out/r2_plain5.log 2>&1 || exit 2
    timeout 1200 ncu --set full --clock-control none --import-source on \
      -k regex:"k_interleave|k_gather_b|k_xfwd|k_yconv_plane|k_xinv_b|k_interp_near" -c 6 -f -o gpurun_out/r2_cfg5 \
      python scripts/ncu_target.py --cfg 5 --nf 32 > gpurun_out/r2_full5.log 2>&1 ;;
  cfg3)
    timeout 300 python scripts/ncu_target.py --cfg 3 --nf 8 > gpurun_out/r2_plain3.log 2>&1 || exit 3
    timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_zconv_tma|k_yfwd" -c 2 -f -o gpurun_out/r2_cfg3 \
      python scripts/ncu_target.py --cfg 3 --nf 8 > gpurun_out/r2_full3.log 2>&1 ;;
esac
echo done
