#!/bin/bash
# A/B session: build, the parity subset ($TESTS), then the cfg5 bench line and
# the serialised per-kernel times for each environment variant in $VARIANTS
# ("name:VAR=value,VAR2=value" entries, space separated; "base:" = defaults).
set -u
mkdir -p gpurun_out
T=${TAG:-ab}
python -m paper_2009_02281_b200.build > gpurun_out/${T}_build.log 2>&1 || { echo build failed; exit 1; }
if [ -n "${TESTS:-}" ]; then
  timeout 1500 python -m pytest ${TESTS} -x -q > gpurun_out/${T}_pytest.log 2>&1
  echo "pytest rc=$?" >> gpurun_out/${T}_pytest.log
fi
for v in ${VARIANTS:-base:}; do
  name=${v%%:*}; envs=${v#*:}
  (
    IFS=','; for kv in $envs; do [ -n "$kv" ] && export "$kv"; done; unset IFS
    timeout 600 python bench.py --no-cpu-baseline ${BENCH_ARGS:---no-secondary} > gpurun_out/${T}_${name}_bench.json 2> gpurun_out/${T}_${name}_bench.err
    echo "bench rc=$?" >> gpurun_out/${T}_${name}_bench.err
    if [ -n "${KT:-}" ]; then
      timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${T}_${name}_kt.csv \
        python scripts/ncu_target.py --cfg ${CFG:-5} --nf ${NF:-32} > gpurun_out/${T}_${name}_kt.log 2>&1
      python scripts/ncu_summary.py launches gpurun_out/${T}_${name}_kt.csv gpurun_out/${T}_${name}_kt.md --hot >> gpurun_out/${T}_${name}_kt.log 2>&1
    fi
  )
done
