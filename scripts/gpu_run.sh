#!/bin/bash
# Dev GPU session: selected GPU tests ($TESTS, pytest -k $K), then the bench
# on the configs in $BENCH (no ncu).  Logs in gpurun_out/$TAG_*.
set -u
mkdir -p gpurun_out
TAG=${TAG:-run}
python -m paper_2009_02281_b200.build > gpurun_out/${TAG}_build.log 2>&1 || { echo build failed; exit 1; }
if [ -n "${TESTS:-}" ]; then
  timeout ${TTIME:-1500} python -m pytest $TESTS -m gpu -x -q --durations=30 ${K:+-k "$K"} > gpurun_out/${TAG}_pytest.log 2>&1
  echo "pytest rc=$?" >> gpurun_out/${TAG}_pytest.log
fi
for c in ${BENCH:-}; do
  timeout 900 python bench.py --config $c --no-cpu-baseline ${BARGS:-} > gpurun_out/${TAG}_b$c.json 2> gpurun_out/${TAG}_b$c.err
  echo "bench rc=$?" >> gpurun_out/${TAG}_b$c.err
done
if [ -n "${PROBE:-}" ]; then
  timeout 900 python scripts/perf_probe.py --configs $PROBE --precs c64 --iters 30 > gpurun_out/${TAG}_probe.jsonl 2> gpurun_out/${TAG}_probe.err
fi
