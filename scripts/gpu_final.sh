#!/bin/bash
# Round-end style session: the whole -m gpu suite (timed), smoke, the default bench.
set -u
mkdir -p gpurun_out
T=${TAG:-fin}
python -m paper_2009_02281_b200.build > gpurun_out/${T}_build.log 2>&1 || exit 1
S=$(date +%s)
timeout 2400 python -m pytest tests -m gpu -x -q --durations=15 > gpurun_out/${T}_pytest.log 2>&1
echo "pytest rc=$? seconds=$(( $(date +%s) - S ))" >> gpurun_out/${T}_pytest.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${T}_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/${T}_smoke.log
timeout 900 python bench.py > gpurun_out/${T}_bench.json 2> gpurun_out/${T}_bench.err; echo "bench rc=$?" >> gpurun_out/${T}_bench.err
