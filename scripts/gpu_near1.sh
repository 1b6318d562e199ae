#!/bin/bash
# Single-column S4+S5 kernel (k_interp_near1): parity tests, then the A/B of
# the single-column stage times against the entry-per-lane kernel.
set -u
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py tests/test_gpu_kop.py tests/test_gpu_solve.py -m gpu -x -q > gpurun_out/near1_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/near1_pytest.log
tail -3 gpurun_out/near1_pytest.log
for o in 0 1; do
  AIMX_NEAR1_OLD=$o python scripts/perf_probe.py --configs 5,3,2 --precs c64 --iters 30 2>/dev/null > gpurun_out/near1_probe_old$o.jsonl
  python - <<P
import json
for l in open("gpurun_out/near1_probe_old$o.jsonl"):
    d = json.loads(l)
    print("old=$o cfg", d["cfg"], "ms/matvec", round(d["ms_per_matvec"], 4), {k: round(v["ms"], 4) for k, v in d["stages"].items()})
P
done
