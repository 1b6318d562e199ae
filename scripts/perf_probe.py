"""Per-config stage timing of the GPU path (development tool; prints JSON lines).

    python scripts/perf_probe.py [--configs 1,2,3,5] [--precs c64,c128] [--iters 50]

Per config: setup time, then `iters` (spectrum + matvec) pairs with the
library's event profiler on, reporting per-stage ms/launch and the modelled
GB/s of each stage (bench.stage_bytes)."""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import aimx_inputs as inp  # noqa: E402
from bench import stage_bytes  # noqa: E402
from paper_2009_02281_b200 import AIMx  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--configs", default="1,2,3,5")
ap.add_argument("--precs", default="c64,c128")
ap.add_argument("--iters", type=int, default=50)
a = ap.parse_args()

for cfg in [int(x) for x in a.configs.split(",")]:
    c = inp.get_config(cfg)
    mesh = inp.make_mesh(cfg)
    for prec in a.precs.split(","):
        if prec == "c128" and cfg in (2, 5):
            continue
        t0 = time.perf_counter()
        op = AIMx(mesh.vertices, mesh.triangles, c.grid_n, prec=prec)
        torch.cuda.synchronize()
        tset = time.perf_counter() - t0
        st = op.stats()
        dt = torch.complex64 if prec == "c64" else torch.complex128
        x = torch.as_tensor(inp.rhs_vector(cfg, 0, op.N)).to(dt).cuda()
        y = torch.empty_like(x)
        for i in range(5):
            op.set_frequency(c.freqs[0])
            op.matvec(x, y)
        torch.cuda.synchronize()
        op.profile_enable(True)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for i in range(a.iters):
            op.set_frequency(c.freqs[i % len(c.freqs)])
            op.matvec(x, y)
        e1.record()
        torch.cuda.synchronize()
        prof = op.profile_read()
        kern = prof.pop("kernels")
        op.profile_enable(False)
        # unprofiled back-to-back matvecs
        op.set_frequency(c.freqs[0])
        torch.cuda.synchronize()
        e2, e3 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e2.record()
        for i in range(a.iters):
            op.matvec(x, y)
        e3.record()
        torch.cuda.synchronize()
        sb = stage_bytes(st, prec)
        fused = prof["yfwd"][1] == 0
        if fused:
            sb["zconv"] = stage_bytes(st, prec, fused_yz=True)["zconv"]
        stages = {k: {"ms": ms / n, "GBps": sb[k] / (ms / n * 1e-3) / 1e9,
                      "MB": sb[k] / 1e6} for k, (ms, n) in prof.items() if n > 0}
        print(json.dumps({"cfg": cfg, "prec": prec, "setup_s": tset, "stats": st,
                          "ms_per_freq_pt_profiled": e0.elapsed_time(e1) / a.iters,
                          "ms_per_matvec": e2.elapsed_time(e3) / a.iters, "kernels_per_freq_pt": kern / a.iters,
                          "stages": stages}),
              flush=True)
        op.close()
        del op
        torch.cuda.empty_cache()
