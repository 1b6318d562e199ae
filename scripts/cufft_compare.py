"""cuFFT comparison point (north star: "cuFFT is reported only as a comparison
point"): per config, our S2 + S3 stages of one device batch (event profiler,
projection gather included) against the same zero-padded convolution done by
cuFFT (torch.fft) on the full padded grid.  Prints JSON lines.

    python scripts/cufft_compare.py [--configs 1,2,3,5] [--iters 20]
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import aimx_inputs as inp  # noqa: E402
from bench import cufft_conv_ms  # noqa: E402
from paper_2009_02281_b200 import AIMx  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--configs", default="1,2,3,5")
ap.add_argument("--iters", type=int, default=20)
a = ap.parse_args()
S3 = ("proj_xfft", "yfwd", "zconv", "yinv", "xinv")
for cfg in [int(x) for x in a.configs.split(",")]:
    c = inp.get_config(cfg)
    m = inp.make_mesh(cfg)
    prec = "c64"
    op = AIMx(m.vertices, m.triangles, c.grid_n, prec=prec)
    B = op.stats()["batch_slots"]
    for cols in sorted({1, B}):
        nf = cols * a.iters
        freqs = [c.freqs[i % len(c.freqs)] for i in range(nf)]
        X = torch.as_tensor(inp.rhs_matrix(cfg, op.N, [i % len(c.freqs) for i in range(nf)])).to(
            torch.complex64).cuda()
        op.sweep(freqs[:cols], X[:cols], batch=cols)
        op.profile_enable(True)
        op.sweep(freqs, X, batch=cols)
        prof = op.profile_read()
        op.profile_enable(False)
        ours = sum(prof[k][0] / prof[k][1] for k in S3 if prof[k][1] > 0)
        cu = cufft_conv_ms(c.grid_n, cols, prec)
        print(json.dumps({"cfg": cfg, "prec": prec, "grid": list(c.grid_n), "columns": cols,
                          "ours_ms": ours, "cufft_ms": cu, "speedup": cu / ours,
                          "ours_stages_ms": {k: prof[k][0] / prof[k][1] for k in S3 if prof[k][1] > 0}}),
              flush=True)
    op.close()
    del op
    torch.cuda.empty_cache()
