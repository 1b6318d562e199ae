"""Per-frequency cost of the conventional AIM vs AIMx on one B200 (the
structure of the paper's tab:prof): for each config, a sweep of
`nf` frequency points (matvec per point, same inputs) in both modes, and the
AIM mode's per-frequency near fill alone.  Prints JSON lines.

    python scripts/aim_probe.py [--configs 1,2,3] [--nf 8]
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import aimx_inputs as inp  # noqa: E402
from paper_2009_02281_b200 import AIMx  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--configs", default="1,2,3")
ap.add_argument("--nf", type=int, default=8)
a = ap.parse_args()


def timed(fn, reps=3):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


for cfg in [int(x) for x in a.configs.split(",")]:
    c = inp.get_config(cfg)
    m = inp.make_mesh(cfg)
    op = AIMx(m.vertices, m.triangles, c.grid_n, prec="c64")
    st = op.stats()
    nf = min(a.nf, len(c.freqs))
    freqs = np.asarray(c.freqs)[np.linspace(0, len(c.freqs) - 1, nf).astype(int)]
    X = torch.as_tensor(np.stack([inp.rhs_vector(cfg, i, op.N) for i in range(nf)])).to(torch.complex64).cuda()
    Y = torch.empty_like(X)
    aimx_ms = timed(lambda: op.sweep(freqs, X, Y))
    op.set_conventional(True)
    aim_ms = timed(lambda: op.sweep(freqs, X, Y))
    fill_ms = timed(lambda: [op.set_frequency(f) for f in freqs]) / nf
    op.set_frequency(freqs[0])
    mv_ms = timed(lambda: op.matvec(X[0], Y[0]), 20)
    op.set_conventional(False)
    print(json.dumps({"cfg": cfg, "N": op.N, "nnz": st["nnz"], "nf": nf,
                      "aimx_ms_per_freq": aimx_ms / nf, "aim_ms_per_freq": aim_ms / nf,
                      "aim_fill_ms_per_freq": fill_ms, "aim_matvec_ms": mv_ms,
                      "speedup_per_freq_one_matvec": aim_ms / aimx_ms}), flush=True)
    op.close()
    del op
    torch.cuda.empty_cache()
