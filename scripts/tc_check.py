"""Quick check of the tensor-core S4+S5 kernel (AIMX_NEAR_TC=1): a 32-point
cfg1 sweep (32 slots) against the oracle, and a cfg5 sweep of one 32-point
batch against the FMA kernel's result saved by a run without the variable.

    AIMX_NEAR_TC=1 python scripts/tc_check.py cfg1
    python scripts/tc_check.py cfg5-save ; AIMX_NEAR_TC=1 python scripts/tc_check.py cfg5-cmp
"""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import aimx_inputs as inp  # noqa: E402
from paper_2009_02281_b200 import AIMx  # noqa: E402

mode = sys.argv[1]
if mode == "cfg1":
    from oracle.aimx import from_config
    m = inp.make_mesh(1)
    orc = from_config(1)
    op = AIMx(m.vertices, m.triangles, (16, 16, 4), prec="c64")
    freqs = np.linspace(30e6, 450e6, 32)
    X = np.stack([inp.rhs_vector(1, i, op.N) for i in range(32)])
    Y = op.sweep(freqs, torch.as_tensor(X).to(torch.complex64).cuda()).cpu().numpy()
    errs = []
    for i, f in enumerate(freqs):
        orc.set_frequency(f)
        z = orc.matvec(X[i].astype(np.complex64).astype(np.complex128))
        errs.append(float(np.linalg.norm(Y[i] - z) / np.linalg.norm(z)))
    print("cfg1 sweep max rel-L2 vs oracle", max(errs), "stats", op.stats().get("batch_slots"))
else:
    c = inp.get_config(5)
    m = inp.make_mesh(5)
    op = AIMx(m.vertices, m.triangles, c.grid_n, prec="c64")
    freqs = np.asarray(c.freqs[:32])
    X = torch.as_tensor(np.stack([inp.rhs_vector(5, i, op.N) for i in range(32)])).to(torch.complex64).cuda()
    Y = op.sweep(freqs, X)
    torch.cuda.synchronize()
    t = time.time()
    for _ in range(10):
        op.sweep(freqs, X, Y)
    torch.cuda.synchronize()
    print("cfg5 32-point sweep ms", (time.time() - t) / 10 * 1e3)
    path = "/tmp/tc_ref.npy"
    if mode == "cfg5-save":
        np.save(path, Y.cpu().numpy())
    else:
        R = np.load(path)
        y = Y.cpu().numpy()
        print("cfg5 max column rel-L2 TC vs FMA", max(float(np.linalg.norm(y[i] - R[i]) / np.linalg.norm(R[i])) for i in range(32)))
