"""cfg3 (closed PEC sphere, 122,880 RWG, 128^3): GMRES to 1e-4 with the EFIE
(frequencies batched) and with the CFIE (eq:CFIEdis; one frequency at a
time).  Seeded complex-Gaussian right-hand sides.  JSON lines."""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import aimx_inputs as inp  # noqa: E402
from paper_2009_02281_b200 import AIMx  # noqa: E402

cfg = 3
c = inp.get_config(cfg)
m = inp.make_mesh(cfg)
freqs = np.asarray(c.freqs)[[0, 5, 10, 15]]
op = AIMx(m.vertices, m.triangles, c.grid_n, prec="c64")
B = torch.as_tensor(inp.rhs_matrix(cfg, op.N, [0, 5, 10, 15])).to(torch.complex64).cuda()
for mode in ("efie", "cfie"):
    if mode == "cfie":
        op.set_cfie(True)
    torch.cuda.synchronize()
    t = time.perf_counter()
    X, its, rr = op.solve(freqs, B, tol=1e-4, restart=30, maxiter=int(sys.argv[1]) if len(sys.argv) > 1 else 600)
    torch.cuda.synchronize()
    print(json.dumps({"mode": mode, "freqs_hz": freqs.tolist(), "iterations": its.tolist(),
                      "relres": rr.tolist(), "seconds": time.perf_counter() - t}), flush=True)
