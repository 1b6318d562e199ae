"""Right-hand sides per second at one frequency: aimx_matvec_multi (batched)
against back-to-back single matvecs, cfg2 and cfg3 (c64).  JSON lines."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import aimx_inputs as inp  # noqa: E402
from paper_2009_02281_b200 import AIMx  # noqa: E402

for cfg in (2, 3):
    c = inp.get_config(cfg)
    m = inp.make_mesh(cfg)
    op = AIMx(m.vertices, m.triangles, c.grid_n, prec="c64")
    S = op.stats()["batch_slots"]
    n = 4 * S
    X = torch.as_tensor(inp.rhs_matrix(cfg, op.N, range(n))).to(torch.complex64).cuda()
    Y = torch.empty_like(X)
    op.set_frequency(c.freqs[0])
    op.matvec_multi(X, Y)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    op.matvec_multi(X, Y)
    e1.record()
    torch.cuda.synchronize()
    multi = e0.elapsed_time(e1)
    e0.record()
    for i in range(n):
        op.matvec(X[i], Y[i])
    e1.record()
    torch.cuda.synchronize()
    single = e0.elapsed_time(e1)
    print(json.dumps({"cfg": cfg, "slots": S, "nrhs": n, "multi_rhs_per_s": n / (multi / 1e3),
                      "single_rhs_per_s": n / (single / 1e3)}), flush=True)
    op.close()
