"""Double-layer operator K on cfg3 (sphere, 122,880 RWG, 128^3): time of
aimx_matvec_kop next to aimx_matvec, and the c64 result against the c128 one
(the fp32 cancellation of the s-weighted channels).  JSON line."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import aimx_inputs as inp  # noqa: E402
from paper_2009_02281_b200 import AIMx  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 3
c = inp.get_config(cfg)
m = inp.make_mesh(cfg)
x = inp.rhs_vector(cfg, 0, 0) if False else None
out = {"cfg": cfg}
res = {}
for prec in ("c128", "c64"):
    op = AIMx(m.vertices, m.triangles, c.grid_n, prec=prec)
    dt = torch.complex64 if prec == "c64" else torch.complex128
    xv = torch.as_tensor(inp.rhs_vector(cfg, 0, op.N)).to(dt).cuda()
    op.set_kop(True)
    op.set_frequency(c.freqs[len(c.freqs) // 2])
    y = op.matvec_kop(xv)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10):
        op.matvec_kop(xv, y)
    e1.record()
    torch.cuda.synchronize()
    out[f"{prec}_kop_ms"] = e0.elapsed_time(e1) / 10
    yl = op.matvec(xv)
    e0.record()
    for _ in range(10):
        op.matvec(xv, yl)
    e1.record()
    torch.cuda.synchronize()
    out[f"{prec}_L_ms"] = e0.elapsed_time(e1) / 10
    res[prec] = y.cpu().numpy().astype(np.complex128)
    op.close()
out["c64_vs_c128_relL2"] = float(np.linalg.norm(res["c64"] - res["c128"]) / np.linalg.norm(res["c128"]))
print(json.dumps(out))
