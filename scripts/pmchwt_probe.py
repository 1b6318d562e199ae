"""cfg4 on the B200: the dielectric cube (eps_r = 4, side 0.5 m, 40,368
triangles, 60,552 RWG per current) with PMCHWT (aimx_matvec_pmchwt) on
BASELINE's 96^3 grid (padded 192, radix 3), K through the gradient-of-kernel
spectra (and the radial form with AIMX_K_RADIAL=1 for comparison): setup
time, PMCHWT matvec time, and c64 against c128.  JSON line."""
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

m = inp.make_mesh(4)
n = (96, 96, 96)
f = 350e6                       # mid-band of cfg4's 100-600 MHz
out = {"mesh": "cfg4 cube", "grid": list(n), "eps_r": 4.0, "f_hz": f}
res = {}
for prec in ("c64", "c128", "c64_radial"):
    if prec == "c64_radial":
        os.environ["AIMX_K_RADIAL"] = "1"
    t0 = time.perf_counter()
    op = AIMx(m.vertices, m.triangles, n, prec=prec[:3] if prec != "c128" else "c128")
    op.set_kop(True)
    out[f"{prec}_kop_grad"] = op.stats()["kop_grad"]
    torch.cuda.synchronize()
    out[f"{prec}_setup_s"] = time.perf_counter() - t0
    N = op.N
    rng = np.random.default_rng(4)
    x = rng.standard_normal(2 * N) + 1j * rng.standard_normal(2 * N)
    x[N:] /= 376.73
    dt = torch.complex128 if prec == "c128" else torch.complex64
    xg = torch.as_tensor(x).to(dt).cuda()
    op.set_frequency(f)
    y = op.matvec_pmchwt(4.0, xg)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5):
        op.matvec_pmchwt(4.0, xg, y)
    e1.record()
    torch.cuda.synchronize()
    out[f"{prec}_pmchwt_ms"] = e0.elapsed_time(e1) / 5
    out["N_rwg"] = N
    res[prec] = y.cpu().numpy().astype(np.complex128)
    op.close()
    del op
    torch.cuda.empty_cache()
N = out["N_rwg"]
for name, sl in (("E", slice(0, N)), ("H", slice(N, 2 * N))):
    for k in ("c64", "c64_radial"):
        out[f"{k}_vs_c128_relL2_{name}"] = float(np.linalg.norm(res[k][sl] - res["c128"][sl]) /
                                                 np.linalg.norm(res["c128"][sl]))
print(json.dumps(out))
