"""Where the end-to-end sweep (aimx_sweep_host) spends its time on cfg
$E2E_CFG (default 2):
copies alone (H2D, D2H, both), the device-resident sweep, and the host sweep
wall time, each averaged over a few repetitions.  Prints one JSON line."""
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

CFG = int(os.environ.get("E2E_CFG", "2"))
c = inp.get_config(CFG)
m = inp.make_mesh(CFG)
op = AIMx(m.vertices, m.triangles, c.grid_n, order=c.order, near_cells=c.near_cells, prec="c64")
freqs = c.freqs
Xh = torch.from_numpy(inp.rhs_matrix(CFG, op.N, np.arange(len(freqs)))).to(torch.complex64).pin_memory()
Yh = torch.empty_like(Xh).pin_memory()
X = Xh.cuda()
Y = torch.empty_like(X)
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def wall(fn, n=10):
    fn()
    torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(n):
        fn()
        torch.cuda.synchronize()
    return 1e3 * (time.perf_counter() - t) / n


def both():
    with torch.cuda.stream(s1):
        X.copy_(Xh, non_blocking=True)
    with torch.cuda.stream(s2):
        Yh.copy_(Y, non_blocking=True)


out = {
    "h2d_ms": wall(lambda: X.copy_(Xh, non_blocking=True)),
    "d2h_ms": wall(lambda: Yh.copy_(Y, non_blocking=True)),
    "both_ms": wall(both),
    "sweep_device_wall_ms": wall(lambda: op.sweep(freqs, X, Y)),
    "sweep_host_wall_ms": wall(lambda: op.sweep_host(freqs, Xh, Yh)),
    "bytes_each_way": int(Xh.numel() * 8),
}
plans = sys.argv[1].split(";") if len(sys.argv) > 1 else ["25,25,25,25", "4,32,32,32", "4,32,32,28,4",
                                                          "8,32,32,28", "2,32,32,32,2", "16,32,32,20", "12,32,32,24"]
for plan in plans:
    os.environ["AIMX_SWEEP_PLAN"] = plan
    out[f"host[{plan}]"] = wall(lambda: op.sweep_host(freqs, Xh, Yh), 20)
    out[f"dev[{plan}]"] = wall(lambda: op.sweep(freqs, X, Y), 20)
    del os.environ["AIMX_SWEEP_PLAN"]
print(json.dumps(out))
