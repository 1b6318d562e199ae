"""Solved frequency points on the GPU (aimx_solve): cfg3 sphere (EFIE converges
with the static diagonal preconditioner), c64, tol 1e-4, restart 30.
Prints JSON: per-frequency iterations, relative residuals, and solved points/s."""
import json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import aimx_inputs as inp
from paper_2009_02281_b200 import AIMx
cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 3
c = inp.get_config(cfg)
m = inp.make_mesh(cfg)
op = AIMx(m.vertices, m.triangles, c.grid_n, prec="c64")
nf = min(len(c.freqs), 16)
freqs = c.freqs[:nf]
B = torch.as_tensor(np.stack([inp.rhs_vector(cfg, i, op.N) for i in range(nf)])).to(torch.complex64).cuda()
op.solve(freqs[:1], B[:1], tol=1e-4, restart=30, maxiter=50)   # warm-up
torch.cuda.synchronize()
t0 = time.perf_counter()
X, its, rr = op.solve(freqs, B, tol=1e-4, restart=30, maxiter=3000)
torch.cuda.synchronize()
dt = time.perf_counter() - t0
print(json.dumps({"cfg": cfg, "nf": nf, "seconds": dt, "solved_freq_pts_per_s": nf / dt,
                  "iterations": its.tolist(), "relres": rr.tolist(), "batch_slots": op.stats()["batch_slots"]}))
