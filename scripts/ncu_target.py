"""Short driver for ncu captures: setup one config, run a short sweep.

    python scripts/ncu_target.py --cfg 3 --nf 2 [--prec c64]
"""
import argparse, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import aimx_inputs as inp
from paper_2009_02281_b200 import AIMx
ap = argparse.ArgumentParser()
ap.add_argument("--cfg", type=int, default=3)
ap.add_argument("--nf", type=int, default=2)
ap.add_argument("--prec", default="c64")
a = ap.parse_args()
c = inp.get_config(a.cfg)
m = inp.make_mesh(a.cfg)
op = AIMx(m.vertices, m.triangles, c.grid_n, prec=a.prec)
dt = torch.complex64 if a.prec == "c64" else torch.complex128
nf = a.nf
X = torch.as_tensor(np.stack([inp.rhs_vector(a.cfg, i, op.N) for i in range(nf)])).to(dt).cuda()
Y = op.sweep(c.freqs[:nf], X)
torch.cuda.synchronize()
print("ok", a.cfg, a.prec, nf, float(Y.abs().sum()))
