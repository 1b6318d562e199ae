"""Small end-to-end run for compute-sanitizer: cfg1 (c64, c128) matvec, parts,
batched sweep, and the 2-rank emulated slab path."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import aimx_inputs as inp
from paper_2009_02281_b200 import AIMx
m = inp.make_mesh(1)
for prec in ("c64", "c128"):
    for slab in (None, ("emulate", 2)):
        op = AIMx(m.vertices, m.triangles, (16, 16, 4), prec=prec, slab=slab)
        dt = torch.complex64 if prec == "c64" else torch.complex128
        x = torch.as_tensor(inp.rhs_vector(1, 0, op.N)).to(dt).cuda()
        op.set_frequency(150e6)
        y = op.matvec(x)
        yA, yP = op.matvec_parts(x)
        X = torch.stack([x] * 5)
        Y = op.sweep(np.linspace(50e6, 300e6, 5), X)
        torch.cuda.synchronize()
        print(prec, slab, float(y.abs().sum()), float(Y.abs().sum()))
        op.close()
print("ok")
