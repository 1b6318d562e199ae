"""Small GPU-vs-oracle check per config / precision (debug helper)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import aimx_inputs as inp
from oracle.aimx import AIMxOracle
from paper_2009_02281_b200 import AIMx
cases = [a.split(":") for a in sys.argv[1:]] or [["ico", "c64"]]
for name, prec in cases:
    if name == "ico":
        m = inp.icosphere_mesh(2); n = (16, 8, 32)
    elif name == "cfg1":
        m = inp.make_mesh(1); n = (16, 16, 4)
    elif name == "strip":   # cfg2-like long thin grid, small
        m = inp.box_mesh(40, 4, 1, (0, 0, 0), (20e-3, 0.2e-3, 0.02e-3)); n = (64, 16, 4)
    elif name == "big":
        m = inp.icosphere_mesh(3); n = (256, 32, 8)
    orc = AIMxOracle(m.vertices, m.triangles, n)
    op = AIMx(m.vertices, m.triangles, n, prec=prec)
    f = 3e8 if name != "strip" else 10e9
    op.set_frequency(f); orc.set_frequency(f)
    x = np.random.default_rng(0).standard_normal(op.N) + 0.3j
    dt = torch.complex64 if prec == "c64" else torch.complex128
    yA, yP = op.matvec_parts(torch.as_tensor(x).to(dt).cuda())
    torch.cuda.synchronize()
    oA, oR = orc.parts(x.astype(np.complex64).astype(np.complex128) if prec == "c64" else x)
    eA = np.linalg.norm(yA.cpu().numpy() - oA) / np.linalg.norm(oA)
    eR = np.linalg.norm(yP.cpu().numpy() + oR) / np.linalg.norm(oR)
    print(name, prec, n, "errA %.2e errPhi %.2e" % (eA, eR), flush=True)
