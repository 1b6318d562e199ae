"""K (gradient / radial form) against the oracle on icospheres (dev tool)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import aimx_inputs as inp
from oracle.aimx import AIMxOracle
from oracle.kop import AIMxK
from tests._parity import make_gpu_op, rel_l2, to_gpu, gpu_input_as_c128
for sub, n in ((2, (16, 16, 16)), (2, (24, 24, 24)), (2, (32, 32, 32)), (2, (48, 48, 48))):
    m = inp.icosphere_mesh(sub, radius=0.5)
    orc = AIMxOracle(m.vertices, m.triangles, n, static=False)
    ak = AIMxK(orc)
    x = np.random.default_rng(11).standard_normal(orc.N) + 1j * np.random.default_rng(12).standard_normal(orc.N)
    for prec in ("c128", "c64"):
        for form in ("grad", "radial"):
            if form == "radial":
                os.environ["AIMX_K_RADIAL"] = "1"
            else:
                os.environ.pop("AIMX_K_RADIAL", None)
            op = make_gpu_op(m, n, prec)
            op.set_kop(True)
            st = op.stats()
            f = 50e6
            op.set_frequency(f)
            k0 = 2 * np.pi * f / 299792458.0
            y = op.matvec_kop(to_gpu(x, prec)).cpu().numpy()
            ref = ak.matvec(gpu_input_as_c128(x, prec), k0)
            print(n, prec, form, st["kop_grad"], st["occupied_planes"], "K err", rel_l2(y, ref), flush=True)
