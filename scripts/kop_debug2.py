"""Locate the 24^3 K mismatch (dev tool)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import aimx_inputs as inp
from oracle.aimx import AIMxOracle
from oracle.kop import AIMxK, K_precorrection_entries, residue_entries, static_K_entries, grid_K
from oracle.static_near import symmetrize
from tests._parity import make_gpu_op, rel_l2, to_gpu, gpu_input_as_c128
for n in ((16, 16, 16), (24, 24, 24), (20, 20, 20), (24, 16, 16), (16, 24, 16), (16, 16, 24)):
    m = inp.icosphere_mesh(2, radius=0.5)
    orc = AIMxOracle(m.vertices, m.triangles, n)
    ak = AIMxK(orc)
    op = make_gpu_op(m, n, "c128")
    rows = np.repeat(np.arange(orc.N), np.diff(orc.rowptr))
    try:
        ck = op.K_static()
        print(n, "C_K err", rel_l2(ck, np.asarray(ak.C[rows, orc.col]).ravel()), flush=True)
    except Exception as e:
        print(n, "C_K failed", e, flush=True)
    x = np.random.default_rng(11).standard_normal(orc.N) + 1j * np.random.default_rng(12).standard_normal(orc.N)
    f = 50e6; k0 = 2 * np.pi * f / 299792458.0
    op.set_frequency(f); orc.set_frequency(f)
    z = op.matvec(to_gpu(x, "c128")).cpu().numpy()
    print(n, "L err", rel_l2(z, orc.matvec(x)), flush=True)
    op.set_kop(True); op.set_frequency(f)
    y = op.matvec_kop(to_gpu(x, "c128")).cpu().numpy()
    g = grid_K(orc, x, k0)
    print(n, "K err", rel_l2(y, ak.matvec(x, k0)), "grid-part-only err", rel_l2(y - ak.C @ x, g), flush=True)
