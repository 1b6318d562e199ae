"""GPU parity of the single-column S4+S5 kernel (k_interp_near1 and its warp-private form
k_interp_near1w: c64, lanes split an entry's rows; eq:LAIMx P:283, eq:EFIEAIMx P:288, W = P^T P:198)
against the fp64 oracle, in both of its chunk-length variants (32-slot
contexts: half-length chunks, 8 CTAs per SM; fewer slots: full-length chunks),
on a planar mesh (3 stored channels) and a closed mesh (4 channels), combined
and in parts, and against the entry-per-lane kernel it replaces
(AIMX_NEAR1_OLD=1 at setup).

Bar: rel-L2 2e-5 per output vector (north_star, c64); the two kernels differ
only in summation order (<= 1e-6).
"""
import numpy as np
import pytest

import aimx_inputs as inp
from tests._parity import TOL, gpu_input_as_c128, make_gpu_op, rel_l2, to_gpu

pytestmark = pytest.mark.gpu

MESHES = {
    "planar": lambda: (inp.make_mesh(1), (16, 16, 4)),
    "closed": lambda: (inp.icosphere_mesh(2), (16, 8, 32)),
}


# (slots, AIMX_NEAR1_WARP): 32 slots -> the warp-private form k_interp_near1w
# (default) or the CTA form k_interp_near1<., HALF>; 8 slots -> k_interp_near1
@pytest.mark.parametrize("slots,warp", [(32, "1"), (32, "0"), (8, "1")])
@pytest.mark.parametrize("which", ["planar", "closed"])
def test_near1_matvec_vs_oracle_and_old_kernel(which, slots, warp, monkeypatch):
    from oracle.aimx import AIMxOracle
    mesh, n = MESHES[which]()
    monkeypatch.setenv("AIMX_BATCH", str(slots))      # read by the library at setup
    monkeypatch.setenv("AIMX_NEAR1_WARP", warp)
    op = make_gpu_op(mesh, n, "c64")
    assert op.stats()["batch_slots"] == slots
    monkeypatch.setenv("AIMX_NEAR1_OLD", "1")
    old = make_gpu_op(mesh, n, "c64")
    orc = AIMxOracle(mesh.vertices, mesh.triangles, n)
    rng = np.random.default_rng(7 + slots)
    for f in (90e6, 310e6):
        x = rng.standard_normal(op.N) * (1 - 0.6j) + 0.4j * rng.standard_normal(op.N)
        xg = to_gpu(x, "c64")
        orc.set_frequency(f)
        ref = orc.matvec(gpu_input_as_c128(x, "c64"))
        op.set_frequency(f)
        old.set_frequency(f)
        y = op.matvec(xg).cpu().numpy()
        yo = old.matvec(xg).cpu().numpy()
        assert rel_l2(y, ref) <= TOL["c64"], (which, slots, f, rel_l2(y, ref))
        assert rel_l2(y, yo) <= 1e-6, (which, slots, f, rel_l2(y, yo))
        # parts (y^A, y^rho unscaled): the PARTS instantiation
        pa, pr = op.matvec_parts(xg)
        qa, qr = old.matvec_parts(xg)
        assert rel_l2(pa.cpu().numpy(), qa.cpu().numpy()) <= 1e-6
        assert rel_l2(pr.cpu().numpy(), qr.cpu().numpy()) <= 1e-6
    op.close()
    old.close()
