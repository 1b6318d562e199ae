"""GPU parity on the 1024-point padded lines of cfg5's grid (1024 x 1024 x 16),
at a size the oracle finishes in seconds: elongated strips on 512 x 16 x 4
and 16 x 512 x 4 grids (padded lines of 1024 points along x, or along y).

* plate strips (one occupied z plane): the planar S3 path, k_xfwd / k_xinv
  <1024> or the planar y pass k_yconv_plane<1024> (cfg5's kernels), and the
  general 3-D path with AIMX_NO_PLANAR=1 (one-plane z pass);
* box strips (closed, 3 occupied planes): the general 3-D path with
  1024-point x passes, or the separate 1024-point y passes and the z pass.

Each against the fp64 oracle at the north_star tolerance, L_A x and L_phi x
separately, plus a 4-column sweep (the batched kernels).  Anchors and the
near CSR are bit-exact.
"""
import numpy as np
import pytest

import aimx_inputs as inp
from tests._parity import TOL, check_structure, gpu_input_as_c128, make_gpu_op, rel_l2, to_gpu

pytestmark = pytest.mark.gpu


def _mesh(kind, axis):
    long_, short = 20.0, 0.5          # metres; h = 20 / 509 from the long axis
    if kind == "plate":
        return (inp.plate_mesh(200, 5, long_, short) if axis == "x" else inp.plate_mesh(5, 200, short, long_))
    if axis == "x":
        return inp.box_mesh(200, 5, 1, (0.0, 0.0, 0.0), (long_, short, 0.04))
    return inp.box_mesh(5, 200, 1, (0.0, 0.0, 0.0), (short, long_, 0.04))


CASES = [("plate", "x", False), ("plate", "y", False), ("plate", "y", True), ("box", "x", False),
         ("box", "y", False)]


@pytest.mark.parametrize("prec", ["c64", "c128"])
@pytest.mark.parametrize("kind,axis,no_planar", CASES)
def test_1024_point_lines_vs_oracle(kind, axis, no_planar, prec, monkeypatch):
    from oracle.aimx import AIMxOracle
    m = _mesh(kind, axis)
    n = (512, 16, 4) if axis == "x" else (16, 512, 4)
    orc = AIMxOracle(m.vertices, m.triangles, n)
    if no_planar:
        monkeypatch.setenv("AIMX_NO_PLANAR", "1")
    op = make_gpu_op(m, n, prec)
    st = op.stats()
    assert st["planar"] == (kind == "plate" and not no_planar)
    check_structure(op, orc)
    for i, f in enumerate((150e6, 900e6)):
        op.set_frequency(f)
        orc.set_frequency(f)
        x = inp.rhs_vector(5, 100 + i, op.N)
        xg = to_gpu(x, prec)
        yA, yP = op.matvec_parts(xg)
        oA, oR = orc.parts(gpu_input_as_c128(x, prec))
        assert rel_l2(yA.cpu().numpy(), oA) <= TOL[prec]
        assert rel_l2(yP.cpu().numpy(), -oR) <= TOL[prec]
        assert rel_l2(op.matvec(xg).cpu().numpy(), orc.combine(oA, oR)) <= TOL[prec]
    # batched kernels: a 4-point sweep against the oracle per column
    freqs = np.array([100e6, 300e6, 500e6, 700e6])
    X = np.stack([inp.rhs_vector(5, 110 + i, op.N) for i in range(4)])
    Y = op.sweep(freqs, to_gpu(X, prec)).cpu().numpy()
    for i, f in enumerate(freqs):
        orc.set_frequency(f)
        assert rel_l2(Y[i], orc.matvec(gpu_input_as_c128(X[i], prec))) <= TOL[prec]
