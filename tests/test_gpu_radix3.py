"""GPU parity on padded FFT lengths 3 * 2^k (48, 96, 192): cfg4's 96^3 grid
pads to 192 points per axis.  The register FFT engine factors them as
R1 x 24 (24 = 3 x 8: a radix-3 stage, fft_reg.cuh dft24); the x passes, the
y passes, the TMA z pass, the planar y pass and the spectrum's even-extension
passes all run on them.  Against the fp64 oracle at the north_star tolerance
(L_A x and L_phi x separately), and cfg4 (the 0.5 m cube, 60,552 RWG, 96^3)
at full size on sampled rows."""
import numpy as np
import pytest

import aimx_inputs as inp
from tests._parity import TOL, check_structure, gpu_input_as_c128, make_gpu_op, rel_l2, to_gpu

pytestmark = pytest.mark.gpu


CASES = [
    ("box", (24, 48, 96)),      # x 48, y 96, z 192 (TMA z pass, separate y passes)
    ("box", (96, 24, 24)),      # x 192, y / z 48
    ("plate", (96, 48, 4)),     # planar: x 192, planar y pass 96
    ("sphere", (24, 24, 24)),   # 48 on every axis, W = 192 not a multiple of the pass's 128 lines
]


def _mesh(kind, n):
    if kind == "sphere":
        return inp.icosphere_mesh(2, radius=0.5)
    if kind == "plate":
        return inp.plate_mesh(40, 20, 1.0, 0.5)
    ext = np.array(n, float) / max(n) * 0.9          # box filling the grid
    return inp.box_mesh(max(2, n[0] // 4), max(2, n[1] // 4), max(2, n[2] // 4), (0.0, 0.0, 0.0), tuple(ext))


@pytest.mark.parametrize("prec", ["c64", "c128"])
@pytest.mark.parametrize("kind,n", CASES)
def test_radix3_lengths_vs_oracle(kind, n, prec):
    from oracle.aimx import AIMxOracle
    m = _mesh(kind, n)
    orc = AIMxOracle(m.vertices, m.triangles, n)
    op = make_gpu_op(m, n, prec)
    check_structure(op, orc)
    for i, f in enumerate((60e6, 240e6)):
        op.set_frequency(f)
        orc.set_frequency(f)
        x = inp.rhs_vector(4, 100 + i, op.N)
        xg = to_gpu(x, prec)
        yA, yP = op.matvec_parts(xg)
        oA, oR = orc.parts(gpu_input_as_c128(x, prec))
        assert rel_l2(yA.cpu().numpy(), oA) <= TOL[prec]
        assert rel_l2(yP.cpu().numpy(), -oR) <= TOL[prec]
    freqs = np.array([80e6, 160e6, 320e6])
    X = np.stack([inp.rhs_vector(4, 110 + i, op.N) for i in range(3)])
    Y = op.sweep(freqs, to_gpu(X, prec)).cpu().numpy()
    for i, f in enumerate(freqs):
        orc.set_frequency(f)
        assert rel_l2(Y[i], orc.matvec(gpu_input_as_c128(X[i], prec))) <= TOL[prec]


def test_cfg4_fullsize_L_c64():
    """cfg4 (the cube, 96^3 grid, padded 192): bit-exact structures over the
    whole problem, C on sampled rows, L_A x / L_phi x / Z x on 32 sampled rows
    (the oracle's grid part on the full grid) at the first and last frequency."""
    from tests.test_gpu_fullsize import _fullsize
    c = inp.get_config(4)
    _fullsize(4, "c64", [c.freqs[0], c.freqs[-1]], 32)
