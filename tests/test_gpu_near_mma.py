"""S4+S5 on the tensor cores (k_interp_near_mma: c64 launches of 8 to 32
columns, mma.sync tf32 with the 3-term split) against the fp64 oracle, one
column per frequency, at every column bucket (8, 16, 32) and ragged counts,
on a planar mesh (3 stored channels) and a closed mesh (4 channels).
The kernel is opt-in (AIMX_NEAR_MMA=1): measured slower than the FMA kernel
on B200, kept with its parity tests as the measured variant.

Bar: rel-L2 2e-5 per output vector (north_star, c64), the same as every c64
path; the tf32 split keeps ~2^-21 relative per product.
"""
import numpy as np
import pytest

import aimx_inputs as inp
from tests._parity import TOL, gpu_input_as_c128, make_gpu_op, rel_l2, to_gpu

pytestmark = pytest.mark.gpu


@pytest.fixture(autouse=True)
def _mma_on(monkeypatch):
    monkeypatch.setenv("AIMX_NEAR_MMA", "1")   # read by the library at setup


def _sweep_vs_oracle(mesh, n, freqs, batches, seed):
    from oracle.aimx import AIMxOracle
    orc = AIMxOracle(mesh.vertices, mesh.triangles, n)
    op = make_gpu_op(mesh, n, "c64")
    nf = len(freqs)
    X = np.random.default_rng(seed).standard_normal((nf, op.N)) * (1 - 0.7j) \
        + 0.3j * np.random.default_rng(seed + 1).standard_normal((nf, op.N))
    Xg = to_gpu(X, "c64")
    Xo = gpu_input_as_c128(X, "c64")
    ref = []
    for i, f in enumerate(freqs):
        orc.set_frequency(f)
        ref.append(orc.matvec(Xo[i]))
    worst = 0.0
    for b in batches:
        Y = op.sweep(freqs, Xg, batch=b).cpu().numpy()
        for i in range(nf):
            e = rel_l2(Y[i], ref[i])
            worst = max(worst, e)
            assert e <= TOL["c64"], (b, i, e)
    op.close()
    return worst


def test_mma_near_planar_mesh_all_buckets():
    """cfg1's planar patch mesh (phi stores x, y, rho): batches 8, 13, 16, 29, 32."""
    freqs = np.linspace(40e6, 420e6, 32)
    _sweep_vs_oracle(inp.make_mesh(1), (16, 16, 4), freqs, (8, 13, 16, 29, 32), 11)


def test_mma_near_closed_mesh_all_buckets():
    """A closed icosphere on a ragged grid (phi stores all four channels)."""
    freqs = np.linspace(30e6, 400e6, 32)
    _sweep_vs_oracle(inp.icosphere_mesh(2), (16, 8, 32), freqs, (9, 16, 32), 21)


def test_mma_near_equals_fma_kernel_to_rounding():
    """The tensor-core kernel against the FMA kernel (single-column launches
    always take the FMA kernel): 32-column sweep vs one column at a time."""
    op = make_gpu_op(inp.make_mesh(1), (16, 16, 4), "c64")
    freqs = np.linspace(50e6, 350e6, 32)
    X = to_gpu(np.stack([inp.rhs_vector(1, 40 + i, op.N) for i in range(32)]), "c64")
    y32 = op.sweep(freqs, X, batch=32).cpu().numpy()
    y1 = op.sweep(freqs, X, batch=1).cpu().numpy()
    for i in range(32):
        assert rel_l2(y32[i], y1[i]) <= 1e-6, i
    op.close()
