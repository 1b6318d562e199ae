"""Slab-decomposed FFT through the C ABI, on one GPU.

The `world` ranks are emulated inside one context (aimx_setup_slab with no
NCCL id): every rank runs its own kernels on its own rows / kx slab, and the
two all-to-all exchanges are device copies between the ranks' exchange
buffers -- the same pack / unpack as the NCCL path.  The NCCL path itself runs
with world = 1 (one GPU).  Bar: the oracle, per north_star tolerance."""
import numpy as np
import pytest

import aimx_inputs as inp
from tests._parity import TOL, gpu_input_as_c128, make_gpu_op, rel_l2, to_gpu

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def orc1():
    from oracle.aimx import from_config
    return from_config(1)


@pytest.mark.parametrize("world", [2, 4])
@pytest.mark.parametrize("prec", ["c64", "c128"])
def test_slab_emulated_cfg1(world, prec, orc1):
    op = make_gpu_op(inp.make_mesh(1), (16, 16, 4), prec, slab=("emulate", world))
    for f in (150e6, 37.5e6):
        op.set_frequency(f)
        orc1.set_frequency(f)
        x = inp.rhs_vector(1, 2, op.N)
        xg = to_gpu(x, prec)
        xo = gpu_input_as_c128(x, prec)
        oA, oR = orc1.parts(xo)
        yA, yP = op.matvec_parts(xg)
        assert rel_l2(yA.cpu().numpy(), oA) <= TOL[prec]
        assert rel_l2(yP.cpu().numpy(), -oR) <= TOL[prec]
        assert rel_l2(op.matvec(xg).cpu().numpy(), orc1.combine(oA, oR)) <= TOL[prec]
    freqs = np.linspace(40e6, 300e6, 6)
    X = np.stack([inp.rhs_vector(1, i, op.N) for i in range(6)])
    Y = op.sweep(freqs, to_gpu(X, prec)).cpu().numpy()
    for i, f in enumerate(freqs):
        orc1.set_frequency(f)
        assert rel_l2(Y[i], orc1.matvec(gpu_input_as_c128(X[i], prec))) <= TOL[prec]


@pytest.mark.parametrize("world", [2, 4, 8])
def test_slab_emulated_ragged_closed_mesh(world):
    """Closed icosphere on a ragged grid: row blocks of 1-2 rows, the halo
    reaching across several ranks, unoccupied rows and planes."""
    from oracle.aimx import AIMxOracle
    m = inp.icosphere_mesh(2)
    n = (16, 8, 32)
    orc = AIMxOracle(m.vertices, m.triangles, n)
    op = make_gpu_op(m, n, "c128", slab=("emulate", world))
    for f in (30e6, 400e6):
        op.set_frequency(f)
        orc.set_frequency(f)
        x = np.random.default_rng(7).standard_normal(op.N) * (1 - 0.25j)
        yA, yP = op.matvec_parts(to_gpu(x, "c128"))
        oA, oR = orc.parts(x)
        assert rel_l2(yA.cpu().numpy(), oA) <= 1e-11
        assert rel_l2(yP.cpu().numpy(), -oR) <= 1e-11


def test_slab_nccl_single_rank(orc1):
    """The NCCL exchange path (grouped send/recv, all-reduce of owned rows)
    with one rank on this GPU."""
    from paper_2009_02281_b200 import nccl_unique_id
    nid = nccl_unique_id()
    op = make_gpu_op(inp.make_mesh(1), (16, 16, 4), "c128", slab=(0, 1, nid))
    op.set_frequency(150e6)
    orc1.set_frequency(150e6)
    x = inp.rhs_vector(1, 3, op.N)
    y = op.matvec(to_gpu(x, "c128")).cpu().numpy()
    assert rel_l2(y, orc1.matvec(x)) <= 1e-11
    freqs = np.linspace(50e6, 250e6, 3)
    X = np.stack([inp.rhs_vector(1, i, op.N) for i in range(3)])
    Y = op.sweep(freqs, to_gpu(X, "c128")).cpu().numpy()
    for i, f in enumerate(freqs):
        orc1.set_frequency(f)
        assert rel_l2(Y[i], orc1.matvec(X[i])) <= 1e-11


def test_slab_matches_single_context_cfg2():
    """Full-size cfg2 (bench configuration) with 4 emulated ranks equals the
    one-context path on the same inputs (both checked against the oracle
    elsewhere), batched sweep included."""
    c = inp.get_config(2)
    m = inp.make_mesh(2)
    one = make_gpu_op(m, c.grid_n, "c64")
    sl = make_gpu_op(m, c.grid_n, "c64", slab=("emulate", 4))
    freqs = c.freqs[:20]
    X = to_gpu(np.stack([inp.rhs_vector(2, i, one.N) for i in range(20)]), "c64")
    Y1 = one.sweep(freqs, X).cpu().numpy()
    Y2 = sl.sweep(freqs, X).cpu().numpy()
    for i in range(20):
        assert rel_l2(Y2[i], Y1[i]) <= 2e-6


def test_slab_cfg5_eight_ranks_vs_single_context():
    """configs[4] (8x8 patch array, 512x512x8 grid, ~400k RWG) with the 8-rank
    slab decomposition SURVEY 8(e) plans for it, emulated on this GPU, equals
    the one-context path (oracle-checked on the other configurations)."""
    c = inp.get_config(5)
    m = inp.make_mesh(5)
    one = make_gpu_op(m, c.grid_n, "c64")
    sl = make_gpu_op(m, c.grid_n, "c64", slab=("emulate", 8))
    freqs = c.freqs[:4]
    X = to_gpu(np.stack([inp.rhs_vector(5, i, one.N) for i in range(4)]), "c64")
    Y1 = one.sweep(freqs, X).cpu().numpy()
    Y2 = sl.sweep(freqs, X).cpu().numpy()
    for i in range(4):
        assert rel_l2(Y2[i], Y1[i]) <= 2e-6
