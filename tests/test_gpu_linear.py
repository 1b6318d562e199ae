"""Linear-term modification on the GPU, through the C ABI, vs the
oracle (oracle/linear_term.py): the overlap pattern bit-exact, C_lin within
fp64 rounding (c128) / fp32 storage (c64), and every output of the modified
matvec, parts, sweep, slab and solve paths within the north_star tolerance."""
import numpy as np
import pytest

import aimx_inputs as inp
from tests._parity import TOL, gpu_input_as_c128, make_gpu_op, rel_l2, to_gpu

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def orc1():
    from oracle.aimx import from_config
    o = from_config(1)
    o.set_linear_term(True)
    return o


@pytest.fixture(scope="module", params=["c128", "c64"])
def gpu1(request):
    op = make_gpu_op(inp.make_mesh(1), (16, 16, 4), request.param)
    return op, request.param


def _dense_lin(orc):
    cols = np.full((orc.N, 5), -1, np.int32)
    ca = np.zeros((orc.N, 5))
    cr = np.zeros((orc.N, 5))
    for m in range(orc.N):
        s = slice(orc.lin_rowptr[m], orc.lin_rowptr[m + 1])
        k = s.stop - s.start
        cols[m, :k] = orc.lin_col[s]
        ca[m, :k] = orc.CAl[s]
        cr[m, :k] = orc.CRl[s]
    return cols, ca, cr


def test_linear_entries(gpu1, orc1):
    op, prec = gpu1
    from paper_2009_02281_b200 import AIMxError
    with pytest.raises(AIMxError):       # AIMX_E_STATE before the first enable
        op.linear_entries()
    assert not op.linear_term
    op.set_linear_term(True)
    assert op.linear_term
    cols, ca, cr = op.linear_entries()
    rc, rca, rcr = _dense_lin(orc1)
    assert np.array_equal(cols, rc)
    tol = 1e-12 if prec == "c128" else 1e-6
    assert rel_l2(ca, rca) <= tol and rel_l2(cr, rcr) <= tol
    op.set_linear_term(False)


@pytest.mark.parametrize("f", [150e6, 37.5e6, 400e6])
def test_linear_matvec_and_parts(gpu1, orc1, f):
    op, prec = gpu1
    op.set_frequency(f)
    orc1.set_frequency(f)
    x = inp.rhs_vector(1, 4, op.N)
    xg = to_gpu(x, prec)
    xo = gpu_input_as_c128(x, prec)
    y_off = op.matvec(xg).cpu().numpy()
    op.set_linear_term(True)
    y = op.matvec(xg).cpu().numpy()
    yA, yP = op.matvec_parts(xg)
    op.set_linear_term(False)
    assert np.array_equal(op.matvec(xg).cpu().numpy(), y_off)   # off again: the unmodified path
    oA, oR = orc1.parts(xo)
    z = orc1.combine(oA, oR)
    assert rel_l2(y, z) <= TOL[prec]
    assert rel_l2(yA.cpu().numpy(), oA) <= TOL[prec]
    assert rel_l2(yP.cpu().numpy(), -oR) <= TOL[prec]
    if prec == "c128":
        # the correction itself (y_on - y_off) to fp64 rounding
        orc1.lin = False
        z_off = orc1.matvec(xo)
        orc1.lin = True
        assert rel_l2(y - y_off, z - z_off) <= 1e-8


@pytest.mark.parametrize("batch", [0, 5])
def test_linear_sweep(gpu1, orc1, batch):
    op, prec = gpu1
    op.set_linear_term(True)
    freqs = np.linspace(20e6, 480e6, 21)
    X = np.stack([inp.rhs_vector(1, 30 + i, op.N) for i in range(21)])
    Y = op.sweep(freqs, to_gpu(X, prec), batch=batch).cpu().numpy()
    op.set_linear_term(False)
    for i, f in enumerate(freqs):
        orc1.set_frequency(f)
        assert rel_l2(Y[i], orc1.matvec(gpu_input_as_c128(X[i], prec))) <= TOL[prec], i


@pytest.mark.parametrize("world", [2, 4])
def test_linear_slab_emulated(orc1, world):
    op = make_gpu_op(inp.make_mesh(1), (16, 16, 4), "c128", slab=("emulate", world))
    op.set_linear_term(True)
    for f in (150e6, 37.5e6):
        op.set_frequency(f)
        orc1.set_frequency(f)
        x = inp.rhs_vector(1, 9, op.N)
        oA, oR = orc1.parts(x)
        yA, yP = op.matvec_parts(to_gpu(x, "c128"))
        assert rel_l2(yA.cpu().numpy(), oA) <= TOL["c128"]
        assert rel_l2(yP.cpu().numpy(), -oR) <= TOL["c128"]
    freqs = np.linspace(40e6, 300e6, 6)
    X = np.stack([inp.rhs_vector(1, i, op.N) for i in range(6)])
    Y = op.sweep(freqs, to_gpu(X, "c128")).cpu().numpy()
    for i, f in enumerate(freqs):
        orc1.set_frequency(f)
        assert rel_l2(Y[i], orc1.matvec(X[i])) <= TOL["c128"]


def test_linear_static_cache(tmp_path, orc1):
    """A context whose static matrices come from a cache rebuilds the geometry
    for C_lin and gives the same entries."""
    m = inp.make_mesh(1)
    a = make_gpu_op(m, (16, 16, 4), "c128")
    path = str(tmp_path / "s.bin")
    a.save_static(path)
    b = make_gpu_op(m, (16, 16, 4), "c128", static_cache=path)
    a.set_linear_term(True)
    b.set_linear_term(True)
    ea, eb = a.linear_entries(), b.linear_entries()
    for u, v in zip(ea, eb):
        assert np.array_equal(u, v)


def test_linear_cfg2_fullsize_rows():
    """cfg2 (bench workload) in its c64 launch configuration with the
    modification on: the 100-point sweep vs the oracle on sampled rows."""
    from oracle.aimx import from_config
    c = inp.get_config(2)
    orc = from_config(2, static=False)
    orc.set_linear_term(True)
    op = make_gpu_op(inp.make_mesh(2), c.grid_n, "c64")
    op.set_linear_term(True)
    cols, ca, cr = op.linear_entries()
    rc, rca, rcr = _dense_lin(orc)
    assert np.array_equal(cols, rc)
    assert rel_l2(ca, rca) <= 1e-6 and rel_l2(cr, rcr) <= 1e-6
    freqs = c.freqs
    X = np.stack([inp.rhs_vector(2, i, op.N) for i in range(len(freqs))])
    Y = op.sweep(freqs, to_gpu(X, "c64")).cpu().numpy()
    rows = np.sort(np.random.default_rng(2).choice(op.N, 6, replace=False))
    for i in (0, 24, 99):
        orc.set_frequency(freqs[i])
        _, _, z = orc.matvec_rows(gpu_input_as_c128(X[i], "c64"), rows)
        assert rel_l2(Y[i][rows], z) <= TOL["c64"], i


def test_linear_solve_cfg1(orc1):
    """aimx_solve with the modification on solves the modified system: the
    library's residual under the ORACLE's modified operator, and the solution
    against the oracle GMRES on the same operator."""
    from oracle.gmres import solve
    op = make_gpu_op(inp.make_mesh(1), (16, 16, 4), "c128")
    op.set_linear_term(True)
    freqs = np.array([60e6, 240e6])
    B = np.stack([inp.rhs_vector(1, 50 + i, op.N) for i in range(2)])
    X, its, rr = op.solve(freqs, to_gpu(B, "c128"), tol=1e-9, restart=20, maxiter=3000)
    X = X.cpu().numpy()
    for i, f in enumerate(freqs):
        x_o, _, _ = solve(orc1, f, B[i], tol=1e-12, restart=40, maxiter=5000)
        orc1.set_frequency(f)
        res = np.linalg.norm(B[i] - orc1.matvec(X[i])) / np.linalg.norm(B[i])
        assert rr[i] <= 1e-9 * (1 + 1e-6) and res <= 1e-9
        assert rel_l2(X[i], x_o) <= 1e-6
