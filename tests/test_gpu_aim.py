"""Conventional AIM mode on the GPU vs the oracle (oracle/aim.py):
the per-frequency near correction D(k0) to fp64 rounding (c128) / fp32
storage (c64), and matvec / parts / sweep outputs within the north_star
tolerance; the mode's exclusions and its switch back to AIMx."""
import numpy as np
import pytest

import aimx_inputs as inp
from tests._parity import TOL, gpu_input_as_c128, make_gpu_op, rel_l2, to_gpu

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def orc1():
    from oracle.aimx import from_config
    return from_config(1)


@pytest.mark.parametrize("prec", ["c128", "c64"])
def test_aim_cfg1(prec, orc1):
    from oracle.aim import ConventionalAIM
    from paper_2009_02281_b200 import AIMxError
    aim = ConventionalAIM(orc1)
    op = make_gpu_op(inp.make_mesh(1), (16, 16, 4), prec)
    op.set_frequency(150e6)
    x = inp.rhs_vector(1, 5, op.N)
    xg = to_gpu(x, prec)
    xo = gpu_input_as_c128(x, prec)
    y_aimx = op.matvec(xg).cpu().numpy()
    with pytest.raises(AIMxError):
        op.aim_entries()                      # mode off
    op.set_conventional(True)                 # fills the bound frequency
    for f in (150e6, 37.5e6, 420e6):
        op.set_frequency(f)
        aim.set_frequency(f)
        da, dr = op.aim_entries()
        # D = L_d,NR - W H_d,NR P cancels: its imaginary part (the -j k0/(4 pi)
        # monopole term of both) is ~1e-4 of the terms', so fp64 rounding of
        # the terms shows up at ~1e-12 of |D|
        tol = 1e-11 if prec == "c128" else 1e-6
        assert rel_l2(da, aim.DA) <= tol and rel_l2(dr, aim.DR) <= tol
        yA, yP = op.matvec_parts(xg)
        oA, oR = aim.parts(xo)
        assert rel_l2(yA.cpu().numpy(), oA) <= TOL[prec]
        assert rel_l2(yP.cpu().numpy(), -oR) <= TOL[prec]
        assert rel_l2(op.matvec(xg).cpu().numpy(), orc1.combine(oA, oR)) <= TOL[prec]
    # a sweep runs frequency by frequency, each with its own near fill
    freqs = np.linspace(40e6, 360e6, 7)
    X = np.stack([inp.rhs_vector(1, 20 + i, op.N) for i in range(7)])
    Y = op.sweep(freqs, to_gpu(X, prec)).cpu().numpy()
    for i, f in enumerate(freqs):
        aim.set_frequency(f)
        assert rel_l2(Y[i], aim.matvec(gpu_input_as_c128(X[i], prec))) <= TOL[prec]
    import torch
    Xh = torch.as_tensor(X).to(op.cdtype).pin_memory()
    Yh = torch.empty_like(Xh).pin_memory()
    op.sweep_host(freqs, Xh, Yh)
    assert np.array_equal(Yh.numpy(), Y)
    # exclusions, and back to AIMx
    with pytest.raises(AIMxError):
        op.set_linear_term(True)
    # GMRES on the conventional-AIM system (one frequency at a time, each with
    # its near fill): the residual under the ORACLE's AIM operator
    Xs, its, rr = op.solve(freqs[:2], to_gpu(X[:2], prec), tol=1e-6 if prec == "c128" else 1e-4,
                           restart=30, maxiter=3000)
    Xs = Xs.cpu().numpy()
    for i in range(2):
        aim.set_frequency(freqs[i])
        b = gpu_input_as_c128(X[i], prec)
        res = np.linalg.norm(b - aim.matvec(Xs[i])) / np.linalg.norm(b)
        assert rr[i] <= (1e-6 if prec == "c128" else 1e-4) * (1 + 1e-6)
        assert res <= (1e-6 if prec == "c128" else 5e-4)
    op.set_conventional(False)
    op.set_frequency(150e6)
    assert np.array_equal(op.matvec(xg).cpu().numpy(), y_aimx)


def test_aim_cfg2_sampled_rows():
    """cfg2 (bench geometry, c64): D(k0) on sampled rows against the oracle's
    pair-by-pair evaluation."""
    from oracle.aim import dynamic_pair_entries, dynamic_precorrection_entries
    from oracle.aimx import from_config
    c = inp.get_config(2)
    orc = from_config(2, static=False)
    op = make_gpu_op(inp.make_mesh(2), c.grid_n, "c64")
    op.set_conventional(True)
    rows = np.sort(np.random.default_rng(9).choice(op.N, 12, replace=False))
    for f in (c.freqs[0], c.freqs[-1]):
        op.set_frequency(f)
        da, dr = op.aim_entries()
        k0 = 2 * np.pi * f / 299792458.0
        for m in rows:
            s = slice(orc.rowptr[m], orc.rowptr[m + 1])
            cols = orc.col[s]
            mm = np.full(cols.shape, m)
            la, yr = dynamic_pair_entries(orc.V, orc.T, orc.rwg, mm, cols, k0)
            pa, pr = dynamic_precorrection_entries(orc.Lam, orc.A, mm, cols, orc.order, orc.grid.h, k0)
            assert rel_l2(da[s], la - pa) <= 1e-5
            assert rel_l2(dr[s], yr - pr) <= 1e-5
