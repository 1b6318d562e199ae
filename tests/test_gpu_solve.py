"""aimx_solve (batched GMRES, static diagonal preconditioner
P:340-359) against the oracle GMRES (oracle/gmres.py, pinned against LU):
the same solutions to the tolerance, comparable iteration counts, and the
library's residual checked with the ORACLE operator."""
import os

import numpy as np
import pytest

import aimx_inputs as inp
from tests._parity import gpu_input_as_c128, make_gpu_op, rel_l2, to_gpu

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def orc1():
    from oracle.aimx import from_config
    return from_config(1)


@pytest.mark.parametrize("prec,tol", [("c128", 1e-9), ("c64", 1e-4)])
def test_solve_cfg1_vs_oracle(prec, tol, orc1):
    from oracle.gmres import solve
    op = make_gpu_op(inp.make_mesh(1), (16, 16, 4), prec)
    freqs = np.array([40e6, 150e6, 290e6])
    B = np.stack([inp.rhs_vector(1, 10 + i, op.N) for i in range(3)])
    X, its, rr = op.solve(freqs, to_gpu(B, prec), tol=tol, restart=20, maxiter=3000)
    X = X.cpu().numpy()
    for i, f in enumerate(freqs):
        b = gpu_input_as_c128(B[i], prec)
        x_o, it_o, _ = solve(orc1, f, b, tol=1e-12, restart=40, maxiter=5000)      # reference solution
        orc1.set_frequency(f)
        res = np.linalg.norm(b - orc1.matvec(X[i])) / np.linalg.norm(b)         # oracle operator
        assert rr[i] <= tol * (1 + 1e-6)
        assert res <= (tol if prec == "c128" else 5 * tol)
        assert rel_l2(X[i], x_o) <= (1e-6 if prec == "c128" else 1e-2)
        _, it_t, _ = solve(orc1, f, b, tol=tol, restart=20, maxiter=3000)
        assert abs(int(its[i]) - it_t) <= max(2, it_t // 10)


def test_solve_cfg2_fixed_iterations_vs_oracle():
    """configs[1] (the bench's geometry: thin strips, electrically small at the
    low end, where the EFIE converges slowly), c64, one 5-point batch, a fixed
    budget of 2 restart cycles: the residual the library reports equals the
    residual of its X under the ORACLE operator, and is close to the oracle
    GMRES's after the same number of iterations."""
    from oracle.aimx import from_config
    from oracle.gmres import solve
    c = inp.get_config(2)
    op = make_gpu_op(inp.make_mesh(2), c.grid_n, "c64")
    freqs = c.freqs[[0, 30, 60, 90, 99]]
    B = np.stack([inp.rhs_vector(2, i, op.N) for i in range(5)])
    X, its, rr = op.solve(freqs, to_gpu(B, "c64"), tol=1e-12, restart=30, maxiter=60)
    assert np.all(its == 60) and np.all(rr < 1.0)
    orc = from_config(2, workers=len(os.sched_getaffinity(0)))   # static fill over the host's cores
    X = X.cpu().numpy()
    for i in (0, 4):
        orc.set_frequency(freqs[i])
        b = gpu_input_as_c128(B[i], "c64")
        res = np.linalg.norm(b - orc.matvec(X[i])) / np.linalg.norm(b)
        assert abs(res - rr[i]) <= 1e-3 * rr[i] + 1e-6
        _, it_o, hist = solve(orc, freqs[i], b, tol=1e-12, restart=30, maxiter=60)
        assert it_o == 60 and abs(hist[-1] - rr[i]) <= 0.2 * hist[-1]


def test_solve_zero_rhs_and_errors():
    import torch
    from paper_2009_02281_b200 import AIMxError
    op = make_gpu_op(inp.make_mesh(1), (16, 16, 4), "c64")
    Z = torch.zeros((2, op.N), dtype=torch.complex64, device="cuda")
    X, its, rr = op.solve([1e8, 2e8], Z)
    assert torch.count_nonzero(X) == 0 and np.all(its == 0)
    with pytest.raises(AIMxError):
        op.solve([0.0], Z[:1])
