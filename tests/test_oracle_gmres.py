"""Pins of the oracle GMRES (oracle/gmres.py) -- independent of its code:
the dense level-0 AIMx matrix of cfg1 (unit-vector matvecs) solved by LU, the
true residual of the returned x, monotone residual estimates, exactness after
N steps on a small system, and the preconditioner's definition on the static
self terms."""
import numpy as np
import pytest

import aimx_inputs as inp


@pytest.fixture(scope="module")
def orc1():
    from oracle.aimx import from_config
    return from_config(1)


def test_small_dense_system_exact_after_n_steps():
    from oracle.gmres import gmres
    rng = np.random.default_rng(1)
    n = 12
    A = rng.standard_normal((n, n)) + 1j * rng.standard_normal((n, n)) + 4 * np.eye(n)
    b = rng.standard_normal(n) + 1j * rng.standard_normal(n)
    Minv = 1.0 / np.diag(A)
    x, it, hist = gmres(lambda v: A @ v, b, Minv, tol=1e-13, restart=n, maxiter=n)
    assert it <= n
    assert np.linalg.norm(x - np.linalg.solve(A, b)) <= 1e-10 * np.linalg.norm(x)
    assert all(h2 <= h1 * (1 + 1e-12) for h1, h2 in zip(hist, hist[1:]))   # minimal residual: monotone


def test_restarted_matches_lu_on_cfg1(orc1):
    """cfg1 at 150 MHz: the dense AIMx matrix (column j = Z e_j) solved by LU
    versus restarted GMRES(20) to 1e-10."""
    from oracle.gmres import solve
    orc1.set_frequency(150e6)
    N = orc1.N
    Z = np.stack([orc1.matvec(np.eye(N)[j]) for j in range(N)], axis=1)
    b = inp.rhs_vector(1, 7, N)
    x_lu = np.linalg.solve(Z, b)
    x, it, hist = solve(orc1, 150e6, b, tol=1e-10, restart=20, maxiter=2000)
    assert np.linalg.norm(b - Z @ x) / np.linalg.norm(b) <= 1e-9      # true residual
    assert np.linalg.norm(x - x_lu) / np.linalg.norm(x_lu) <= 1e-6
    assert it < 2000


def test_preconditioner_is_static_self_terms(orc1):
    from oracle.gmres import preconditioner, static_diagonal
    from oracle.kernels import MU0
    orc1.set_frequency(150e6)
    dA, dR = static_diagonal(orc1)
    LA = orc1.LA_NR
    for m in (0, 17, orc1.N - 1):
        lo, hi = orc1.rowptr[m], orc1.rowptr[m + 1]
        k = lo + list(orc1.col[lo:hi]).index(m)
        assert dA[m] == LA[k] and dR[m] == orc1.YR_NR[k]
    assert np.all(dA > 0)                                   # self terms of L_A are positive
    M = preconditioner(orc1, dA, dR)
    k0 = orc1.k0
    assert np.allclose(M, -1j * orc1.omega * MU0 * (dA - dR / k0 ** 2), rtol=0, atol=0)


def test_zero_rhs(orc1):
    from oracle.gmres import solve
    x, it, hist = solve(orc1, 150e6, np.zeros(orc1.N, complex))
    assert it == 0 and not np.any(x)
