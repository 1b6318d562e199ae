"""Pins for oracle/kop.py (AIMx for the double-layer operator K, P:400-474;
SURVEY 8(f) NEXT #1 groundwork, oracle only this round).

* grad G against central differences of G (eq:ghgf) and the paper's Taylor
  coefficients (eq:ghgftaylor); grad G_d against grad G - grad G_s;
* the closed-form Q(r) = int (r - r')/R^3 against Duffy quadrature;
* the static PV entries of far pairs against a 7 x 7 product rule, and the
  symmetry of the exact PV part (the antisymmetric quadrature error shrinks
  under refinement);
* the residue term: antisymmetric, zero on the diagonal;
* K_s,P against the dense definition with explicit grid matrices;
* the grid convolution against the dense O(N_g^2) sum;
* AIMx K against the dense direct K on a closed icosphere (rel-L2 <= 1e-2);
* eq:gH00's printed scalar is the coefficient of rhat in the r -> 0 limit of
  grad G_d (so the vector self term is direction dependent and its +-rhat
  average, reading R23's 0, is the symmetric value); the gh00="literal" flag
  changes the grid K by exactly the self term's contribution.
"""
import numpy as np
import pytest

import aimx_inputs as inp
from oracle.kernels import G
from oracle.kop import (EPS3, AIMxK, DirectK, K_precorrection_entries, gH00_literal, grad_G, grad_G_d, grad_G_s,
                        grid_K, residue_entries, static_K_entries, triangle_Q)


@pytest.fixture(scope="module")
def sph():
    from oracle.aimx import AIMxOracle
    m = inp.icosphere_mesh(1, radius=0.5)
    return AIMxOracle(m.vertices, m.triangles, (8, 8, 8))


def test_grad_G_vs_central_differences():
    k0 = 3.0
    rv = np.random.default_rng(0).standard_normal((6, 3)) * 0.4
    e = 1e-6
    fd = np.stack([(G(k0, np.linalg.norm(rv + e * np.eye(3)[a], axis=-1))
                    - G(k0, np.linalg.norm(rv - e * np.eye(3)[a], axis=-1))) / (2 * e) for a in range(3)], -1)
    assert np.abs(grad_G(k0, rv) - fd).max() <= 1e-8 * np.abs(fd).max()
    assert np.abs(grad_G_d(k0, rv) - (grad_G(k0, rv) - grad_G_s(rv))).max() <= 1e-13 * np.abs(fd).max()


@pytest.mark.parametrize("k0,r", [(2.0, 1e-2), (5.0, 3e-3)])
def test_grad_G_taylor(k0, r):
    # eq:ghgftaylor: grad G = -rhat/(4 pi) (1/r^2 - (-j k0)^2/2! - 2 (-j k0)^3 r/3! + O(r^2))
    rhat = np.array([0.6, 0.0, 0.8])
    g = grad_G(k0, r * rhat)
    series = -(1 / r ** 2 - (-1j * k0) ** 2 / 2 - 2 * (-1j * k0) ** 3 * r / 6) / (4 * np.pi)
    assert np.allclose(g, series * rhat, rtol=(k0 * r) ** 2, atol=0)
    gd = grad_G_d(k0, r * rhat)                          # the frequency-dependent terms only
    assert np.allclose(gd, (series + 1 / (4 * np.pi * r * r)) * rhat, rtol=(k0 * r) ** 2 * 10, atol=0)


def _duffy(r, v0, v1, v2, f, q):
    x, w = np.polynomial.legendre.leggauss(q)
    x = 0.5 * (x + 1)
    w = 0.5 * w
    n = np.cross(v1 - v0, v2 - v0)
    n /= np.linalg.norm(n)
    rho = r - np.dot(r - v0, n) * n
    tot = 0.0
    for a, b in ((v0, v1), (v1, v2), (v2, v0)):
        a2 = np.dot(np.cross(a - rho, b - rho), n)
        U, Vv = np.meshgrid(x, x, indexing="ij")
        W = np.outer(w, w) * U * a2
        P = rho + U[..., None] * ((a - rho) + Vv[..., None] * (b - a))
        tot = tot + np.tensordot(W, f(P, r), axes=([0, 1], [0, 1]))
    return tot


@pytest.mark.parametrize("r", [[0.4, 0.3, 0.5], [2.0, 1.0, 0.3], [0.4, 0.35, 0.05], [-0.5, 0.2, 0.01],
                               [1.5, 1.5, 0.0]])
def test_Q_vs_duffy(r):
    v0, v1, v2 = np.array([0.0, 0, 0]), np.array([1.0, 0.1, 0]), np.array([0.3, 0.9, 0.05])
    r = np.array(r)
    q = triangle_Q(r[None], v0[None], v1[None], v2[None])[0]
    ref = _duffy(r, v0, v1, v2, lambda P, x: (x - P) / np.linalg.norm(x - P, axis=-1)[..., None] ** 3, 200)
    assert np.linalg.norm(q - ref) <= 1e-10 * np.linalg.norm(ref)


def test_static_far_pairs_vs_product_rule_and_symmetry(sph):
    from oracle.direct import _points
    op = sph
    pts, w, f, div = _points(op.V, op.T, op.rwg)
    P, W, F = pts.reshape(op.N, 14, 3), w.reshape(op.N, 14), f.reshape(op.N, 14, 3)

    def prod(a, b):
        g = grad_G_s(P[a][:, None, :] - P[b][None, :, :])
        return -np.einsum("i,ic,ijc,j->", W[a], F[a], np.cross(g, F[b][None, :, :]), W[b])
    far = [(0, 100), (7, 60), (30, 111)]
    for a, b in far:
        k = static_K_entries(op.V, op.T, op.rwg, [a, b], [b, a])
        assert k[0] == pytest.approx(prod(a, b), rel=1e-4)
        assert k[1] == pytest.approx(k[0], rel=1e-4)                 # symmetric
    # touching pairs: the antisymmetric part is quadrature error; refinement shrinks it
    N = op.N
    rows = np.repeat(np.arange(N), np.diff(op.rowptr))
    errs = []
    for ns in (1, 8):
        k = static_K_entries(op.V, op.T, op.rwg, rows, op.col, nsub_touch=ns)
        from oracle.static_near import transpose_perm
        kt = k[transpose_perm(op.rowptr, op.col)]
        errs.append(np.linalg.norm(k - kt) / np.linalg.norm(k))
    assert errs[1] < 0.3 * errs[0]


def test_residue_antisymmetric(sph):
    op = sph
    N = op.N
    m, n = np.meshgrid(np.arange(N), np.arange(N), indexing="ij")
    R = residue_entries(op.V, op.T, op.rwg, m.ravel(), n.ravel()).reshape(N, N)
    assert np.abs(R + R.T).max() <= 1e-14 * np.abs(R).max()
    assert np.abs(np.diag(R)).max() <= 1e-14 * np.abs(R).max() and np.count_nonzero(R) > 0


def test_K_precorrection_vs_dense_definition(sph):
    op = sph
    g = op.grid
    idx = np.arange(g.ng)
    ijk = np.stack([idx % g.n[0], (idx // g.n[0]) % g.n[1], idx // (g.n[0] * g.n[1])], axis=1)
    Hg = grad_G_s(g.h * (ijk[:, None, :] - ijk[None, :, :]).astype(float))      # [Ng, Ng, 3]
    Pd = [op.P[c].toarray() for c in range(3)]
    M = np.zeros((op.N, op.N))
    for c in range(3):
        for a in range(3):
            for b in range(3):
                if EPS3[c, a, b]:
                    M -= EPS3[c, a, b] * Pd[c].T @ Hg[..., a] @ Pd[b]
    rows = np.repeat(np.arange(op.N), np.diff(op.rowptr))
    kp = K_precorrection_entries(op.Lam, op.A, rows, op.col, op.order, g.h)
    assert np.abs(kp - M[rows, op.col]).max() <= 1e-12 * np.abs(M).max()


def test_grid_K_vs_dense_sum(sph):
    op = sph
    k0 = 2 * np.pi * 1.5e8 / 299792458.0
    g = op.grid
    idx = np.arange(g.ng)
    ijk = np.stack([idx % g.n[0], (idx // g.n[0]) % g.n[1], idx // (g.n[0] * g.n[1])], axis=1)
    Hg = grad_G(k0, g.h * (ijk[:, None, :] - ijk[None, :, :]).astype(float))
    x = np.random.default_rng(1).standard_normal(op.N) * (1 + 0.5j)
    Pd = [op.P[c].toarray() for c in range(3)]
    y = np.zeros(op.N, complex)
    for c in range(3):
        for a in range(3):
            for b in range(3):
                if EPS3[c, a, b]:
                    y -= EPS3[c, a, b] * Pd[c].T @ (Hg[..., a] @ (Pd[b] @ x))
    yk = grid_K(op, x, k0)
    assert np.linalg.norm(yk - y) <= 1e-12 * np.linalg.norm(y)


def test_aimx_K_vs_direct(sph):
    op = sph
    d = DirectK(op.V, op.T, op.rwg)
    ak = AIMxK(op)
    rng = np.random.default_rng(4)
    for f in (50e6, 150e6):
        k0 = 2 * np.pi * f / 299792458.0
        d.set_frequency(k0)
        for _ in range(3):
            x = rng.standard_normal(op.N) + 1j * rng.standard_normal(op.N)
            assert np.linalg.norm(ak.matvec(x, k0) - d.K @ x) <= 1e-2 * np.linalg.norm(d.K @ x)


def test_grid_K_through_the_radial_kernel(sph):
    # the planned device form: the curl of the gradient-kernel
    # convolution from two even-kernel convolutions, J and s x J
    from oracle.kop import grid_K_radial
    op = sph
    x = np.random.default_rng(6).standard_normal(op.N) * (1 - 0.3j)
    for f in (30e6, 300e6):
        k0 = 2 * np.pi * f / 299792458.0
        a, b = grid_K(op, x, k0), grid_K_radial(op, x, k0)
        assert np.linalg.norm(a - b) <= 1e-12 * np.linalg.norm(a)


def test_pmchwt_equal_media_reduces_to_doubled_blocks(sph):
    # eps_r = 1: both media are free space, so y_E = 2 Z J - 2 K_pv M and
    # y_H = 2 K_pv J + 2 Z / eta0^2 M (reading R27; the residues cancel)
    from oracle.kernels import C0, MU0
    from oracle.kop import pmchwt_matvec
    op = sph
    ak = AIMxK(op)
    rng = np.random.default_rng(9)
    x = rng.standard_normal(2 * op.N) + 1j * rng.standard_normal(2 * op.N)
    f = 120e6
    y = pmchwt_matvec(op, ak, f, 1.0, x)
    op.set_frequency(f)
    J, M = x[:op.N], x[op.N:]
    eta0 = MU0 * C0
    k0 = op.k0
    Kj, Km = ak.matvec(J, k0, residue=False), ak.matvec(M, k0, residue=False)
    assert np.linalg.norm(y[:op.N] - (2 * op.matvec(J) - 2 * Km)) <= 1e-12 * np.linalg.norm(y[:op.N])
    assert np.linalg.norm(y[op.N:] - (2 * Kj + 2 * op.matvec(M) / eta0 ** 2)) <= 1e-12 * np.linalg.norm(y[op.N:])


def test_rows_variants_equal_the_full_operators(sph):
    # the sampled-row forms used by the full-size GPU parity tests (cfg4):
    # C_K row by row and the grid part on the full grid give the same rows
    from oracle.kop import kop_rows, pmchwt_matvec, pmchwt_rows, static_K_rows
    op = sph
    ak = AIMxK(op)
    rows = np.array([0, 7, 33, op.N - 1])
    kr = static_K_rows(op, rows)
    rng = np.random.default_rng(17)
    x = rng.standard_normal(op.N) + 1j * rng.standard_normal(op.N)
    k0 = 2 * np.pi * 120e6 / 299792458.0
    for res in (True, False):
        full = ak.matvec(x, k0, residue=res)
        assert np.linalg.norm(kop_rows(op, kr, x, k0, residue=res) - full[rows]) <= 1e-12 * np.linalg.norm(full[rows])
    x2 = rng.standard_normal(2 * op.N) + 1j * rng.standard_normal(2 * op.N)
    y = pmchwt_matvec(op, ak, 120e6, 4.0, x2)
    yE, yH = pmchwt_rows(op, kr, 120e6, 4.0, x2)
    assert np.linalg.norm(yE - y[rows]) <= 1e-12 * np.linalg.norm(y[rows])
    assert np.linalg.norm(yH - y[op.N + rows]) <= 1e-12 * np.linalg.norm(y[op.N + rows])


@pytest.mark.parametrize("k0", [1.0, 7.5])
def test_gH00_printed_scalar_is_the_rhat_coefficient_of_the_limit(k0):
    """eq:gH00: (-j k0)^2 / (4 pi 2!) = lim_{r->0} grad G_d . rhat for
    every direction (eq:ghgftaylor's second term), while grad G_d itself tends
    to that scalar times rhat: opposite directions give opposite vectors, so
    the only direction-free value is their average, 0 (reading R23)."""
    s = gH00_literal(k0)
    assert np.isclose(s, -k0 * k0 / (8 * np.pi), rtol=1e-15, atol=0)
    rng = np.random.default_rng(5)
    for _ in range(5):
        rhat = rng.standard_normal(3)
        rhat /= np.linalg.norm(rhat)
        for eps in (1e-4, 1e-5):
            g = grad_G_d(k0, eps * rhat)
            assert np.allclose(g, s * rhat, rtol=10 * (k0 * eps), atol=0)
            gm = grad_G_d(k0, -eps * rhat)
            assert np.allclose(0.5 * (g + gm), 0.0, atol=abs(s) * 10 * (k0 * eps))


def test_grid_K_literal_gH00_flag_adds_exactly_the_self_term(sph):
    """gh00="literal" puts eq:gH00's scalar in every component of H_grad(0):
    Phi_c gains s sum_{a,b} eps_cab g_b, so y changes by
    -sum_c P_c^T (s sum_{a,b} eps_cab P_b x)."""
    op = sph
    k0 = 2 * np.pi * 3e8 / 299792458.0
    x = np.random.default_rng(9).standard_normal(op.N) * (1 - 0.25j)
    d = grid_K(op, x, k0, gh00="literal") - grid_K(op, x, k0)
    s = gH00_literal(k0)
    gb = [op.P[b] @ x for b in range(3)]
    ref = np.zeros(op.N, complex)
    for c in range(3):
        phi = sum(EPS3[c, a, b] * s * gb[b] for a in range(3) for b in range(3) if EPS3[c, a, b])
        ref -= op.P[c].T @ phi
    assert np.linalg.norm(d - ref) <= 1e-10 * np.linalg.norm(ref)
    with pytest.raises(ValueError):
        grid_K(op, x, k0, gh00="half")
