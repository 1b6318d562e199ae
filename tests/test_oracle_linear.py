"""Pins for oracle/linear_term.py (the linear-term modification).

* G_lin against the paper's Taylor coefficient (eq:linterm, golden) and the
  remainder G_d - k0^2 G_lin against the next Taylor terms (a wrong sign or
  factor leaves an O(k0^2 r) remainder);
* the closed-form R potentials against brute-force Duffy quadrature;
* the overlap pattern against a brute-force triangle intersection;
* the lin precorrection against the dense definition W H_lin P;
* the assembled entries (analytic inner) against the same outer rule with a
  brute-force inner integral;
* the self-term error with and without the modification against the dense
  direct reference (fig:selferrors P:643-646).
"""
import json
import os

import numpy as np
import pytest

import aimx_inputs as inp
from oracle.kernels import G_d
from oracle.linear_term import (G_lin, H_lin_block, lin_pair_entries, lin_precorrection_entries, overlap_csr,
                                triangle_R_potentials)
from oracle.mesh import build_rwg
from oracle.static_near import RADON7_BARY, RADON7_W, _rwg_triangles

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "paper_fixed_points.json")))


def test_G_lin_is_the_taylor_r_term():
    # eq:hgftaylor P:217 coefficient of r^1 at k0 = 2 (golden, l = 2)
    k0 = GOLD["taylor_coefficients"]["k0"]
    c2 = [c for c in GOLD["taylor_coefficients"]["coef"] if c["l"] == 2][0]
    assert k0 * k0 * G_lin(1.0) == pytest.approx(c2["re"], rel=1e-14)
    assert c2["im"] == 0.0


@pytest.mark.parametrize("k0,r", [(1.0, 1e-2), (3.0, 2e-3), (20.0, 1e-3)])
def test_remainder_after_lin_is_cubic_and_higher(k0, r):
    # G_d - k0^2 G_lin = -j k0/(4 pi) + j k0^3 r^2/(24 pi) + k0^4 r^3/(96 pi) + O(r^4)
    rem = G_d(k0, r) - k0 * k0 * G_lin(r) - (-1j * k0 / (4 * np.pi))
    x = k0 * r
    assert rem.imag == pytest.approx(k0 ** 3 * r * r / (24 * np.pi), rel=x * x / 10 + 1e-9)
    assert rem.real == pytest.approx(k0 ** 4 * r ** 3 / (96 * np.pi), rel=x * x / 10 + 1e-7)


def _duffy(r, v0, v1, v2, f, q):
    x, w = np.polynomial.legendre.leggauss(q)
    x = 0.5 * (x + 1)
    w = 0.5 * w
    n = np.cross(v1 - v0, v2 - v0)
    n /= np.linalg.norm(n)
    rho = r - np.dot(r - v0, n) * n
    tot = 0.0
    for a, b in ((v0, v1), (v1, v2), (v2, v0)):
        a2 = np.dot(np.cross(a - rho, b - rho), n)       # signed 2 x area of (rho, a, b)
        U, Vv = np.meshgrid(x, x, indexing="ij")
        W = np.outer(w, w) * U * a2
        P = rho + U[..., None] * ((a - rho) + Vv[..., None] * (b - a))
        tot = tot + np.tensordot(W, f(P, r, rho), axes=([0, 1], [0, 1]))
    return tot


TRI = (np.array([0.0, 0.0, 0.0]), np.array([1.0, 0.1, 0.0]), np.array([0.3, 0.9, 0.05]))


@pytest.mark.parametrize("r,q,tol", [
    ("centroid", 48, 1e-12),
    ("above", 48, 1e-12),
    ("vertex", 48, 1e-12),
    ("edge_mid", 48, 1e-12),
    ([2.0, 2.0, 0.3], 48, 1e-12),
    ([-0.5, 0.2, 0.01], 150, 1e-12),
    ("near_edge", 400, 1e-9),
])
def test_R_potentials_vs_duffy(r, q, tol):
    v0, v1, v2 = TRI
    c = (v0 + v1 + v2) / 3
    r = {"centroid": c, "above": c + np.array([0, 0, 0.2]), "vertex": v0, "edge_mid": 0.5 * (v0 + v1),
         "near_edge": 0.5 * (v0 + v1) + np.array([0, 0, 1e-3])}.get(r, r) if isinstance(r, str) else np.array(r)
    J0, J1, rho = triangle_R_potentials(r[None], v0[None], v1[None], v2[None])
    b0 = _duffy(r, v0, v1, v2, lambda P, r, rho: np.linalg.norm(P - r, axis=-1), q)
    b1 = _duffy(r, v0, v1, v2, lambda P, r, rho: (P - rho) * np.linalg.norm(P - r, axis=-1)[..., None], q)
    assert J0[0] == pytest.approx(b0, rel=tol)
    assert np.linalg.norm(J1[0] - b1) <= tol * np.linalg.norm(b1) + 1e-15


def test_overlap_pattern_bruteforce():
    m = inp.make_mesh(1)
    r = build_rwg(m.vertices, m.triangles)
    rowptr, col = overlap_csr(r)
    for i in range(r.n):
        ti = {int(r.tp[i]), int(r.tm[i])}
        ref = [j for j in range(r.n) if ti & {int(r.tp[j]), int(r.tm[j])}]
        assert list(col[rowptr[i]:rowptr[i + 1]]) == ref
        assert i in ref and len(ref) <= 5


def test_lin_precorrection_equals_dense_definition(cfg1_oracle):
    import scipy.sparse as sp
    op = cfg1_oracle
    rowptr, col = overlap_csr(op.rwg)
    rows = np.repeat(np.arange(op.N), np.diff(rowptr))
    la, yr = lin_precorrection_entries(op.Lam, op.A, rows, col, op.order, op.grid.h)
    # dense H_lin on the grid: H_lin[g, g'] = -h |i - i'| / (8 pi)
    g = op.grid
    idx = np.arange(g.ng)
    ijk = np.stack([idx % g.n[0], (idx // g.n[0]) % g.n[1], idx // (g.n[0] * g.n[1])], axis=1)
    D = np.sqrt(((ijk[:, None, :] - ijk[None, :, :]) ** 2).sum(-1)) * g.h
    H = -D / (8 * np.pi)
    Pd = [op.P[c].toarray() for c in range(4)]
    LAd = sum(Pd[c].T @ H @ Pd[c] for c in range(3))
    YRd = Pd[3].T @ H @ Pd[3]
    assert np.max(np.abs(la - LAd[rows, col])) <= 1e-12 * np.abs(LAd).max()
    assert np.max(np.abs(yr - YRd[rows, col])) <= 1e-12 * np.abs(YRd).max()
    # the block form: H_lin(0) = 0 and H_lin symmetric in the offset
    B = H_lin_block(np.array([0, 0, 0]), op.order, op.grid.h)
    assert np.all(np.diag(B) == 0) and np.array_equal(B, B.T)


def test_lin_entries_vs_bruteforce_inner():
    m = inp.make_mesh(1)
    V, T = m.vertices, m.triangles
    r = build_rwg(V, T)
    rowptr, col = overlap_csr(r)
    pairs = [(0, c) for c in col[rowptr[0]:rowptr[1]]] + [(7, 7), (40, int(col[rowptr[40] + 1]))]
    rows = np.array([p[0] for p in pairs])
    cols = np.array([p[1] for p in pairs])
    la, yr = lin_pair_entries(V, T, r, rows, cols)
    verts, area, free, coef, div = _rwg_triangles(np.asarray(V, float), np.asarray(T), r)
    for i, (mm, nn) in enumerate(pairs):
        ra = rr = 0.0
        for sm in range(2):
            pts = RADON7_BARY @ verts[mm, sm]
            for q in range(7):
                wq = RADON7_W[q] * area[mm, sm]
                fm = coef[mm, sm] * (pts[q] - free[mm, sm])
                for sn in range(2):
                    v0, v1, v2 = verts[nn, sn]
                    Rf = lambda P, x, rho: np.linalg.norm(P - x, axis=-1)
                    j0 = _duffy(pts[q], v0, v1, v2, Rf, 60)
                    jf = _duffy(pts[q], v0, v1, v2,
                                lambda P, x, rho: (P - free[nn, sn]) * np.linalg.norm(P - x, axis=-1)[..., None], 60)
                    ra += wq * np.dot(fm, coef[nn, sn] * jf) * (-1 / (8 * np.pi))
                    rr += wq * div[mm, sm] * div[nn, sn] * j0 * (-1 / (8 * np.pi))
        assert la[i] == pytest.approx(ra, rel=1e-8, abs=1e-12 * abs(rr))
        assert yr[i] == pytest.approx(rr, rel=1e-8)
    # |r - r'| is conditionally negative definite and an RWG's charge sums to
    # zero, so int int div f div f R < 0 and the scalar self term (kernel -R/(8 pi)) is > 0
    assert np.all(yr[rows == cols] > 0)


@pytest.fixture(scope="module")
def cfg1_direct_split(cfg1_oracle):
    from oracle.direct import DirectEFIE
    return DirectEFIE(cfg1_oracle.V, cfg1_oracle.T, cfg1_oracle.rwg, lin_split=True)


def _diag_parts(op):
    a_d = np.empty(op.N, complex)
    r_d = np.empty(op.N, complex)
    for m in range(op.N):
        e = np.zeros(op.N, complex)
        e[m] = 1
        a, r = op.parts(e)
        a_d[m], r_d[m] = a[m], r[m]
    return a_d, r_d


def _delta_L(op, d):
    a, r = _diag_parts(op)
    da = np.max(np.abs(a - np.diag(d.LA)) / np.abs(np.diag(d.LA)))
    dr = np.max(np.abs(r - np.diag(d.YR)) / np.abs(np.diag(d.YR)))
    return max(da, dr)


@pytest.mark.parametrize("f_hz", [50e6, 150e6])
def test_self_term_error_with_linear_term(cfg1_oracle, cfg1_direct_split, f_hz):
    # the modification reduces the self-term error, "below 1e-5"
    # on the fine end (mean edge 0.019 lambda0 at 50 MHz); at 150 MHz (0.057
    # lambda0) the gain is still > 30x
    from oracle.aimx import from_config
    op = from_config(1)
    d = cfg1_direct_split
    d.set_frequency(f_hz)
    op.set_frequency(f_hz)
    base = _delta_L(op, d)
    op.set_linear_term(True)
    lin = _delta_L(op, d)
    assert base < GOLD["self_term_error"]["max_rel_diag_error"]
    if f_hz <= 50e6:
        assert lin < GOLD["self_term_error_lin"]["max_rel_diag_error"]
    assert lin * 30 < base


def test_direct_split_agrees_with_plain_direct(cfg1_oracle, cfg1_direct, cfg1_direct_split):
    # the same operator with a different quadrature of the r term: the 7 x 7
    # product rule's kink error is O(k0^2 h^3) relative
    d1 = cfg1_direct_split
    d1.set_frequency(150e6)
    assert np.linalg.norm(d1.LA - cfg1_direct.LA) <= 1e-3 * np.linalg.norm(d1.LA)
    assert np.linalg.norm(d1.YR - cfg1_direct.YR) <= 1e-3 * np.linalg.norm(d1.YR)
