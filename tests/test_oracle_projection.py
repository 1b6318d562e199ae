"""Pins for oracle/projection.py (not gpu).

P:561 moment matching == polynomial interpolation: the projected point
sources reproduce every tensor moment x^a y^b z^c (a, b, c <= n) of the basis
function.  The reference integrals use an INDEPENDENT rule (collapsed
Gauss-Legendre from numpy.polynomial.legendre), not the oracle's monomial
expansion.
"""
import numpy as np
import pytest

import aimx_inputs as inp
from oracle import grid as G
from oracle.mesh import build_rwg
from oracle.projection import projection_weights


def _tri_rule(q):
    x, w = np.polynomial.legendre.leggauss(q)
    u = 0.5 * (x + 1)
    wu = 0.5 * w
    U, Vv = np.meshgrid(u, u, indexing="ij")
    WU, WV = np.meshgrid(wu, wu, indexing="ij")
    l1 = U.ravel()
    l2 = (Vv * (1 - U)).ravel()
    ww = (WU * WV * (1 - U)).ravel() * 2.0     # weights sum to 1 over the triangle
    return l1, l2, ww


def _moments(V, T, r, grid, A, n_idx, order):
    """int f_c t_x^a t_y^b t_z^c dS and int div f (...) by the independent rule."""
    l1, l2, ww = _tri_rule(10)
    p = order + 1
    out = np.zeros((4, p, p, p))
    for tri, sign, area, free in ((r.tp[n_idx], 1.0, r.area_p[n_idx], r.pp[n_idx]),
                                  (r.tm[n_idx], -1.0, r.area_m[n_idx], r.pm[n_idx])):
        v0, v1, v2 = V[T[tri]]
        pts = v0 + l1[:, None] * (v1 - v0) + l2[:, None] * (v2 - v0)
        t = (pts - grid.origin) / grid.h - A[n_idx]
        f = sign * r.length[n_idx] / (2 * area) * (pts - V[free])
        div = sign * r.length[n_idx] / area
        for a in range(p):
            for b in range(p):
                for c in range(p):
                    mono = t[:, 0] ** a * t[:, 1] ** b * t[:, 2] ** c
                    for ch in range(3):
                        out[ch, a, b, c] += area * np.sum(ww * f[:, ch] * mono)
                    out[3, a, b, c] += area * np.sum(ww * div * mono)
    return out


@pytest.mark.parametrize("cfg", [1, 3])
def test_projection_reproduces_tensor_moments(cfg):
    if cfg == 3:
        m = inp.icosphere_mesh(3)
        n = (24, 24, 24)
    else:
        m = inp.make_mesh(1)
        n = (16, 16, 4)
    r = build_rwg(m.vertices, m.triangles)
    g = G.grid_spec(m.vertices, n, 2)
    A = G.anchors(m.vertices, r, g)
    sel = np.arange(0, r.n, max(1, r.n // 40))
    from oracle.mesh import RWG
    Lam = projection_weights(m.vertices, m.triangles, r, g, A)
    p = 3
    s = np.arange(p ** 3)
    ti, tj, tk = s % p, (s // p) % p, s // (p * p)
    for nn in sel:
        ref = _moments(m.vertices, m.triangles, r, g, A, nn, 2)
        scale = np.abs(ref).max()
        for a in range(p):
            for b in range(p):
                for c in range(p):
                    mono = ti ** a * tj ** b * tk ** c
                    got = Lam[nn] @ mono
                    assert np.allclose(got, ref[:, a, b, c], rtol=0, atol=1e-13 * scale), (nn, a, b, c)


def test_projection_charge_neutral_and_planar_z_weights(cfg1_oracle):
    Lam = cfg1_oracle.Lam
    # sum_s Lambda^rho = int div f = 0
    assert np.max(np.abs(Lam[:, 3, :].sum(-1))) < 1e-15 * np.abs(Lam[:, 3]).max() * 30
    # planar mesh on node plane z = 1: z-Lagrange factors are exactly (0, 1, 0)
    p = 3
    k = np.arange(27) // 9
    assert np.all(Lam[:, :, k != 1] == 0.0)


def test_point_source_on_node_weights():
    # a tiny RWG centred on a node: weight concentrates on that node
    eps = 1e-5
    c = np.array([5.0, 5.0, 5.0])
    V = np.array([c + [0, -eps, 0], c + [0, eps, 0], c + [eps, 0, 0], c + [-eps, 0, 0]])
    T = np.array([[0, 1, 3], [1, 0, 2]])
    r = build_rwg(V, T)
    g = G.Grid((12, 12, 12), 2, 1.0, np.zeros(3))
    A = G.anchors(V, r, g)
    Lam = projection_weights(V, T, r, g, A)
    tot = np.abs(Lam[0, 0]).sum()
    centre = 1 + 3 * (1 + 3 * 1)
    # the x-current moment int f_x dS sits on the centre node up to O(eps)
    assert abs(Lam[0, 0, centre]) / tot > 1 - 1e-4
