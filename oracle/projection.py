"""Moment-matched projection weights P^(A), P^(phi) (oracle).  TEST INFRASTRUCTURE ONLY.

P:109-110  grid currents/charges "are chosen via moment-matching to generate
           approximately the same fields in the far region"
P:198      "P^(L) projects sources from the mesh to the AIM grid, ...
           W^(L) interpolates the computed potentials back onto the mesh"
P:561      "The moment-matching procedure of the AIM is equivalent to polynomial
           interpolation of the kernel"

Reading (R6-R7; AMB-5, AMB-6, AMB-7): the full tensor moment set
0 <= a, b, c <= n is matched on the (n+1)^3 stencil, a square system whose
solution is the Lagrange form

    Lambda^c_{n,(i,j,k)}   = integral over T+ u T- of f_{n,c}(r) l_i(x) l_j(y) l_k(z) dS
    Lambda^rho_{n,(i,j,k)} = integral over T+ u T- of (div f_n)  l_i(x) l_j(y) l_k(z) dS

with l_i the 1-D Lagrange polynomials on the stencil nodes (local coordinate
t = (x - o)/h - A, nodes t = 0..n).  W = P^T per channel (Galerkin testing).

The integrand is a polynomial of degree <= 3n + 1 in the barycentric
coordinates, so it is integrated EXACTLY by monomial expansion:
    integral_T lambda_1^a lambda_2^b dS = 2 A a! b! / (a + b + 2)!
(the CUDA library uses collapsed Gauss-Legendre quadrature instead; the two
share no code).  Output Lambda[N_b, 4, (n+1)^3], channels (x, y, z, rho),
node s = i + (n+1)(j + (n+1) k).
"""
from __future__ import annotations

import math

import numpy as np

from .grid import Grid
from .mesh import RWG


def _polymul(P: np.ndarray, Q: np.ndarray) -> np.ndarray:
    """Bivariate polynomial product; coefficient arrays [..., a, b] of
    lambda_1^a lambda_2^b."""
    dp = P.shape[-1] - 1
    dq = Q.shape[-1] - 1
    shape = np.broadcast_shapes(P.shape[:-2], Q.shape[:-2]) + (dp + dq + 1, dp + dq + 1)
    R = np.zeros(shape, dtype=np.float64)
    for a in range(dp + 1):
        for b in range(dp + 1 - a):
            R[..., a:a + dq + 1, b:b + dq + 1] += P[..., a:a + 1, b:b + 1] * Q
    return R


def _linear(c0, c1, c2) -> np.ndarray:
    P = np.zeros(np.shape(c0) + (2, 2))
    P[..., 0, 0] = c0
    P[..., 1, 0] = c1
    P[..., 0, 1] = c2
    return P


def _monomial_integrals(deg: int) -> np.ndarray:
    """M[a, b] = integral_T lambda_1^a lambda_2^b dS / (2A) = a! b! / (a+b+2)!."""
    M = np.zeros((deg + 1, deg + 1))
    for a in range(deg + 1):
        for b in range(deg + 1 - a):
            M[a, b] = math.factorial(a) * math.factorial(b) / math.factorial(a + b + 2)
    return M


def _lagrange_polys(t: np.ndarray, order: int) -> np.ndarray:
    """t: linear polys [B, 2, 2] -> l_i(t) as polys [B, n+1, n+1, n+1]."""
    p = order + 1
    B = t.shape[0]
    out = np.zeros((B, p, order + 1, order + 1))
    for i in range(p):
        acc = np.zeros((B, 1, 1))
        acc[:, 0, 0] = 1.0
        for j in range(p):
            if j == i:
                continue
            fac = t.copy()
            fac[:, 0, 0] -= j
            fac /= (i - j)
            acc = _polymul(acc, fac)
        out[:, i, : acc.shape[1], : acc.shape[2]] = acc
    return out


def _triangle_weights(V, tri_v, sigma, length, area, free_v, grid: Grid, A, order):
    """Weights of one triangle of each RWG in the batch: [B, 4, p^3]."""
    p = order + 1
    v0, v1, v2 = V[tri_v[:, 0]], V[tri_v[:, 1]], V[tri_v[:, 2]]
    B = v0.shape[0]
    lag = []
    for a in range(3):
        t0 = (v0[:, a] - grid.origin[a]) / grid.h - A[:, a]
        t1 = (v1[:, a] - grid.origin[a]) / grid.h - A[:, a]
        t2 = (v2[:, a] - grid.origin[a]) / grid.h - A[:, a]
        lag.append(_lagrange_polys(_linear(t0, t1 - t0, t2 - t0), order))
    # Q_{ijk} = l_i(x) l_j(y) l_k(z), as polys of degree 3n
    Lx = lag[0][:, None, None, :, :, :]   # index i last among stencil axes
    Ly = lag[1][:, None, :, None, :, :]
    Lz = lag[2][:, :, None, None, :, :]
    Q = _polymul(_polymul(Lz, Ly), Lx)    # [B, k, j, i, D, D]
    D = Q.shape[-1] - 1
    M = _monomial_integrals(D + 1)
    two_a = (2.0 * area)[:, None, None, None]
    m0 = np.einsum("bkjiuv,uv->bkji", Q, M[: D + 1, : D + 1]) * two_a
    m1 = np.einsum("bkjiuv,uv->bkji", Q, M[1: D + 2, : D + 1]) * two_a
    m2 = np.einsum("bkjiuv,uv->bkji", Q, M[: D + 1, 1: D + 2]) * two_a
    m0 = m0.reshape(B, p ** 3)   # flattening (k, j, i) gives s = i + p (j + p k)
    m1 = m1.reshape(B, p ** 3)
    m2 = m2.reshape(B, p ** 3)
    W = np.zeros((B, 4, p ** 3))
    pv = V[free_v]
    coef = sigma * length / (2.0 * area)
    for c in range(3):
        g0 = v0[:, c] - pv[:, c]
        g1 = v1[:, c] - v0[:, c]
        g2 = v2[:, c] - v0[:, c]
        W[:, c, :] = coef[:, None] * (g0[:, None] * m0 + g1[:, None] * m1 + g2[:, None] * m2)
    W[:, 3, :] = (sigma * length / area)[:, None] * m0
    return W


def projection_weights(V: np.ndarray, T: np.ndarray, rwg: RWG, grid: Grid,
                       A: np.ndarray, chunk: int = 8192) -> np.ndarray:
    V = np.asarray(V, dtype=np.float64)
    T = np.asarray(T, dtype=np.int64)
    p = grid.order + 1
    out = np.zeros((rwg.n, 4, p ** 3))
    for s in range(0, rwg.n, chunk):
        e = min(rwg.n, s + chunk)
        sl = slice(s, e)
        Wp = _triangle_weights(V, T[rwg.tp[sl]], 1.0, rwg.length[sl], rwg.area_p[sl],
                               rwg.pp[sl], grid, A[sl], grid.order)
        Wm = _triangle_weights(V, T[rwg.tm[sl]], -1.0, rwg.length[sl], rwg.area_m[sl],
                               rwg.pm[sl], grid, A[sl], grid.order)
        out[sl] = Wp + Wm
    return out
