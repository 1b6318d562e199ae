"""Static near-region matrix L_s,NR by direct integration with G_s (oracle).
TEST INFRASTRUCTURE ONLY.

P:265-269  eq:Lmatdecomp2: the singularity of G is contained entirely in the
           sparse, frequency-independent L_s,NR, "computed accurately with
           direct integration"
P:297      change (a): L_s,NR and L_s,P "must be assembled using the kernel G_s"
P:312,317  singularity "subtraction or cancellation techniques"
P:184      the gradient is transferred to the testing function, so the scalar
           part pairs div f_m with div f_n

Entries (AMB-13: L_phi = -y^rho):
    L^A_s[m,n]   = sum_{T in m, T' in n} int_T f_m(r) . int_T' f_n(r') G_s(R) dS' dS
    y^rho_s[m,n] = sum_{T in m, T' in n} int_T div f_m int_T' div f_n G_s(R) dS' dS

Recipe (paper silent, AMB-9, R9): the inner integral over the
source triangle is analytic for every pair (the closed-form potential integrals
of 1/R and (rho' - rho)/R over a flat triangle, Wilton et al. / Graglia form),
using
    int_T' (r' - p') / R dS' = I1 + (rho - p') I0,
rho the projection of r onto the plane of T'; the outer integral uses the
7-point degree-5 symmetric rule; the result is symmetrised,
L <- (L + L^T) / 2.  The log terms use ln(R + s) = ln(R0^2 / (R - s)) for
s < 0 (cancellation-free) and are dropped when R0 = 0 (their factor is 0).
"""
from __future__ import annotations

import math

import numpy as np

from .kernels import FOUR_PI
from .mesh import RWG

# 7-point degree-5 rule on a triangle (barycentric points, weights sum to 1)
_S15 = math.sqrt(15.0)
_A1 = (6.0 - _S15) / 21.0
_A2 = (6.0 + _S15) / 21.0
_W1 = (155.0 - _S15) / 1200.0
_W2 = (155.0 + _S15) / 1200.0
RADON7_BARY = np.array([
    [1 / 3, 1 / 3, 1 / 3],
    [_A1, _A1, 1 - 2 * _A1], [_A1, 1 - 2 * _A1, _A1], [1 - 2 * _A1, _A1, _A1],
    [_A2, _A2, 1 - 2 * _A2], [_A2, 1 - 2 * _A2, _A2], [1 - 2 * _A2, _A2, _A2],
])
RADON7_W = np.array([9.0 / 40.0, _W1, _W1, _W1, _W2, _W2, _W2])


def _dot(a, b):
    return np.einsum("...i,...i->...", a, b)


def _logsum(R, s, R0sq, live):
    """ln(R + s), cancellation-free; 0 where the factor in front is 0 (~live)."""
    pos = s >= 0.0
    arg = np.where(pos, R + s, R0sq / np.where(pos, 1.0, R - s))
    arg = np.where(live, arg, 1.0)
    return np.log(arg)


def triangle_potentials(r, v0, v1, v2):
    """Closed-form I0 = int_T 1/R dS' and I1 = int_T (rho' - rho)/R dS' over the
    flat triangle (v0, v1, v2) for observation points r (all arrays [..., 3]).
    Returns (I0, I1, rho)."""
    e1 = v1 - v0
    e2 = v2 - v0
    nrm = np.cross(e1, e2)
    nhat = nrm / np.linalg.norm(nrm, axis=-1, keepdims=True)
    d = _dot(r - v0, nhat)
    rho = r - d[..., None] * nhat
    ad = np.abs(d)
    I0 = np.zeros(d.shape)
    I1 = np.zeros(r.shape)
    for va, vb in ((v0, v1), (v1, v2), (v2, v0)):
        ev = vb - va
        L = np.linalg.norm(ev, axis=-1)
        shat = ev / L[..., None]
        mhat = np.cross(shat, nhat)            # outward in-plane edge normal
        sm = _dot(va - rho, shat)
        sp_ = _dot(vb - rho, shat)
        t0 = _dot(va - rho, mhat)              # > 0 when rho is inside
        R0sq = t0 * t0 + d * d
        Rm = np.linalg.norm(r - va, axis=-1)
        Rp = np.linalg.norm(r - vb, axis=-1)
        live = R0sq > (1e-14 * L) ** 2
        f2 = _logsum(Rp, sp_, R0sq, live) - _logsum(Rm, sm, R0sq, live)
        hasd = ad > 0.0
        den_p = np.where(hasd, R0sq + ad * Rp, 1.0)
        den_m = np.where(hasd, R0sq + ad * Rm, 1.0)
        beta = np.where(hasd, np.arctan(t0 * sp_ / den_p) - np.arctan(t0 * sm / den_m), 0.0)
        I0 = I0 + t0 * f2 - ad * beta
        I1 = I1 + 0.5 * mhat * (R0sq * f2 + sp_ * Rp - sm * Rm)[..., None]
    return I0, I1, rho


def _rwg_triangles(V, T, rwg: RWG):
    """Per RWG and side (0 = T+, 1 = T-): vertices [N,2,3,3], sign, free vertex,
    coefficient l/(2A) and divergence sigma l / A."""
    tri = np.stack([T[rwg.tp], T[rwg.tm]], axis=1)        # [N,2,3]
    verts = V[tri]                                         # [N,2,3,3]
    sign = np.array([1.0, -1.0])
    area = np.stack([rwg.area_p, rwg.area_m], axis=1)
    free = np.stack([V[rwg.pp], V[rwg.pm]], axis=1)        # [N,2,3]
    coef = sign[None, :] * rwg.length[:, None] / (2.0 * area)   # sigma l/(2A)
    div = sign[None, :] * rwg.length[:, None] / area            # sigma l/A
    return verts, area, free, coef, div


def static_pair_entries(V, T, rwg: RWG, rows, cols):
    """Unsymmetrised entries (outer integral on the test RWG m = rows, inner on
    the source RWG n = cols).  Returns (LA, Yrho) float64 arrays."""
    V = np.asarray(V, np.float64)
    T = np.asarray(T, np.int64)
    verts, area, free, coef, div = _rwg_triangles(V, T, rwg)
    rows = np.asarray(rows)
    cols = np.asarray(cols)
    LA = np.zeros(rows.shape[0])
    YR = np.zeros(rows.shape[0])
    for sm in range(2):          # test triangle of m
        tv = verts[rows, sm]     # [P,3,3]
        rq = np.einsum("qk,pkc->pqc", RADON7_BARY, tv)     # [P,7,3] outer points
        wq = RADON7_W[None, :] * area[rows, sm][:, None]   # [P,7]
        fm = coef[rows, sm][:, None, None] * (rq - free[rows, sm][:, None, :])
        for sn in range(2):      # source triangle of n
            # inner integrals at all outer points
            sv = verts[cols, sn][:, None, :, :]            # [P,1,3,3]
            I0, I1, rho = triangle_potentials(rq, sv[..., 0, :], sv[..., 1, :], sv[..., 2, :])
            inner = coef[cols, sn][:, None, None] * (I1 + (rho - free[cols, sn][:, None, :]) * I0[..., None])
            LA += (wq * _dot(fm, inner)).sum(axis=1) / FOUR_PI
            YR += div[rows, sm] * div[cols, sn] * (wq * I0).sum(axis=1) / FOUR_PI
    return LA, YR


def _chunk_job(args):
    V, T, rwg, rows, cols = args
    return static_pair_entries(V, T, rwg, rows, cols)


def static_near_matrices(V, T, rwg: RWG, rowptr, col, chunk: int = 200000, workers: int = 1):
    """Symmetrised L^A_s,NR and y^rho_s,NR on the near pattern, as CSR data
    arrays aligned with (rowptr, col).  `workers` > 1 evaluates chunks of
    pairs in a process pool (same per-pair arithmetic)."""
    N = rwg.n
    rows = np.repeat(np.arange(N), np.diff(rowptr))
    LA = np.empty(col.shape[0])
    YR = np.empty(col.shape[0])
    spans = [(s, min(col.shape[0], s + chunk)) for s in range(0, col.shape[0], chunk)]
    if workers > 1 and len(spans) > 1:
        import multiprocessing as mp
        ctx = mp.get_context("fork")
        with ctx.Pool(workers) as pool:
            res = pool.map(_chunk_job, [(V, T, rwg, rows[s:e], col[s:e]) for s, e in spans])
        for (s, e), (a, r) in zip(spans, res):
            LA[s:e], YR[s:e] = a, r
    else:
        for s, e in spans:
            LA[s:e], YR[s:e] = static_pair_entries(V, T, rwg, rows[s:e], col[s:e])
    return symmetrize(rowptr, col, LA), symmetrize(rowptr, col, YR)


def transpose_perm(rowptr, col):
    """For a CSR pattern that is symmetric, perm[k] = position of entry (n, m)
    when position k holds (m, n)."""
    N = rowptr.shape[0] - 1
    rows = np.repeat(np.arange(N), np.diff(rowptr))
    return np.lexsort((rows, col))


def symmetrize(rowptr, col, vals):
    """(L + L^T)/2 on the (symmetric) near pattern."""
    perm = transpose_perm(rowptr, col)
    return 0.5 * (vals + vals[perm])
