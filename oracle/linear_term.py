"""Linear-term accuracy modification (oracle).  TEST INFRASTRUCTURE ONLY.

P:363-366  eq:linterm   k0^2 G_lin = (-j k0)^2 / (4 pi 2!) r,  i.e.
                        G_lin(r) = -r / (8 pi)
P:382-385  G_d <- G - G_s - k0^2 G_lin
P:386-389  eq:Lmatdecomplin  L(k0) = L_s + k0^2 L_lin + L_d(k0)
P:390-393  "for L_lin, direct integration is only required for entries
           corresponding to overlapping basis and test functions.  The
           remaining entries of L_s and L_lin are approximated with grid-based
           FFTs."  "L_lin is accounted for on-the-fly during the matrix-vector
           product, scaled by the appropriate value of k0^2."
P:396      O(N) extra time and memory.

Reading (R21): "overlapping" = the supports share a triangle (a
positive-area intersection), so each row holds at most 5 such columns.  The
grid operator W H(k0) P is unchanged (its samples at |delta| > 0 are G, which
contains k0^2 G_lin; at delta = 0 G_lin(0) = 0 and G_d(0) is unchanged), so
on an overlapping pair the grid's share of k0^2 L_lin, k0^2 W H_lin P with
H_lin(delta) = G_lin(h |delta|), is replaced by the direct entry:

    y^A   += k0^2 C^A_lin x,    C^A_lin   = L^A_lin   - sum_c W^c H_lin P^c
    y^rho += k0^2 C^rho_lin x,  C^rho_lin = y^rho_lin - W^rho H_lin P^rho

on overlapping pairs only.  Entries use the static recipe (R9): analytic inner
integrals of R and (rho' - rho) R over the flat source triangle, 7-point outer
rule, symmetrised.

Closed forms (surface divergence theorem in the source plane, u = rho' - rho,
R^2 = d^2 + |u|^2, t0_i the signed distance of rho to edge i, m_i its outward
in-plane normal, R0_i^2 = t0_i^2 + d^2, s the coordinate along edge i):
    div_s(u R) = 3 R - d^2 / R            =>  int_T R = (d^2 I0 + sum_i t0_i int_i R ds) / 3
    grad_s R^3 = 3 R u                     =>  int_T u R = (1/3) sum_i m_i int_i R^3 ds
    int R ds   = [s R + R0^2 ln(s + R)] / 2
    int R^3 ds = s R^3 / 4 + 3 R0^2 s R / 8 + 3 R0^4 ln(s + R) / 8
"""
from __future__ import annotations

import math

import numpy as np

from .mesh import RWG
from .static_near import RADON7_BARY, RADON7_W, _dot, _logsum, _rwg_triangles, symmetrize, triangle_potentials

EIGHT_PI = 8.0 * math.pi


def G_lin(r):
    """eq:linterm P:363-366 without the k0^2: G_lin(r) = -r / (8 pi)."""
    return -np.asarray(r, np.float64) / EIGHT_PI


def triangle_R_potentials(r, v0, v1, v2):
    """J0 = int_T R dS' and J1 = int_T (rho' - rho) R dS' over the flat triangle
    for observation points r (arrays [..., 3]).  Returns (J0, J1, rho)."""
    I0, _, rho = triangle_potentials(r, v0, v1, v2)
    e1 = v1 - v0
    e2 = v2 - v0
    nrm = np.cross(e1, e2)
    nhat = nrm / np.linalg.norm(nrm, axis=-1, keepdims=True)
    d = _dot(r - v0, nhat)
    J0 = d * d * I0
    J1 = np.zeros(r.shape)
    for va, vb in ((v0, v1), (v1, v2), (v2, v0)):
        ev = vb - va
        L = np.linalg.norm(ev, axis=-1)
        shat = ev / L[..., None]
        mhat = np.cross(shat, nhat)
        sm = _dot(va - rho, shat)
        sp_ = _dot(vb - rho, shat)
        t0 = _dot(va - rho, mhat)
        R0sq = t0 * t0 + d * d
        Rm = np.linalg.norm(r - va, axis=-1)
        Rp = np.linalg.norm(r - vb, axis=-1)
        live = R0sq > (1e-14 * L) ** 2
        f2 = _logsum(Rp, sp_, R0sq, live) - _logsum(Rm, sm, R0sq, live)
        f2 = np.where(live, f2, 0.0)
        K1 = 0.5 * (sp_ * Rp - sm * Rm + R0sq * f2)
        K3 = (sp_ * Rp ** 3 - sm * Rm ** 3) / 4.0 + 3.0 * R0sq * (sp_ * Rp - sm * Rm) / 8.0 \
            + 3.0 * R0sq * R0sq * f2 / 8.0
        J0 = J0 + t0 * K1
        J1 = J1 + mhat * K3[..., None]
    return J0 / 3.0, J1 / 3.0, rho


def overlap_csr(rwg: RWG):
    """Pairs (m, n) whose supports share a triangle (R21), CSR with sorted
    columns; the diagonal is always present."""
    N = rwg.n
    by_tri: dict[int, list[int]] = {}
    for n in range(N):
        by_tri.setdefault(int(rwg.tp[n]), []).append(n)
        by_tri.setdefault(int(rwg.tm[n]), []).append(n)
    rowptr = [0]
    col: list[int] = []
    for m in range(N):
        cs = sorted(set(by_tri[int(rwg.tp[m])]) | set(by_tri[int(rwg.tm[m])]))
        col.extend(cs)
        rowptr.append(len(col))
    return np.array(rowptr, np.int64), np.array(col, np.int64)


def lin_pair_entries(V, T, rwg: RWG, rows, cols):
    """Unsymmetrised L^A_lin and y^rho_lin (outer on the test RWG m = rows,
    analytic inner on the source RWG n = cols), kernel G_lin = -R/(8 pi)."""
    V = np.asarray(V, np.float64)
    T = np.asarray(T, np.int64)
    verts, area, free, coef, div = _rwg_triangles(V, T, rwg)
    rows = np.asarray(rows)
    cols = np.asarray(cols)
    LA = np.zeros(rows.shape[0])
    YR = np.zeros(rows.shape[0])
    for sm in range(2):
        tv = verts[rows, sm]
        rq = np.einsum("qk,pkc->pqc", RADON7_BARY, tv)
        wq = RADON7_W[None, :] * area[rows, sm][:, None]
        fm = coef[rows, sm][:, None, None] * (rq - free[rows, sm][:, None, :])
        for sn in range(2):
            sv = verts[cols, sn][:, None, :, :]
            J0, J1, rho = triangle_R_potentials(rq, sv[..., 0, :], sv[..., 1, :], sv[..., 2, :])
            inner = coef[cols, sn][:, None, None] * (J1 + (rho - free[cols, sn][:, None, :]) * J0[..., None])
            LA -= (wq * _dot(fm, inner)).sum(axis=1) / EIGHT_PI
            YR -= div[rows, sm] * div[cols, sn] * (wq * J0).sum(axis=1) / EIGHT_PI
    return LA, YR


def H_lin_block(D: np.ndarray, order: int, h: float) -> np.ndarray:
    """B_D[s, s'] = H_lin(s - s' - D) = G_lin(h |s - s' - D|) (H_lin(0) = 0)."""
    from .precorrection import stencil_offsets
    off = stencil_offsets(order)
    delta = off[:, None, :] - off[None, :, :] - D[None, None, :]
    return G_lin(h * np.sqrt((delta * delta).sum(axis=-1).astype(np.float64)))


def lin_precorrection_entries(Lam, A, rows, cols, order: int, h: float):
    """W H_lin P on the listed pairs: (sum_c Lambda^c_m B Lambda^c_n, Lambda^rho_m B Lambda^rho_n)."""
    LA = np.zeros(len(rows))
    YR = np.zeros(len(rows))
    for i, (m, n) in enumerate(zip(rows, cols)):
        B = H_lin_block(A[n] - A[m], order, h)
        t = np.einsum("cs,st,ct->c", Lam[m], B, Lam[n])
        LA[i] = t[0] + t[1] + t[2]
        YR[i] = t[3]
    return LA, YR


def lin_correction(V, T, rwg: RWG, Lam, A, order: int, h: float):
    """(rowptr, col, C^A_lin, C^rho_lin, L^A_lin, y^rho_lin) on the overlapping pairs."""
    rowptr, col = overlap_csr(rwg)
    rows = np.repeat(np.arange(rwg.n), np.diff(rowptr))
    la, yr = lin_pair_entries(V, T, rwg, rows, col)
    la = symmetrize(rowptr, col, la)
    yr = symmetrize(rowptr, col, yr)
    pa, pr = lin_precorrection_entries(Lam, A, rows, col, order, h)
    return rowptr, col, la - pa, yr - pr, la, yr


def lin_dense(V, T, rwg: RWG):
    """Dense symmetrised (L^A_lin, y^rho_lin) over all pairs (small meshes)."""
    N = rwg.n
    m, n = np.meshgrid(np.arange(N), np.arange(N), indexing="ij")
    LA, YR = lin_pair_entries(V, T, rwg, m.ravel(), n.ravel())
    LA = LA.reshape(N, N)
    YR = YR.reshape(N, N)
    return 0.5 * (LA + LA.T), 0.5 * (YR + YR.T)
