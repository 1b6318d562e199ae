"""Conventional AIM, per-frequency near region (oracle).  TEST INFRASTRUCTURE ONLY.

P:188-191  eq:aimL    L(k0) = L_NR(k0) + L_FR(k0), L_NR "computed using direct
                      integration"
P:196-198  eq:aimLFR  L_FR(k0) ~= W H(k0) P - L_P(k0)
P:204-206  eq:aimLP   L_P(k0) = W H_NR(k0) P
P:210      "Both L_NR(k0) and L_P(k0) must be generated for each frequency"

Written as a correction of the AIMx operator on the near pattern (reading R22):
with G = G_s + G_d,
    L_NR(k0) = L_s,NR + L_d,NR(k0),   L_P(k0) = L_s,P + W H_d,NR(k0) P,
so  L_AIM(k0) = L_AIMx(k0) + D(k0),   D = L_d,NR(k0) - W H_d,NR(k0) P
on the near pairs, 0 elsewhere.  H is the same grid operator (its samples at
|delta| > 0 are G; its self term -j k0/(4 pi), eq:Hmm, and the static one 0,
eq:Hsmm, enter W H P and L_P identically on near pairs, so they cancel there,
and far pairs never reach delta = 0).  L_d,NR uses the direct reference's
recipe for G_d (7-point x 7-point product rule, direct.py), so the AIM operator
reproduces the direct entries on every near pair.
"""
from __future__ import annotations

import numpy as np
import scipy.sparse as sp

from .kernels import G_d


def dynamic_pair_entries(V, T, rwg, rows, cols, k0: float, chunk: int = 20000):
    """L^A_d and y^rho_d (kernel G_d) for the listed pairs by the 7 x 7 product
    rule over the 2 x 2 triangle combinations."""
    from .direct import _points
    pts, w, f, div = _points(np.asarray(V, np.float64), np.asarray(T, np.int64), rwg)
    N = rwg.n
    P = pts.reshape(N, 14, 3)
    W = w.reshape(N, 14)
    F = f.reshape(N, 14, 3)
    D = div.reshape(N, 14)
    rows = np.asarray(rows)
    cols = np.asarray(cols)
    LA = np.empty(rows.shape[0], np.complex128)
    YR = np.empty(rows.shape[0], np.complex128)
    for s in range(0, rows.shape[0], chunk):
        m, n = rows[s:s + chunk], cols[s:s + chunk]
        R = np.linalg.norm(P[m][:, :, None, :] - P[n][:, None, :, :], axis=-1)    # [p, 14, 14]
        G = G_d(k0, R) * W[m][:, :, None] * W[n][:, None, :]
        LA[s:s + chunk] = np.einsum("pij,pic,pjc->p", G, F[m], F[n])
        YR[s:s + chunk] = np.einsum("pij,pi,pj->p", G, D[m], D[n])
    return LA, YR


def H_d_block(D: np.ndarray, order: int, h: float, k0: float) -> np.ndarray:
    """B_D[s, s'] = H_d(s - s' - D) = G_d(k0, h |s - s' - D|), with
    H_d(0) = -j k0/(4 pi) (eq:Hdmm)."""
    from .precorrection import stencil_offsets
    off = stencil_offsets(order)
    delta = off[:, None, :] - off[None, :, :] - D[None, None, :]
    return G_d(k0, h * np.sqrt((delta * delta).sum(axis=-1).astype(np.float64)))


def dynamic_precorrection_entries(Lam, A, rows, cols, order: int, h: float, k0: float):
    """W H_d,NR(k0) P on the listed pairs, grouped by anchor offset."""
    rows = np.asarray(rows)
    cols = np.asarray(cols)
    Dv = A[cols] - A[rows]
    LA = np.zeros(rows.shape[0], np.complex128)
    YR = np.zeros(rows.shape[0], np.complex128)
    uniq, inv = np.unique(Dv, axis=0, return_inverse=True)
    inv = inv.ravel()
    for g in range(uniq.shape[0]):
        idx = np.flatnonzero(inv == g)
        B = H_d_block(uniq[g], order, h, k0)
        t = np.einsum("pcs,st,pct->pc", Lam[rows[idx]], B, Lam[cols[idx]])
        LA[idx] = t[:, 0] + t[:, 1] + t[:, 2]
        YR[idx] = t[:, 3]
    return LA, YR


class ConventionalAIM:
    """The conventional AIM operator at one frequency, on top of an AIMxOracle
    (same grid, weights, near pattern and static matrices)."""

    def __init__(self, op):
        self.op = op
        self.rows = np.repeat(np.arange(op.N), np.diff(op.rowptr))

    @property
    def N(self) -> int:
        return self.op.N

    def set_frequency(self, f_hz: float):
        op = self.op
        op.set_frequency(f_hz)
        la, yr = dynamic_pair_entries(op.V, op.T, op.rwg, self.rows, op.col, op.k0)
        pa, pr = dynamic_precorrection_entries(op.Lam, op.A, self.rows, op.col, op.order, op.grid.h, op.k0)
        self.DA, self.DR = la - pa, yr - pr
        shape = (op.N, op.N)
        self.DA_mat = sp.csr_matrix((self.DA, op.col, op.rowptr), shape=shape)
        self.DR_mat = sp.csr_matrix((self.DR, op.col, op.rowptr), shape=shape)

    def parts(self, x):
        x = np.asarray(x, np.complex128)
        yA, yR = self.op.parts(x)
        return yA + self.DA_mat @ x, yR + self.DR_mat @ x

    def matvec(self, x):
        yA, yR = self.parts(x)
        return self.op.combine(yA, yR)
