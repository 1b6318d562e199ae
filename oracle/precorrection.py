"""Near-region precorrection L_s,P = W H_s,NR P (oracle).  TEST INFRASTRUCTURE ONLY.

P:274-280  eq:aimLPs  L_s,P = W^(L) H_s,NR P^(L); "H_s,NR is the convolution
           matrix for near-region precorrections, and encodes G_s"
P:303-309  eq:Hmn     H^(m,n) = G(k0, r_m, r_n) (here with G_s)
P:320-322  eq:Hsmm    H_s^(m,m) = H_s,NR^(m,m) = 0

For a near pair (m, n) with anchor difference D = A_n - A_m, node s of m's
stencil and node s' of n's stencil are (s - s' - D) cells apart, so
    L^A_s,P[m,n]   = sum_{c in x,y,z} Lambda^c_m^T B_D Lambda^c_n
    y^rho_s,P[m,n] = Lambda^rho_m^T B_D Lambda^rho_n
    B_D[s, s'] = H_s(s - s' - D),  H_s(delta) = 1 / (4 pi h |delta|),  H_s(0) = 0.
Pairs are grouped by D (a plain re-ordering of the sum over the pattern).
"""
from __future__ import annotations

import numpy as np

from .kernels import FOUR_PI


def stencil_offsets(order: int) -> np.ndarray:
    p = order + 1
    s = np.arange(p ** 3)
    return np.stack([s % p, (s // p) % p, s // (p * p)], axis=1)   # [p^3, 3] (i,j,k)


def H_s_block(D: np.ndarray, order: int, h: float) -> np.ndarray:
    off = stencil_offsets(order)
    delta = off[:, None, :] - off[None, :, :] - D[None, None, :]
    r2 = (delta * delta).sum(axis=-1).astype(np.float64)
    out = np.zeros(r2.shape)
    nz = r2 > 0
    out[nz] = 1.0 / (FOUR_PI * h * np.sqrt(r2[nz]))
    return out


def precorrection_entries(Lam: np.ndarray, A: np.ndarray, rows, col, order: int, h: float):
    """L^A_s,P and y^rho_s,P for the listed (row, col) pairs."""
    D = A[col] - A[rows]
    LA = np.zeros(col.shape[0])
    YR = np.zeros(col.shape[0])
    uniq, inv = np.unique(D, axis=0, return_inverse=True)
    inv = inv.ravel()
    order_k = np.argsort(inv, kind="stable")
    ks = inv[order_k]
    starts = np.flatnonzero(np.r_[True, ks[1:] != ks[:-1]])
    ends = np.r_[starts[1:], ks.shape[0]]
    for s, e in zip(starts, ends):
        idx = order_k[s:e]
        B = H_s_block(D[idx[0]], order, h)
        Lm = Lam[rows[idx]]            # [P, 4, p^3]
        Ln = Lam[col[idx]]
        t = np.einsum("pcs,pcs->pc", Lm @ B, Ln)
        LA[idx] = t[:, 0] + t[:, 1] + t[:, 2]
        YR[idx] = t[:, 3]
    return LA, YR


def _pc_job(args):
    return precorrection_entries(*args)


def precorrection(Lam: np.ndarray, A: np.ndarray, rowptr, col, order: int, h: float,
                  workers: int = 1, chunk: int = 1000000):
    """Returns (LA_P, Yrho_P) aligned with the CSR pattern."""
    N = A.shape[0]
    rows = np.repeat(np.arange(N), np.diff(rowptr))
    if workers <= 1 or col.shape[0] <= chunk:
        return precorrection_entries(Lam, A, rows, col, order, h)
    import multiprocessing as mp
    spans = [(s, min(col.shape[0], s + chunk)) for s in range(0, col.shape[0], chunk)]
    with mp.get_context("fork").Pool(workers) as pool:
        res = pool.map(_pc_job, [(Lam, A, rows[s:e], col[s:e], order, h) for s, e in spans])
    return np.concatenate([r[0] for r in res]), np.concatenate([r[1] for r in res])


def precorrection_dense(Lam: np.ndarray, A: np.ndarray, grid, rowptr, col):
    """Definition written out with explicit dense matrices (tiny grids only):
    P_c [N_g x N_b], H_s [N_g x N_g]; (P_c^T H_s P_c) restricted to the pattern."""
    from .grid import stencil_nodes
    Ng = grid.ng
    N = A.shape[0]
    nodes = stencil_nodes(A, grid)
    Nx, Ny, Nz = grid.n
    lin = np.arange(Ng)
    xyz = np.stack([lin % Nx, (lin // Nx) % Ny, lin // (Nx * Ny)], axis=1)
    dd = xyz[:, None, :] - xyz[None, :, :]
    r2 = (dd * dd).sum(-1).astype(np.float64)
    Hs = np.zeros((Ng, Ng))
    nz = r2 > 0
    Hs[nz] = 1.0 / (FOUR_PI * grid.h * np.sqrt(r2[nz]))
    rows = np.repeat(np.arange(N), np.diff(rowptr))
    out = []
    for c in range(4):
        P = np.zeros((Ng, N))
        np.add.at(P, (nodes, np.repeat(np.arange(N)[:, None], nodes.shape[1], 1)), Lam[:, c, :])
        M = P.T @ Hs @ P
        out.append(M[rows, col])
    return out[0] + out[1] + out[2], out[3]
