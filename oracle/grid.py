"""AIM grid, stencil anchors and near-region map (oracle).  TEST INFRASTRUCTURE ONLY.

P:188   "a regular grid is superimposed on the bounding box associated with S"
P:576   "a stencil which has n+1 points in each direction"
P:192   L_NR "contains the near-region entries" (size only shown graphically)

Readings (R3-R5; AMB-3, AMB-4, AMB-8):

* grid: margin m = ceil(n/2) nodes; isotropic h = max_a ext_a / (N_a - 1 - 2m)
  with ext_a = max - min of vertex coordinate a; origin o_a = min_a - m h.
  Node (i, j, k) is at o + h (i, j, k); linear index i + N_x (j + N_y k).
* stencil centre of an RWG = mean of its two triangle centroids, evaluated as
  ((v_a + v_b) * 2 + (p+ + p-)) / 6 in exactly this operation order with no
  fused multiply-add; u = (c - o) / h; even n: anchor = floor(u + 0.5) - n/2,
  odd n: floor(u) - (n-1)/2; the stencil is nodes anchor + {0..n} per axis.
* near pair (m, n): per-axis stencil gap g_a = max(0, |A_m,a - A_n,a| - n);
  near iff g_x^2 + g_y^2 + g_z^2 <= T^2 (T = near threshold in cells).
"""
from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np
import scipy.sparse as sp
from scipy.spatial import cKDTree

from .mesh import RWG


class GridError(ValueError):
    pass


@dataclass
class Grid:
    n: tuple        # (N_x, N_y, N_z)
    order: int
    h: float
    origin: np.ndarray  # float64 [3]

    @property
    def ng(self) -> int:
        return int(self.n[0] * self.n[1] * self.n[2])


def grid_spec(V: np.ndarray, n: tuple, order: int) -> Grid:
    V = np.asarray(V, dtype=np.float64)
    m = (order + 1) // 2               # ceil(n/2)
    lo = V.min(axis=0)
    hi = V.max(axis=0)
    h = 0.0
    for a in range(3):
        ext = hi[a] - lo[a]
        span = n[a] - 1 - 2 * m
        if n[a] < order + 1:
            raise GridError("grid too small for the stencil")
        if ext > 0.0:
            if span <= 0:
                raise GridError("grid too small for the mesh extent")
            h = max(h, ext / span)
    if not h > 0.0:
        raise GridError("zero-extent mesh")
    origin = np.array([lo[a] - m * h for a in range(3)])
    return Grid(tuple(int(x) for x in n), int(order), float(h), origin)


def stencil_centres(V: np.ndarray, rwg: RWG) -> np.ndarray:
    """((v_a + v_b) * 2 + (p+ + p-)) / 6, one IEEE op at a time (no FMA)."""
    s1 = V[rwg.a] + V[rwg.b]
    s1 = s1 * 2.0
    s2 = V[rwg.pp] + V[rwg.pm]
    c = s1 + s2
    return c / 6.0


def anchors(V: np.ndarray, rwg: RWG, grid: Grid) -> np.ndarray:
    c = stencil_centres(V, rwg)
    u = (c - grid.origin) / grid.h
    n = grid.order
    if n % 2 == 0:
        A = np.floor(u + 0.5) - n // 2
    else:
        A = np.floor(u) - (n - 1) // 2
    A = A.astype(np.int64)
    hi = np.asarray(grid.n) - 1 - n
    if np.any(A < 0) or np.any(A > hi):
        raise GridError("stencil does not fit in the grid")
    return A


def stencil_nodes(A: np.ndarray, grid: Grid) -> np.ndarray:
    """Linear grid index of each of the (n+1)^3 stencil nodes, ordered
    s = i + (n+1)(j + (n+1) k) with i along x.  Shape [N_b, (n+1)^3]."""
    p = grid.order + 1
    ii, jj, kk = np.meshgrid(np.arange(p), np.arange(p), np.arange(p), indexing="ij")
    # s = i + p (j + p k): flatten with k slowest
    off_i = ii.transpose(2, 1, 0).ravel()
    off_j = jj.transpose(2, 1, 0).ravel()
    off_k = kk.transpose(2, 1, 0).ravel()
    Nx, Ny, _ = grid.n
    x = A[:, 0:1] + off_i[None, :]
    y = A[:, 1:2] + off_j[None, :]
    z = A[:, 2:3] + off_k[None, :]
    return x + Nx * (y + Ny * z)


def near_gap_sq(Am: np.ndarray, An: np.ndarray, order: int) -> np.ndarray:
    g = np.maximum(0, np.abs(Am - An) - order)
    return (g * g).sum(axis=-1)


def near_csr(A: np.ndarray, order: int, T: int):
    """Near-region CSR (rows in RWG order, columns ascending).  Candidates from
    a Chebyshev ball |dA|_inf <= n + T (library kd-tree), then the exact integer
    test g^2 <= T^2.  Returns (rowptr int64, col int64)."""
    N = A.shape[0]
    tree = cKDTree(A.astype(np.float64))
    pairs = tree.query_pairs(r=order + T + 0.5, p=np.inf, output_type="ndarray")
    if pairs.size:
        keep = near_gap_sq(A[pairs[:, 0]], A[pairs[:, 1]], order) <= T * T
        pairs = pairs[keep]
    rows = np.concatenate([np.arange(N), pairs[:, 0], pairs[:, 1]])
    cols = np.concatenate([np.arange(N), pairs[:, 1], pairs[:, 0]])
    M = sp.csr_matrix((np.ones(rows.shape[0], dtype=np.int8), (rows, cols)), shape=(N, N))
    M.sort_indices()
    return M.indptr.astype(np.int64), M.indices.astype(np.int64)


def near_csr_bruteforce(A: np.ndarray, order: int, T: int):
    """O(N^2) definition, for small pins."""
    N = A.shape[0]
    g2 = near_gap_sq(A[:, None, :], A[None, :, :], order)
    near = g2 <= T * T
    rowptr = np.r_[0, np.cumsum(near.sum(axis=1))].astype(np.int64)
    col = np.nonzero(near)[1].astype(np.int64)
    return rowptr, col
