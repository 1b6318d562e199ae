"""The AIMx EFIE matrix-vector product (oracle).  TEST INFRASTRUCTURE ONLY.

P:281-285  eq:LAIMx   L(k0) ~= L_s,NR - L_s,P + W^(L) H(k0) P^(L)
P:286-290  eq:EFIEAIMx  -j w mu0 [ L^A_s,NR - L^A_s,P + W^(A) H P^(A)
                          + k0^-2 (L^phi_s,NR - L^phi_s,P + W^(phi) H P^(phi)) ] J
P:293      the static matrices "need only be computed once"

Step by step:
  S0  setup: RWG -> grid -> anchors -> near map -> Lambda -> L_s,NR -> L_s,P
      -> C_A = L^A_s,NR - L^A_s,P, C_rho = y^rho_s,NR - y^rho_s,P; H_hat_s
  S1  set_frequency: H_hat(k0) = H_hat_s + DFT3(K_d(k0))
  S2  g_c = P_c x                      (c = x, y, z, rho)
  S3  phi_c = IDFT3(H_hat DFT3(pad g_c)) cropped
  S4  y^A = sum_{c=x,y,z} P_c^T phi_c ;  y^rho = P_rho^T phi_rho     (W = P^T)
  S5  y^A += C_A x ; y^rho += C_rho x ; Z x = -j w mu0 (y^A - k0^-2 y^rho)
Parts: L_A x = y^A, L_phi x = -y^rho (AMB-13).
Optional (set_linear_term): y^A += k0^2 C^A_lin x, y^rho +=
k0^2 C^rho_lin x on overlapping pairs (linear_term).
"""
from __future__ import annotations

import math

import numpy as np
import scipy.sparse as sp

from . import convolution as conv
from .grid import Grid, anchors, grid_spec, near_csr, stencil_nodes
from .kernels import MU0, wavenumber
from .mesh import build_rwg
from .precorrection import precorrection
from .projection import projection_weights
from .static_near import static_near_matrices, static_pair_entries


class AIMxOracle:
    def __init__(self, V, T, n, order: int = 2, near_cells: int = 2,
                 grid: Grid | None = None, static: bool = True, workers: int = 1):
        self.V = np.asarray(V, np.float64)
        self.T = np.asarray(T, np.int64)
        self.rwg = build_rwg(self.V, self.T)
        self.grid = grid if grid is not None else grid_spec(self.V, tuple(n), order)
        self.order = self.grid.order
        self.near_cells = near_cells
        self.A = anchors(self.V, self.rwg, self.grid)
        self.rowptr, self.col = near_csr(self.A, self.order, near_cells)
        self.Lam = projection_weights(self.V, self.T, self.rwg, self.grid, self.A)
        self.nodes = stencil_nodes(self.A, self.grid)
        N, Ng = self.rwg.n, self.grid.ng
        p3 = self.nodes.shape[1]
        rr = np.repeat(np.arange(N), p3)
        self.P = [sp.csr_matrix((self.Lam[:, c, :].ravel(), (self.nodes.ravel(), rr)),
                                shape=(Ng, N)) for c in range(4)]
        self.Hs_hat = conv.spectrum_static(self.grid.n, self.grid.h)
        self.CA = self.CR = None
        self.workers = workers
        if static:
            self.build_static()
        self.k0 = None
        self.lin = False
        self.CAl_mat = self.CRl_mat = None

    def set_linear_term(self, on: bool = True):
        """treat k0^2 G_lin separately on overlapping pairs."""
        from .linear_term import lin_correction
        self.lin = bool(on)
        if self.lin and self.CAl_mat is None:
            rp, cl, ca, cr, _, _ = lin_correction(self.V, self.T, self.rwg, self.Lam, self.A, self.order,
                                                  self.grid.h)
            shape = (self.N, self.N)
            self.lin_rowptr, self.lin_col, self.CAl, self.CRl = rp, cl, ca, cr
            self.CAl_mat = sp.csr_matrix((ca, cl, rp), shape=shape)
            self.CRl_mat = sp.csr_matrix((cr, cl, rp), shape=shape)

    @property
    def N(self) -> int:
        return self.rwg.n

    # ---------------------------------------------------------------- S0
    def build_static(self):
        LA_NR, YR_NR = static_near_matrices(self.V, self.T, self.rwg, self.rowptr, self.col,
                                            workers=self.workers)
        LA_P, YR_P = precorrection(self.Lam, self.A, self.rowptr, self.col, self.order, self.grid.h,
                                   workers=self.workers)
        self.LA_NR, self.YR_NR, self.LA_P, self.YR_P = LA_NR, YR_NR, LA_P, YR_P
        self.CA = LA_NR - LA_P
        self.CR = YR_NR - YR_P
        shape = (self.N, self.N)
        self.CA_mat = sp.csr_matrix((self.CA, self.col, self.rowptr), shape=shape)
        self.CR_mat = sp.csr_matrix((self.CR, self.col, self.rowptr), shape=shape)

    def static_rows(self, rows):
        """C_A and C_rho restricted to the given rows (symmetrised entries
        computed pair by pair in both orientations) -> list of (cols, CA, CR)."""
        out = []
        for m in rows:
            cols = self.col[self.rowptr[m]:self.rowptr[m + 1]]
            mm = np.full(cols.shape, m)
            a1, r1 = static_pair_entries(self.V, self.T, self.rwg, mm, cols)
            a2, r2 = static_pair_entries(self.V, self.T, self.rwg, cols, mm)
            la = 0.5 * (a1 + a2)
            yr = 0.5 * (r1 + r2)
            lap, yrp = _precorr_row(self, m, cols)
            out.append((cols, la - lap, yr - yrp))
        return out

    # ---------------------------------------------------------------- S1
    def set_frequency(self, f_hz: float):
        if not (f_hz > 0 and math.isfinite(f_hz)):
            raise ValueError("frequency must be finite and > 0")
        self.f = float(f_hz)
        self.k0 = wavenumber(f_hz)
        self.omega = 2.0 * math.pi * f_hz
        self.H_hat = conv.spectrum(self.grid.n, self.grid.h, self.k0, self.Hs_hat)

    # ---------------------------------------------------------------- S2-S4
    def grid_potentials(self, x):
        Nx, Ny, Nz = self.grid.n
        g = np.stack([(self.P[c] @ x).reshape(Nz, Ny, Nx) for c in range(4)])
        return conv.convolve(self.H_hat, g)

    def grid_parts(self, x):
        """W H P x per part, no near correction: (y^A_grid, y^rho_grid)."""
        phi = self.grid_potentials(np.asarray(x, np.complex128))
        yA = sum(self.P[c].T @ phi[c].ravel() for c in range(3))
        yR = self.P[3].T @ phi[3].ravel()
        return yA, yR

    # ---------------------------------------------------------------- S5
    def parts(self, x):
        """(y^A, y^rho): L_A x = y^A, L_phi x = -y^rho."""
        x = np.asarray(x, np.complex128)
        yA, yR = self.grid_parts(x)
        yA = yA + self.CA_mat @ x
        yR = yR + self.CR_mat @ x
        if self.lin:
            k2 = self.k0 * self.k0
            yA = yA + k2 * (self.CAl_mat @ x)
            yR = yR + k2 * (self.CRl_mat @ x)
        return yA, yR

    def combine(self, yA, yR):
        return -1j * self.omega * MU0 * (yA - yR / (self.k0 * self.k0))

    def matvec(self, x):
        yA, yR = self.parts(x)
        return self.combine(yA, yR)

    def matvec_rows(self, x, rows):
        """Z x on selected rows only (full grid path, near rows pair by pair)."""
        x = np.asarray(x, np.complex128)
        yA, yR = self.grid_parts(x)
        res = []
        for m, (cols, ca, cr) in zip(rows, self.static_rows(rows)):
            a = yA[m] + ca @ x[cols]
            r = yR[m] + cr @ x[cols]
            if self.lin:
                k2 = self.k0 * self.k0
                a += k2 * (self.CAl_mat.getrow(m) @ x)[0]
                r += k2 * (self.CRl_mat.getrow(m) @ x)[0]
            res.append((a, r))
        a = np.array([t[0] for t in res])
        r = np.array([t[1] for t in res])
        return a, r, self.combine(a, r)

    def sweep(self, freqs, X):
        Y = np.empty_like(np.asarray(X, np.complex128))
        for i, f in enumerate(freqs):
            self.set_frequency(f)
            Y[i] = self.matvec(X[i])
        return Y


def _precorr_row(op: AIMxOracle, m: int, cols):
    from .precorrection import H_s_block
    la = np.zeros(cols.shape[0])
    yr = np.zeros(cols.shape[0])
    for j, n in enumerate(cols):
        B = H_s_block(op.A[n] - op.A[m], op.order, op.grid.h)
        t = np.einsum("cs,st,ct->c", op.Lam[m], B, op.Lam[n])
        la[j] = t[0] + t[1] + t[2]
        yr[j] = t[3]
    return la, yr


def from_config(cfg: int, static: bool = True, workers: int = 1) -> AIMxOracle:
    import aimx_inputs as inp
    c = inp.get_config(cfg)
    mesh = inp.make_mesh(cfg)
    return AIMxOracle(mesh.vertices, mesh.triangles, c.grid_n, c.order, c.near_cells,
                      static=static, workers=workers)
