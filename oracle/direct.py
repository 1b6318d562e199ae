"""Dense direct-integration MoM EFIE matrix (oracle).  TEST INFRASTRUCTURE ONLY.

The paper's "direct integration" reference mode ("direct integration
with factorization"; eq:EFIEdis P:179-181):

    Z_dir = -j w mu0 (L_A + k0^-2 L_phi),
    L_A[m,n]   = int int f_m . f_n G dS' dS,
    L_phi[m,n] = - int int div f_m div f_n G dS' dS      (AMB-13),

with G = G_s + G_d (eq:hgfdecomp0 P:222): the singular static part uses the
same analytic-inner recipe as static_near (every pair, symmetrised); the
bounded dynamic part G_d (continuous, G_d(0) = -j k0/(4 pi)) uses the
7 x 7 product rule.  Small meshes only (dense N x N).

lin_split=True: G_d is split further into k0^2 G_lin (eq:linterm,
non-smooth at r = 0; analytic inner integrals on every pair, linear_term) and
the remainder G_d - k0^2 G_lin (its first non-smooth term is O(k0^4 r^3)),
which keeps the 7 x 7 rule.  This is the tighter reference the modification's
error is measured against (fig:selferrors P:643-646).
"""
from __future__ import annotations

import numpy as np

from .kernels import G_d, MU0
from .mesh import RWG
from .linear_term import G_lin, lin_dense
from .static_near import RADON7_BARY, RADON7_W, static_pair_entries


def _points(V, T, rwg: RWG):
    tri = np.stack([T[rwg.tp], T[rwg.tm]], axis=1)            # [N,2,3]
    verts = V[tri]                                             # [N,2,3,3]
    area = np.stack([rwg.area_p, rwg.area_m], axis=1)          # [N,2]
    free = np.stack([V[rwg.pp], V[rwg.pm]], axis=1)            # [N,2,3]
    sign = np.array([1.0, -1.0])
    pts = np.einsum("qk,nskc->nsqc", RADON7_BARY, verts)       # [N,2,7,3]
    w = RADON7_W[None, None, :] * area[:, :, None]             # [N,2,7]
    f = (sign[None, :] * rwg.length[:, None] / (2 * area))[:, :, None, None] * (pts - free[:, :, None, :])
    div = np.broadcast_to((sign[None, :] * rwg.length[:, None] / area)[:, :, None], w.shape)
    return pts, w, f, div


def static_dense(V, T, rwg: RWG):
    N = rwg.n
    m, n = np.meshgrid(np.arange(N), np.arange(N), indexing="ij")
    LA, YR = static_pair_entries(V, T, rwg, m.ravel(), n.ravel())
    LA = LA.reshape(N, N)
    YR = YR.reshape(N, N)
    return 0.5 * (LA + LA.T), 0.5 * (YR + YR.T)


def dynamic_dense(V, T, rwg: RWG, k0: float, minus_lin: bool = False):
    pts, w, f, div = _points(V, T, rwg)
    N = rwg.n
    P = pts.reshape(-1, 3)
    R = np.linalg.norm(P[:, None, :] - P[None, :, :], axis=-1)
    Gd = G_d(k0, R)
    if minus_lin:
        Gd = Gd - k0 * k0 * G_lin(R)
    M = P.shape[0]
    owner = np.repeat(np.arange(N), 14)
    LA = np.zeros((N, N), dtype=np.complex128)
    for c in range(3):
        U = np.zeros((N, M))
        U[owner, np.arange(M)] = (w * f[..., c]).ravel()
        LA += U @ Gd @ U.T
    U = np.zeros((N, M))
    U[owner, np.arange(M)] = (w * div).ravel()
    YR = U @ Gd @ U.T
    return LA, YR


class DirectEFIE:
    def __init__(self, V, T, rwg: RWG, lin_split: bool = False):
        self.V = np.asarray(V, np.float64)
        self.T = np.asarray(T, np.int64)
        self.rwg = rwg
        self.lin_split = lin_split
        self.LA_s, self.YR_s = static_dense(self.V, self.T, rwg)
        if lin_split:
            self.LA_lin, self.YR_lin = lin_dense(self.V, self.T, rwg)

    def set_frequency(self, f_hz: float):
        from .kernels import wavenumber
        self.k0 = wavenumber(f_hz)
        self.omega = 2.0 * np.pi * f_hz
        LAd, YRd = dynamic_dense(self.V, self.T, self.rwg, self.k0, minus_lin=self.lin_split)
        self.LA = self.LA_s + LAd
        self.YR = self.YR_s + YRd
        if self.lin_split:
            k2 = self.k0 * self.k0
            self.LA = self.LA + k2 * self.LA_lin
            self.YR = self.YR + k2 * self.YR_lin
        self.Z = -1j * self.omega * MU0 * (self.LA - self.YR / self.k0 ** 2)
