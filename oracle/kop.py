"""The double-layer operator K and its AIMx form (oracle).  TEST INFRASTRUCTURE ONLY.

SURVEY 8(f) NEXT #1: the oracle side of AIMx for K (the library's
aimx_matvec_kop is checked against it, tests/test_gpu_kop.py).

R25  the static PV entries use the analytic inner integral with the 7-point
     outer rule, subdivided 8 x 8 on triangle pairs that touch (the inner
     field is log-singular along a shared edge), and are symmetrised like the
     L entries (R9): the exact PV part is symmetric.

P:408  eq:opK        K[X](r) = int_S grad G(r - r') x X(r') dS'
P:412  eq:ghgf       grad G = -rhat (1 + j k0 r) e^{-j k0 r} / (4 pi r^2),
                     rhat = (r - r')/r
P:429  eq:ghgftaylor grad G = -rhat/(4 pi) (1/r^2 - (-j k0)^2/2! - 2 (-j k0)^3 r/3! + ...)
P:445  eq:ghgfs      grad G_s = -rhat / (4 pi r^2);  eq:ghgfd  grad G_d = grad G - grad G_s
P:457  eq:KAIMx      K ~= K_s,NR - K_s,P + W^(K) H_grad(k0) P^(K)
P:463  eq:gH00       self term of H_grad (reading R23)
P:474  "direct integration ... in a principal value sense, while the
       self-interactions ... are accounted for with an analytical residue term"

Readings:
 R23 (AMB-16)  eq:gH00 gives one scalar for a vector kernel; grad G_d has no
               limit at r = 0 (its direction is rhat).  H_grad(0) = 0 per
               Cartesian component (the odd symmetry of d_a G); the static
               H_grad,s(0) = 0 likewise, so near pairs are unaffected.
 R24           the discrete K (eq:CFIEdis P:424: "the discretized n x n x K
               operator") tested with f_m, exterior limit:
                 Kmat[m,n] = int f_m . (n x n x K[f_n])^+ dS
                           = -int f_m . PV K[f_n] dS  +  1/2 int f_m . (n x f_n) dS
               (f_m is tangential, so f_m . (n (n . v) - v) = -f_m . v; the
               residue is n x H^+ = J/2 + n x PV K[J]).  n = outward normal
               (vertex order).  The residue sign follows this exterior-limit
               reading.  It is pinned by the field of a uniformly magnetised
               sphere (tests/test_oracle_kop_physics.py: Kmat x = +b/3 within
               2%, the other sign gives -2b/3).

AIMx for K, channel form: with the current channels g_b = P^b x (b = x, y, z),
    Phi_c = sum_{a,b} eps_{cab} (H_grad,a (*) g_b),   y_K = -sum_c W^c Phi_c + (K_s,NR - K_s,P) x,
H_grad,a(delta) = d_a G(k0, r) at r = h delta (the test node minus the source
node), W = P^T.  Inner integrals of the static part in closed form:
    int_T (r - r')/R^3 dS' = sum_i m_i f2_i + n sgn(d) Omega,
with f2_i = ln((R_+ + s_+)/(R_- + s_-)) on edge i and Omega the solid angle
of T seen from r (the beta sum of the 1/R potential, static_near); and
(r - r') x (r' - p) = (r - r') x (r - p), so
    int_T grad G_s(r - r') x c (r' - p) dS' = -(c / 4 pi) Q(r) x (r - p).
Coplanar contributions vanish: the inner vector is then normal to the plane
and f_m is tangential.
"""
from __future__ import annotations

import math

import numpy as np

from .kernels import FOUR_PI
from .mesh import RWG
from .static_near import RADON7_BARY, RADON7_W, _dot, _logsum, _rwg_triangles

EPS3 = np.zeros((3, 3, 3))
EPS3[0, 1, 2] = EPS3[1, 2, 0] = EPS3[2, 0, 1] = 1.0
EPS3[0, 2, 1] = EPS3[2, 1, 0] = EPS3[1, 0, 2] = -1.0


def grad_G(k0, rv):
    """eq:ghgf: grad_r G(r - r') at rv = r - r' (array [..., 3]); 0 at rv = 0."""
    rv = np.asarray(rv, np.float64)
    r = np.linalg.norm(rv, axis=-1)
    z = r == 0.0
    rr = np.where(z, 1.0, r)
    f = -(1.0 + 1j * k0 * rr) * np.exp(-1j * k0 * rr) / (FOUR_PI * rr ** 3)
    return np.where(z[..., None], 0.0, f[..., None] * rv)


def grad_G_s(rv):
    """eq:ghgfs: -rhat/(4 pi r^2) = -rv/(4 pi r^3); 0 at rv = 0."""
    rv = np.asarray(rv, np.float64)
    r = np.linalg.norm(rv, axis=-1)
    z = r == 0.0
    rr = np.where(z, 1.0, r)
    return np.where(z[..., None], 0.0, -rv / (FOUR_PI * rr[..., None] ** 3))


def grad_G_d(k0, rv):
    """eq:ghgfd, evaluated without cancellation:
    grad G_d = -rv/(4 pi r^3) ((1 + j x) e^{-j x} - 1), x = k0 r, with
    (1 + j x) e^{-j x} - 1 = (cos x + x sin x - 1) + j (x cos x - sin x);
    0 at rv = 0 (R23)."""
    rv = np.asarray(rv, np.float64)
    r = np.linalg.norm(rv, axis=-1)
    z = r == 0.0
    rr = np.where(z, 1.0, r)
    x = k0 * rr
    s2 = np.sin(0.5 * x)
    re = -2.0 * s2 * s2 + x * np.sin(x)                 # cos x - 1 + x sin x
    small = x < 1e-2                                      # x cos x - sin x = -x^3/3 + x^5/30 - ...
    im = np.where(small, -x ** 3 / 3.0 + x ** 5 / 30.0, x * np.cos(x) - np.sin(x))
    f = -(re + 1j * im) / (FOUR_PI * rr ** 3)
    return np.where(z[..., None], 0.0, f[..., None] * rv)


def triangle_Q(r, v0, v1, v2):
    """Q(r) = int_T (r - r')/R^3 dS' over the flat triangle (arrays [..., 3]);
    principal value in the plane (d = 0)."""
    e1 = v1 - v0
    e2 = v2 - v0
    nrm = np.cross(e1, e2)
    nhat = nrm / np.linalg.norm(nrm, axis=-1, keepdims=True)
    d = _dot(r - v0, nhat)
    # a point in the plane up to rounding is IN the plane: the normal part
    # jumps by +-2 pi across it and belongs to the residue, not the PV (R24)
    scale = (np.linalg.norm(e1, axis=-1) + np.linalg.norm(e2, axis=-1))
    d = np.where(np.abs(d) <= 1e-12 * scale, 0.0, d)
    rho = r - d[..., None] * nhat
    ad = np.abs(d)
    Q = np.zeros(np.broadcast_shapes(r.shape, v0.shape))
    omega = np.zeros(d.shape)
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
        f2 = np.where(live, _logsum(Rp, sp_, R0sq, live) - _logsum(Rm, sm, R0sq, live), 0.0)
        hasd = ad > 0.0
        den_p = np.where(hasd, R0sq + ad * Rp, 1.0)
        den_m = np.where(hasd, R0sq + ad * Rm, 1.0)
        beta = np.where(hasd, np.arctan(t0 * sp_ / den_p) - np.arctan(t0 * sm / den_m), 0.0)
        Q = Q + mhat * f2[..., None]
        omega = omega + beta
    return Q + (np.sign(d) * omega)[..., None] * nhat


def triangle_normals(V, T):
    n = np.cross(V[T[:, 1]] - V[T[:, 0]], V[T[:, 2]] - V[T[:, 0]])
    return n / np.linalg.norm(n, axis=1, keepdims=True)


def residue_entries(V, T, rwg: RWG, rows, cols):
    """1/2 int f_m . (n x f_n) dS over the triangles m and n share (R24);
    exact for the linear integrand by the 7-point rule."""
    V = np.asarray(V, np.float64)
    T = np.asarray(T, np.int64)
    verts, area, free, coef, div = _rwg_triangles(V, T, rwg)
    tri = np.stack([rwg.tp, rwg.tm], axis=1)
    nrm = triangle_normals(V, T)
    out = np.zeros(len(rows))
    for i, (m, n) in enumerate(zip(rows, cols)):
        for sm in range(2):
            for sn in range(2):
                if tri[m, sm] != tri[n, sn]:
                    continue
                pts = RADON7_BARY @ verts[m, sm]
                fm = coef[m, sm] * (pts - free[m, sm])
                fn = coef[n, sn] * (pts - free[n, sn])
                out[i] += 0.5 * area[m, sm] * np.sum(RADON7_W * _dot(fm, np.cross(nrm[tri[m, sm]], fn)))
    return out


def subdivided_rule(nsub: int):
    """Barycentric points / weights (sum 1) of the 7-point rule on each of the
    nsub^2 congruent sub-triangles of the reference triangle."""
    pts, wts = [], []
    for i in range(nsub):
        for j in range(nsub - i):
            corners = [((i, j), (i + 1, j), (i, j + 1))]
            if i + j + 1 < nsub:
                corners.append(((i + 1, j + 1), (i, j + 1), (i + 1, j)))
            for c in corners:
                B = np.array([[1.0 - (u + v) / nsub, u / nsub, v / nsub] for u, v in c])   # [3 corners, 3 bary]
                pts.append(RADON7_BARY @ B)
                wts.append(RADON7_W / nsub ** 2)
    return np.concatenate(pts), np.concatenate(wts)


def static_K_entries(V, T, rwg: RWG, rows, cols, nsub_touch: int = 8):
    """PV part of K_s on the listed pairs: -int f_m . int grad G_s x f_n,
    analytic inner (triangle_Q); outer 7-point rule, subdivided nsub_touch^2
    times on triangle pairs that touch without coinciding (the inner field is
    log-singular along a shared edge; reading R25)."""
    V = np.asarray(V, np.float64)
    T = np.asarray(T, np.int64)
    verts, area, free, coef, div = _rwg_triangles(V, T, rwg)
    tri = np.stack([rwg.tp, rwg.tm], axis=1)
    rows = np.asarray(rows)
    cols = np.asarray(cols)
    K = np.zeros(rows.shape[0])
    rules = {1: (RADON7_BARY, RADON7_W), nsub_touch: subdivided_rule(nsub_touch)}
    for sm in range(2):
        for sn in range(2):
            tm_, tn_ = tri[rows, sm], tri[cols, sn]
            touch = np.array([len(set(T[a]) & set(T[b])) > 0 for a, b in zip(tm_, tn_)]) & (tm_ != tn_)
            for ns, sel in ((1, ~touch), (nsub_touch, touch)):
                idx = np.flatnonzero(sel & (tm_ != tn_))   # coinciding triangles: PV part 0
                if idx.size == 0:
                    continue
                bary, wb = rules[ns]
                m, n = rows[idx], cols[idx]
                rq = np.einsum("qk,pkc->pqc", bary, verts[m, sm])
                wq = wb[None, :] * area[m, sm][:, None]
                fm = coef[m, sm][:, None, None] * (rq - free[m, sm][:, None, :])
                sv = verts[n, sn][:, None, :, :]
                Q = triangle_Q(rq, sv[..., 0, :], sv[..., 1, :], sv[..., 2, :])
                inner = -(coef[n, sn] / FOUR_PI)[:, None, None] * np.cross(Q, rq - free[n, sn][:, None, :])
                K[idx] -= (wq * _dot(fm, inner)).sum(axis=1)
    return K


def _points(V, T, rwg):
    from .direct import _points as pts
    return pts(np.asarray(V, np.float64), np.asarray(T, np.int64), rwg)


def dynamic_K_dense(V, T, rwg: RWG, k0: float):
    """-int f_m . int grad G_d x f_n over all pairs, 7 x 7 product rule."""
    pts, w, f, div = _points(V, T, rwg)
    N = rwg.n
    P = pts.reshape(N, 14, 3)
    W = w.reshape(N, 14)
    F = f.reshape(N, 14, 3)
    K = np.zeros((N, N), np.complex128)
    for m in range(N):
        g = grad_G_d(k0, P[m][None, :, None, :] - P[:, None, :, :])      # [N, 14, 14, 3]
        cr = np.cross(g, F[:, None, :, :])                                # grad G_d x f_n(r')
        K[m] = -np.einsum("i,ic,nijc,nj->n", W[m], F[m], cr, W)
    return K


def static_K_dense(V, T, rwg: RWG):
    """Symmetrised PV part of K_s over all pairs (the exact one is symmetric:
    grad G_s is odd and a . (b x c) = -c . (b x a); reading R25)."""
    N = rwg.n
    m, n = np.meshgrid(np.arange(N), np.arange(N), indexing="ij")
    K = static_K_entries(V, T, rwg, m.ravel(), n.ravel()).reshape(N, N)
    return 0.5 * (K + K.T)


class DirectK:
    """Dense direct-integration Kmat (R24): static PV part analytic-inner,
    dynamic part 7 x 7, plus the residue."""

    def __init__(self, V, T, rwg: RWG):
        self.V = np.asarray(V, np.float64)
        self.T = np.asarray(T, np.int64)
        self.rwg = rwg
        N = rwg.n
        self.Ks = static_K_dense(self.V, self.T, rwg)
        m, n = np.meshgrid(np.arange(N), np.arange(N), indexing="ij")
        self.Res = residue_entries(self.V, self.T, rwg, m.ravel(), n.ravel()).reshape(N, N)

    def set_frequency(self, k0: float):
        self.k0 = k0
        self.K = self.Ks + dynamic_K_dense(self.V, self.T, self.rwg, k0) + self.Res


# ---------------------------------------------------------------- AIMx for K
def gH00_literal(k0: float) -> complex:
    """eq:gH00 as printed: (-j k0)^2 / (4 pi 2!).  It is the coefficient
    of rhat in the r -> 0 limit of grad G_d (eq:ghgftaylor P:429), not a value
    of the vector kernel; the default reading R23 uses 0 (the average over
    +-rhat).  Kept behind gh00="literal" (AMB-16)."""
    return (-1j * k0) ** 2 / (FOUR_PI * 2.0)


def gradient_kernel_samples(n: tuple, h: float, k0: float | None, gh00: str = "zero"):
    """H_grad,a on the padded grid [2Nz, 2Ny, 2Nx] (wrap slot 0, R10): d_a G at
    r = h * offset (k0 None: the static kernel).  Returns [3, ...] (a = x, y, z).
    gh00: self term H_grad,a(0): "zero" (R23), or "literal" (eq:gH00's scalar in
    every component)."""
    offs = []
    wrap = []
    for N in (n[2], n[1], n[0]):
        i = np.arange(2 * N)
        offs.append(np.where(i < N, i, i - 2 * N))
        wrap.append(i == N)
    oz, oy, ox = np.meshgrid(*offs, indexing="ij")
    wz, wy, wx = np.meshgrid(*wrap, indexing="ij")
    rv = h * np.stack([ox, oy, oz], axis=-1).astype(np.float64)
    g = grad_G_s(rv) if k0 is None else grad_G(k0, rv)
    g[wz | wy | wx] = 0.0
    if gh00 == "literal" and k0 is not None:
        g[0, 0, 0, :] = gH00_literal(k0)
    elif gh00 != "zero":
        raise ValueError(f"gh00 must be 'zero' or 'literal', not {gh00!r}")
    return np.moveaxis(g, -1, 0)


def grid_K(op, x, k0: float, gh00: str = "zero"):
    """-sum_c W^c sum_{a,b} eps_cab (H_grad,a (*) P^b x) on the op's grid
    (gh00: the self-term reading, see gradient_kernel_samples)."""
    import scipy.fft as sfft
    Nx, Ny, Nz = op.grid.n
    g = np.stack([(op.P[b] @ x).reshape(Nz, Ny, Nx) for b in range(3)])
    from .convolution import WORKERS
    G = sfft.fftn(g, s=(2 * Nz, 2 * Ny, 2 * Nx), axes=(-3, -2, -1), workers=WORKERS)
    Hh = sfft.fftn(gradient_kernel_samples(op.grid.n, op.grid.h, k0, gh00), axes=(-3, -2, -1), workers=WORKERS)
    y = np.zeros(op.N, np.complex128)
    for c in range(3):
        acc = np.zeros_like(G[0])
        for a in range(3):
            for b in range(3):
                if EPS3[c, a, b] != 0.0:
                    acc += EPS3[c, a, b] * Hh[a] * G[b]
        phi = sfft.ifftn(acc, workers=WORKERS)[:Nz, :Ny, :Nx]
        y -= op.P[c].T @ phi.ravel()
    return y


def radial_F_samples(n: tuple, h: float, k0: float):
    """F(r) = (1 + j k0 r) e^{-j k0 r} / (4 pi r^3) at r = h |offset| on the
    padded grid (0 at offset 0 and on the wrap slots): grad G(r) = -r F(r)."""
    from .convolution import padded_distances
    r, wrap = padded_distances(n, h)
    F = np.zeros(r.shape, np.complex128)
    nz = (r > 0) & ~wrap
    F[nz] = (1.0 + 1j * k0 * r[nz]) * np.exp(-1j * k0 * r[nz]) / (FOUR_PI * r[nz] ** 3)
    return F


def grid_K_radial(op, x, k0: float):
    """The same grid operator as grid_K through the EVEN radial kernel F only:
    with node coordinates s (in cells),
        sum_{a,b} eps_cab (d_a G (*) J_b) = -h [ s x (F (*) J) - F (*) (s x J) ]_c,
    because d_a G(h delta) = -h delta_a F(h |delta|) and
    sum_s' (s - s')_a F(s - s') J(s') = s_a (F (*) J)(s) - (F (*) (s_a J))(s).
    (the planned device form of NEXT #1.)"""
    import scipy.fft as sfft
    Nx, Ny, Nz = op.grid.n
    J = np.stack([(op.P[b] @ x).reshape(Nz, Ny, Nx) for b in range(3)])
    kz, ky, kx = np.meshgrid(np.arange(Nz), np.arange(Ny), np.arange(Nx), indexing="ij")
    S = np.stack([kx, ky, kz]).astype(np.float64)                    # node coordinates s (x, y, z)
    SxJ = np.cross(S, J, axis=0)
    Fh = sfft.fftn(radial_F_samples(op.grid.n, op.grid.h, k0))

    def conv(g):
        G_ = sfft.fftn(g, s=(2 * Nz, 2 * Ny, 2 * Nx), axes=(-3, -2, -1))
        return sfft.ifftn(G_ * Fh, axes=(-3, -2, -1))[..., :Nz, :Ny, :Nx]
    Phi = -op.grid.h * (np.cross(S, conv(J), axis=0) - conv(SxJ))
    return -sum(op.P[c].T @ Phi[c].ravel() for c in range(3))


def K_precorrection_entries(Lam, A, rows, cols, order: int, h: float):
    """K_s,P on the listed pairs: -sum_{c,a,b} eps_cab Lam^c_m B^a_D Lam^b_n,
    B^a_D[s, s'] = d_a G_s(h (s - s' - D))."""
    from .precorrection import stencil_offsets
    off = stencil_offsets(order)
    out = np.zeros(len(rows))
    for i, (m, n) in enumerate(zip(rows, cols)):
        D = A[n] - A[m]
        delta = off[:, None, :] - off[None, :, :] - D[None, None, :]
        B = grad_G_s(h * delta.astype(np.float64))                   # [p3, p3, 3]
        t = 0.0
        for c in range(3):
            for a in range(3):
                for b in range(3):
                    if EPS3[c, a, b] != 0.0:
                        t += EPS3[c, a, b] * Lam[m, c] @ B[..., a] @ Lam[n, b]
        out[i] = -t
    return out


class AIMxK:
    """eq:KAIMx on top of an AIMxOracle (same grid, weights, near pattern)."""

    def __init__(self, op):
        self.op = op
        from .static_near import symmetrize
        rows = np.repeat(np.arange(op.N), np.diff(op.rowptr))
        ks = symmetrize(op.rowptr, op.col, static_K_entries(op.V, op.T, op.rwg, rows, op.col))
        res = residue_entries(op.V, op.T, op.rwg, rows, op.col)
        kp = K_precorrection_entries(op.Lam, op.A, rows, op.col, op.order, op.grid.h)
        import scipy.sparse as sp
        self.C = sp.csr_matrix((ks + res - kp, op.col, op.rowptr), shape=(op.N, op.N))
        self.Cpv = sp.csr_matrix((ks - kp, op.col, op.rowptr), shape=(op.N, op.N))

    def matvec(self, x, k0: float, residue: bool = True):
        x = np.asarray(x, np.complex128)
        return (self.C if residue else self.Cpv) @ x + grid_K(self.op, x, k0)


def pmchwt_matvec(op, ak: AIMxK, f_hz: float, eps_r: float, x):
    """PMCHWT for a homogeneous dielectric body (
    reading R27, AMB-17: the paper names PMCHWT, but never states
    it): unknowns x = [J; M] (electric and magnetic surface currents), media
    0 (outside, k0, eta0) and 1 (inside, k1 = k0 sqrt(eps_r), eta1 = eta0 /
    sqrt(eps_r), mu_r = 1):
        y_E = (Z0 + Z1) J - (K0 + K1) M
        y_H = (K0 + K1) J + (Z0 / eta0^2 + Z1 / eta1^2) M
    Z_i = -j w mu0 (L_A(k_i) + k_i^-2 L_phi(k_i)) (w the physical frequency),
    K_i the tested PV operator (the exterior and interior residues cancel in
    the sum).  The same static matrices serve both media (G_s is medium-free).
    M is n x E (so y_H is +int f . H_inc for the incident fields); the
    composition and both media's scalings are pinned by the extinction
    theorem (tests/test_oracle_kop_physics.py)."""
    from .kernels import MU0, C0
    x = np.asarray(x, np.complex128)
    N = op.N
    J, M = x[:N], x[N:]
    w = 2 * np.pi * f_hz
    eta0 = MU0 * C0
    eta1 = eta0 / np.sqrt(eps_r)
    out_E = np.zeros(N, complex)
    out_H = np.zeros(N, complex)
    Ksum_J = np.zeros(N, complex)
    Ksum_M = np.zeros(N, complex)
    for i, fi in enumerate((f_hz, f_hz * np.sqrt(eps_r))):
        op.set_frequency(fi)
        k = op.k0
        zJ = (lambda a, r: -1j * w * MU0 * (a - r / (k * k)))(*op.parts(J))
        zM = (lambda a, r: -1j * w * MU0 * (a - r / (k * k)))(*op.parts(M))
        out_E += zJ
        out_H += zM / (eta0 ** 2 if i == 0 else eta1 ** 2)
        Ksum_J += ak.matvec(J, k, residue=False)
        Ksum_M += ak.matvec(M, k, residue=False)
    return np.concatenate([out_E - Ksum_M, out_H + Ksum_J])


# ---------------------------------------------------------------- sampled rows (full-size parity)
def static_K_rows(op, rows):
    """C_K on the near columns of the given rows, entry by entry: the
    symmetrised PV part (both orientations, reading R25), + residue, - K_s,P.
    Returns a list of (row, cols, C_K row, C_K row without the residue)."""
    out = []
    for m in rows:
        cols = op.col[op.rowptr[m]:op.rowptr[m + 1]]
        mm = np.full(cols.shape, m)
        pv = 0.5 * (static_K_entries(op.V, op.T, op.rwg, mm, cols) + static_K_entries(op.V, op.T, op.rwg, cols, mm))
        res = residue_entries(op.V, op.T, op.rwg, mm, cols)
        kp = K_precorrection_entries(op.Lam, op.A, mm, cols, op.order, op.grid.h)
        out.append((m, cols, pv + res - kp, pv - kp))
    return out


def kop_rows(op, krows, x, k0: float, residue: bool = True):
    """(Kmat x) on the rows of krows (= static_K_rows(op, rows)): AIMxK.matvec
    with the grid part on the full grid and C_K only on those rows."""
    x = np.asarray(x, np.complex128)
    g = grid_K(op, x, k0)
    return np.array([g[m] + (ck if residue else cpv) @ x[cols] for m, cols, ck, cpv in krows])


def pmchwt_rows(op, krows, f_hz: float, eps_r: float, x):
    """pmchwt_matvec on the rows of krows (y_E rows, y_H rows), with the L
    parts from op.matvec_rows (the oracle's row-wise near part) and K from
    kop_rows; the same composition and scalings (reading R27)."""
    from .kernels import MU0, C0
    x = np.asarray(x, np.complex128)
    N = op.N
    J, M = x[:N], x[N:]
    rows = [m for m, _, _, _ in krows]
    w = 2 * np.pi * f_hz
    eta0 = MU0 * C0
    eta1 = eta0 / np.sqrt(eps_r)
    yE = np.zeros(len(rows), complex)
    yH = np.zeros(len(rows), complex)
    for i, fi in enumerate((f_hz, f_hz * np.sqrt(eps_r))):
        op.set_frequency(fi)
        k = op.k0
        aJ, rJ, _ = op.matvec_rows(J, rows)
        aM, rM, _ = op.matvec_rows(M, rows)
        yE += -1j * w * MU0 * (aJ - rJ / (k * k))
        yH += -1j * w * MU0 * (aM - rM / (k * k)) / (eta0 ** 2 if i == 0 else eta1 ** 2)
        yE -= kop_rows(op, krows, M, k, residue=False)
        yH += kop_rows(op, krows, J, k, residue=False)
    return yE, yH
