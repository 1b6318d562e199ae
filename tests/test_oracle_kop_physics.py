"""Physics pins for the two oracle parts that round 1 left "parity unpinned"
(oracle/kop.py, readings R24 and R27).

Both pins compare the oracle's AIMx operators on a closed icosphere with
fields known in closed form.  They hold to the discretisation error of the
RWG basis (a few per cent here).  A flipped sign or a wrong medium scaling
moves the result by O(1).

1. The sign of the residue term of the tested K ("principal value ...
   analytical residue term"; reading R24: exterior limit).  The surface
   current J = M z x r_hat on a sphere is the bound current of a uniformly
   magnetised ball.  Its field H = curl A (what eq:opK's K[J] computes,
   P:408) is (2/3) M z inside and the dipole field (M/3)(3 cos(theta) r_hat - z)
   outside (textbook magnetostatics).  Tangential to the surface:
       H+_t = -(1/3) z_t,   H-_t = (2/3) z_t,   PV K[J]_t = (H+_t + H-_t)/2 = (1/6) z_t,
   so with b_m = int f_m . z dS (f_m is tangential):
       -int f_m . PV K[J]           = -b/6   (the PV part, k0 -> 0)
       int f_m . (n x n x H+)       = +b/3   (Kmat: PV part + residue)
   The opposite residue sign would give -2b/3.
2. The PMCHWT composition and its medium scalings (P:92 and P:159 only name
   PMCHWT; reading R27).  Extinction theorem: the currents n x H_inc and
   n x E_inc of a plane wave, radiating in the plane wave's own medium, give
   a field whose tangential principal value on S is -E_inc/2 (and
   +H_inc/2 for the H row in R27's sign convention, M = n x E).  So, with
   tE = int f . E_inc and tH = int f . H_inc:
   * eps_r = 1 (both media free space): y = [-tE; +tH];
   * the interior medium alone, A1 = pmchwt(eps_r) - pmchwt(1)/2, on a plane
     wave of medium 1 (k1 = 2 k0, eta1 = eta0/2 at eps_r = 4): A1 x = [-tE/2; +tH/2].
     This pins k1 and the eta1^-2 weight of the interior H row (a wrong weight
     changes that row's magnetic term by a factor 4).
"""
import numpy as np
import pytest

import aimx_inputs as inp
from oracle.aimx import AIMxOracle
from oracle.direct import _points
from oracle.kernels import C0, MU0
from oracle.kop import AIMxK, pmchwt_matvec, residue_entries, triangle_normals


class Sphere:
    def __init__(self):
        m = inp.icosphere_mesh(2, 1.0)                    # 320 triangles, 480 RWG
        self.op = op = AIMxOracle(m.vertices, m.triangles, (16, 16, 16))
        self.ak = AIMxK(op)
        N = op.N
        self.pts, self.w, self.f, _ = _points(op.V, op.T, op.rwg)   # [N, 2, 7, 3] (7-point rule)
        tri = np.stack([op.rwg.tp, op.rwg.tm], 1)
        self.nrm = triangle_normals(op.V, op.T)[tri]                # [N, 2, 3]
        # Gram matrix <f_m, f_n> (shared triangles; the 7-point rule is exact)
        self.gram = np.zeros((N, N))
        for a in range(N):
            for sa in range(2):
                t = tri[a, sa]
                for b in np.flatnonzero((tri[:, 0] == t) | (tri[:, 1] == t)):
                    sb = 0 if tri[b, 0] == t else 1
                    self.gram[a, b] += np.sum(self.w[a, sa] * np.einsum("qc,qc->q", self.f[a, sa], self.f[b, sb]))

    def tested(self, field):
        """int f_m . field dS for field(points, normals) -> [..., 3]."""
        v = field(self.pts, np.broadcast_to(self.nrm[:, :, None, :], self.pts.shape))
        return np.einsum("nsq,nsqc,nsqc->n", self.w, self.f, v)

    def project(self, field):
        """RWG coefficients of a tangential field (Galerkin projection)."""
        return np.linalg.solve(self.gram, self.tested(field))


@pytest.fixture(scope="module")
def sph():
    return Sphere()


def _rel(a, b):
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


def test_K_residue_sign_magnetised_sphere(sph):
    op, ak = sph.op, sph.ak
    z = np.array([0.0, 0.0, 1.0])
    x = sph.project(lambda p, n: np.cross(z, p / np.linalg.norm(p, axis=-1, keepdims=True)))
    b = sph.tested(lambda p, n: np.broadcast_to(z, p.shape))
    k0 = 1e-4                                              # static limit
    ext = ak.matvec(x, k0)                                 # PV + residue (R24)
    pv = ak.matvec(x, k0, residue=False)
    assert _rel(pv, -b / 6) <= 0.05                        # measured 0.025
    assert _rel(ext, b / 3) <= 0.05                        # measured 0.017
    # the other residue sign is far off: PV - residue = -2b/3
    rows = np.repeat(np.arange(op.N), np.diff(op.rowptr))
    res = residue_entries(op.V, op.T, op.rwg, rows, op.col)
    import scipy.sparse as sp
    R = sp.csr_matrix((res, op.col, op.rowptr), shape=(op.N, op.N))
    assert _rel(pv - R @ x, b / 3) >= 1.0
    assert _rel(ext - pv, b / 2) <= 0.05                   # the residue alone: 1/2 int f . (n x J)


def _plane_wave(sph, k, eta):
    ex, ey = np.array([1.0, 0.0, 0.0]), np.array([0.0, 1.0, 0.0])
    E = lambda p, n: ex * np.exp(-1j * k * p[..., 2:3])
    H = lambda p, n: ey / eta * np.exp(-1j * k * p[..., 2:3])
    J = sph.project(lambda p, n: np.cross(n, H(p, n)))
    M = sph.project(lambda p, n: np.cross(n, E(p, n)))     # R27's convention: M = n x E
    return J, M, sph.tested(E), sph.tested(H)


def test_pmchwt_extinction_equal_media(sph):
    op, ak, N = sph.op, sph.ak, sph.op.N
    f = C0 / (2 * np.pi)                                   # k0 a = 1
    k0, eta0 = 1.0, MU0 * C0
    J, M, tE, tH = _plane_wave(sph, k0, eta0)
    y = pmchwt_matvec(op, ak, f, 1.0, np.concatenate([J, M]))
    assert _rel(y[:N], -tE) <= 0.06                        # measured 0.022
    assert _rel(y[N:], tH) <= 0.06                         # measured 0.027
    # the opposite magnetic-current convention fails both rows
    y2 = pmchwt_matvec(op, ak, f, 1.0, np.concatenate([J, -M]))
    assert _rel(y2[:N], -tE) >= 0.5 and _rel(y2[N:], tH) >= 0.5


def test_pmchwt_interior_medium_scalings(sph):
    op, ak, N = sph.op, sph.ak, sph.op.N
    f, eps_r = C0 / (2 * np.pi), 4.0
    k1, eta1 = 2.0, MU0 * C0 / 2.0                         # k0 sqrt(eps_r), eta0 / sqrt(eps_r)
    J, M, tE, tH = _plane_wave(sph, k1, eta1)
    x = np.concatenate([J, M])
    y = pmchwt_matvec(op, ak, f, eps_r, x) - 0.5 * pmchwt_matvec(op, ak, f, 1.0, x)   # medium 1 alone
    assert _rel(y[:N], -tE / 2) <= 0.08                    # measured 0.031
    assert _rel(y[N:], tH / 2) <= 0.08                     # measured 0.045
