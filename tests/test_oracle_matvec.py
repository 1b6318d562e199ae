"""Pins for oracle/convolution.py and the whole oracle AIMx matvec (not gpu)."""
import json
import os

import numpy as np
import pytest

import aimx_inputs as inp
from oracle import convolution as conv
from oracle import kernels as K
from oracle.aimx import AIMxOracle
from oracle.grid import Grid

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "paper_fixed_points.json")))


# ---------------------------------------------------------------- S3 convolution
@pytest.mark.parametrize("k0", [0.0, 0.7, 9.0])
def test_fft_convolution_equals_bruteforce_toeplitz(k0):
    # eq:Hmn P:305 applied as an O(N^2) sum vs the zero-padded FFT path
    n = (5, 4, 3)
    h = 0.21
    rng = np.random.default_rng(1)
    g = rng.standard_normal((3, 4, 5)) + 1j * rng.standard_normal((3, 4, 5))
    Hhat = conv.spectrum(n, h, k0)
    fft = conv.convolve(Hhat, g)
    bf = conv.convolve_bruteforce(g, h, lambda r: K.G(k0, r), -1j * k0 / (4 * np.pi))
    assert np.max(np.abs(fft - bf)) <= 1e-12 * np.abs(bf).max()


@pytest.mark.parametrize("n", [(512, 2, 2), (2, 512, 2)])
def test_fft_convolution_1024_point_lines(n):
    # the padded 1024-point lines of cfg5's grid (1024 x 1024 x 16), along x
    # and along y, against the O(N^2) definition on a thin grid (2048 nodes)
    h, k0 = 0.013, 3.1
    rng = np.random.default_rng(5)
    g = np.zeros((n[2], n[1], n[0]), complex)
    m = rng.random(g.shape) < 0.3                      # sparse sources, as on a grid
    g[m] = rng.standard_normal(m.sum()) + 1j * rng.standard_normal(m.sum())
    fft = conv.convolve(conv.spectrum(n, h, k0), g)
    bf = conv.convolve_bruteforce(g, h, lambda r: K.G(k0, r), -1j * k0 / (4 * np.pi))
    assert np.max(np.abs(fft - bf)) <= 1e-12 * np.abs(bf).max()


def test_unit_impulse_returns_kernel_samples():
    n = (6, 5, 4)
    h = 0.5
    k0 = 1.3
    g = np.zeros((4, 5, 6), complex)
    g[0, 0, 0] = 1.0
    phi = conv.convolve(conv.spectrum(n, h, k0), g)
    z, y, x = np.meshgrid(np.arange(4), np.arange(5), np.arange(6), indexing="ij")
    r = h * np.sqrt(x ** 2 + y ** 2 + z ** 2)
    ref = np.where(r > 0, K.G(k0, np.where(r > 0, r, 1.0)), -1j * k0 / (4 * np.pi))
    assert np.max(np.abs(phi - ref)) < 1e-14 * np.abs(ref).max()
    # the self entry is the paper's modified H^(m,m) = -j k0/(4 pi) (eq:Hmm P:335)
    assert phi[0, 0, 0] == pytest.approx(-1j * k0 / (4 * np.pi), abs=1e-15)


def test_static_spectrum_split_and_octant_symmetry():
    n = (8, 6, 4)
    h = 0.1
    k0 = 2.0
    Hs = conv.spectrum_static(n, h)
    H = conv.spectrum(n, h, k0, Hs)
    r, wrap = conv.padded_distances(n, h)
    Kfull = np.where(r > 0, K.G(k0, np.where(r > 0, r, 1.0)), -1j * k0 / (4 * np.pi))
    Kfull[wrap] = 0
    import scipy.fft as sfft
    assert np.max(np.abs(H - sfft.fftn(Kfull))) < 1e-13 * np.abs(H).max()
    # static kernel is real and even -> static spectrum real and even per axis
    assert np.max(np.abs(Hs.imag)) < 1e-12 * np.abs(Hs).max()
    for ax in range(3):
        Nax = H.shape[ax]
        idx = (-np.arange(Nax)) % Nax
        assert np.max(np.abs(np.take(H, idx, axis=ax) - H)) < 1e-13 * np.abs(H).max()


# ---------------------------------------------------------------- whole matvec
def _dense_level0(op: AIMxOracle, k0):
    """Level-0 definition of eq:LAIMx with explicit dense matrices."""
    N, Ng = op.N, op.grid.ng
    Nx, Ny, Nz = op.grid.n
    lin = np.arange(Ng)
    xyz = np.stack([lin % Nx, (lin // Nx) % Ny, lin // (Nx * Ny)], 1)
    d = xyz[:, None, :] - xyz[None, :, :]
    r = op.grid.h * np.sqrt((d * d).sum(-1).astype(float))
    H = np.where(r > 0, K.G(k0, np.where(r > 0, r, 1.0)), -1j * k0 / (4 * np.pi))
    P = [p.toarray() for p in op.P]
    CA = op.CA_mat.toarray()
    CR = op.CR_mat.toarray()
    LA = sum(P[c].T @ H @ P[c] for c in range(3)) + CA
    YR = P[3].T @ H @ P[3] + CR
    return LA, YR


def test_fft_sparse_oracle_equals_dense_level0(cfg1_oracle):
    op = cfg1_oracle
    op.set_frequency(150e6)
    LA, YR = _dense_level0(op, op.k0)
    for i in range(3):
        x = inp.rhs_vector(1, i, op.N)
        yA, yR = op.parts(x)
        assert np.linalg.norm(yA - LA @ x) <= 1e-13 * np.linalg.norm(LA @ x)
        assert np.linalg.norm(yR - YR @ x) <= 1e-13 * np.linalg.norm(YR @ x)


def test_complex_symmetry_linearity_zero(cfg1_oracle):
    op = cfg1_oracle
    op.set_frequency(150e6)
    rng = np.random.default_rng(2)
    u = rng.standard_normal(op.N) + 1j * rng.standard_normal(op.N)
    v = rng.standard_normal(op.N) + 1j * rng.standard_normal(op.N)
    Zu, Zv = op.matvec(u), op.matvec(v)
    znorm = np.abs(Zu).max() * np.sqrt(op.N)
    assert abs(u @ Zv - v @ Zu) <= 1e-13 * np.linalg.norm(u) * np.linalg.norm(v) * znorm
    assert np.all(op.matvec(np.zeros(op.N)) == 0)
    a, b = 0.3 - 1.1j, 2.0 + 0.5j
    assert np.linalg.norm(op.matvec(a * u + b * v) - a * Zu - b * Zv) <= 1e-13 * np.linalg.norm(Zu) * 3


def test_static_matrices_frequency_independent(cfg1_oracle):
    op = cfg1_oracle
    ca, cr = op.CA.copy(), op.CR.copy()
    for f in (10e6, 150e6, 400e6):
        op.set_frequency(f)
        op.matvec(np.ones(op.N))
    assert op.CA.tobytes() == ca.tobytes() and op.CR.tobytes() == cr.tobytes()


def test_dynamic_grid_term_vanishes_as_k0_to_zero(cfg1_oracle):
    # W (H - H_s) P -> 0 as k0 -> 0 (G_d -> 0)
    op = cfg1_oracle
    x = inp.rhs_vector(1, 0, op.N)
    op.set_frequency(150e6)
    Hs = op.Hs_hat
    errs = []
    for f in (1e6, 1e4, 1e2):
        op.set_frequency(f)
        yA, yR = op.grid_parts(x)
        H = op.H_hat
        op.H_hat = Hs
        sA, sR = op.grid_parts(x)
        op.H_hat = H
        errs.append(np.linalg.norm(yR - sR) / np.linalg.norm(sR))
    assert errs[0] < 1e-3 and errs[1] < 1e-5 and errs[2] < 1e-7
    assert errs[0] > errs[1] > errs[2]


def test_near_far_structural_identities(cfg1_oracle):
    # eq:Lmatdecomp3 / eq:LAIMx: far pair -> L[m,n] = W_m H P_n exactly;
    # near pair -> L[m,n] - L_s,NR[m,n] = W_m H_d P_n (dynamic grid part only).
    op = cfg1_oracle
    op.set_frequency(150e6)
    cols = [0, 137]
    for n in cols:
        e = np.zeros(op.N, complex)
        e[n] = 1.0
        yA, yR = op.parts(e)
        gA, gR = op.grid_parts(e)
        H = op.H_hat
        op.H_hat = H - op.Hs_hat        # grid with the dynamic kernel only
        dA, dR = op.grid_parts(e)
        op.H_hat = H
        near_rows = set()
        for m in range(op.N):
            cs = op.col[op.rowptr[m]:op.rowptr[m + 1]]
            if n in cs:
                near_rows.add(m)
                k = op.rowptr[m] + np.searchsorted(cs, n)
                assert abs((yA[m] - op.LA_NR[k]) - dA[m]) <= 1e-13 * abs(yA[m]) + 1e-22
                assert abs((yR[m] - op.YR_NR[k]) - dR[m]) <= 1e-13 * abs(yR[m]) + 1e-20
            else:
                assert yA[m] == gA[m] and yR[m] == gR[m]
        assert 0 < len(near_rows) < op.N


def test_integer_cell_shift_invariance():
    m = inp.make_mesh(1)
    from oracle.grid import grid_spec
    g0 = grid_spec(m.vertices, (16, 16, 4), 2)
    g = Grid((20, 20, 6), 2, g0.h, g0.origin)
    base = AIMxOracle(m.vertices, m.triangles, None, grid=g)
    shift = g.h * np.array([2.0, 1.0, 1.0])
    V2 = m.vertices + shift
    moved = AIMxOracle(V2, m.triangles, None, grid=Grid(g.n, g.order, g.h, g.origin))
    assert np.array_equal(moved.A - base.A, np.tile([2, 1, 1], (base.N, 1)))
    assert np.array_equal(moved.col, base.col)
    x = inp.rhs_vector(1, 3, base.N)
    base.set_frequency(150e6)
    moved.set_frequency(150e6)
    y1, y2 = base.matvec(x), moved.matvec(x)
    assert np.linalg.norm(y1 - y2) <= 1e-12 * np.linalg.norm(y1)


# ---------------------------------------------------------------- vs direct MoM
def test_aimx_vs_dense_direct_within_paper_error(cfg1_oracle, cfg1_direct):
    # S:446 / eq:Lbounds P:592: rel-L2 <= 1e-2 over 20 seeded x; per part too
    op, d = cfg1_oracle, cfg1_direct
    op.set_frequency(150e6)
    worst = 0.0
    for i in range(20):
        x = inp.rhs_vector(1, i, op.N)
        yA, yR = op.parts(x)
        z = op.combine(yA, yR)
        zd = d.Z @ x
        worst = max(worst, np.linalg.norm(z - zd) / np.linalg.norm(zd),
                    np.linalg.norm(yA - d.LA @ x) / np.linalg.norm(d.LA @ x),
                    np.linalg.norm(yR - d.YR @ x) / np.linalg.norm(d.YR @ x))
    assert worst <= 1e-2


def test_self_term_error_below_one_percent(cfg1_oracle, cfg1_direct):
    # P:645 "the error in the proposed method remains below 1%" (diag of L_A and L_phi)
    op, d = cfg1_oracle, cfg1_direct
    op.set_frequency(150e6)
    lim = GOLD["self_term_error"]["max_rel_diag_error"]
    LA_diag = np.empty(op.N, complex)
    YR_diag = np.empty(op.N, complex)
    for m in range(op.N):
        e = np.zeros(op.N, complex)
        e[m] = 1
        a, r = op.parts(e)
        LA_diag[m], YR_diag[m] = a[m], r[m]
    assert np.max(np.abs(LA_diag - np.diag(d.LA)) / np.abs(np.diag(d.LA))) < lim
    assert np.max(np.abs(YR_diag - np.diag(d.YR)) / np.abs(np.diag(d.YR))) < lim
