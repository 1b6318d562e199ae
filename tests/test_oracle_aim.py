"""Pins for oracle/aim.py (the conventional AIM).

The conventional AIM's near entries are direct integration (eq:aimL P:190),
its far entries the grid operator (eq:aimLFR P:197): so on cfg1 its matrix
must equal the dense direct reference on every near pair and the AIMx operator
on every far pair.  The dynamic pair entries are checked against the dense
direct code (a different evaluation of the same product rule) and the
dynamic precorrection against the dense definition P^T H_d P."""
import numpy as np
import pytest

from oracle.aim import ConventionalAIM, H_d_block, dynamic_pair_entries, dynamic_precorrection_entries
from oracle.kernels import G_d


def _columns(fn, N):
    A = np.empty((N, N), complex)
    R = np.empty((N, N), complex)
    E = np.eye(N)
    for m in range(N):
        A[:, m], R[:, m] = fn(E[m])
    return A, R


def test_aim_near_is_direct_far_is_aimx(cfg1_oracle, cfg1_direct):
    op, d = cfg1_oracle, cfg1_direct        # cfg1_direct is bound to 150 MHz
    op.lin = False
    aim = ConventionalAIM(op)
    aim.set_frequency(150e6)
    A, R = _columns(aim.parts, op.N)
    A0, R0 = _columns(op.parts, op.N)
    near = np.zeros((op.N, op.N), bool)
    near[np.repeat(np.arange(op.N), np.diff(op.rowptr)), op.col] = True
    assert np.abs(A - d.LA)[near].max() <= 1e-12 * np.abs(d.LA).max()
    assert np.abs(R - d.YR)[near].max() <= 1e-12 * np.abs(d.YR).max()
    assert np.array_equal(A[~near], A0[~near]) and np.array_equal(R[~near], R0[~near])
    # and it differs from AIMx on the near pairs (the point of the method)
    assert np.abs(A0 - d.LA)[near].max() > 1e-4 * np.abs(d.LA).max()


def test_dynamic_entries_vs_dense_direct(cfg1_oracle):
    from oracle.direct import dynamic_dense
    op = cfg1_oracle
    k0 = 2 * np.pi * 2e8 / 299792458.0
    LA, YR = dynamic_dense(op.V, op.T, op.rwg, k0)
    rng = np.random.default_rng(3)
    rows = rng.integers(0, op.N, 400)
    cols = rng.integers(0, op.N, 400)
    la, yr = dynamic_pair_entries(op.V, op.T, op.rwg, rows, cols, k0)
    assert np.max(np.abs(la - LA[rows, cols])) <= 1e-13 * np.abs(LA).max()
    assert np.max(np.abs(yr - YR[rows, cols])) <= 1e-13 * np.abs(YR).max()


def test_dynamic_precorrection_vs_dense_definition(cfg1_oracle):
    op = cfg1_oracle
    k0 = 2 * np.pi * 3e8 / 299792458.0
    g = op.grid
    idx = np.arange(g.ng)
    ijk = np.stack([idx % g.n[0], (idx // g.n[0]) % g.n[1], idx // (g.n[0] * g.n[1])], axis=1)
    Hd = G_d(k0, g.h * np.sqrt(((ijk[:, None, :] - ijk[None, :, :]) ** 2).sum(-1)))
    assert Hd[0, 0] == pytest.approx(-1j * k0 / (4 * np.pi))          # eq:Hdmm
    Pd = [op.P[c].toarray() for c in range(4)]
    rows = np.repeat(np.arange(op.N), np.diff(op.rowptr))
    pa, pr = dynamic_precorrection_entries(op.Lam, op.A, rows, op.col, op.order, g.h, k0)
    LAd = sum(Pd[c].T @ Hd @ Pd[c] for c in range(3))
    YRd = Pd[3].T @ Hd @ Pd[3]
    assert np.max(np.abs(pa - LAd[rows, op.col])) <= 1e-12 * np.abs(LAd).max()
    assert np.max(np.abs(pr - YRd[rows, op.col])) <= 1e-12 * np.abs(YRd).max()
    B = H_d_block(np.array([0, 0, 0]), op.order, g.h, k0)
    assert np.array_equal(B, B.T) and np.all(np.diag(B) == -1j * k0 / (4 * np.pi))


def test_aim_correction_vanishes_at_low_frequency(cfg1_oracle):
    # G_d -> 0 as k0 -> 0 (|G_d| <= k0 / 4 pi), so D = O(k0) and AIM -> AIMx
    op = cfg1_oracle
    aim = ConventionalAIM(op)
    sizes = []
    for f in (1e6, 1e5):
        aim.set_frequency(f)
        sizes.append(max(np.abs(aim.DA).max(), np.abs(aim.DR).max()))
    assert sizes[1] < 0.2 * sizes[0]
