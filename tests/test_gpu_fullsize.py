"""Full-size parity at BASELINE.json's configs, in bench.py's launch
configuration: integer structures bit-exact over the WHOLE problem; static
matrices and outputs on seeded sampled rows that the oracle computes one by one
(the grid part of the oracle runs on the full grid)."""
import numpy as np
import pytest

import aimx_inputs as inp
from tests._parity import TOL, check_structure, gpu_input_as_c128, make_gpu_op, oracle_config, rel_l2, to_gpu

pytestmark = pytest.mark.gpu


def _fullsize(cfg, prec, freqs, nrows, orc=None):
    c = inp.get_config(cfg)
    orc = orc if orc is not None else oracle_config(cfg)
    op = make_gpu_op(inp.make_mesh(cfg), c.grid_n, prec)
    check_structure(op, orc)
    lam = op.weights()
    # two different exact integrations (reading R8) agree to rounding: measured
    # 1.4e-13 of max |Lambda| on cfg5 (401,088 RWG), below 1e-13 elsewhere
    assert np.max(np.abs(lam - orc.Lam)) <= 5e-13 * np.abs(orc.Lam).max()
    rng = np.random.default_rng(cfg)
    rows = np.sort(rng.choice(op.N, nrows, replace=False))
    st = op.static()
    sr = orc.static_rows(rows)
    for m, (cols, ca, cr) in zip(rows, sr):
        sl = slice(orc.rowptr[m], orc.rowptr[m + 1])
        assert rel_l2(st["CA"][sl], ca) <= 1e-12
        assert rel_l2(st["CR"][sl], cr) <= 1e-12
    for fi, f in enumerate(freqs):
        op.set_frequency(f)
        orc.set_frequency(f)
        x = inp.rhs_vector(cfg, fi, op.N)
        xg = to_gpu(x, prec)
        y = op.matvec(xg).cpu().numpy()
        yA, yP = op.matvec_parts(xg)
        a, r, z = orc.matvec_rows(gpu_input_as_c128(x, prec), rows)
        assert rel_l2(yA.cpu().numpy()[rows], a) <= TOL[prec]
        assert rel_l2(yP.cpu().numpy()[rows], -r) <= TOL[prec]
        assert rel_l2(y[rows], z) <= TOL[prec]
    return op


def test_cfg2_fullsize_c64():
    c = inp.get_config(2)
    _fullsize(2, "c64", [c.freqs[0], c.freqs[-1]], 48)


@pytest.mark.parametrize("prec", ["c64", "c128"])
def test_cfg3_fullsize(prec):
    c = inp.get_config(3)
    _fullsize(3, prec, [c.freqs[0], c.freqs[-1]], 24)


def test_cfg2_sweep_matches_per_frequency_matvecs():
    c = inp.get_config(2)
    op = make_gpu_op(inp.make_mesh(2), c.grid_n, "c64")
    freqs = c.freqs[:8]
    X = to_gpu(np.stack([inp.rhs_vector(2, i, op.N) for i in range(8)]), "c64")
    Y = op.sweep(freqs, X)
    for i, f in enumerate(freqs):
        op.set_frequency(f)
        assert rel_l2(op.matvec(X[i].contiguous()).cpu().numpy(), Y[i].cpu().numpy()) <= 1e-6


def test_cfg2_bench_sweep_vs_oracle_rows():
    """bench.py's launch configuration (cfg2, c64, the 100-point sweep in
    device batches of 32, 32, 32 and 4 points, 32- and 4-column kernels)
    against the oracle on seeded sampled rows."""
    c = inp.get_config(2)
    op = make_gpu_op(inp.make_mesh(2), c.grid_n, "c64")
    assert op.stats()["batch_slots"] == 32      # 100 points -> device batches 32, 32, 32, 4
    orc = oracle_config(2)
    X = np.stack([inp.rhs_vector(2, i, op.N) for i in range(len(c.freqs))])
    Y = op.sweep(c.freqs, to_gpu(X, "c64")).cpu().numpy()
    rows = np.sort(np.random.default_rng(22).choice(op.N, 32, replace=False))
    sr = orc.static_rows(rows)                       # near rows, pair by pair (once)
    for i in (0, 31, 32, 95, 96, 99):    # first / last points of the batches
        orc.set_frequency(c.freqs[i])
        x = gpu_input_as_c128(X[i], "c64")
        gA, gR = orc.grid_parts(x)
        a = np.array([gA[m] + ca @ x[cols] for m, (cols, ca, cr) in zip(rows, sr)])
        r = np.array([gR[m] + cr @ x[cols] for m, (cols, ca, cr) in zip(rows, sr)])
        assert rel_l2(Y[i][rows], orc.combine(a, r)) <= TOL["c64"]


@pytest.fixture(scope="module")
def orc5():
    return oracle_config(5)        # grid part on the full 1024 x 1024 x 16 padded grid


def test_cfg5_fullsize_c64(orc5):
    """cfg5 (401,088 RWG, 78.4 M near pairs, 1024-point x and y lines, the
    planar S3 path): RWG table, anchors and near CSR bit-exact over the whole
    problem; weights; C on 48 seeded rows; L_A x, L_phi x and Z x on those rows
    at the first and last frequency."""
    c = inp.get_config(5)
    op = _fullsize(5, "c64", [c.freqs[0], c.freqs[-1]], 48, orc=orc5)
    assert op.stats()["planar"]


def test_cfg5_bench_sweep_vs_oracle_rows(orc5):
    """bench.py's launch configuration (cfg5, c64, the 64-point sweep in two
    device batches of 32 points, 32-column kernels) against the oracle on
    seeded sampled rows at the first / last points of both batches."""
    c = inp.get_config(5)
    op = make_gpu_op(inp.make_mesh(5), c.grid_n, "c64")
    assert op.stats()["batch_slots"] == 32
    X = np.stack([inp.rhs_vector(5, i, op.N) for i in range(len(c.freqs))])
    Y = op.sweep(c.freqs, to_gpu(X, "c64")).cpu().numpy()
    rows = np.sort(np.random.default_rng(55).choice(op.N, 48, replace=False))
    sr = orc5.static_rows(rows)
    for i in (0, 31, 32, 63):
        orc5.set_frequency(c.freqs[i])
        x = gpu_input_as_c128(X[i], "c64")
        gA, gR = orc5.grid_parts(x)
        a = np.array([gA[m] + ca @ x[cols] for m, (cols, ca, cr) in zip(rows, sr)])
        r = np.array([gR[m] + cr @ x[cols] for m, (cols, ca, cr) in zip(rows, sr)])
        assert rel_l2(Y[i][rows], orc5.combine(a, r)) <= TOL["c64"]
