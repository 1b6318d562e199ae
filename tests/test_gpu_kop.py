"""NEXT #1 groundwork on the device: the static near part of the double-layer
operator K (C_K = sym(K_s,PV) + residue - K_s,P, readings R23-R25) computed
by the setup kernels in fp64, against the oracle (oracle/kop.py) on closed
icospheres."""
import numpy as np
import pytest

import aimx_inputs as inp
from tests._parity import make_gpu_op, rel_l2

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("subdiv,n", [(1, (8, 8, 8)), (2, (16, 16, 16))])
def test_K_static_vs_oracle(subdiv, n):
    from oracle.aimx import AIMxOracle
    from oracle.kop import K_precorrection_entries, residue_entries, static_K_entries
    from oracle.static_near import symmetrize
    m = inp.icosphere_mesh(subdiv, radius=0.5)
    orc = AIMxOracle(m.vertices, m.triangles, n, static=False)
    op = make_gpu_op(m, n, "c128")
    rp, col = op.near_csr()
    assert np.array_equal(rp, orc.rowptr) and np.array_equal(col, orc.col)
    rows = np.repeat(np.arange(orc.N), np.diff(orc.rowptr))
    ks = symmetrize(orc.rowptr, orc.col, static_K_entries(orc.V, orc.T, orc.rwg, rows, orc.col))
    res = residue_entries(orc.V, orc.T, orc.rwg, rows, orc.col)
    kp = K_precorrection_entries(orc.Lam, orc.A, rows, orc.col, orc.order, orc.grid.h)
    ck = op.K_static()
    assert rel_l2(ck, ks + res - kp) <= 1e-12
    assert rel_l2(ck, ks + res) > 1e-6          # the precorrection is not negligible


_KORC = {}   # oracle K per (icosphere, grid), shared by precisions and forms


@pytest.mark.parametrize("form", ["grad", "radial"])
@pytest.mark.parametrize("prec", ["c128", "c64"])
@pytest.mark.parametrize("subdiv,n", [(1, (8, 8, 8)), (2, (16, 16, 16)), (2, (24, 24, 24))])
def test_K_matvec_vs_oracle(prec, subdiv, n, form, monkeypatch):
    """aimx_matvec_kop against the oracle's AIMx K (odd gradient spectra) on
    closed icospheres.  grad: the device's gradient-of-kernel form (one
    forward / inverse transform pair, the spectral cross product in the fused
    short y/z pass (8^3 c64) or the TMA z pass; 24^3: padded 48, radix 3);
    radial (AIMX_K_RADIAL=1): the radial factor F, two passes."""
    from oracle.aimx import AIMxOracle
    from oracle.kop import AIMxK
    from paper_2009_02281_b200 import AIMxError
    from tests._parity import TOL, gpu_input_as_c128, to_gpu
    if form == "radial":
        monkeypatch.setenv("AIMX_K_RADIAL", "1")
    m = inp.icosphere_mesh(subdiv, radius=0.5)
    if (subdiv, n) not in _KORC:
        orc = AIMxOracle(m.vertices, m.triangles, n, static=False)
        _KORC[(subdiv, n)] = (orc, AIMxK(orc))
    orc, ak = _KORC[(subdiv, n)]
    op = make_gpu_op(m, n, prec)
    x = np.random.default_rng(11).standard_normal(op.N) + 1j * np.random.default_rng(12).standard_normal(op.N)
    with pytest.raises(AIMxError):
        op.matvec_kop(to_gpu(x, prec))            # not enabled
    op.set_kop(True)
    assert op.stats()["kop_grad"] == (form == "grad")
    for f in (50e6, 300e6):
        op.set_frequency(f)
        k0 = 2 * np.pi * f / 299792458.0
        y = op.matvec_kop(to_gpu(x, prec)).cpu().numpy()
        ref = ak.matvec(gpu_input_as_c128(x, prec), k0)
        assert rel_l2(y, ref) <= TOL[prec], (f, rel_l2(y, ref))


@pytest.fixture(scope="module")
def k3():
    from oracle.aimx import AIMxOracle
    from oracle.kop import AIMxK
    m = inp.icosphere_mesh(2, radius=0.5)
    orc = AIMxOracle(m.vertices, m.triangles, (32, 32, 32), static=False)
    return m, AIMxK(orc)


@pytest.mark.parametrize("prec", ["c128", "c64"])
def test_K_matvec_long_transforms(prec, k3):
    """A 32^3 grid: the y / z transforms are too long for the fused kernel and
    every z plane is occupied, so K runs the separate y passes and the TMA z
    pass (with the spectral cross product)."""
    from tests._parity import TOL, gpu_input_as_c128, to_gpu
    m, ak = k3
    op = make_gpu_op(m, (32, 32, 32), prec)
    op.set_kop(True)
    x = np.random.default_rng(21).standard_normal(op.N) * (1 + 0.4j)
    for f in (80e6, 400e6):
        op.set_frequency(f)
        y = op.matvec_kop(to_gpu(x, prec)).cpu().numpy()
        ref = ak.matvec(gpu_input_as_c128(x, prec), 2 * np.pi * f / 299792458.0)
        assert rel_l2(y, ref) <= TOL[prec], (f, rel_l2(y, ref))


@pytest.mark.parametrize("prec", ["c128", "c64"])
def test_cfie_matvec_sweep_solve(prec):
    """CFIE (eq:CFIEdis): matvec = Z x - eta0 Kmat x against the oracle's
    parts; a sweep and a GMRES solve in CFIE mode, residuals under the oracle
    CFIE operator."""
    from oracle.aimx import AIMxOracle
    from oracle.kop import AIMxK
    from tests._parity import TOL, gpu_input_as_c128, to_gpu
    m = inp.icosphere_mesh(2, radius=0.5)
    n = (16, 16, 16)
    orc = AIMxOracle(m.vertices, m.triangles, n)
    ak = AIMxK(orc)
    eta0 = 1.25663706212e-6 * 299792458.0

    def cfie(x, f):
        orc.set_frequency(f)
        return orc.matvec(x) - eta0 * ak.matvec(x, orc.k0)
    op = make_gpu_op(m, n, prec)
    op.set_cfie(True)
    x = np.random.default_rng(31).standard_normal(op.N) * (1 - 0.2j)
    for f in (60e6, 250e6):
        op.set_frequency(f)
        y = op.matvec(to_gpu(x, prec)).cpu().numpy()
        assert rel_l2(y, cfie(gpu_input_as_c128(x, prec), f)) <= TOL[prec]
    freqs = np.array([80e6, 200e6, 320e6])
    X = np.stack([np.random.default_rng(40 + i).standard_normal(op.N) + 0j for i in range(3)])
    Y = op.sweep(freqs, to_gpu(X, prec)).cpu().numpy()
    for i, f in enumerate(freqs):
        assert rel_l2(Y[i], cfie(gpu_input_as_c128(X[i], prec), f)) <= TOL[prec]
    tol = 1e-6 if prec == "c128" else 1e-4
    Xs, its, rr = op.solve(freqs, to_gpu(X, prec), tol=tol, restart=30, maxiter=2000)
    Xs = Xs.cpu().numpy()
    for i, f in enumerate(freqs):
        b = gpu_input_as_c128(X[i], prec)
        res = np.linalg.norm(b - cfie(Xs[i], f)) / np.linalg.norm(b)
        assert rr[i] <= tol * (1 + 1e-6) and res <= 5 * tol, (i, its[i], rr[i], res)


@pytest.mark.parametrize("prec", ["c128", "c64"])
def test_pmchwt_vs_oracle(prec):
    """PMCHWT (reading R27) for a dielectric sphere, eps_r = 4: the library's
    composite of L and principal-value K in both media against the oracle's."""
    from oracle.aimx import AIMxOracle
    from oracle.kop import AIMxK, pmchwt_matvec
    from tests._parity import TOL, gpu_input_as_c128, to_gpu
    m = inp.icosphere_mesh(2, radius=0.25)
    n = (16, 16, 16)
    orc = AIMxOracle(m.vertices, m.triangles, n)
    ak = AIMxK(orc)
    op = make_gpu_op(m, n, prec)
    op.set_kop(True)
    x = np.random.default_rng(51).standard_normal(2 * op.N) * (1 + 0.3j)
    x[op.N:] /= 376.73                       # M ~ eta0 J
    for f in (100e6, 300e6):
        op.set_frequency(f)
        y = op.matvec_pmchwt(4.0, to_gpu(x, prec)).cpu().numpy()
        ref = pmchwt_matvec(orc, ak, f, 4.0, gpu_input_as_c128(x, prec))
        N = op.N
        for sl in (slice(0, N), slice(N, 2 * N)):   # each equation on its own scale
            assert rel_l2(y[sl], ref[sl]) <= TOL[prec], (f, sl, rel_l2(y[sl], ref[sl]))


def test_kop_api_edges():
    """States and exclusions of the K / CFIE / PMCHWT calls."""
    import torch
    from paper_2009_02281_b200 import AIMxError
    from tests._parity import to_gpu
    m = inp.icosphere_mesh(1, radius=0.5)
    op = make_gpu_op(m, (8, 8, 8), "c128")
    x = to_gpu(np.ones(op.N), "c128")
    x2 = to_gpu(np.ones(2 * op.N), "c128")
    with pytest.raises(AIMxError):
        op.matvec_pmchwt(4.0, x2)                  # K not built
    op.set_kop(True)
    with pytest.raises(AIMxError):
        op.matvec_kop(x)                           # no frequency bound
    op.set_frequency(100e6)
    y = op.matvec_kop(x)
    assert torch.isfinite(torch.view_as_real(y)).all()
    with pytest.raises(AIMxError):
        op.matvec_pmchwt(0.5, x2)                  # eps_r < 1
    with pytest.raises(AIMxError):
        op.matvec_kop(x, x)                        # aliasing
    op.set_cfie(True)
    with pytest.raises(AIMxError):
        op.set_kop(False)                          # CFIE needs K
    with pytest.raises(AIMxError):
        op.set_conventional(True)                  # CFIE and conventional AIM are exclusive
    with pytest.raises(AIMxError):
        op.matvec_pmchwt(4.0, x2)                  # PMCHWT runs the AIMx operators
    op.set_cfie(False)
    yp = op.matvec_pmchwt(4.0, x2)
    assert yp.shape[0] == 2 * op.N
    # zero input -> zero output
    z = op.matvec_kop(torch.zeros_like(x))
    assert torch.count_nonzero(z) == 0
    s = make_gpu_op(m, (8, 8, 8), "c128", slab=("emulate", 2))
    with pytest.raises(AIMxError):
        s.set_kop(True)


@pytest.mark.parametrize("prec", ["c64", "c128"])
def test_pmchwt_flat_faced_cube_vs_oracle(prec):
    """PMCHWT (eps_r = 4) on a cube (flat faces, cfg4's body at a small size,
    grid 24^3 padded 48): with the gradient-of-kernel spectra the c64 path
    meets the north_star bar on both equations (the radial form's fp32
    cancellation on flat faces missed it: 2.8e-5 on the H rows)."""
    from oracle.aimx import AIMxOracle
    from oracle.kop import AIMxK, pmchwt_matvec
    from tests._parity import TOL, gpu_input_as_c128, to_gpu
    m = inp.box_mesh(8, 8, 8, (0.0, 0.0, 0.0), (0.5, 0.5, 0.5))
    n = (24, 24, 24)
    if "cube" not in _KORC:
        orc = AIMxOracle(m.vertices, m.triangles, n)
        _KORC["cube"] = (orc, AIMxK(orc))
    orc, ak = _KORC["cube"]
    op = make_gpu_op(m, n, prec)
    op.set_kop(True)
    assert op.stats()["kop_grad"]
    x = np.random.default_rng(61).standard_normal(2 * op.N) * (1 - 0.4j)
    x[op.N:] /= 376.73
    for f in (100e6, 400e6):
        op.set_frequency(f)
        y = op.matvec_pmchwt(4.0, to_gpu(x, prec)).cpu().numpy()
        ref = pmchwt_matvec(orc, ak, f, 4.0, gpu_input_as_c128(x, prec))
        for sl in (slice(0, op.N), slice(op.N, 2 * op.N)):
            assert rel_l2(y[sl], ref[sl]) <= TOL[prec], (f, sl, rel_l2(y[sl], ref[sl]))


def test_cfg4_pmchwt_fullsize_c64():
    """cfg4 as BASELINE.json names it: the dielectric cube (eps_r = 4, 0.5 m,
    60,552 RWG -> 121,104 unknowns [J; M]), grid 96^3 (padded 192: radix 3),
    K via the gradient-of-kernel spectra, c64.  The PMCHWT matvec against the
    oracle on 24 seeded rows of each equation (the oracle's grid parts on the
    full grid, its near parts row by row) at the first and last frequency."""
    from oracle.kop import pmchwt_rows, static_K_rows
    from tests._parity import TOL, gpu_input_as_c128, oracle_config, to_gpu
    c = inp.get_config(4)
    orc = oracle_config(4)
    op = make_gpu_op(inp.make_mesh(4), c.grid_n, "c64")
    op.set_kop(True)
    assert op.stats()["kop_grad"] and op.N == 60552
    rows = np.sort(np.random.default_rng(44).choice(op.N, 24, replace=False))
    kr = static_K_rows(orc, rows)
    rng = np.random.default_rng(45)
    x = (rng.standard_normal(2 * op.N) + 1j * rng.standard_normal(2 * op.N))
    x[op.N:] /= 376.73
    for f in (c.freqs[0], c.freqs[-1]):
        op.set_frequency(f)
        y = op.matvec_pmchwt(4.0, to_gpu(x, "c64")).cpu().numpy()
        yE, yH = pmchwt_rows(orc, kr, f, 4.0, gpu_input_as_c128(x, "c64"))
        assert rel_l2(y[rows], yE) <= TOL["c64"]
        assert rel_l2(y[op.N + rows], yH) <= TOL["c64"]


@pytest.mark.parametrize("prec", ["c128", "c64"])
def test_K_on_planar_grid_vs_oracle(prec):
    """K on a planar mesh (cfg1's plate): the EFIE passes of the context store
    3 channels (Lambda^z = 0), K's radial passes 4 (s x J has a z part) in their
    own buffers; K and then the EFIE matvec against the oracle."""
    from oracle.aimx import AIMxOracle
    from oracle.kop import AIMxK
    from tests._parity import TOL, gpu_input_as_c128, to_gpu
    m = inp.make_mesh(1)
    n = (16, 16, 4)
    orc = AIMxOracle(m.vertices, m.triangles, n)
    ak = AIMxK(orc)
    op = make_gpu_op(m, n, prec)
    op.set_kop(True)
    st = op.stats()
    assert st["planar"] and st["grid_channels"] == 3 and not st["kop_grad"]
    x = np.random.default_rng(31).standard_normal(op.N) * (1 - 0.2j)
    f = 150e6
    op.set_frequency(f)
    orc.set_frequency(f)
    xo = gpu_input_as_c128(x, prec)
    y = op.matvec_kop(to_gpu(x, prec)).cpu().numpy()
    assert rel_l2(y, ak.matvec(xo, 2 * np.pi * f / 299792458.0)) <= TOL[prec]
    z = op.matvec(to_gpu(x, prec)).cpu().numpy()
    assert rel_l2(z, orc.matvec(xo)) <= TOL[prec]
