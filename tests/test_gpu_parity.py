"""GPU (CUDA, through the C ABI) vs the fp64 oracle on the same seeded inputs.

Bar (north_star): integer structures bit-exact; Z x, L_A x and
L_phi x each within rel-L2 1e-11 (complex128 path) / 2e-5 (complex64 path).
"""
import numpy as np
import pytest

import aimx_inputs as inp
from tests._parity import (TOL, check_structure, gpu_input_as_c128, make_gpu_op, rel_l2,
                           to_gpu)

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def orc1():
    from oracle.aimx import from_config
    return from_config(1)


@pytest.fixture(scope="module", params=["c128", "c64"])
def gpu1(request):
    return make_gpu_op(inp.make_mesh(1), (16, 16, 4), request.param), request.param


def test_cfg1_structures_bit_exact(gpu1, orc1):
    op, prec = gpu1
    check_structure(op, orc1)


def test_cfg1_weights_and_static(gpu1, orc1):
    op, prec = gpu1
    lam = op.weights()
    assert np.max(np.abs(lam - orc1.Lam)) <= 1e-14 * np.abs(orc1.Lam).max() * 10
    s = op.static()
    for key, ref in (("LA_NR", orc1.LA_NR), ("YR_NR", orc1.YR_NR), ("LA_P", orc1.LA_P),
                     ("YR_P", orc1.YR_P), ("CA", orc1.CA), ("CR", orc1.CR)):
        assert rel_l2(s[key], ref) <= 1e-12, key


def _octant_ref(op, H):
    """The oracle's padded spectrum H [2Nz, 2Ny, 2Nx] in the library's layout
    [ky, kz, kx]: the octant, or for planar contexts the dz = 0 slice's 2-D
    spectrum, sum over kz of H / (2 N_z) (the inverse z-DFT at dz = 0)."""
    Nz2, Ny2, Nx2 = H.shape
    Nx, Ny, Nz = Nx2 // 2, Ny2 // 2, Nz2 // 2
    if op.stats()["planar"]:
        H = H.sum(axis=0, keepdims=True) / Nz2
        Nz = 0
    return np.transpose(H[: Nz + 1, : Ny + 1, : Nx + 1], (1, 0, 2))


def test_cfg1_static_spectrum(gpu1, orc1):
    op, prec = gpu1
    assert op.stats()["planar"]          # the plate: one occupied z plane
    assert rel_l2(op.spectrum(0), _octant_ref(op, orc1.Hs_hat)) <= 1e-13


@pytest.mark.parametrize("fi", [0, 1])
def test_cfg1_matvec_parts_and_combined(gpu1, orc1, fi):
    op, prec = gpu1
    f = 150e6 if fi == 0 else 37.5e6
    op.set_frequency(f)
    orc1.set_frequency(f)
    assert rel_l2(op.spectrum(1), _octant_ref(op, orc1.H_hat)) <= (1e-13 if prec == "c128" else 1e-6)
    for i in range(3):
        x = inp.rhs_vector(1, i, op.N)
        xg = to_gpu(x, prec)
        xo = gpu_input_as_c128(x, prec)
        y = op.matvec(xg).cpu().numpy()
        yA, yP = op.matvec_parts(xg)
        yA, yP = yA.cpu().numpy(), yP.cpu().numpy()
        oA, oR = orc1.parts(xo)
        z = orc1.combine(oA, oR)
        assert rel_l2(yA, oA) <= TOL[prec]
        assert rel_l2(yP, -oR) <= TOL[prec]
        assert rel_l2(y, z) <= TOL[prec]


def test_cfg1_edge_cases(gpu1):
    import torch
    op, prec = gpu1
    from paper_2009_02281_b200 import AIMxError
    op.set_frequency(150e6)
    z = torch.zeros(op.N, dtype=op.cdtype, device="cuda")
    assert torch.count_nonzero(op.matvec(z)) == 0
    x = to_gpu(inp.rhs_vector(1, 5, op.N), prec)
    y1 = op.matvec(x).clone()
    y2 = op.matvec(x).clone()
    assert torch.equal(y1, y2)                   # deterministic, no atomics
    a = 0.5 - 2.0j
    ya = op.matvec((x * a).contiguous())
    assert rel_l2(ya.cpu().numpy(), (y1 * a).cpu().numpy()) <= TOL[prec]
    with pytest.raises(AIMxError):
        op.set_frequency(0.0)
    with pytest.raises(AIMxError):
        op.set_frequency(float("nan"))
    with pytest.raises(AIMxError):
        op.matvec(x, x)                           # aliasing


def test_matvec_before_frequency_is_state_error():
    from paper_2009_02281_b200 import AIMxError
    op = make_gpu_op(inp.make_mesh(1), (16, 16, 4), "c64")
    x = to_gpu(np.ones(op.N), "c64")
    with pytest.raises(AIMxError) as e:
        op.matvec(x)
    assert e.value.status == 4


def test_setup_errors():
    from paper_2009_02281_b200 import AIMxError
    m = inp.make_mesh(1)
    with pytest.raises(AIMxError) as e:           # grid too small for the stencil fit
        make_gpu_op(m, (16, 16, 2), "c64")
    assert e.value.status == 3
    with pytest.raises(AIMxError) as e:           # FFT length 2*12 not compiled
        make_gpu_op(m, (12, 16, 4), "c64")
    assert e.value.status == 7
    V = np.array([[0, 0, 0], [1, 0, 0], [0, 1, 0], [1, 1, 0]], float)
    bad = inp.Mesh(V, np.array([[0, 1, 2], [1, 2, 3]], np.int32))
    with pytest.raises(AIMxError) as e:           # inconsistent orientation
        make_gpu_op(bad, (8, 8, 4), "c64")
    assert e.value.status == 2
    deg = inp.Mesh(V, np.array([[0, 1, 1]], np.int32))
    with pytest.raises(AIMxError) as e:
        make_gpu_op(deg, (8, 8, 4), "c64")
    assert e.value.status == 2


@pytest.mark.parametrize("prec", ["c64", "c128"])
def test_sweep_equals_matvec_loop_and_host_sweep(prec):
    import torch
    op = make_gpu_op(inp.make_mesh(1), (16, 16, 4), prec)
    freqs = np.linspace(50e6, 300e6, 5)
    X = np.stack([inp.rhs_vector(1, i, op.N) for i in range(5)])
    Xg = to_gpu(X, prec)
    Y = op.sweep(freqs, Xg).cpu()
    tol = 1e-6 if prec == "c64" else 1e-14
    for i, f in enumerate(freqs):
        op.set_frequency(f)
        yi = op.matvec(Xg[i].contiguous()).cpu()
        assert rel_l2(yi.numpy(), Y[i].numpy()) <= tol
    Xh = Xg.cpu().pin_memory()
    Yh = torch.empty_like(Xh).pin_memory()
    op.sweep_host(freqs, Xh, Yh, batch=2)
    assert torch.equal(Yh, op.sweep(freqs, Xg, batch=2).cpu())


@pytest.mark.parametrize("prec", ["c64", "c128"])
def test_small_closed_mesh_ragged_grid(prec):
    """Closed icosphere on a ragged non-cubic grid (several tiles + tails)."""
    from oracle.aimx import AIMxOracle
    m = inp.icosphere_mesh(2)
    n = (16, 8, 32)
    orc = AIMxOracle(m.vertices, m.triangles, n)
    op = make_gpu_op(m, n, prec)
    check_structure(op, orc)
    for f in (30e6, 400e6):
        op.set_frequency(f)
        orc.set_frequency(f)
        x = np.random.default_rng(3).standard_normal(op.N) * (1 + 0.5j)
        xg = to_gpu(x, prec)
        yA, yP = op.matvec_parts(xg)
        oA, oR = orc.parts(gpu_input_as_c128(x, prec))
        assert rel_l2(yA.cpu().numpy(), oA) <= TOL[prec]
        assert rel_l2(yP.cpu().numpy(), -oR) <= TOL[prec]


@pytest.mark.parametrize("order", [1, 3])
def test_other_stencil_orders(order):
    from oracle.aimx import AIMxOracle
    m = inp.icosphere_mesh(2)
    n = (16, 16, 16)
    orc = AIMxOracle(m.vertices, m.triangles, n, order=order)
    op = make_gpu_op(m, n, "c128", order=order)
    check_structure(op, orc)
    op.set_frequency(200e6)
    orc.set_frequency(200e6)
    x = np.random.default_rng(4).standard_normal(op.N) + 0j
    yA, yP = op.matvec_parts(to_gpu(x, "c128"))
    oA, oR = orc.parts(x)
    assert rel_l2(yA.cpu().numpy(), oA) <= 1e-11
    assert rel_l2(yP.cpu().numpy(), -oR) <= 1e-11


@pytest.mark.parametrize("prec", ["c64", "c128"])
def test_sweep_results_independent_of_batch_size(prec):
    """Deterministic (bitwise) for a fixed batch size; across batch sizes the
    near-row reduction is partitioned differently, so results agree to rounding."""
    import torch
    op = make_gpu_op(inp.make_mesh(1), (16, 16, 4), prec)
    assert op.stats()["batch_slots"] >= 20
    freqs = np.linspace(20e6, 400e6, 11)
    X = to_gpu(np.stack([inp.rhs_vector(1, i, op.N) for i in range(11)]), prec)
    ref = op.sweep(freqs, X, batch=1).clone()
    tol = 1e-6 if prec == "c64" else 1e-14
    for b in (2, 3, 4, 16, 11 + 9):
        y = op.sweep(freqs, X, batch=b).clone()
        assert torch.equal(op.sweep(freqs, X, batch=b), y)
        assert rel_l2(y.cpu().numpy(), ref.cpu().numpy()) <= tol


@pytest.mark.parametrize("R,order", [(4, 0), (4, 1), (8, 0), (8, 1), (16, 0), (16, 1)])
@pytest.mark.parametrize("prec", ["c64", "c128"])
def test_near_row_group_layouts(R, order, prec, monkeypatch):
    """Every row-group layout of the near matrix (R rows per group, anchor
    linear or Morton row order) against the oracle: parts at one column, and
    a batched sweep (16-column SpMM bucket) per frequency."""
    from oracle.aimx import AIMxOracle
    monkeypatch.setenv("AIMX_NEAR_R", str(R))
    monkeypatch.setenv("AIMX_NEAR_ORDER", str(order))
    m = inp.icosphere_mesh(2)
    n = (16, 8, 32)
    orc = AIMxOracle(m.vertices, m.triangles, n)
    op = make_gpu_op(m, n, prec)
    st = op.stats()
    assert st["near_group_rows"] == R and st["near_row_order"] == order
    assert st["nnz"] <= st["near_union"] * R
    x = np.random.default_rng(5).standard_normal(op.N) * (0.3 - 1j)
    op.set_frequency(250e6)
    orc.set_frequency(250e6)
    yA, yP = op.matvec_parts(to_gpu(x, prec))
    oA, oR = orc.parts(gpu_input_as_c128(x, prec))
    assert rel_l2(yA.cpu().numpy(), oA) <= TOL[prec]
    assert rel_l2(yP.cpu().numpy(), -oR) <= TOL[prec]
    freqs = np.linspace(40e6, 500e6, 11)
    X = np.stack([inp.rhs_vector(1, i, op.N) for i in range(11)])
    Y = op.sweep(freqs, to_gpu(X, prec), batch=11).cpu().numpy()       # 16-column kernels
    for i, f in enumerate(freqs):
        orc.set_frequency(f)
        z = orc.matvec(gpu_input_as_c128(X[i], prec))
        assert rel_l2(Y[i], z) <= TOL[prec]
    freqs = np.linspace(40e6, 500e6, 21)
    X = np.stack([inp.rhs_vector(1, i, op.N) for i in range(21)])
    Y = op.sweep(freqs, to_gpu(X, prec), batch=21).cpu().numpy()       # 32-column kernels
    for i in (0, 7, 20):
        orc.set_frequency(freqs[i])
        assert rel_l2(Y[i], orc.matvec(gpu_input_as_c128(X[i], prec))) <= TOL[prec]


@pytest.mark.parametrize("prec", ["c64", "c128"])
def test_static_cache_roundtrip(prec, tmp_path):
    """aimx_save_static / aimx_setup_cached: the cached context
    reproduces the computed one bit for bit; a cache of another mesh is refused."""
    import torch
    from paper_2009_02281_b200 import AIMxError
    m = inp.make_mesh(1)
    op = make_gpu_op(m, (16, 16, 4), prec)
    path = str(tmp_path / "cfg1.aimxstat")
    op.save_static(path)
    op2 = make_gpu_op(m, (16, 16, 4), prec, static_cache=path)
    for k in ("CA", "CR", "LA_NR"):
        assert np.array_equal(op.static()[k], op2.static()[k])
    freqs = np.linspace(50e6, 300e6, 5)
    X = to_gpu(np.stack([inp.rhs_vector(1, i, op.N) for i in range(5)]), prec)
    assert torch.equal(op.sweep(freqs, X), op2.sweep(freqs, X))
    other = inp.icosphere_mesh(2)
    with pytest.raises(AIMxError):
        make_gpu_op(other, (16, 8, 32), prec, static_cache=path)


@pytest.mark.parametrize("prec", ["c64", "c128"])
def test_sweep_overlapped_near_equals_serial(prec, monkeypatch):
    """The sweep pipeline runs S4+S5 of batch i on its own stream while the
    grid part of batch i+1 runs (double-buffered phi); the same kernels run
    serially with AIMX_NO_OVERLAP: bit-identical results, device and host
    buffers, with the linear-term correction on too."""
    import torch
    op = make_gpu_op(inp.make_mesh(1), (16, 16, 4), prec)
    freqs = np.linspace(30e6, 450e6, 37)
    X = to_gpu(np.stack([inp.rhs_vector(1, 70 + i, op.N) for i in range(37)]), prec)
    for lin in (False, True):
        op.set_linear_term(lin)
        for b in (0, 5):
            a = op.sweep(freqs, X, batch=b).clone()
            Xh = X.cpu().pin_memory()
            Yh = torch.empty_like(Xh).pin_memory()
            op.sweep_host(freqs, Xh, Yh, batch=b)
            monkeypatch.setenv("AIMX_NO_OVERLAP", "1")
            s = op.sweep(freqs, X, batch=b).clone()
            monkeypatch.delenv("AIMX_NO_OVERLAP")
            assert torch.equal(a, s)
            if b > 0:   # same batches: bit for bit
                assert torch.equal(Yh, a.cpu())
            else:       # the host sweep's shorter first batch: equal to rounding
                assert rel_l2(Yh.numpy(), a.cpu().numpy()) <= (1e-6 if prec == "c64" else 1e-13)


def test_sweep_plan_shapes():
    """Sweep batch plans (full slots, remainder last): one point, exactly the
    slots, slots + 1 (a 1-point last batch), an explicit batch size; every
    point equals the single-frequency matvec."""
    import torch
    op = make_gpu_op(inp.make_mesh(1), (16, 16, 4), "c128")
    S = op.stats()["batch_slots"]
    for nf, b in ((1, 0), (S, 0), (S + 1, 0), (S + 1, 7)):
        freqs = np.linspace(50e6, 400e6, nf)
        X = to_gpu(np.stack([inp.rhs_vector(1, 90 + i, op.N) for i in range(nf)]), "c128")
        Y = op.sweep(freqs, X, batch=b).cpu().numpy()
        for i in (0, nf - 1):
            op.set_frequency(freqs[i])
            assert rel_l2(op.matvec(X[i].contiguous()).cpu().numpy(), Y[i]) <= 1e-13
    Y0 = op.sweep(np.zeros(0), torch.zeros(0, op.N, dtype=op.cdtype, device="cuda"))
    assert Y0.shape[0] == 0


@pytest.mark.parametrize("prec", ["c64", "c128"])
def test_matvec_graph_replay_bit_identical(prec, monkeypatch):
    """A matvec whose (buffers, mode, frequency) repeat is captured into a
    CUDA graph and replayed: bit-identical to the eager launches, for the
    combined and the parts outputs, across frequency changes and with the
    linear-term switch (which drops the captured graphs)."""
    import torch
    op = make_gpu_op(inp.make_mesh(1), (16, 16, 4), prec)
    x = to_gpu(inp.rhs_vector(1, 3, op.N), prec)
    y = torch.empty_like(x)
    a, b = torch.empty_like(x), torch.empty_like(x)
    for lin in (False, True):
        op.set_linear_term(lin)
        for f in (150e6, 60e6, 150e6):
            op.set_frequency(f)
            outs = []
            for _ in range(4):                     # eager, capture, replay, replay
                op.matvec(x, y)
                op.matvec_parts(x)
                outs.append((y.clone(),) + tuple(t.clone() for t in op.matvec_parts(x)))
            monkeypatch.setenv("AIMX_NO_GRAPH", "1")
            op.matvec(x, y)
            ref = (y.clone(),) + tuple(t.clone() for t in op.matvec_parts(x))
            monkeypatch.delenv("AIMX_NO_GRAPH")
            for o in outs:
                for u, v in zip(o, ref):
                    assert torch.equal(u, v)


@pytest.mark.parametrize("prec", ["c64", "c128"])
@pytest.mark.parametrize("path", ["planar", "3d", "slab2"])
def test_planar_single_plane_z_pass(prec, path, monkeypatch):
    """A planar mesh occupies ONE z plane.  planar: the 2-D form of S3 (x fwd,
    y fwd * H_hat2 * y inv with the dz = 0 kernel slice, x inv); 3d
    (AIMX_NO_PLANAR=1) and slab2 (emulated slab ranks, kx-slab offsets): the
    general path, whose z pass takes its one-plane form (a multiply by the
    kernel's z-sum) on a grid whose y transform is too long for the fused y/z
    kernel.  Each against the oracle."""
    from oracle.aimx import AIMxOracle
    m = inp.make_mesh(1)
    n = (16, 32, 4)
    orc = AIMxOracle(m.vertices, m.triangles, n)
    if path == "3d":
        monkeypatch.setenv("AIMX_NO_PLANAR", "1")
    op = make_gpu_op(m, n, prec, slab=None if path != "slab2" else ("emulate", 2))
    assert op.stats()["occupied_planes"] == 1
    assert op.stats()["planar"] == (path == "planar")
    for f in (150e6, 600e6):
        op.set_frequency(f)
        orc.set_frequency(f)
        x = inp.rhs_vector(1, 8, op.N)
        yA, yP = op.matvec_parts(to_gpu(x, prec))
        oA, oR = orc.parts(gpu_input_as_c128(x, prec))
        assert rel_l2(yA.cpu().numpy(), oA) <= TOL[prec]
        assert rel_l2(yP.cpu().numpy(), -oR) <= TOL[prec]


@pytest.mark.parametrize("prec", ["c64", "c128"])
def test_matvec_multi_equals_single(prec):
    """Several right-hand sides at one frequency (batched kernels, one spectrum
    for all columns) against single matvecs, across a batch boundary, with the
    linear term on too."""
    op = make_gpu_op(inp.make_mesh(1), (16, 16, 4), prec)
    S = op.stats()["batch_slots"]
    n = S + 3
    X = to_gpu(np.stack([inp.rhs_vector(1, 200 + i, op.N) for i in range(n)]), prec)
    tol = 1e-6 if prec == "c64" else 1e-13
    for lin in (False, True):
        op.set_linear_term(lin)
        op.set_frequency(210e6)
        Y = op.matvec_multi(X).cpu().numpy()
        for i in (0, S - 1, S, n - 1):
            assert rel_l2(Y[i], op.matvec(X[i].contiguous()).cpu().numpy()) <= tol


def test_calls_on_several_streams_are_ordered():
    """Calls on different streams share the context's buffers; the library
    orders them with events (include/aimx.h).  Interleave matvecs, parts and
    sweeps on two side streams and the default stream with no host sync in
    between; every result must equal the serial one bit for bit."""
    import torch
    op = make_gpu_op(inp.make_mesh(2), (256, 16, 4), "c64")
    c = inp.get_config(2)
    xs = [to_gpu(inp.rhs_vector(2, 300 + i, op.N), "c64") for i in range(6)]
    X = to_gpu(np.stack([inp.rhs_vector(2, 310 + i, op.N) for i in range(8)]), "c64")
    op.set_frequency(c.freqs[3])
    ref_mv = [op.matvec(x).clone() for x in xs]
    ref_pa = [tuple(t.clone() for t in op.matvec_parts(x)) for x in xs[:2]]
    ref_sw = op.sweep(c.freqs[:8], X).clone()
    torch.cuda.synchronize()
    sa, sb = torch.cuda.Stream(), torch.cuda.Stream()
    outs = []
    for rep in range(3):
        for i, x in enumerate(xs):
            st = (sa, sb, torch.cuda.current_stream())[i % 3]
            with torch.cuda.stream(st):
                outs.append(("mv", i, op.matvec(x)))
                if i < 2:
                    outs.append(("pa", i, op.matvec_parts(x)))
                if i == 3:
                    outs.append(("sw", 0, op.sweep(c.freqs[:8], X)))
    torch.cuda.synchronize()
    for kind, i, v in outs:
        if kind == "mv":
            assert torch.equal(v, ref_mv[i])
        elif kind == "pa":
            assert all(torch.equal(a, b) for a, b in zip(v, ref_pa[i]))
        else:
            assert torch.equal(v, ref_sw)


def test_planar_z_channel_skip_is_exact(monkeypatch):
    """A planar mesh (z = 0) has Lambda^z = 0 exactly, so the grid passes
    store and transform three channels (x, y, rho); the results equal the
    four-channel run (AIMX_NO_ZSKIP=1) bit for bit, single-column and sweep."""
    import torch
    m = inp.patch_array_mesh(2, 2, 30e-3, 40e-3, 50e-3, 12, 16)
    n = (64, 64, 4)
    freqs = np.linspace(2e9, 6e9, 8)
    outs = []
    for skip in (True, False):
        if not skip:
            monkeypatch.setenv("AIMX_NO_ZSKIP", "1")
        op = make_gpu_op(m, n, "c64")
        assert op.stats()["planar"] and op.stats()["grid_channels"] == (3 if skip else 4)
        X = to_gpu(np.stack([inp.rhs_vector(5, 400 + i, op.N) for i in range(8)]), "c64")
        Y = op.sweep(freqs, X).clone()
        op.set_frequency(freqs[3])
        outs.append((Y, op.matvec(X[3].contiguous()).clone()) + tuple(t.clone() for t in op.matvec_parts(X[3].contiguous())))
        op.close()
    for a, b in zip(outs[0], outs[1]):
        assert torch.equal(a, b)


def test_sweep_status_flags_nonfinite_columns():
    """aimx_sweep_status: 0 for finite sweep outputs, 1 for a column with a NaN."""
    import torch
    op = make_gpu_op(inp.make_mesh(1), (16, 16, 4), "c64")
    X = to_gpu(np.stack([inp.rhs_vector(1, 500 + i, op.N) for i in range(4)]), "c64")
    Y = op.sweep([1e8, 2e8, 3e8, 4e8], X)
    assert np.array_equal(op.sweep_status(Y), [0, 0, 0, 0])
    X[2, 5] = float("nan")
    Y = op.sweep([1e8, 2e8, 3e8, 4e8], X)
    assert np.array_equal(op.sweep_status(Y), [0, 0, 1, 0])
    assert torch.isfinite(torch.view_as_real(Y[[0, 1, 3]])).all()


@pytest.mark.parametrize("prec", ["c64", "c128"])
def test_profiled_serial_sweep_equals_pipelined(prec):
    """bench.py's stage breakdown runs a sweep with every stage bracketed by
    events and its device batches on one stream (AIMX_PROFILE_SERIAL): the
    same kernels on the same batches, so bit-identical to the pipelined sweep;
    every stage of the S1-S5 path is bracketed at least once per batch."""
    import torch
    op = make_gpu_op(inp.make_mesh(1), (16, 16, 4), prec)
    freqs = np.linspace(30e6, 450e6, 37)
    X = to_gpu(np.stack([inp.rhs_vector(1, 90 + i, op.N) for i in range(37)]), prec)
    a = op.sweep(freqs, X, batch=8).clone()
    op.profile_enable(True, serial=True)
    s = op.sweep(freqs, X, batch=8).clone()
    prof = op.profile_read()
    op.profile_enable(False)
    assert torch.equal(a, s)
    nbat = (37 + 7) // 8
    assert prof["spectrum"][1] >= nbat and prof["interp_near"][1] >= nbat
    assert prof["kernels"] > 0 and all(ms >= 0 for ms, n in (prof[k] for k in op.STAGES))


def test_planar_mesh_near_rows_in_linear_order(monkeypatch):
    """One-plane meshes group the near rows in linear anchor order (measured
    faster than Morton on cfg5); AIMX_NEAR_ORDER still overrides, and both
    layouts give the same operator to rounding."""
    m = inp.make_mesh(1)
    op = make_gpu_op(m, (16, 16, 4), "c128")
    assert op.stats()["near_row_order"] == 0
    monkeypatch.setenv("AIMX_NEAR_ORDER", "1")
    op1 = make_gpu_op(m, (16, 16, 4), "c128")
    monkeypatch.delenv("AIMX_NEAR_ORDER")
    assert op1.stats()["near_row_order"] == 1
    x = to_gpu(inp.rhs_vector(1, 3, op.N), "c128")
    op.set_frequency(150e6)
    op1.set_frequency(150e6)
    assert rel_l2(op.matvec(x).cpu().numpy(), op1.matvec(x).cpu().numpy()) <= 1e-13
