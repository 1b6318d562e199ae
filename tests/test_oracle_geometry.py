"""Pins for oracle mesh/grid/near-map code (not gpu)."""
import json
import os

import numpy as np
import pytest

import aimx_inputs as inp
from oracle import grid as G
from oracle.mesh import MeshError, build_rwg

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "paper_fixed_points.json")))


def test_closed_mesh_edge_count_rule():
    # a closed mesh of 3,080 triangles has 4,620 edges (E = 3T/2)
    g = GOLD["closed_mesh_counts"]
    assert g["edges"] * 2 == g["triangles"] * 3
    for m in (inp.icosphere_mesh(2), inp.box_mesh(3, 2, 1, (0, 0, 0), (1, 0.5, 0.2))):
        rwg = build_rwg(m.vertices, m.triangles)
        assert rwg.n * 2 == m.nt * 3


@pytest.mark.parametrize("cfg", [1, 2])
def test_config_counts(cfg):
    c = inp.get_config(cfg)
    m = inp.make_mesh(cfg)
    assert m.nt == c.expected_tri
    assert build_rwg(m.vertices, m.triangles).n == c.expected_rwg


def test_rwg_orientation_and_charge_neutrality():
    m = inp.make_mesh(1)
    r = build_rwg(m.vertices, m.triangles)
    # sorted lexicographically, a < b
    assert np.all(r.a < r.b)
    key = r.a * 10**6 + r.b
    assert np.all(np.diff(key) > 0)
    # T+ contains a->b in its cyclic order, T- contains b->a
    T = m.triangles
    for n in range(r.n):
        tp, tm = list(T[r.tp[n]]), list(T[r.tm[n]])
        ia = tp.index(r.a[n])
        assert tp[(ia + 1) % 3] == r.b[n]
        ib = tm.index(r.b[n])
        assert tm[(ib + 1) % 3] == r.a[n]
    # integral of div f over the support = l/A+ A+ - l/A- A- = 0
    tot = r.length / r.area_p * r.area_p - r.length / r.area_m * r.area_m
    assert np.max(np.abs(tot)) < 1e-15


def test_mesh_errors():
    V = np.array([[0, 0, 0], [1, 0, 0], [0, 1, 0], [1, 1, 0]], float)
    with pytest.raises(MeshError):  # inconsistent orientation
        build_rwg(V, np.array([[0, 1, 2], [1, 2, 3]]))
    with pytest.raises(MeshError):  # degenerate
        build_rwg(V, np.array([[0, 1, 1]]))
    with pytest.raises(MeshError):  # index out of range
        build_rwg(V, np.array([[0, 1, 9]]))
    V5 = np.vstack([V, [[0, 0, 1], [0, 0, -1]]])
    with pytest.raises(MeshError):  # non-manifold edge 0-1 in three triangles
        build_rwg(V5, np.array([[0, 1, 2], [1, 0, 4], [0, 1, 5]]))


@pytest.mark.parametrize("cfg,expect", [
    (2, 0.02e-3 / 253), (3, 2.0 / 125), (4, 0.5 / 93), (5, 0.39 / 509)])
def test_grid_spacing_rule(cfg, expect):
    # SURVEY C.3 reading: h = max ext_a / (N_a - 1 - 2m)
    m = inp.make_mesh(cfg)
    c = inp.get_config(cfg)
    g = G.grid_spec(m.vertices, c.grid_n, c.order)
    if cfg == 2:
        expect = 20e-3 / 253
    assert g.h == pytest.approx(expect, rel=1e-12)


def test_cfg1_grid_and_planar_nodes():
    m = inp.make_mesh(1)
    g = G.grid_spec(m.vertices, (16, 16, 4), 2)
    ext = m.vertices.max(0) - m.vertices.min(0)
    assert g.h == max(ext[0] / 13, ext[1] / 13)
    # the plane z = 0 sits exactly on node z = 1 (u_z = m = 1)
    assert (0.0 - g.origin[2]) / g.h == 1.0


def _brute_min_node_distance(Am, An, order, h):
    # explicit geometric min distance between the two (n+1)^3 node sets
    off = np.stack(np.meshgrid(*[np.arange(order + 1)] * 3, indexing="ij"), -1).reshape(-1, 3)
    Pm = (Am + off) * h
    Pn = (An + off) * h
    d = np.linalg.norm(Pm[:, None, :] - Pn[None, :, :], axis=-1)
    return d.min()


def test_near_map_against_geometric_brute_force():
    rng = np.random.default_rng(11)
    A = rng.integers(0, 12, size=(150, 3))
    h = 0.37
    rp, col = G.near_csr(A, 2, 2)
    rpb, colb = G.near_csr_bruteforce(A, 2, 2)
    assert np.array_equal(rp, rpb) and np.array_equal(col, colb)
    near = set()
    for m in range(A.shape[0]):
        for c in col[rp[m]:rp[m + 1]]:
            near.add((m, int(c)))
    for m in range(0, 150, 7):
        for n in range(150):
            d = _brute_min_node_distance(A[m], A[n], 2, h)
            assert ((m, n) in near) == (d <= 2 * h * (1 + 1e-12))


def test_cfg1_near_map_properties(cfg1_oracle):
    op = cfg1_oracle
    rp, col = op.rowptr, op.col
    N = op.N
    M = np.zeros((N, N), bool)
    for m in range(N):
        M[m, col[rp[m]:rp[m + 1]]] = True
        assert np.all(np.diff(col[rp[m]:rp[m + 1]]) > 0)
    assert np.array_equal(M, M.T)
    assert np.all(np.diag(M))
    # SURVEY Appendix A (same readings, independent script): 24,978 pairs
    assert col.shape[0] == 24978
    # every stencil inside the grid
    assert op.A.min() >= 0
    assert np.all(op.A.max(0) <= np.array(op.grid.n) - 1 - op.order)


def test_anchor_rule_ties_round_half_up():
    # u exactly x.5 -> floor(u + 0.5) rounds up (reading R4)
    from oracle.mesh import build_rwg as br
    h = 1.0
    V = np.array([[2.0, 2.0, 2.0], [3.0, 2.0, 2.0], [2.5, 3.5, 2.0], [2.5, 0.5, 2.0]])
    T = np.array([[0, 1, 2], [1, 0, 3]])
    r = br(V, T)
    g = G.Grid((10, 10, 10), 2, h, np.zeros(3))
    c = G.stencil_centres(V, r)
    assert np.allclose(c, [[2.5, 2.0, 2.0]])
    A = G.anchors(V, r, g)
    assert A.tolist() == [[2, 1, 1]]


@pytest.mark.parametrize("mesh", [inp.icosphere_mesh(3), inp.box_mesh(5, 3, 2, (0, 0, 0), (1, .5, .2))])
def test_closed_inputs_are_outward_oriented(mesh):
    V, T = mesh.vertices, mesh.triangles
    v0, v1, v2 = V[T[:, 0]], V[T[:, 1]], V[T[:, 2]]
    # signed volume (divergence theorem) > 0 for outward orientation
    vol = np.einsum("ij,ij->i", v0, np.cross(v1, v2)).sum() / 6.0
    assert vol > 0
    build_rwg(V, T)   # consistent orientation or MeshError


def test_icosphere_counts_at_config_size():
    m = inp.icosphere_mesh(3)
    assert m.nv == 642 and m.nt == 1280
