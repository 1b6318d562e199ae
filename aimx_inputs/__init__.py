"""Seeded synthetic inputs shared by the oracle and the CUDA path.

This module holds NONE of the method's arithmetic: it only emits meshes
(vertex coordinates + consistently oriented triangle index triples), the AIM
grid *size* and stencil order chosen by each BASELINE.json config, frequency
lists and seeded complex-Gaussian RWG coefficient vectors.  Everything the
AIMx method computes from these (RWG basis, grid spacing/origin, stencils,
near lists, weights, integrals, spectra, matvecs) lives separately in
``oracle/`` (CPU, fp64, test-only) and ``paper_2009_02281_b200`` (CUDA).

Recipes:

* cfg1 -- 1 m x 1 m PEC plate, 11x11 vertices at 0.1 m pitch, z = 0, every
  vertex jittered in-plane by U(-0.02, 0.02) x 0.1 m (AMB-20); each square
  (i,j) split along (i,j)->(i+1,j+1): 200 triangles, 280 interior RWGs.
  Grid 16x16x4, order 2, near threshold 2 cells, f = 150 MHz.
* cfg2 -- two closed PEC boxes 20 x 0.2 x 0.02 mm at y in [0,0.2] and
  [0.4,0.6] mm, structured faces 333x4x1: 13,352 triangles, 20,028 RWGs.
  Grid 256x16x4, 100 frequencies linspace(1, 50) GHz.
* cfg3 -- PEC sphere r = 1 m, icosahedron midpoint-subdivided 6x and projected
  to the sphere: 40,962 vertices, 81,920 triangles, 122,880 RWGs.  Grid 128^3,
  16 frequencies linspace(50, 300) MHz.
* cfg4 -- closed cube 0.5 m, 58x58 squares per face: 40,368 triangles,
  60,552 RWGs (PMCHWT needs the K operator: SURVEY §8(f) NEXT #1).
* cfg5 -- 8x8 PEC patches 30 (x) x 40 (y) mm at 50 mm pitch, z = 0, each
  40x53 squares: 271,360 triangles, 401,088 RWGs.  Grid 512x512x8,
  64 frequencies linspace(2, 6) GHz.

Seeds: mesh jitter ``default_rng(SeedSequence([2009, 2281, cfg]))``; the RWG
coefficient vector for frequency index i ``default_rng(SeedSequence([2009,
2281, cfg, 1, i]))`` with ``x = standard_normal(N) + 1j*standard_normal(N)``
(AMB-19).  Planar meshes are oriented +z, closed meshes outward.
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

__all__ = [
    "Mesh", "Config", "CONFIGS", "get_config", "make_mesh", "rhs_vector",
    "plate_mesh", "box_mesh", "icosphere_mesh", "patch_array_mesh",
]


@dataclass(frozen=True)
class Mesh:
    vertices: np.ndarray   # float64 [nv, 3], metres
    triangles: np.ndarray  # int32 [nt, 3], 0-based, consistently oriented

    @property
    def nv(self) -> int:
        return int(self.vertices.shape[0])

    @property
    def nt(self) -> int:
        return int(self.triangles.shape[0])


@dataclass(frozen=True)
class Config:
    cfg: int
    name: str
    grid_n: tuple          # (N_x, N_y, N_z) unpadded AIM grid points
    order: int             # stencil order n (n+1 points per axis)
    near_cells: int        # near threshold T in grid cells
    freqs: np.ndarray = field(repr=False)  # Hz
    precisions: tuple = ("c64",)
    expected_rwg: int = 0
    expected_tri: int = 0


def _seed(*k: int) -> np.random.Generator:
    return np.random.default_rng(np.random.SeedSequence([2009, 2281, *k]))


# --------------------------------------------------------------------------- plates
def _grid_quads_to_tris(idx: np.ndarray) -> np.ndarray:
    """idx[i, j] = vertex index of lattice point (i, j) (i along x, j along y).
    Every square (i, j) is split along (i,j)->(i+1,j+1) into two +z oriented
    triangles, emitted square by square in (j, i) order."""
    ni, nj = idx.shape[0] - 1, idx.shape[1] - 1
    tris = []
    for j in range(nj):
        for i in range(ni):
            a, b = idx[i, j], idx[i + 1, j]
            c, d = idx[i + 1, j + 1], idx[i, j + 1]
            tris.append((a, b, c))
            tris.append((a, c, d))
    return np.asarray(tris, dtype=np.int32)


def plate_mesh(nx: int, ny: int, lx: float, ly: float, x0: float = 0.0,
               y0: float = 0.0, jitter=None) -> Mesh:
    """Structured planar rectangle at z = 0 with (nx x ny) squares."""
    xs = x0 + lx * np.arange(nx + 1) / nx
    ys = y0 + ly * np.arange(ny + 1) / ny
    V = np.zeros(((nx + 1) * (ny + 1), 3))
    idx = np.zeros((nx + 1, ny + 1), dtype=np.int64)
    k = 0
    for j in range(ny + 1):
        for i in range(nx + 1):
            V[k] = (xs[i], ys[j], 0.0)
            idx[i, j] = k
            k += 1
    if jitter is not None:
        V[:, :2] += jitter
    return Mesh(V, _grid_quads_to_tris(idx))


def patch_array_mesh(npx: int, npy: int, lx: float, ly: float, pitch: float,
                     nx: int, ny: int) -> Mesh:
    verts, tris, off = [], [], 0
    for py in range(npy):
        for px in range(npx):
            m = plate_mesh(nx, ny, lx, ly, x0=px * pitch, y0=py * pitch)
            verts.append(m.vertices)
            tris.append(m.triangles + off)
            off += m.nv
    return Mesh(np.concatenate(verts), np.concatenate(tris).astype(np.int32))


# --------------------------------------------------------------------------- boxes
def box_mesh(nx: int, ny: int, nz: int, lo, hi) -> Mesh:
    """Closed axis-aligned box surface, structured (nx, ny, nz) divisions,
    every quad split into two outward-oriented triangles."""
    lo = np.asarray(lo, float)
    hi = np.asarray(hi, float)
    n = (nx, ny, nz)
    coords = [lo[a] + (hi[a] - lo[a]) * np.arange(n[a] + 1) / n[a] for a in range(3)]
    index = {}
    V = []
    for k in range(nz + 1):
        for j in range(ny + 1):
            for i in range(nx + 1):
                if i in (0, nx) or j in (0, ny) or k in (0, nz):
                    index[(i, j, k)] = len(V)
                    V.append((coords[0][i], coords[1][j], coords[2][k]))
    V = np.asarray(V)
    T = []

    def quad(a, b, c, d):  # corners counter-clockwise about the outward normal
        T.append((index[a], index[b], index[c]))
        T.append((index[a], index[c], index[d]))

    for j in range(ny):          # z faces
        for i in range(nx):
            quad((i, j, 0), (i, j + 1, 0), (i + 1, j + 1, 0), (i + 1, j, 0))
            quad((i, j, nz), (i + 1, j, nz), (i + 1, j + 1, nz), (i, j + 1, nz))
    for k in range(nz):          # y faces
        for i in range(nx):
            quad((i, 0, k), (i + 1, 0, k), (i + 1, 0, k + 1), (i, 0, k + 1))
            quad((i, ny, k), (i, ny, k + 1), (i + 1, ny, k + 1), (i + 1, ny, k))
    for k in range(nz):          # x faces
        for j in range(ny):
            quad((0, j, k), (0, j, k + 1), (0, j + 1, k + 1), (0, j + 1, k))
            quad((nx, j, k), (nx, j + 1, k), (nx, j + 1, k + 1), (nx, j, k + 1))
    return Mesh(V, np.asarray(T, dtype=np.int32))


def merge_meshes(*ms: Mesh) -> Mesh:
    verts, tris, off = [], [], 0
    for m in ms:
        verts.append(m.vertices)
        tris.append(m.triangles + off)
        off += m.nv
    return Mesh(np.concatenate(verts), np.concatenate(tris).astype(np.int32))


# --------------------------------------------------------------------------- sphere
def icosphere_mesh(subdiv: int, radius: float = 1.0) -> Mesh:
    """Icosahedron, midpoint-subdivided ``subdiv`` times, vertices projected
    onto the sphere; outward orientation preserved by the subdivision."""
    t = (1.0 + 5.0 ** 0.5) / 2.0
    V = [(-1, t, 0), (1, t, 0), (-1, -t, 0), (1, -t, 0),
         (0, -1, t), (0, 1, t), (0, -1, -t), (0, 1, -t),
         (t, 0, -1), (t, 0, 1), (-t, 0, -1), (-t, 0, 1)]
    F = [(0, 11, 5), (0, 5, 1), (0, 1, 7), (0, 7, 10), (0, 10, 11),
         (1, 5, 9), (5, 11, 4), (11, 10, 2), (10, 7, 6), (7, 1, 8),
         (3, 9, 4), (3, 4, 2), (3, 2, 6), (3, 6, 8), (3, 8, 9),
         (4, 9, 5), (2, 4, 11), (6, 2, 10), (8, 6, 7), (9, 8, 1)]
    V = [np.asarray(v, float) / np.linalg.norm(v) for v in V]
    for _ in range(subdiv):
        mid = {}
        F2 = []

        def midpoint(a, b):
            key = (a, b) if a < b else (b, a)
            if key not in mid:
                p = V[a] + V[b]
                V.append(p / np.linalg.norm(p))
                mid[key] = len(V) - 1
            return mid[key]

        for (a, b, c) in F:
            ab, bc, ca = midpoint(a, b), midpoint(b, c), midpoint(c, a)
            F2 += [(a, ab, ca), (b, bc, ab), (c, ca, bc), (ab, bc, ca)]
        F = F2
    return Mesh(np.asarray(V) * radius, np.asarray(F, dtype=np.int32))


# --------------------------------------------------------------------------- configs
CONFIGS = {
    1: Config(1, "plate", (16, 16, 4), 2, 2, np.array([150e6]),
              ("c128", "c64"), 280, 200),
    2: Config(2, "strips", (256, 16, 4), 2, 2, np.linspace(1e9, 50e9, 100),
              ("c64",), 20028, 13352),
    3: Config(3, "sphere", (128, 128, 128), 2, 2, np.linspace(50e6, 300e6, 16),
              ("c64", "c128"), 122880, 81920),
    4: Config(4, "cube", (96, 96, 96), 2, 2, np.linspace(100e6, 600e6, 32),
              ("c64",), 60552, 40368),
    5: Config(5, "patches", (512, 512, 8), 2, 2, np.linspace(2e9, 6e9, 64),
              ("c64",), 401088, 271360),
}


def get_config(cfg: int) -> Config:
    return CONFIGS[int(cfg)]


def make_mesh(cfg: int) -> Mesh:
    cfg = int(cfg)
    if cfg == 1:
        rng = _seed(1)
        jit = rng.uniform(-0.02, 0.02, size=(121, 2)) * 0.1
        return plate_mesh(10, 10, 1.0, 1.0, jitter=jit)
    if cfg == 2:
        a = box_mesh(333, 4, 1, (0.0, 0.0, 0.0), (20e-3, 0.2e-3, 0.02e-3))
        b = box_mesh(333, 4, 1, (0.0, 0.4e-3, 0.0), (20e-3, 0.6e-3, 0.02e-3))
        return merge_meshes(a, b)
    if cfg == 3:
        return icosphere_mesh(6, 1.0)
    if cfg == 4:
        return box_mesh(58, 58, 58, (0.0, 0.0, 0.0), (0.5, 0.5, 0.5))
    if cfg == 5:
        return patch_array_mesh(8, 8, 30e-3, 40e-3, 50e-3, 40, 53)
    raise ValueError(f"unknown config {cfg}")


def rhs_vector(cfg: int, i: int, n: int) -> np.ndarray:
    """Seeded complex128 i.i.d. N(0,1) RWG coefficients for frequency index i."""
    rng = _seed(int(cfg), 1, int(i))
    return rng.standard_normal(n) + 1j * rng.standard_normal(n)


def rhs_matrix(cfg: int, n: int, idx) -> np.ndarray:
    return np.stack([rhs_vector(cfg, i, n) for i in idx])
