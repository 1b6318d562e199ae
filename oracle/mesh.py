"""RWG basis on a triangle mesh (oracle).  TEST INFRASTRUCTURE ONLY.

P:177-178: the current is expanded with Rao-Wilton-Glisson (RWG) functions
"defined on pairs of adjacent triangles".  The paper is silent on ordering and
sign (AMB-2); the reading adopted (R2):

* interior edge = unordered vertex pair {a < b} shared by exactly two
  triangles; a pair in more than two triangles is a mesh error; an edge in one
  triangle is a boundary edge and carries no RWG (open surfaces are allowed);
* RWGs are numbered in ascending lexicographic (a, b);
* T+ is the triangle whose cyclic vertex order contains a->b, T- contains
  b->a; both containing a->b is an orientation error;
* f_n(r) = +(l / 2A+)(r - p+) on T+, -(l / 2A-)(r - p-) on T-, so
  div f_n = +l/A+ on T+ and -l/A- on T-.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np


class MeshError(ValueError):
    pass


@dataclass
class RWG:
    a: np.ndarray      # int64 [N]  edge vertex (a < b)
    b: np.ndarray      # int64 [N]
    tp: np.ndarray     # int64 [N]  triangle T+
    tm: np.ndarray     # int64 [N]  triangle T-
    pp: np.ndarray     # int64 [N]  free vertex of T+
    pm: np.ndarray     # int64 [N]  free vertex of T-
    length: np.ndarray  # float64 [N]
    area_p: np.ndarray  # float64 [N]
    area_m: np.ndarray  # float64 [N]

    @property
    def n(self) -> int:
        return int(self.a.shape[0])


def triangle_areas(V: np.ndarray, T: np.ndarray) -> np.ndarray:
    e1 = V[T[:, 1]] - V[T[:, 0]]
    e2 = V[T[:, 2]] - V[T[:, 0]]
    return 0.5 * np.linalg.norm(np.cross(e1, e2), axis=1)


def build_rwg(V: np.ndarray, T: np.ndarray) -> RWG:
    V = np.asarray(V, dtype=np.float64)
    T = np.asarray(T, dtype=np.int64)
    if T.ndim != 2 or T.shape[1] != 3 or V.ndim != 2 or V.shape[1] != 3:
        raise MeshError("bad array shapes")
    if T.size and (T.min() < 0 or T.max() >= V.shape[0]):
        raise MeshError("triangle index out of range")
    if np.any((T[:, 0] == T[:, 1]) | (T[:, 1] == T[:, 2]) | (T[:, 0] == T[:, 2])):
        raise MeshError("triangle with repeated vertex")
    area = triangle_areas(V, T)
    if np.any(area <= 0.0):
        raise MeshError("degenerate (zero-area) triangle")
    # directed edges u->v of each triangle, with the free (opposite) vertex
    u = T[:, [0, 1, 2]].ravel()
    v = T[:, [1, 2, 0]].ravel()
    free = T[:, [2, 0, 1]].ravel()
    tri = np.repeat(np.arange(T.shape[0]), 3)
    lo = np.minimum(u, v)
    hi = np.maximum(u, v)
    fwd = u < v                      # directed a->b with a < b
    order = np.lexsort((~fwd, hi, lo))   # group by (lo, hi)
    lo, hi, fwd, tri, free = lo[order], hi[order], fwd[order], tri[order], free[order]
    key = lo * (V.shape[0] + 1) + hi
    starts = np.flatnonzero(np.r_[True, key[1:] != key[:-1]])
    counts = np.diff(np.r_[starts, key.shape[0]])
    if np.any(counts > 2):
        raise MeshError("non-manifold edge (more than two triangles)")
    s2 = starts[counts == 2]
    f0, f1 = fwd[s2], fwd[s2 + 1]
    if np.any(f0 == f1):
        raise MeshError("inconsistent triangle orientation")
    # sorted with ~fwd as the last key -> the forward (a->b) entry comes first
    ip, im = s2, s2 + 1
    a, b = lo[ip], hi[ip]
    tp, tm = tri[ip], tri[im]
    pp, pm = free[ip], free[im]
    length = np.linalg.norm(V[b] - V[a], axis=1)
    return RWG(a, b, tp, tm, pp, pm, length, area[tp], area[tm])
