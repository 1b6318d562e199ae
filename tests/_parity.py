"""Shared helpers for GPU-vs-oracle parity (tests and smoke only)."""
from __future__ import annotations

import numpy as np

import aimx_inputs as inp

TOL = {"c128": 1e-11, "c64": 2e-5}   # north_star: rel-L2 per output vector


def rel_l2(a, b) -> float:
    a = np.asarray(a)
    b = np.asarray(b)
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


def make_gpu_op(mesh, n, prec, order=2, near_cells=2, **kw):
    from paper_2009_02281_b200 import AIMx
    return AIMx(mesh.vertices, mesh.triangles, n, order=order, near_cells=near_cells, prec=prec, **kw)


def to_gpu(x, prec):
    import torch
    dt = torch.complex64 if prec == "c64" else torch.complex128
    return torch.as_tensor(np.asarray(x)).to(dt).cuda().contiguous()


def gpu_input_as_c128(x, prec):
    """The exact values the GPU consumes, upcast (c64 path: rounded to complex64)."""
    if prec == "c64":
        return np.asarray(x).astype(np.complex64).astype(np.complex128)
    return np.asarray(x, np.complex128)


def check_structure(op_gpu, op_orc):
    """Bit-exact integer structures: RWG table, anchors, near CSR."""
    ab, tpm, fpm = op_gpu.rwg()
    r = op_orc.rwg
    assert np.array_equal(ab[:, 0], r.a) and np.array_equal(ab[:, 1], r.b)
    assert np.array_equal(tpm[:, 0], r.tp) and np.array_equal(tpm[:, 1], r.tm)
    assert np.array_equal(fpm[:, 0], r.pp) and np.array_equal(fpm[:, 1], r.pm)
    assert np.array_equal(op_gpu.anchors(), op_orc.A)
    rp, col = op_gpu.near_csr()
    assert np.array_equal(rp, op_orc.rowptr) and np.array_equal(col, op_orc.col)
    st = op_gpu.stats()
    assert st["h"] == op_orc.grid.h
    assert np.array_equal(np.array(st["origin"]), op_orc.grid.origin)


_ORC = {}


def oracle_config(cfg: int):
    """The oracle of a config with its grid part only (static=False), built
    once per test session (cfg5 takes ~40 s) and shared by the full-size tests."""
    if cfg not in _ORC:
        from oracle.aimx import from_config
        _ORC[cfg] = from_config(cfg, static=False)
    return _ORC[cfg]
