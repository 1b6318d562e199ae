"""B200-native AIMx matrix-vector product (arxiv 2009.02281), Python binding.

Thin ctypes marshalling over the C ABI in ``include/aimx.h`` (libaimx.so,
hand-written sm_100a kernels).  Every step of the path runs in the library's
kernels; PyTorch is used only for device memory and streams.  There is NO CPU
fallback: if the shared library is missing or no CUDA device is present the
calls raise.

    op = AIMx(vertices, triangles, n=(16, 16, 4), prec="c128")
    op.set_frequency(150e6)
    y = op.matvec(x)               # x: complex torch tensor on cuda
    yA, yPhi = op.matvec_parts(x)  # L_A x, L_phi x
    Y = op.sweep(freqs, X)         # Y[i] = Z(f_i) X[i]
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

__all__ = ["AIMx", "AIMxError", "load_library", "library_path", "ABI_FUNCTIONS"]

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB = None

AIMX_C64, AIMX_C128 = 0, 1


class AIMxError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"aimx status {status}: {msg}")
        self.status = status


class _Mesh(C.Structure):
    _fields_ = [("nv", C.c_int64), ("vertices", C.POINTER(C.c_double)),
                ("nt", C.c_int64), ("triangles", C.POINTER(C.c_int32))]


class _Grid(C.Structure):
    _fields_ = [("n", C.c_int32 * 3), ("order", C.c_int32), ("near_cells", C.c_int32),
                ("h", C.c_double), ("origin", C.c_double * 3)]


class _Stats(C.Structure):
    _fields_ = [("num_unknowns", C.c_int64), ("nnz", C.c_int64), ("occupied_nodes", C.c_int64),
                ("occupied_lines", C.c_int64), ("occupied_planes", C.c_int64),
                ("projection_entries", C.c_int64), ("device_bytes", C.c_int64), ("batch_slots", C.c_int64),
                ("setup_seconds", C.c_double),
                ("n", C.c_int32 * 3), ("order", C.c_int32), ("h", C.c_double),
                ("origin", C.c_double * 3), ("near_group_rows", C.c_int32), ("near_row_order", C.c_int32),
                ("near_union", C.c_int64), ("planar", C.c_int32), ("kop_grad", C.c_int32),
                ("grid_channels", C.c_int32), ("reserved", C.c_int32)]


_P = C.c_void_p
ABI_FUNCTIONS = {
    "aimx_setup": (C.c_int, [C.POINTER(_Mesh), C.POINTER(_Grid), C.c_int, C.c_int, _P, C.POINTER(_P)]),
    "aimx_set_frequency": (C.c_int, [_P, C.c_double]),
    "aimx_set_linear_term": (C.c_int, [_P, C.c_int]),
    "aimx_get_linear_term": (C.c_int, [_P, C.POINTER(C.c_int)]),
    "aimx_set_conventional": (C.c_int, [_P, C.c_int]),
    "aimx_get_aim_entries": (C.c_int, [_P, _P, _P]),
    "aimx_get_kop_static": (C.c_int, [_P, _P]),
    "aimx_set_kop": (C.c_int, [_P, C.c_int]),
    "aimx_set_cfie": (C.c_int, [_P, C.c_int]),
    "aimx_matvec_multi": (C.c_int, [_P, C.c_int64, _P, _P, _P]),
    "aimx_matvec_pmchwt": (C.c_int, [_P, C.c_double, _P, _P, _P]),
    "aimx_matvec_kop": (C.c_int, [_P, _P, _P, _P]),
    "aimx_matvec": (C.c_int, [_P, _P, _P, _P]),
    "aimx_matvec_parts": (C.c_int, [_P, _P, _P, _P, _P]),
    "aimx_sweep": (C.c_int, [_P, C.c_int64, C.POINTER(C.c_double), _P, _P, C.c_int32, _P]),
    "aimx_sweep_host": (C.c_int, [_P, C.c_int64, C.POINTER(C.c_double), _P, _P, C.c_int32, _P]),
    "aimx_num_unknowns": (C.c_int64, [_P]),
    "aimx_get_stats": (C.c_int, [_P, C.POINTER(_Stats)]),
    "aimx_get_rwg": (C.c_int, [_P, _P, _P, _P]),
    "aimx_get_anchors": (C.c_int, [_P, _P]),
    "aimx_get_near_csr": (C.c_int, [_P, _P, _P, C.POINTER(C.c_int64)]),
    "aimx_get_static": (C.c_int, [_P, _P, _P, _P, _P, _P, _P]),
    "aimx_get_linear_entries": (C.c_int, [_P, _P, _P, _P]),
    "aimx_get_weights": (C.c_int, [_P, _P]),
    "aimx_get_spectrum": (C.c_int, [_P, C.c_int, _P]),
    "aimx_profile_enable": (C.c_int, [_P, C.c_int]),
    "aimx_profile_read": (C.c_int, [_P, _P, _P, C.POINTER(C.c_int64)]),
    "aimx_profile_stages": (C.c_int, [_P, C.c_int32]),
    "aimx_destroy": (None, [_P]),
    "aimx_status_string": (C.c_char_p, [C.c_int]),
    "aimx_last_error": (C.c_char_p, [_P]),
    "aimx_last_setup_error": (C.c_char_p, []),
    "aimx_version": (C.c_char_p, []),
    "aimx_slab_plan": (C.c_int, [_P, C.c_int32, C.c_int32, C.c_int32, _P]),
    "aimx_setup_slab": (C.c_int, [C.POINTER(_Mesh), C.POINTER(_Grid), C.c_int, C.c_int, C.c_int32,
                                  C.c_int32, _P, _P, C.POINTER(_P)]),
    "aimx_nccl_unique_id": (C.c_int, [_P]),
    "aimx_sync": (C.c_int, [_P, C.c_double]),
    "aimx_sweep_status": (C.c_int, [_P, C.c_int64, _P, _P, _P]),
    "aimx_save_static": (C.c_int, [_P, C.c_char_p]),
    "aimx_solve": (C.c_int, [_P, C.c_int64, C.POINTER(C.c_double), _P, _P, C.c_double, C.c_int32, C.c_int32,
                             C.POINTER(C.c_int32), C.POINTER(C.c_double), _P]),
    "aimx_setup_cached": (C.c_int, [C.POINTER(_Mesh), C.POINTER(_Grid), C.c_int, C.c_int, C.c_char_p, _P,
                                    C.POINTER(_P)]),
}


def slab_plan(n, order: int, world: int, rank: int) -> dict:
    """Host-only slab decomposition of the grid (aimx_slab_plan; no GPU)."""
    lib = load_library()
    nn = (C.c_int32 * 3)(*[int(v) for v in n])
    out = (C.c_int32 * 6)()
    _check(lib, lib.aimx_slab_plan(C.cast(nn, _P), int(order), int(world), int(rank), C.cast(out, _P)))
    return {"rows": (out[0], out[1]), "phi_rows": (out[0], out[2]), "kx": (out[3], out[4])}


def nccl_unique_id() -> bytes:
    """128-byte ncclUniqueId for aimx_setup_slab (call on rank 0, broadcast)."""
    lib = load_library()
    buf = (C.c_uint8 * 128)()
    _check(lib, lib.aimx_nccl_unique_id(C.cast(buf, _P)))
    return bytes(buf)


def library_path() -> str:
    return os.path.join(_HERE, "libaimx.so")


def load_library():
    """Load libaimx.so (built in-tree by ``python -m paper_2009_02281_b200.build``
    or ``__graft_entry__.build()``).  Raises if it is missing."""
    global _LIB
    if _LIB is not None:
        return _LIB
    path = library_path()
    if not os.path.exists(path):
        raise ImportError(f"libaimx.so not built at {path}; run __graft_entry__.build() "
                          "(there is no CPU fallback)")
    lib = C.CDLL(path)
    for name, (res, args) in ABI_FUNCTIONS.items():
        f = getattr(lib, name)
        f.restype = res
        f.argtypes = args
    _LIB = lib
    return lib


def _torch():
    import torch
    return torch


def _check(lib, st, ctx=None):
    if st != 0:
        msg = (lib.aimx_last_error(ctx) if ctx else lib.aimx_last_setup_error()) or b""
        raise AIMxError(st, f"{lib.aimx_status_string(st).decode()}: {msg.decode()}")


class AIMx:
    """One AIMx operator context on one CUDA device (S0 setup in __init__)."""

    def __init__(self, vertices, triangles, n, order: int = 2, near_cells: int = 2,
                 h: float = 0.0, origin=(0.0, 0.0, 0.0), prec: str = "c64",
                 device: int | None = None, stream=None, slab=None, static_cache: str | None = None):
        """slab: None (one GPU), ("emulate", world) (slab-decomposed FFT with
        `world` ranks emulated on this GPU), or (rank, world, nccl_id) (this
        process is one rank of the slab-decomposed FFT, NCCL).  static_cache: path of
        an aimx_save_static file to load the static matrices from (one context)."""
        torch = _torch()
        if not torch.cuda.is_available():
            raise RuntimeError("AIMx needs a CUDA device (no CPU fallback)")
        self.lib = load_library()
        self.prec = prec
        self.cdtype = {"c64": torch.complex64, "c128": torch.complex128}[prec]
        self.device = torch.cuda.current_device() if device is None else int(device)
        V = np.ascontiguousarray(vertices, dtype=np.float64)
        T = np.ascontiguousarray(triangles, dtype=np.int32)
        mesh = _Mesh(V.shape[0], V.ctypes.data_as(C.POINTER(C.c_double)),
                     T.shape[0], T.ctypes.data_as(C.POINTER(C.c_int32)))
        g = _Grid()
        for a in range(3):
            g.n[a] = int(n[a])
            g.origin[a] = float(origin[a])
        g.order, g.near_cells, g.h = int(order), int(near_cells), float(h)
        with torch.cuda.device(self.device):
            s = stream if stream is not None else torch.cuda.current_stream()
            self._stream = s
            ctx = _P()
            pc = AIMX_C64 if prec == "c64" else AIMX_C128
            if slab is None and static_cache is not None:
                st = self.lib.aimx_setup_cached(C.byref(mesh), C.byref(g), pc, self.device,
                                                os.fsencode(static_cache), _P(s.cuda_stream), C.byref(ctx))
            elif slab is None:
                st = self.lib.aimx_setup(C.byref(mesh), C.byref(g), pc, self.device,
                                         _P(s.cuda_stream), C.byref(ctx))
            elif slab[0] == "emulate":
                st = self.lib.aimx_setup_slab(C.byref(mesh), C.byref(g), pc, self.device, 0,
                                              int(slab[1]), None, _P(s.cuda_stream), C.byref(ctx))
            else:
                rank, world, nid = slab
                idb = (C.c_uint8 * 128).from_buffer_copy(bytes(nid))
                st = self.lib.aimx_setup_slab(C.byref(mesh), C.byref(g), pc, self.device, int(rank),
                                              int(world), C.cast(idb, _P), _P(s.cuda_stream),
                                              C.byref(ctx))
        _check(self.lib, st)
        self.ctx = ctx
        self.N = int(self.lib.aimx_num_unknowns(ctx))
        self.freq = None

    # ----------------------------------------------------------- lifecycle
    def save_static(self, path: str):
        """Write the static matrices (aimx_save_static) for AIMx(..., static_cache=path)."""
        _check(self.lib, self.lib.aimx_save_static(self.ctx, os.fsencode(path)), self.ctx)

    def sync(self, timeout_s: float = 0.0):
        """Wait for every call enqueued on the context (aimx_sync); NCCL
        contexts abort their communicator on an asynchronous NCCL error or
        after timeout_s seconds (> 0) and raise."""
        _check(self.lib, self.lib.aimx_sync(self.ctx, float(timeout_s)), self.ctx)

    def close(self):
        if getattr(self, "ctx", None):
            self.lib.aimx_destroy(self.ctx)
            self.ctx = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _s(self, stream):
        torch = _torch()
        s = stream if stream is not None else torch.cuda.current_stream(self.device)
        return _P(s.cuda_stream)

    def _dev(self):
        return _torch().device("cuda", self.device)

    def _vec(self, x, shape):
        torch = _torch()
        if not (isinstance(x, torch.Tensor) and x.is_cuda and x.dtype == self.cdtype
                and x.is_contiguous() and tuple(x.shape) == shape):
            raise ValueError(f"expected contiguous {self.cdtype} cuda tensor of shape {shape}")
        if x.device.index != self.device:
            raise ValueError(f"tensor on cuda:{x.device.index}, the context is on cuda:{self.device}")
        return _P(x.data_ptr())

    # ----------------------------------------------------------- hot path
    def set_frequency(self, f_hz: float):
        _check(self.lib, self.lib.aimx_set_frequency(self.ctx, float(f_hz)), self.ctx)
        self.freq = float(f_hz)

    def set_linear_term(self, on: bool = True):
        """Linear-term accuracy modification: k0^2 G_lin integrated
        directly on overlapping pairs for every later matvec / sweep / solve."""
        _check(self.lib, self.lib.aimx_set_linear_term(self.ctx, int(bool(on))), self.ctx)

    def set_conventional(self, on: bool = True):
        """Conventional AIM mode: the near region regenerated by
        direct integration at every frequency (the method AIMx is compared with)."""
        _check(self.lib, self.lib.aimx_set_conventional(self.ctx, int(bool(on))), self.ctx)

    def set_kop(self, on: bool = True):
        """Enable the double-layer operator K (aimx_set_kop)."""
        _check(self.lib, self.lib.aimx_set_kop(self.ctx, int(bool(on))), self.ctx)

    def set_cfie(self, on: bool = True):
        """CFIE (eq:CFIEdis): matvec / sweep / solve apply -j w mu0 L - eta0 K."""
        _check(self.lib, self.lib.aimx_set_cfie(self.ctx, int(bool(on))), self.ctx)

    def matvec_pmchwt(self, eps_r: float, x, y=None, stream=None):
        """PMCHWT [y_E; y_H] for x = [J; M] (2N), interior eps_r (aimx_matvec_pmchwt)."""
        torch = _torch()
        if y is None:
            y = torch.empty(2 * self.N, dtype=self.cdtype, device=self._dev())
        _check(self.lib, self.lib.aimx_matvec_pmchwt(self.ctx, float(eps_r), self._vec(x, (2 * self.N,)),
                                                     self._vec(y, (2 * self.N,)), self._s(stream)), self.ctx)
        return y

    def matvec_kop(self, x, y=None, stream=None):
        """y = Kmat x at the bound frequency (aimx_matvec_kop)."""
        torch = _torch()
        if y is None:
            y = torch.empty(self.N, dtype=self.cdtype, device=self._dev())
        _check(self.lib, self.lib.aimx_matvec_kop(self.ctx, self._vec(x, (self.N,)), self._vec(y, (self.N,)),
                                                  self._s(stream)), self.ctx)
        return y

    def K_static(self):
        """C_K of the double-layer operator on the near pattern (CSR order), fp64
        (NEXT #1 groundwork: the device static near fill)."""
        nnz = C.c_int64()
        _check(self.lib, self.lib.aimx_get_near_csr(self.ctx, None, None, C.byref(nnz)), self.ctx)
        ck = np.empty(nnz.value)
        _check(self.lib, self.lib.aimx_get_kop_static(self.ctx, _P(ck.ctypes.data)), self.ctx)
        return ck

    def aim_entries(self):
        """(D_A, D_rho) complex128 [nnz] in CSR order, at the bound frequency."""
        nnz = C.c_int64()
        _check(self.lib, self.lib.aimx_get_near_csr(self.ctx, None, None, C.byref(nnz)), self.ctx)
        da = np.empty(nnz.value, np.complex128)
        dr = np.empty(nnz.value, np.complex128)
        _check(self.lib, self.lib.aimx_get_aim_entries(self.ctx, _P(da.ctypes.data), _P(dr.ctypes.data)), self.ctx)
        return da, dr

    @property
    def linear_term(self) -> bool:
        v = C.c_int()
        _check(self.lib, self.lib.aimx_get_linear_term(self.ctx, C.byref(v)), self.ctx)
        return bool(v.value)

    def matvec(self, x, y=None, stream=None):
        torch = _torch()
        if y is None:
            y = torch.empty(self.N, dtype=self.cdtype, device=self._dev())
        _check(self.lib, self.lib.aimx_matvec(self.ctx, self._vec(x, (self.N,)),
                                              self._vec(y, (self.N,)), self._s(stream)), self.ctx)
        return y

    def matvec_multi(self, X, Y=None, stream=None):
        """Y[i] = Z(k0) X[i] for several right-hand sides at the bound frequency."""
        torch = _torch()
        n = X.shape[0]
        if Y is None:
            Y = torch.empty((n, self.N), dtype=self.cdtype, device=self._dev())
        _check(self.lib, self.lib.aimx_matvec_multi(self.ctx, n, self._vec(X, (n, self.N)), self._vec(Y, (n, self.N)),
                                                    self._s(stream)), self.ctx)
        return Y

    def matvec_parts(self, x, stream=None):
        torch = _torch()
        yA = torch.empty(self.N, dtype=self.cdtype, device=self._dev())
        yP = torch.empty(self.N, dtype=self.cdtype, device=self._dev())
        _check(self.lib, self.lib.aimx_matvec_parts(self.ctx, self._vec(x, (self.N,)),
                                                    self._vec(yA, (self.N,)),
                                                    self._vec(yP, (self.N,)), self._s(stream)),
               self.ctx)
        return yA, yP

    def sweep(self, freqs, X, Y=None, batch: int = 0, stream=None):
        torch = _torch()
        f = np.ascontiguousarray(freqs, dtype=np.float64)
        nf = f.shape[0]
        if Y is None:
            Y = torch.empty((nf, self.N), dtype=self.cdtype, device=self._dev())
        _check(self.lib, self.lib.aimx_sweep(self.ctx, nf, f.ctypes.data_as(C.POINTER(C.c_double)),
                                             self._vec(X, (nf, self.N)), self._vec(Y, (nf, self.N)),
                                             int(batch), self._s(stream)), self.ctx)
        return Y

    def solve(self, freqs, RHS, X=None, tol: float = 1e-4, restart: int = 30, maxiter: int = 1000,
              stream=None):
        """GMRES solve Z(f_i) X[i] = RHS[i] (aimx_solve); returns (X, iterations, relative residuals)."""
        torch = _torch()
        f = np.ascontiguousarray(freqs, dtype=np.float64)
        nf = f.shape[0]
        if X is None:
            X = torch.empty((nf, self.N), dtype=self.cdtype, device=self._dev())
        its = np.zeros(nf, np.int32)
        rr = np.zeros(nf, np.float64)
        _check(self.lib, self.lib.aimx_solve(self.ctx, nf, f.ctypes.data_as(C.POINTER(C.c_double)),
                                             self._vec(RHS, (nf, self.N)), self._vec(X, (nf, self.N)),
                                             float(tol), int(restart), int(maxiter),
                                             its.ctypes.data_as(C.POINTER(C.c_int32)),
                                             rr.ctypes.data_as(C.POINTER(C.c_double)), self._s(stream)), self.ctx)
        return X, its, rr

    def sweep_status(self, Y, stream=None):
        """Per-frequency status of a sweep / solve result Y [nf, N] (device):
        0 = all finite, 1 = a NaN or infinity (aimx_sweep_status)."""
        nf = int(Y.shape[0])
        st = np.zeros(nf, dtype=np.int32)
        _check(self.lib, self.lib.aimx_sweep_status(self.ctx, nf, self._vec(Y, (nf, self.N)),
                                                    _P(st.ctypes.data), self._s(stream)), self.ctx)
        return st

    def sweep_host(self, freqs, X, Y, batch: int = 0, stream=None):
        """X, Y: host (CPU) torch tensors [nf, N] (pinned for best speed)."""
        torch = _torch()
        f = np.ascontiguousarray(freqs, dtype=np.float64)
        nf = f.shape[0]
        for t in (X, Y):
            if not (isinstance(t, torch.Tensor) and not t.is_cuda and t.dtype == self.cdtype
                    and t.is_contiguous() and tuple(t.shape) == (nf, self.N)):
                raise ValueError("sweep_host expects contiguous host tensors [nf, N]")
        _check(self.lib, self.lib.aimx_sweep_host(self.ctx, nf, f.ctypes.data_as(C.POINTER(C.c_double)),
                                                  _P(X.data_ptr()), _P(Y.data_ptr()), int(batch),
                                                  self._s(stream)), self.ctx)
        return Y

    # ----------------------------------------------------------- introspection
    def stats(self) -> dict:
        s = _Stats()
        _check(self.lib, self.lib.aimx_get_stats(self.ctx, C.byref(s)), self.ctx)
        return {"num_unknowns": s.num_unknowns, "nnz": s.nnz, "occupied_nodes": s.occupied_nodes,
                "occupied_lines": s.occupied_lines, "occupied_planes": s.occupied_planes,
                "projection_entries": s.projection_entries, "device_bytes": s.device_bytes,
                "batch_slots": s.batch_slots, "setup_seconds": s.setup_seconds,
                "n": tuple(s.n), "order": s.order, "h": s.h, "origin": tuple(s.origin),
                "near_group_rows": s.near_group_rows, "near_row_order": s.near_row_order,
                "near_union": s.near_union, "planar": bool(s.planar),
                "kop_grad": bool(s.kop_grad), "grid_channels": s.grid_channels}

    STAGES = ("spectrum", "proj_xfft", "yfwd", "zconv", "yinv", "xinv", "interp_near")

    def profile_enable(self, on: bool = True, stages=None, serial: bool = False):
        """stages: names (AIMx.STAGES) to bracket with events; None = all.
        serial: sweeps run their batches on one stream (each stage's own time)."""
        mask = 0x7F if stages is None else sum(1 << self.STAGES.index(k) for k in stages)
        mask |= 0x80 if serial else 0
        _check(self.lib, self.lib.aimx_profile_stages(self.ctx, int(mask)), self.ctx)
        _check(self.lib, self.lib.aimx_profile_enable(self.ctx, int(bool(on))), self.ctx)

    def profile_read(self) -> dict:
        """{stage: (device ms, bracketed launches)} plus "kernels": total kernel
        launches since profile_enable / the previous read."""
        ms = np.zeros(7)
        n = np.zeros(7, np.int64)
        k = C.c_int64()
        _check(self.lib, self.lib.aimx_profile_read(self.ctx, _P(ms.ctypes.data), _P(n.ctypes.data),
                                                    C.byref(k)), self.ctx)
        out = {s: (float(ms[i]), int(n[i])) for i, s in enumerate(self.STAGES)}
        out["kernels"] = int(k.value)
        return out

    def rwg(self):
        ab = np.empty((self.N, 2), np.int32)
        tpm = np.empty((self.N, 2), np.int32)
        fpm = np.empty((self.N, 2), np.int32)
        _check(self.lib, self.lib.aimx_get_rwg(self.ctx, _P(ab.ctypes.data), _P(tpm.ctypes.data),
                                               _P(fpm.ctypes.data)), self.ctx)
        return ab, tpm, fpm

    def anchors(self):
        a = np.empty((self.N, 3), np.int32)
        _check(self.lib, self.lib.aimx_get_anchors(self.ctx, _P(a.ctypes.data)), self.ctx)
        return a

    def near_csr(self):
        nnz = C.c_int64()
        _check(self.lib, self.lib.aimx_get_near_csr(self.ctx, None, None, C.byref(nnz)), self.ctx)
        rp = np.empty(self.N + 1, np.int64)
        col = np.empty(nnz.value, np.int32)
        _check(self.lib, self.lib.aimx_get_near_csr(self.ctx, _P(rp.ctypes.data), _P(col.ctypes.data),
                                                    C.byref(nnz)), self.ctx)
        return rp, col

    def static(self):
        nnz = C.c_int64()
        _check(self.lib, self.lib.aimx_get_near_csr(self.ctx, None, None, C.byref(nnz)), self.ctx)
        out = [np.empty(nnz.value) for _ in range(6)]
        _check(self.lib, self.lib.aimx_get_static(self.ctx, *[_P(a.ctypes.data) for a in out]), self.ctx)
        return dict(zip(["CA", "CR", "LA_NR", "YR_NR", "LA_P", "YR_P"], out))

    def linear_entries(self):
        """(cols [N][5], C^A_lin [N][5], C^rho_lin [N][5]) of the linear-term modification."""
        cols = np.empty((self.N, 5), np.int32)
        ca = np.empty((self.N, 5))
        cr = np.empty((self.N, 5))
        _check(self.lib, self.lib.aimx_get_linear_entries(self.ctx, _P(cols.ctypes.data), _P(ca.ctypes.data),
                                                          _P(cr.ctypes.data)), self.ctx)
        return cols, ca, cr

    def weights(self):
        st = self.stats()
        p3 = (st["order"] + 1) ** 3
        lam = np.empty((self.N, 4, p3))
        _check(self.lib, self.lib.aimx_get_weights(self.ctx, _P(lam.ctypes.data)), self.ctx)
        return lam

    def spectrum(self, which: int = 0):
        st = self.stats()
        nx, ny, nz = st["n"]
        nz1 = 1 if st["planar"] else nz + 1   # planar: the dz = 0 slice's 2-D spectrum
        out = np.empty((ny + 1) * (nx + 1) * nz1 * 2)
        _check(self.lib, self.lib.aimx_get_spectrum(self.ctx, int(which), _P(out.ctypes.data)), self.ctx)
        return out.view(np.complex128).reshape(ny + 1, nz1, nx + 1)
