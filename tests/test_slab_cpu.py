"""Slab decomposition on the CPU (no GPU): the library's host-only plan
(aimx_slab_plan) partitions rows and kx slabs exactly, with the halo the
stencils need; a 2-rank gloo run of the decomposed FFT convolution -- x
transform on each rank's rows, all-to-all to kx slabs, y/z transforms and the
spectrum product, all-to-all back with the halo rows, x inverse -- equals the
undecomposed convolution (the exchange geometry of slab mode)."""
import os
import socket

import numpy as np
import pytest


def _plans(n, order, world):
    from paper_2009_02281_b200 import slab_plan
    return [slab_plan(n, order, world, r) for r in range(world)]


@pytest.mark.parametrize("n,world", [((16, 16, 4), 2), ((16, 16, 4), 4), ((512, 512, 8), 8),
                                     ((16, 8, 32), 8), ((256, 16, 4), 2)])
def test_plan_partitions(n, world):
    pl = _plans(n, 2, world)
    rows = [p["rows"] for p in pl]
    assert rows[0][0] == 0 and rows[-1][1] == n[1]
    for a, b in zip(rows, rows[1:]):
        assert a[1] == b[0] and a[1] > a[0]
    for p in pl:
        assert p["phi_rows"][0] == p["rows"][0]
        assert p["phi_rows"][1] == min(p["rows"][1] + 2, n[1])   # stencil rows of anchors in the block
    kx = [p["kx"] for p in pl]
    assert kx[0][0] == 0 and kx[-1][1] == 2 * n[0]
    w = kx[0][1] - kx[0][0]
    assert all(b - a == w for a, b in kx) and (w & (w - 1)) == 0


def test_plan_rejects():
    from paper_2009_02281_b200 import AIMxError, slab_plan
    with pytest.raises(AIMxError):
        slab_plan((16, 16, 4), 2, 3, 0)       # 32 kx not divisible into 3 slabs
    with pytest.raises(AIMxError):
        slab_plan((12, 16, 4), 2, 2, 0)       # slab of 12 kx: not a power of two
    with pytest.raises(AIMxError):
        slab_plan((16, 2, 4), 2, 4, 0)        # fewer rows than ranks


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _exchange(recv, send, rank):
    """Grouped point-to-point exchange (the library's ncclSend / ncclRecv
    pattern; gloo has no all-to-all)."""
    import torch
    import torch.distributed as dist
    reqs = []
    for q, (r, t) in enumerate(zip(recv, send)):
        if q == rank:
            r.copy_(t)
            continue
        reqs.append(dist.isend(torch.view_as_real(t).contiguous(), q))
        reqs.append(dist.irecv(torch.view_as_real(r), q))
    for w in reqs:
        w.wait()


def _worker(rank, world, port, n, plans, K, g, out):
    import torch
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    Nx, Ny, Nz = n
    p = plans[rank]
    y0, y1 = p["rows"]
    yh1 = p["phi_rows"][1]
    k0, k1 = p["kx"]
    # rows: zero-padded x transform of the rank's rows
    A = np.fft.fft(g[:, y0:y1, :], n=2 * Nx, axis=2)                 # [z][y][kx]
    send = [torch.from_numpy(np.ascontiguousarray(A[:, :, q["kx"][0]:q["kx"][1]])) for q in plans]
    recv = [torch.zeros((Nz, q["rows"][1] - q["rows"][0], k1 - k0), dtype=torch.complex128) for q in plans]
    _exchange(recv, send, rank)
    col = np.zeros((Nz, Ny, k1 - k0), complex)
    for q, t in zip(plans, recv):
        col[:, q["rows"][0]:q["rows"][1], :] = t.numpy()
    F = np.fft.fft(np.fft.fft(col, n=2 * Ny, axis=1), n=2 * Nz, axis=0)   # [kz][ky][kx slab]
    F *= K[:, :, k0:k1]
    G = np.fft.ifft(np.fft.ifft(F, axis=0)[:Nz], axis=1)[:, :Ny, :]
    send = [torch.from_numpy(np.ascontiguousarray(G[:, q["phi_rows"][0]:q["phi_rows"][1], :])) for q in plans]
    recv = [torch.zeros((Nz, yh1 - y0, q["kx"][1] - q["kx"][0]), dtype=torch.complex128) for q in plans]
    _exchange(recv, send, rank)
    rowsbuf = np.zeros((Nz, yh1 - y0, 2 * Nx), complex)
    for q, t in zip(plans, recv):
        rowsbuf[:, :, q["kx"][0]:q["kx"][1]] = t.numpy()
    phi = np.fft.ifft(rowsbuf, axis=2)[:, :, :Nx]
    np.save(out % rank, phi)
    dist.barrier()
    dist.destroy_process_group()


def test_gloo_two_rank_slab_convolution(tmp_path):
    import torch.multiprocessing as mp
    n = (8, 6, 4)
    world = 2
    plans = _plans(n, 2, world)
    rng = np.random.default_rng(5)
    Nx, Ny, Nz = n
    g = rng.standard_normal((Nz, Ny, Nx)) + 1j * rng.standard_normal((Nz, Ny, Nx))
    K = np.fft.fftn(rng.standard_normal((2 * Nz, 2 * Ny, 2 * Nx)))
    out = str(tmp_path / "phi_%d.npy")
    mp.spawn(_worker, args=(world, _free_port(), n, plans, K, g, out), nprocs=world, join=True)
    ref = np.fft.ifftn(K * np.fft.fftn(g, s=(2 * Nz, 2 * Ny, 2 * Nx)))[:Nz, :Ny, :Nx]
    for r, p in enumerate(plans):
        phi = np.load(out % r)
        y0, yh1 = p["phi_rows"]
        assert np.abs(phi - ref[:, y0:yh1, :]).max() <= 1e-12 * np.abs(ref).max()
