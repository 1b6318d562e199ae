"""N > 1 host-side logic on CPU with the gloo backend (world size 2): the
frequency sharding of the weak-scaling sweep (disjoint contiguous blocks of a
100*N-point band, RHS seeded by global index) and the max-over-ranks timing
reduction used by bench.py."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import aimx_inputs as inp
    import bench
    c = inp.get_config(2)
    freqs, idx = bench.rank_freqs(c, rank, world)
    local_ms = 10.0 * (rank + 1)
    tmax = bench.max_over_ranks(local_ms, device="cpu")
    x0 = inp.rhs_vector(2, int(idx[0]), 64)
    q.put((rank, freqs.tolist(), idx.tolist(), tmax, x0.tolist()))
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_sharding_and_max_reduction():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted([q.get(timeout=120) for _ in range(world)])
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    import aimx_inputs as inp
    c = inp.get_config(2)
    band = np.linspace(c.freqs[0], c.freqs[-1], 100 * world)
    got = np.concatenate([np.array(r[1]) for r in res])
    assert np.array_equal(got, band)                       # disjoint, contiguous, complete
    assert [len(r[1]) for r in res] == [100, 100]          # weak scaling: fixed work per rank
    assert res[1][2][0] == 100                             # global index drives the RHS seed
    assert np.allclose(res[1][4], inp.rhs_vector(2, 100, 64))
    assert all(r[3] == 20.0 for r in res)                  # max over ranks
