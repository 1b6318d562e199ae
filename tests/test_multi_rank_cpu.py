"""N > 1 host-side logic on CPU with the gloo backend (world size 2): the
frequency sharding of bench.py (the config's own list in
contiguous blocks of ceil(nf / N) per rank, RHS seeded by global index), the
max-over-ranks timing reduction, and bench.py's self-spawn of N ranks
(`--gpus 2` without torchrun, `--dry-run`: no GPU)."""
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
    freqs, idx = bench.rank_freqs(c, rank, world)       # strong scaling (default)
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
    got = np.concatenate([np.array(r[1]) for r in res])
    assert np.array_equal(got, c.freqs)                    # disjoint, contiguous, complete
    assert [len(r[1]) for r in res] == [50, 50]            # ceil(100 / 2) per rank
    assert res[1][2][0] == 50                              # global index drives the RHS seed
    assert np.allclose(res[1][4], inp.rhs_vector(2, 50, 64))
    assert all(r[3] == 20.0 for r in res)                  # max over ranks


def test_rank_blocks_cover_the_list():
    import aimx_inputs as inp
    import bench
    for cfg, world in ((2, 8), (5, 8), (3, 4), (5, 3)):
        c = inp.get_config(cfg)
        blocks = [bench.rank_freqs(c, r, world)[1] for r in range(world)]
        assert np.array_equal(np.concatenate(blocks), np.arange(len(c.freqs)))
        assert max(len(b) for b in blocks) == -(-len(c.freqs) // world)
    c = inp.get_config(5)
    f, i = bench.rank_freqs(c, 1, 4, "weak")
    assert np.array_equal(i, np.arange(64))                # weak: the full list on every rank


def test_bench_self_spawns_ranks_dry_run():
    import json
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = {k: v for k, v in os.environ.items() if k not in ("RANK", "WORLD_SIZE", "LOCAL_RANK")}
    p = subprocess.run([sys.executable, os.path.join(root, "bench.py"), "--gpus", "2", "--dry-run", "--config", "5"],
                       capture_output=True, text=True, timeout=300, env=env, cwd=root)
    assert p.returncode == 0, p.stderr[-2000:]
    lines = [json.loads(x) for x in p.stdout.splitlines() if x.startswith("{")]
    assert len(lines) == 1                                 # rank 0 prints one line
    d = lines[0]
    assert d["n_gpus"] == 2 and d["freq_pts_per_rank"] == [32, 32] and d["max_over_ranks"] == 2.0
