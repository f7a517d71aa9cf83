"""Multi-process sharding (world_size 2, gloo, CPU): every problem is owned
by exactly one rank, shards are work-balanced, and the gathered results come
back in problem order."""

import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2309_15417_b200 import shard


def test_shard_bounds_partition_and_balance():
    rng = np.random.default_rng(0)
    for n in (0, 1, 2, 7, 100, 1000):
        w = rng.uniform(0.1, 10.0, n)
        for world in (1, 2, 3, 8):
            cuts = [shard.shard_bounds(w, r, world) for r in range(world)]
            assert cuts[0][0] == 0 and cuts[-1][1] == n
            for (a, b), (c, d) in zip(cuts, cuts[1:]):
                assert b == c and a <= b
            if n >= 100:
                loads = [w[a:b].sum() for a, b in cuts]
                assert max(loads) <= w.sum() / world + w.max() + 1e-9


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, n, out_dir):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        w = np.arange(1, n + 1, dtype=float)
        lo, hi = shard.shard_bounds(w, rank, world)
        local = [("result", i, rank) for i in range(lo, hi)]  # stands in for BatchResult.result(i)
        full = shard.gather_results(local, lo, n)
        assert [r[1] for r in full] == list(range(n))
        owners = sorted({r[2] for r in full})
        np.save(os.path.join(out_dir, f"rank{rank}.npy"), np.array([lo, hi, len(owners)]))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("n", [1, 9, 64])
def test_two_rank_gather_with_gloo(tmp_path, n):
    port = _free_port()
    mp.start_processes(_worker, args=(2, port, n, str(tmp_path)), nprocs=2, join=True,
                       start_method="spawn")
    r0 = np.load(tmp_path / "rank0.npy")
    r1 = np.load(tmp_path / "rank1.npy")
    assert r0[0] == 0 and r0[1] == r1[0] and r1[1] == n
