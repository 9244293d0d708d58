"""Multi-rank host logic on CPU (gloo, world size 2): shard ranges and the
ordered all-gather of per-rank results (paper_2505_03728_b200/shard.py)."""

import os
import socket

import numpy as np
import pytest

from paper_2505_03728_b200.shard import gather_rows, shard_range


def test_shard_range_partitions():
    for total in (0, 1, 7, 1000, 1001):
        for world in (1, 2, 3, 8):
            spans = [shard_range(total, world, r) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == total
            assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))
            sizes = [e - s for s, e in spans]
            assert max(sizes) - min(sizes) <= 1
    with pytest.raises(ValueError):
        shard_range(10, 2, 2)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, total, q):
    import torch
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    s, e = shard_range(total, world, rank)
    # stand-in per-target result: a deterministic function of the GLOBAL index
    idx = torch.arange(s, e, dtype=torch.float64)
    local = torch.stack([idx, idx * 0.5, idx ** 2], dim=1)
    full = gather_rows(local, total)
    dist.barrier()
    q.put((rank, full.numpy()))
    dist.destroy_process_group()


@pytest.mark.parametrize("total", [11, 64])
def test_gloo_two_rank_gather_matches_single_rank(total):
    import multiprocessing as mp

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, total, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    idx = np.arange(total, dtype=float)
    expect = np.stack([idx, idx * 0.5, idx ** 2], axis=1)
    for r in (0, 1):
        assert np.array_equal(res[r], expect)
