"""The N>1 replica path on CPU: world_size-2 gloo processes (no GPU needed)."""

import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2505_08491_b200.replicas import aggregate_throughput, shard


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        systems = list(range(16))
        mine = shard(systems, rank, world)
        # rank r pretends its replica took (r + 1) * 100 ms for len(mine) solves
        value, ms, total = aggregate_throughput((rank + 1) * 100.0, len(mine))
        out[rank] = (mine, value, ms, total)
    finally:
        dist.destroy_process_group()


def test_shard_balanced_and_complete():
    items = list(range(17))
    parts = [shard(items, r, 4) for r in range(4)]
    assert sum(parts, []) == items
    assert max(map(len, parts)) - min(map(len, parts)) <= 1
    with pytest.raises(ValueError):
        shard(items, 4, 4)


def test_two_rank_gloo_aggregation():
    world = 2
    port = _free_port()
    with mp.Manager() as mgr:
        out = mgr.dict()
        mp.spawn(_worker, args=(world, port, out), nprocs=world, join=True)
        res = dict(out)
    assert res[0][0] == list(range(8)) and res[1][0] == list(range(8, 16))
    for r in range(world):
        value, ms, total = res[r][1:]
        assert ms == 200.0            # slowest rank's device time
        assert total == 16            # all ranks' solves
        assert value == pytest.approx(16 / 0.2)


def test_single_process_fallback():
    value, ms, total = aggregate_throughput(50.0, 3)
    assert (ms, total) == (50.0, 3) and value == pytest.approx(60.0)
