"""Multi-process host logic with the gloo backend on CPU (world size 2):
request sharding covers the batch exactly once and the step time reported is
the max over ranks (bench.py's contract)."""

import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import bench


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        count, first = bench.shard_requests(64, world, rank)
        local_ms = 1.0 + rank           # rank 1 is the slow one
        out[rank] = (count, first, bench.allmax(world, local_ms), bench.allsum(world, count))
    finally:
        dist.destroy_process_group()


def test_sharding_partitions_batch():
    for world in (1, 2, 3, 4, 8):
        seen = []
        for r in range(world):
            n, first = bench.shard_requests(64, world, r)
            seen.extend(range(first, first + n))
        assert seen == list(range(64))
    with pytest.raises(SystemExit):
        bench.shard_requests(2, 4, 3)


def test_gloo_world2_max_over_ranks():
    port = _free_port()
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(2, port, out), nprocs=2, join=True)
    assert out[0][:2] == (32, 0) and out[1][:2] == (32, 32)
    assert out[0][2] == out[1][2] == 2.0          # max over ranks
    assert out[0][3] == out[1][3] == 64.0         # every request timed once
