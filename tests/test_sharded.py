"""Multi-GPU partition and the final gather on the CPU:
plan_shards covers every (request, KV-head) unit exactly once, and the
gather over a world-2 gloo group reassembles outputs and ragged C2 lists in
global (request, q-head) order."""

import os
import socket
from types import SimpleNamespace

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2506_15704_b200.session import CNT_C2
from paper_2506_15704_b200.sharded import ShardedSession, plan_shards


@pytest.mark.parametrize("batch,hkv,world", [(64, 8, 1), (64, 8, 2), (64, 8, 8), (4, 8, 8),
                                             (1, 8, 2), (1, 8, 8), (1, 8, 3), (2, 8, 5),
                                             (3, 2, 4)])
def test_plan_covers_units_once(batch, hkv, world):
    plan = plan_shards(batch, hkv, world)
    assert [s.rank for s in plan] == list(range(world))
    seen = [(b, h) for s in plan for b in range(s.b0, s.b0 + s.nb) for h in range(s.h0, s.h0 + s.nh)]
    assert sorted(seen) == [(b, h) for b in range(batch) for h in range(hkv)]
    assert all(s.units >= 1 for s in plan)
    if batch >= world:
        assert all(s.nh == hkv for s in plan)           # request split: every KV head local
    else:
        assert all(s.nb == 1 for s in plan)             # KV-head split
    sizes = [s.units for s in plan]
    assert max(sizes) - min(sizes) <= max(1, hkv // 2 + 1)


def test_plan_rejects_more_ranks_than_units():
    with pytest.raises(ValueError):
        plan_shards(1, 2, 3)


def _fake(batch, hkv, G, d, world, rank, cap=16):
    """A ShardedSession whose local session is a stub with deterministic
    outputs / counts / C2 lists (value encodes the global session)."""
    ss = object.__new__(ShardedSession)
    ss.B, ss.Hkv, ss.G, ss.d, ss.Hq = batch, hkv, G, d, hkv * G
    ss.rank, ss.world, ss.pg = rank, world, None
    ss.plan = plan_shards(batch, hkv, world)
    ss.shard = sh = ss.plan[rank]
    ss.device = torch.device("cpu")
    out = torch.empty(sh.nb, sh.nh * G, d)
    counts = torch.zeros(sh.nb, sh.nh * G, 8, dtype=torch.int32)
    c2 = torch.full((sh.nb, sh.nh * G, cap), -1, dtype=torch.int32)
    for bl in range(sh.nb):
        for ql in range(sh.nh * G):
            b, qh = sh.b0 + bl, sh.h0 * G + ql
            s = b * ss.Hq + qh
            out[bl, ql] = s + torch.arange(d) / 1000.0
            k = (s * 7) % cap
            counts[bl, ql, CNT_C2] = k
            c2[bl, ql, :k] = torch.arange(k) * 3 + s
    ss.sess = SimpleNamespace(out=out, counts=counts, c2_idx=c2)
    return ss


def _check(ss, out, cnt, lists, cap=16):
    for b in range(ss.B):
        for qh in range(ss.Hq):
            s = b * ss.Hq + qh
            assert torch.equal(out[b, qh], s + torch.arange(ss.d) / 1000.0)
            k = (s * 7) % cap
            assert int(cnt[b, qh]) == k
            assert lists[b][qh].tolist() == [i * 3 + s for i in range(k)]


def test_gather_single_rank():
    ss = _fake(3, 2, 4, 8, 1, 0)
    _check(ss, *ss.gather())


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, shape, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        ss = _fake(*shape, world, rank)
        res = ss.gather()
        _check(ss, *res)
        out[rank] = True
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("shape,world", [((4, 2, 4, 8), 2), ((1, 8, 4, 8), 2), ((1, 8, 2, 8), 3)])
def test_gloo_gather_reassembles_batch(shape, world):
    port = _free_port()
    out = mp.Manager().dict()
    mp.spawn(_worker, args=(world, port, shape, out), nprocs=world, join=True)
    assert all(out[r] for r in range(world))
