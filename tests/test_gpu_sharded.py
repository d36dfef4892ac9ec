"""Multi-GPU LFPS on one B200: 2 or 3 ranks (processes,
gloo for the gather since they share the one device) each step their shard
of the batch with no collective, then gather outputs and C2 lists; the
gathered step is bit-identical to the same batch run by one rank -- for the
request split (B >= P) and the KV-head split (B < P, the C1 case)."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu

STEPS = 4


def _spec(batch, hkv):
    from paper_2506_15704_b200.workload import GqaSpec
    return GqaSpec(batch=batch, kv_heads=hkv, group=4, d=128, n_prefill=3000, steps=STEPS,
                   seed=61, slash_offsets=(64, 65), band_width=6)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _rank(rank, world, port, batch, hkv, path):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2506_15704_b200.config import LfpsConfig
        from paper_2506_15704_b200.sharded import ShardedSession, populate_sharded
        spec = _spec(batch, hkv)
        ss = ShardedSession(LfpsConfig(d=128), batch, hkv, 4, n_max=3100, rank=rank,
                            world=world, device="cuda:0")
        stream = populate_sharded(ss, spec)
        got = []
        for t in range(STEPS):
            ss.decode_step(stream.q[t], stream.k_new[t], stream.v_new[t], 0.05, check=True)
            out, cnt, lists = ss.gather()
            got.append((out.cpu(), cnt.cpu(), lists))
        if rank == 0:
            torch.save(got, path)
        ss.sess.close()
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("batch,hkv,world", [(2, 2, 2), (1, 4, 2), (1, 4, 3)])
def test_sharded_gather_matches_single_rank(batch, hkv, world, tmp_path):
    from paper_2506_15704_b200.config import LfpsConfig
    from paper_2506_15704_b200.session import CNT_C2, BatchedSession
    from paper_2506_15704_b200.workload import populate
    path = str(tmp_path / "gathered.pt")
    mp.spawn(_rank, args=(world, _free_port(), batch, hkv, path), nprocs=world, join=True)
    got = torch.load(path, weights_only=False)
    spec = _spec(batch, hkv)
    sess = BatchedSession(LfpsConfig(d=128), batch, hkv, 4, n_max=3100, device="cuda:0")
    stream = populate(sess, spec)
    for t in range(STEPS):
        sess.decode_step(stream.q[t], stream.k_new[t], stream.v_new[t], 0.05, check=True)
        out, cnt, lists = got[t]
        assert torch.equal(out, sess.out.cpu()), t          # bit-identical outputs
        assert torch.equal(cnt, sess.counts[..., CNT_C2].cpu())
        for b in range(batch):
            for qh in range(hkv * 4):
                np.testing.assert_array_equal(lists[b][qh].numpy(), sess.c2_list(b, qh))
