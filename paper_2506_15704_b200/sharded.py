"""Multi-GPU LFPS: (request, KV-head) units partitioned over ranks.

SURVEY.md §8(e): the (request, KV-head) units of a decode step are fully
independent -- no unit reads another's K/V rows, tables or priors
 -- so the step shards with NO collective on the
decode path.  One process per GPU (torch.distributed, NCCL):

* ``plan_shards``: when the batch covers the ranks (B >= P), each rank takes
  a contiguous range of requests with all their KV heads (robust to ragged
  contexts, SURVEY §8(e) "C4: requests"); when B < P (C1: one request on up
  to 8 GPUs), each request's KV heads are split over the ranks assigned to
  it ("When B<P: KV heads").
* ``ShardedSession``: the rank's ``BatchedSession`` over its units, fed the
  rank's slice of each step's inputs.
* ``gather``: the north star's one collective, AFTER the decode step: the
  outputs [B, Hq, d] (fixed size per shard) and the ragged C2 index lists --
  counts first, then the payload, padded to the largest shard -- all-gathered
  and reassembled in global (request, q-head) order.

The reference has no multi-process path (its only
parallelism is a thread pool over heads, bench.py:145-164); what must carry
over is that results do not depend on the partition (test_report_cli.py:
61-67) -- the gathered step is identical to the single-GPU step.
"""

from __future__ import annotations

from dataclasses import dataclass

import torch

from .config import LfpsConfig
from .session import CNT_C2, BatchedSession


@dataclass(frozen=True)
class Shard:
    """The units one rank owns: requests [b0, b0 + nb) x KV heads [h0, h0 + nh)."""

    rank: int
    b0: int
    nb: int
    h0: int
    nh: int

    @property
    def units(self) -> int:
        return self.nb * self.nh


def _split(n: int, parts: int, i: int) -> tuple[int, int]:
    """Contiguous split of range(n) into `parts` near-equal pieces: (start, count) of piece i."""
    base, extra = divmod(n, parts)
    return i * base + min(i, extra), base + (1 if i < extra else 0)


def plan_shards(batch: int, kv_heads: int, world: int) -> list[Shard]:
    """Partition the batch's (request, KV-head) units over `world` ranks.

    B >= P: requests split contiguously, every KV head local.  B < P: the
    ranks are split over the requests (contiguously), and each request's KV
    heads over its ranks; needs P <= B * Hkv (every rank gets a unit)."""
    if batch < 1 or kv_heads < 1 or world < 1:
        raise ValueError("batch, kv_heads and world must be >= 1")
    if world > batch * kv_heads:
        raise ValueError(f"{world} ranks exceed the {batch * kv_heads} (request, KV-head) units")
    shards = []
    if batch >= world:
        for r in range(world):
            b0, nb = _split(batch, world, r)
            shards.append(Shard(r, b0, nb, 0, kv_heads))
        return shards
    for b in range(batch):
        r0, nr = _split(world, batch, b)       # ranks of request b
        for j in range(nr):
            h0, nh = _split(kv_heads, nr, j)
            shards.append(Shard(r0 + j, b, 1, h0, nh))
    return shards


class ShardedSession:
    """This rank's part of a batched LFPS layer (see module docstring).

    ``decode_step`` takes the FULL step inputs (q [B, Hq, d], k_new / v_new
    [B, Hkv, d], on this rank's device) and steps this rank's units on their
    slice; ``decode_step_local`` takes the slice directly.  No collective runs
    inside either.  ``gather`` assembles the whole batch's outputs and C2 sets
    on every rank."""

    def __init__(self, cfg: LfpsConfig, batch: int, kv_heads: int, group: int, n_max: int,
                 rank: int, world: int, device=None, group_pg=None, **session_kw):
        self.cfg, self.B, self.Hkv, self.G, self.d = cfg, batch, kv_heads, group, cfg.d
        self.Hq = kv_heads * group
        self.rank, self.world = rank, world
        self.pg = group_pg
        self.plan = plan_shards(batch, kv_heads, world)
        self.shard = self.plan[rank]
        sh = self.shard
        self.sess = BatchedSession(cfg, sh.nb, sh.nh, group, n_max, device=device, **session_kw)
        self.device = self.sess.device

    # -- slicing ---------------------------------------------------------------
    def local_q(self, q: torch.Tensor) -> torch.Tensor:
        sh, G = self.shard, self.G
        return q[sh.b0:sh.b0 + sh.nb, sh.h0 * G:(sh.h0 + sh.nh) * G].contiguous()

    def local_kv(self, x: torch.Tensor) -> torch.Tensor:
        sh = self.shard
        return x[sh.b0:sh.b0 + sh.nb, sh.h0:sh.h0 + sh.nh].contiguous()

    def owns(self, b: int, h: int) -> bool:
        sh = self.shard
        return sh.b0 <= b < sh.b0 + sh.nb and sh.h0 <= h < sh.h0 + sh.nh

    # -- decode ----------------------------------------------------------------
    def decode_step(self, q, k_new, v_new, k_fraction: float, **kw):
        return self.sess.decode_step(self.local_q(q), self.local_kv(k_new), self.local_kv(v_new),
                                     k_fraction, **kw)

    def decode_step_local(self, q_local, k_local, v_local, k_fraction: float, **kw):
        return self.sess.decode_step(q_local, k_local, v_local, k_fraction, **kw)

    # -- the final gather ----------------------------------------------------------
    def _comm_device(self):
        import torch.distributed as dist
        if not dist.is_initialized() or self.world == 1:
            return self.device
        return self.device if dist.get_backend(self.pg) == "nccl" else torch.device("cpu")

    def _all_gather(self, t: torch.Tensor) -> torch.Tensor:
        """[world, *t.shape] (t has the same shape on every rank)."""
        import torch.distributed as dist
        if self.world == 1:
            return t[None]
        flat = t.contiguous().reshape(-1)
        out = torch.empty(self.world * flat.numel(), dtype=t.dtype, device=t.device)
        dist.all_gather_into_tensor(out, flat, group=self.pg)
        return out.reshape((self.world,) + tuple(t.shape))

    def gather(self, with_c2: bool = True):
        """All-gather this step's outputs and (optionally) C2 sets.

        Returns (out [B, Hq, d] f32, c2 counts [B, Hq] i32, c2 lists) on every
        rank, where c2 lists is a [B, Hq] nested list of int32 CPU tensors (or
        None without ``with_c2``).  Outputs travel as one fixed-size buffer per
        rank (padded to the largest shard); C2 goes counts first, then one
        payload buffer padded to the largest rank total."""
        dev = self._comm_device()
        G, d = self.G, self.d
        max_units = max(s.units for s in self.plan)
        sess, sh = self.sess, self.shard
        ns = sh.units * G
        out_buf = torch.zeros(max_units * G, d, dtype=torch.float32, device=dev)
        out_buf[:ns] = sess.out.reshape(ns, d).to(dev)
        cnt_buf = torch.zeros(max_units * G, dtype=torch.int32, device=dev)
        cnt_buf[:ns] = sess.counts.reshape(ns, -1)[:, CNT_C2].to(dev)
        g_out = self._all_gather(out_buf)
        g_cnt = self._all_gather(cnt_buf)
        out = torch.empty(self.B, self.Hq, d, dtype=torch.float32, device=dev)
        cnt = torch.empty(self.B, self.Hq, dtype=torch.int32, device=dev)
        for s in self.plan:
            n = s.units * G
            out[s.b0:s.b0 + s.nb, s.h0 * G:(s.h0 + s.nh) * G] = \
                g_out[s.rank, :n].reshape(s.nb, s.nh * G, d)
            cnt[s.b0:s.b0 + s.nb, s.h0 * G:(s.h0 + s.nh) * G] = \
                g_cnt[s.rank, :n].reshape(s.nb, s.nh * G)
        if not with_c2:
            return out, cnt, None
        # payload: this rank's lists back to back in session order
        totals = g_cnt.to(torch.int64).sum(dim=1)
        cap = int(totals.max())
        mine = sess.counts.reshape(ns, -1)[:, CNT_C2].to(torch.int64)
        pay = torch.zeros(max(cap, 1), dtype=torch.int32, device=dev)
        if int(mine.sum()):
            idx = sess.c2_idx.reshape(ns, -1)
            pos = torch.arange(idx.shape[1], device=idx.device)
            keep = pos[None, :] < mine.to(idx.device)[:, None]
            pay[:int(mine.sum())] = idx[keep].to(dev)
        g_pay = self._all_gather(pay).cpu()
        g_cnt_h = g_cnt.cpu().to(torch.int64)
        lists = [[None] * self.Hq for _ in range(self.B)]
        for s in self.plan:
            off = 0
            for i in range(s.units * G):
                k = int(g_cnt_h[s.rank, i])
                b = s.b0 + i // (s.nh * G)
                qh = s.h0 * G + i % (s.nh * G)
                lists[b][qh] = g_pay[s.rank, off:off + k].clone()
                off += k
        return out, cnt, lists


def populate_sharded(ss: ShardedSession, spec, device=None):
    """Fill this rank's units with the spec's synthetic prefill (the units of
    workload.populate, generated per unit from the same seeds, so the union
    over ranks is exactly the single-GPU batch) and return the FULL step
    inputs (q [T, B, Hq, d], k_new / v_new [T, B, Hkv, d]) -- each rank
    slices its part per step.  Harness input, not part of the decode path."""
    from .workload import StepStream, gen_unit
    dev = device or ss.device
    B, Hkv, G, d = spec.batch, spec.kv_heads, spec.group, spec.d
    n0, T = spec.n_prefill, spec.steps
    sh, sess = ss.shard, ss.sess
    q = torch.zeros(T, B, Hkv * G, d, dtype=torch.bfloat16, device=dev)
    kn = torch.zeros(T, B, Hkv, d, dtype=torch.bfloat16, device=dev)
    vn = torch.zeros(T, B, Hkv, d, dtype=torch.bfloat16, device=dev)
    finals = torch.zeros(sh.nb, sh.nh * G, d, dtype=torch.bfloat16, device=dev)
    for b in range(sh.b0, sh.b0 + sh.nb):
        for h in range(sh.h0, sh.h0 + sh.nh):
            u = gen_unit(spec, b, h, device=dev)
            bl, hl = b - sh.b0, h - sh.h0
            sess.load_unit(bl, hl, u.keys[:n0], u.values[:n0])
            sess.bootstrap_tables((bl * sh.nh + hl) * G, u.weights)
            q[:, b, h * G:(h + 1) * G] = u.queries.transpose(0, 1)
            kn[:, b, h] = u.keys[n0:n0 + T]
            vn[:, b, h] = u.values[n0:n0 + T]
            finals[bl, hl * G:(hl + 1) * G] = u.final_query
    sess.bootstrap_stats(finals)
    torch.cuda.synchronize(dev)
    sess.check_errors("bootstrap")
    return StepStream(q=q, k_new=kn, v_new=vn)
