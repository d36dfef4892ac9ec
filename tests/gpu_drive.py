"""Drive the device path and the devmath oracle side by side (GPU tests)."""

from __future__ import annotations

import numpy as np
import torch

from oracle import lfps_oracle as lo
from paper_2506_15704_b200.session import (CNT_C0, CNT_C1, CNT_C2, CNT_CLAMP, CNT_DROP,
                                           CNT_K, CNT_PROBE, BatchedSession)


def bf16(x) -> torch.Tensor:
    return torch.as_tensor(np.ascontiguousarray(x, dtype=np.float32)).to(torch.bfloat16)


class Pair:
    """One unit-batch on the GPU plus its oracle mirror.

    keys/values: f32 (bf16 values) [B, Hkv, n_total, d]; weights f32
    [B, Hkv, G, s, n0 - S]; finals [B, Hkv, G, d]."""

    def __init__(self, cfg, keys, values, weights, finals, n0, n_max=None, m_cap=None,
                 paged=False, block_rows=None):
        B, Hkv, _, d = keys.shape
        G = weights.shape[2]
        self.cfg, self.B, self.Hkv, self.G, self.d, self.n0 = cfg, B, Hkv, G, d, n0
        self.host_io = False
        self.weights, self.finals = weights, finals
        n_max = n_max or keys.shape[2] + 8
        kv_blocks = None
        if block_rows:
            # a vLLM-style block-table cache: blocks of `block_rows` rows of all
            # KV heads, handed out in a random order
            max_blocks = -(-n_max // block_rows)
            nblk = B * max_blocks + 3
            perm = torch.randperm(nblk, generator=torch.Generator().manual_seed(7))[:B * max_blocks]
            table = perm.reshape(B, max_blocks).to(torch.int32).cuda()
            kp = torch.zeros(nblk, block_rows, Hkv, d, dtype=torch.bfloat16, device="cuda")
            kv_blocks = (kp, torch.zeros_like(kp), table, block_rows)
            m_cap = m_cap or n_max - cfg.sink_count + 2
        self.sess = BatchedSession(cfg, B, Hkv, G, n_max=n_max, m_cap=m_cap, device="cuda",
                                   export_sets=True, paged=paged, kv_blocks=kv_blocks)
        for b in range(B):
            self.sess.load_prefill(b, bf16(keys[b, :, :n0]).cuda(), bf16(values[b, :, :n0]).cuda())
        w = torch.as_tensor(np.ascontiguousarray(weights, dtype=np.float32))
        self.sess.bootstrap_tables(0, w.reshape(B * Hkv * G, cfg.s, n0 - cfg.sink_count).cuda())
        self.sess.bootstrap_stats(bf16(finals.reshape(B, Hkv * G, d)).cuda())
        torch.cuda.synchronize()
        self.sess.check_errors("bootstrap")
        self.units = []
        for b in range(B):
            for h in range(Hkv):
                kv, trs, prs = lo.bootstrap_unit(keys[b, h, :n0], values[b, h, :n0],
                                                 weights[b, h], finals[b, h], cfg, lo.DevArith)
                self.units.append((kv, trs, prs))

    def step(self, q, k_new, v_new, frac, cfg=None):
        """q [B, Hkv, G, d]; k_new/v_new [B, Hkv, d] (f32 bf16-valued).
        ``cfg`` overrides the configuration for this step only (the
        reference's decode_step takes a config per call, engine.py:97)."""
        B, Hkv, G, d = self.B, self.Hkv, self.G, self.d
        cfg = cfg or self.cfg
        saved, self.sess.cfg = self.sess.cfg, cfg
        try:
            res = self._device_step(q, k_new, v_new, frac)
        finally:
            self.sess.cfg = saved
        outs = []
        for b in range(B):
            for h in range(Hkv):
                kv, trs, prs = self.units[b * Hkv + h]
                outs.append(lo.unit_step(kv, trs, prs, q[b, h], k_new[b, h], v_new[b, h], frac,
                                         cfg, lo.DevArith, "fp32"))
        return res, outs

    def _device_step(self, q, k_new, v_new, frac):
        B, Hkv, G, d = self.B, self.Hkv, self.G, self.d
        pre = getattr(self, "prefetch", False)
        if pre:                   # lfps_decode_prefetch, then the step with LFPS_FLAG_PREFETCHED
            self.sess.prefetch()
        if self.host_io:          # lfps_decode_step_host_io: packed pinned inputs, host output
            packed = self.sess.pack_step_inputs(bf16(q.reshape(B, Hkv * G, d)), bf16(k_new),
                                                bf16(v_new))
            host = torch.full(tuple(self.sess.out.shape), float("nan")).pin_memory()
            if getattr(self, "reuse_host", False):
                # one input and one output buffer for the whole run (a decode
                # loop's pattern): new contents, same tensors every step
                if not hasattr(self, "_host_bufs"):
                    self._host_bufs = (torch.empty_like(packed).pin_memory(),
                                       torch.empty_like(host).pin_memory())
                self._host_bufs[0].copy_(packed)
                self._host_bufs[1].fill_(float("nan"))
                packed, host = self._host_bufs
            res = self.sess.decode_step_host(packed, frac, out_host=host, check=True,
                                             prefetched=pre)
            assert torch.equal(host, self.sess.out.cpu())
        else:
            res = self.sess.decode_step(bf16(q.reshape(B, Hkv * G, d)).cuda(),
                                        bf16(k_new).cuda(), bf16(v_new).cuda(), frac, check=True,
                                        prefetched=pre)
        return res

    def compare_step(self, res, outs, out_tol=1e-5, tables=True, bitmaps=True):
        """Assert bit-exact sets/scalars/tables and toleranced outputs."""
        counts = res.counts.cpu().numpy()
        rho = res.rho.cpu().numpy()
        byp = res.bypassed.cpu().numpy()
        out = res.output.cpu().numpy()
        G = self.G
        worst = 0.0
        for u, unit_outs in enumerate(outs):
            b, h = divmod(u, self.Hkv)
            for g, o in enumerate(unit_outs):
                qh = h * G + g
                s = b * self.Hkv * G + qh
                tag = f"b{b} qh{qh}"
                assert bool(byp[b, qh]) == o.bypassed, tag
                assert rho[b, qh] == o.rho, (tag, rho[b, qh], o.rho)
                if not o.bypassed:
                    c = counts[b, qh]
                    assert c[CNT_C0] == o.c0.size, (tag, "c0", c[CNT_C0], o.c0.size)
                    assert c[CNT_C1] == o.c1.size, (tag, "c1")
                    assert c[CNT_PROBE] == o.probe.size, (tag, "probe", c[CNT_PROBE], o.probe.size)
                    assert c[CNT_DROP] == o.c0_dropped, (tag, "drop")
                    assert c[CNT_K] == o.budget_k, (tag, "k")
                    assert c[CNT_C2] == o.c2.size, (tag, "c2")
                    assert c[CNT_CLAMP] == o.clamps, (tag, "clamps")
                    np.testing.assert_array_equal(self.sess.probe_list(b, qh), o.probe, err_msg=tag)
                    if bitmaps:
                        np.testing.assert_array_equal(self.sess.c0_list(b, qh), o.c0,
                                                      err_msg=tag + " c0")
                        np.testing.assert_array_equal(self.sess.c1_list(b, qh), o.c1,
                                                      err_msg=tag + " c1")
                    np.testing.assert_array_equal(self.sess.c2_list(b, qh), o.c2, err_msg=tag)
                ref = o.output
                err = np.linalg.norm(out[b, qh] - ref) / max(np.linalg.norm(ref), 1e-12)
                worst = max(worst, err)
                assert err <= out_tol, (tag, err)
                if tables:
                    kv, trs, prs = self.units[u]
                    tr = trs[g]
                    ver, sla, sc = self.sess.session_tables(s)
                    assert sc == tr.scale, (tag, sc, tr.scale)
                    np.testing.assert_array_equal(ver, tr.ver_view(), err_msg=tag + " ver")
                    np.testing.assert_array_equal(sla, tr.sla_view(), err_msg=tag + " sla")
        return worst


def gqa_pair(batch=2, kv_heads=2, group=4, n0=3000, steps=8, d=128, seed=3, spec_kw=None,
              paged=False, n_max=None, block_rows=None, **cfg_kw):
    from paper_2506_15704_b200.config import LfpsConfig
    from paper_2506_15704_b200.workload import GqaSpec, gen_unit
    kw = dict(slash_offsets=(64, 65), band_width=6)
    kw.update(spec_kw or {})
    spec = GqaSpec(batch=batch, kv_heads=kv_heads, group=group, d=d, n_prefill=n0, steps=steps,
                   seed=seed, **kw)
    cfg = LfpsConfig(d=d, **cfg_kw)
    K, V, W, F, Q = [], [], [], [], []
    for b in range(batch):
        kr, vr, wr, fr, qr = [], [], [], [], []
        for h in range(kv_heads):
            u = gen_unit(spec, b, h, device="cpu")
            kr.append(u.keys.float().numpy())
            vr.append(u.values.float().numpy())
            wr.append(u.weights.numpy())
            fr.append(u.final_query.float().numpy())
            qr.append(u.queries.float().numpy())
        K.append(kr); V.append(vr); W.append(wr); F.append(fr); Q.append(qr)
    K, V, W, F, Q = (np.asarray(x) for x in (K, V, W, F, Q))
    return Pair(cfg, K, V, W, F, n0, paged=paged, n_max=n_max, block_rows=block_rows), K, V, Q
