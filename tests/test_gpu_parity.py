"""Device parity: the sm_100a path against the devmath oracle and the
reference's own golden vectors.

Bar: candidate sets C0/C1/probe bit-exact, Top-k sets
identical (same fp32 scores, lower-index ties), bypass decisions and rho
bit-exact, tracker tables bit-exact (phys values and lazy scale) after every
step, attention output within 1e-5 relative L2 of the fp64 oracle fed the
same fp32 scores.
"""

import numpy as np
import pytest
import torch

from golden_io import load, names
from gpu_drive import Pair
from oracle_run import golden_config
from paper_2506_15704_b200.session import CNT_K, CNT_PROBE

pytestmark = pytest.mark.gpu


def _golden_pair(g):
    cfg = golden_config(g)
    keys = g.keys[None, None]
    values = g.values[None, None]
    weights = g.weights[None, None]
    finals = g.finals[None, None]
    return Pair(cfg, keys, values, weights, finals, g.n0, n_max=g.n0 + g.steps + 8)


@pytest.mark.parametrize("name", names())
def test_golden_trajectory_bit_exact(name):
    g = load(name)
    pair = _golden_pair(g)
    # seeded tables and priors
    kv, trs, prs = pair.units[0]
    for gi in range(g.G):
        ver, sla, sc = pair.sess.session_tables(gi)
        np.testing.assert_array_equal(ver, trs[gi].ver_view())
        np.testing.assert_array_equal(sla, trs[gi].sla_view())
    np.testing.assert_array_equal(pair.sess.sigma_hat_sq.cpu().numpy(),
                                  [p.sigma_hat_sq for p in prs])
    np.testing.assert_array_equal(pair.sess.mean_key[0].cpu().numpy(), prs[0].mean_key)
    ref_c2 = g.sets("c2")
    ref_probe = g.sets("probe")
    for t in range(g.steps):
        q = g.queries[t][None, None]
        res, outs = pair.step(q, g.keys[g.n0 + t][None, None], g.values[g.n0 + t][None, None],
                              g.frac)
        pair.compare_step(res, outs)
        # and the reference's own selections (golden vectors)
        for gi in range(g.G):
            rec = t * g.G + gi
            if not g.raw["bypassed"][rec]:
                np.testing.assert_array_equal(pair.sess.c2_list(0, gi), ref_c2[rec])
                np.testing.assert_array_equal(pair.sess.probe_list(0, gi), ref_probe[rec])


from gpu_drive import gqa_pair as _gqa_pair  # noqa: E402


@pytest.mark.parametrize("frac", [0.05, 0.01])
def test_gqa_batch_bit_exact(frac):
    pair, K, V, Q = _gqa_pair()
    n0 = pair.n0
    for t in range(8):
        res, outs = pair.step(Q[:, :, :, t], K[:, :, n0 + t], V[:, :, n0 + t], frac)
        pair.compare_step(res, outs)


def test_exhaustive_and_mean_only_modes():
    pair, K, V, Q = _gqa_pair(batch=1, kv_heads=2, n0=1500, steps=4, exhaustive_fallback=True,
                              epsilon=1.0)
    for t in range(4):
        res, outs = pair.step(Q[:, :, :, t], K[:, :, 1500 + t], V[:, :, 1500 + t], 0.03)
        pair.compare_step(res, outs)


@pytest.mark.parametrize("d,group", [(128, 4), (64, 8), (256, 2), (32, 1)])
def test_exact_path_matches_oracle_and_overlap(d, group):
    from oracle import lfps_oracle as lo
    pair, K, V, Q = _gqa_pair(batch=1, kv_heads=2, group=group, n0=4000, steps=2, d=d)
    sess = pair.sess
    frac = 0.05
    q = Q[:, :, :, 0]
    import gpu_drive
    qd = gpu_drive.bf16(q.reshape(1, -1, pair.d)).cuda()
    res = sess.exact_topk_step(qd, frac)
    torch.cuda.synchronize()
    exact_idx = res.c2_idx.clone()
    exact_cnt = res.counts.clone()
    for h in range(pair.Hkv):
        kv, trs, prs = pair.units[h]
        for g in range(pair.G):
            qh = h * pair.G + g
            k = max(1, round(frac * kv.n))
            sel, out = lo.exact_topk_step(kv, q[0, h, g], k, pair.cfg, score="fp32")
            np.testing.assert_array_equal(sess.c2_list(0, qh), sel)
            # topk_oracle (full stable sort) agrees too
            np.testing.assert_array_equal(sel, lo.topk_oracle(kv, q[0, h, g], k, 4, "fp32"))
            got = res.output[0, qh].cpu().numpy()
            assert np.linalg.norm(got - out) / np.linalg.norm(out) <= 1e-5
    # LFPS step then eta against the exact set
    res2, outs = pair.step(q, K[:, :, 4000], V[:, :, 4000], frac)
    pair.compare_step(res2, outs)
    eta = sess.overlap(res2.c2_idx, res2.counts, exact_idx, exact_cnt).cpu().numpy()
    for h in range(pair.Hkv):
        for g in range(pair.G):
            qh = h * pair.G + g
            o = outs[h][g]
            if o.bypassed:
                continue
            want = lo.overlap_ratio(o.c2, exact_idx[0, qh, :int(exact_cnt[0, qh, 5])].cpu().numpy(),
                                    int(exact_cnt[0, qh, 5]))
            assert eta[0, qh] == pytest.approx(want, abs=0)


@pytest.mark.parametrize("n0,frac,dup", [(6000, 0.05, 0), (6000, 0.05, 700), (6000, 0.3, 0),
                                         (6000, 1.0, 0), (20000, 0.05, 0), (20000, 0.05, 1500),
                                         (20000, 0.01, 0)])
def test_exact_topk_ties_and_budgets(n0, frac, dup):
    """Exact path against topk_oracle (full stable sort, attention.py:100-113)
    with planted exact ties: `dup` rows get the same key, so the k-th score
    is shared by many rows and the lower-index rule decides (attention.py:
    34-47); frac 1.0 selects every non-sink row.  n0 = 20000 takes the
    sampled-window selection (k_topk.cu), 6000 the histogram path."""
    from oracle import lfps_oracle as lo
    import gpu_drive
    pair, K, V, Q = _gqa_pair(batch=1, kv_heads=2, n0=n0, steps=1, seed=9)
    if dup:
        rng = np.random.default_rng(5)
        rows = rng.choice(np.arange(4, n0), size=dup, replace=False)
        for h in range(pair.Hkv):
            K[0, h, rows] = K[0, h, rows[0]]
        pair = _rebuild(pair, K, V)
    sess = pair.sess
    q = Q[:, :, :, 0]
    qd = gpu_drive.bf16(q.reshape(1, -1, pair.d)).cuda()
    res = sess.exact_topk_step(qd, frac)
    torch.cuda.synchronize()
    for h in range(pair.Hkv):
        kv, trs, prs = pair.units[h]
        for g in range(pair.G):
            qh = h * pair.G + g
            k = max(1, round(frac * kv.n))
            want = lo.topk_oracle(kv, q[0, h, g], k, 4, "fp32")
            np.testing.assert_array_equal(sess.c2_list(0, qh), want)
            _, out = lo.exact_topk_step(kv, q[0, h, g], k, pair.cfg, score="fp32")
            got = res.output[0, qh].cpu().numpy()
            assert np.linalg.norm(got - out) / np.linalg.norm(out) <= 1e-5


def _rebuild(pair, K, V):
    """A fresh Pair over modified keys/values (same weights and finals)."""
    from gpu_drive import Pair
    return Pair(pair.cfg, K, V, pair.weights, pair.finals, pair.n0)


def test_long_trajectory_crosses_slash_blocks():
    """1100 steps: the slash window start crosses two 512-slot block
    boundaries and the vertical window grows into new blocks, so the
    persistent block summaries are rebuilt, re-merged and re-segmented many
    times (k_select.cu).  Sets and outputs are compared every step against
    the oracle, the tables every tenth step."""
    pair, K, V, Q = _gqa_pair(batch=1, kv_heads=1, group=2, d=32, n0=700, steps=1100, seed=33)
    n0 = pair.n0
    for t in range(1100):
        res, outs = pair.step(Q[:, :, :, t], K[:, :, n0 + t], V[:, :, n0 + t], 0.05)
        pair.compare_step(res, outs, tables=(t % 10 == 0))


@pytest.mark.parametrize("split,steps,host_io", [(True, 2, False), (False, 2, False),
                                                 (True, 24, False), (True, 12, True),
                                                 (False, 4, True)])
def test_split_streams_bit_exact(split, steps, host_io):
    """LFPS_FLAG_SPLIT at 1024 sessions (32 requests x 8 KV heads x 4): two
    session groups on internal streams, each with its stats kernel beside its
    gate, and PDL between the later kernels; without the flag (256 sessions)
    the gate runs on an internal stream beside the stats -> select -> finish
    chain.  Results are identical to the oracle over many steps (no
    cross-step or cross-stream races).  host_io: every step through
    lfps_decode_step_host_io (the input copy on its own stream, the output
    copied back to pinned host memory, bit-identical to the device output)."""
    pair, K, V, Q = _gqa_pair(batch=32 if split else 8, kv_heads=8, group=4, d=64, n0=700,
                              steps=steps, seed=41)
    pair.sess.split = split
    pair.host_io = host_io
    n0 = pair.n0
    for t in range(steps):
        res, outs = pair.step(Q[:, :, :, t], K[:, :, n0 + t], V[:, :, n0 + t], 0.05)
        pair.compare_step(res, outs, tables=(t % 8 == 1 or t == steps - 1))


def test_full_attention_matches_oracle():
    """N4: full softmax attention over every row on the device against the
    reference's full_attention_oracle arithmetic (fp64, attention.py:88-97)."""
    import math
    import gpu_drive
    pair, K, V, Q = _gqa_pair(batch=1, kv_heads=2, n0=3000, steps=1, seed=13)
    q = Q[:, :, :, 0]
    out = pair.sess.full_attention(gpu_drive.bf16(q.reshape(1, -1, pair.d)).cuda()).cpu().numpy()
    for h in range(pair.Hkv):
        kv = pair.units[h][0]
        keys, values = kv.keys[:kv.n], kv.values[:kv.n]
        for g in range(pair.G):
            z = keys @ q[0, h, g] / math.sqrt(pair.d)
            w = np.exp(z - z.max())
            w /= w.sum()
            ref = w @ values
            got = out[0, h * pair.G + g]
            assert np.linalg.norm(got - ref) / np.linalg.norm(ref) <= 1e-5


def test_failed_step_commits_nothing_then_recovers():
    """A data error in one session (a non-finite query -> non-finite gate
    logits, engine.py:8-9) fails the whole step: nothing is committed, the
    error is reported; the next good step commits exactly as if the failed
    call never happened (the err[0] call stamp needs no clearing kernel)."""
    import gpu_drive
    pair, K, V, Q = _gqa_pair(batch=2, kv_heads=2, n0=900, steps=3, seed=29)
    sess = pair.sess
    n0 = pair.n0
    res, outs = pair.step(Q[:, :, :, 0], K[:, :, n0], V[:, :, n0], 0.05)
    pair.compare_step(res, outs)
    before = [t.clone() for t in (sess.ver, sess.sla, sess.scale, sess.sla_base, sess.n_ctx)]
    n_before = list(sess.n_host)
    qbad = Q[:, :, :, 1].copy()
    qbad[1, 0, 2, 5] = np.inf                      # session 1 * 8 + 0 * 4 + 2
    with pytest.raises(ValueError, match="session 10"):
        sess.decode_step(gpu_drive.bf16(qbad.reshape(2, -1, pair.d)).cuda(),
                         gpu_drive.bf16(K[:, :, n0 + 1]).cuda(),
                         gpu_drive.bf16(V[:, :, n0 + 1]).cuda(), 0.05, check=True)
    assert list(sess.n_host) == n_before
    after = (sess.ver, sess.sla, sess.scale, sess.sla_base, sess.n_ctx)
    assert all(torch.equal(x, y) for x, y in zip(before, after))
    # the good step (same new row) commits and matches the oracle
    res, outs = pair.step(Q[:, :, :, 1], K[:, :, n0 + 1], V[:, :, n0 + 1], 0.05)
    pair.compare_step(res, outs)
    res, outs = pair.step(Q[:, :, :, 2], K[:, :, n0 + 2], V[:, :, n0 + 2], 0.05)
    pair.compare_step(res, outs)


def test_decode_step_host_output():
    """lfps_decode_step_host_out: the output lands in pinned host memory
    (copied beside the commit kernel) bit-identical to the device output,
    and the step is otherwise the same step (oracle parity)."""
    pair, K, V, Q = _gqa_pair(batch=2, kv_heads=2, n0=900, steps=2, seed=31)
    import gpu_drive
    sess = pair.sess
    n0 = pair.n0
    res, outs = pair.step(Q[:, :, :, 0], K[:, :, n0], V[:, :, n0], 0.05)
    pair.compare_step(res, outs)
    host = torch.empty(tuple(sess.out.shape), dtype=torch.float32).pin_memory()
    host.fill_(float("nan"))
    B, Hkv, G, d = pair.B, pair.Hkv, pair.G, pair.d
    res = sess.decode_step(gpu_drive.bf16(Q[:, :, :, 1].reshape(B, Hkv * G, d)).cuda(),
                           gpu_drive.bf16(K[:, :, n0 + 1]).cuda(),
                           gpu_drive.bf16(V[:, :, n0 + 1]).cuda(), 0.05, out_host=host)
    torch.cuda.current_stream().synchronize()
    sess.check_errors("host-output step")
    assert torch.equal(host, sess.out.cpu())
    with pytest.raises(ValueError):
        sess.decode_step(gpu_drive.bf16(Q[:, :, :, 1].reshape(B, Hkv * G, d)).cuda(),
                         gpu_drive.bf16(K[:, :, n0 + 1]).cuda(),
                         gpu_drive.bf16(V[:, :, n0 + 1]).cuda(), 0.05,
                         out_host=torch.empty(3, dtype=torch.float32))


def test_decode_step_host_io_small_and_rejects():
    """lfps_decode_step_host_io on a small batch (oracle parity for several
    steps, output bit-identical in host memory) and its argument checks."""
    pair, K, V, Q = _gqa_pair(batch=2, kv_heads=2, n0=900, steps=3, seed=37)
    pair.host_io = True
    n0 = pair.n0
    for t in range(3):
        res, outs = pair.step(Q[:, :, :, t], K[:, :, n0 + t], V[:, :, n0 + t], 0.05)
        pair.compare_step(res, outs)
    sess = pair.sess
    nb = sess.step_input_bytes()
    assert nb == (sess.B * sess.Hq + 2 * sess.B * sess.Hkv) * sess.d * 2
    with pytest.raises(ValueError):       # wrong size
        sess.decode_step_host(torch.zeros(nb // 2 - 1, dtype=torch.bfloat16), 0.05)
    with pytest.raises(ValueError):       # wrong dtype
        sess.decode_step_host(torch.zeros(nb // 2, dtype=torch.float16), 0.05)
    with pytest.raises(ValueError):       # bad output buffer
        sess.decode_step_host(torch.zeros(nb // 2, dtype=torch.bfloat16), 0.05,
                              out_host=torch.empty(3, dtype=torch.float32))


def test_decode_step_host_io_reused_buffers():
    """A decode loop's pattern: the same pinned input and output buffers every
    step with new contents (decode_step_host caches their checks per tensor),
    bit-exact against the oracle through graph replays; a buffer of the
    wrong size at a cached tensor's address is still rejected."""
    pair, K, V, Q = _gqa_pair(batch=2, kv_heads=2, n0=900, steps=5, seed=41)
    pair.host_io = True
    pair.reuse_host = True
    pair.sess.graph = True
    n0 = pair.n0
    for t in range(5):
        res, outs = pair.step(Q[:, :, :, t], K[:, :, n0 + t], V[:, :, n0 + t], 0.05)
        pair.compare_step(res, outs)
    sess = pair.sess
    inp, out = pair._host_bufs
    with pytest.raises(ValueError):       # a view of the cached input buffer, the wrong size
        sess.decode_step_host(inp[:-1], 0.05, out_host=out)
    with pytest.raises(ValueError):       # the cached output tensor, resized in place
        out.resize_(out.numel() - 1)
        sess.decode_step_host(inp, 0.05, out_host=out)


def test_paged_kv_pool_bit_exact_across_a_page():
    """N4 paged-KV caller: K/V in a KvPool (virtual [B, Hkv, n_max, d], 2 MiB
    pages mapped as contexts grow).  The prefill ends 3 rows before the first
    page boundary (8192 rows at d=128), so the appended rows of the 6 steps
    land on BOTH pages and the probe / exact / full reads straddle it; every
    step matches the oracle, through decode_step and the host-io entry point.
    Releasing a request returns its pages and blocks further steps until it
    is reloaded; after load_prefill + bootstrap the reloaded request decodes
    again in the same batch (the other request continuing its trajectory)."""
    from oracle import lfps_oracle as lo
    from paper_2506_15704_b200 import kv_pool
    import gpu_drive
    rows = kv_pool.page_rows(128)
    n0 = rows - 3
    pair, K, V, Q = _gqa_pair(batch=2, kv_heads=2, n0=n0, steps=12, seed=53, paged=True,
                              n_max=2 * rows)
    sess = pair.sess
    assert sess.kv_pool is not None and sess.n_max == 2 * rows
    page = kv_pool.page_bytes()
    assert sess.kv_mapped_bytes() == 2 * 2 * 2 * 2 * page        # K+V x B x Hkv, 2 pages (slack)
    for t in range(6):
        pair.host_io = t % 2 == 1
        res, outs = pair.step(Q[:, :, :, t], K[:, :, n0 + t], V[:, :, n0 + t], 0.05)
        pair.compare_step(res, outs)
    for h in range(2):                                # rows rows-3 .. rows+2 were appended
        kr, _ = sess.kv_rows(0, h, n0 + 6)
        np.testing.assert_array_equal(kr.float().cpu().numpy()[rows - 3:], K[0, h, rows - 3:n0 + 6])
    q = gpu_drive.bf16(Q[:, :, :, 5].reshape(2, -1, 128)).cuda()
    sess.exact_topk_step(q, 0.05)
    torch.cuda.synchronize()
    sess.check_errors("exact on paged rows")
    for h in range(2):
        kv = pair.units[h][0]
        for g in range(4):
            k = max(1, round(0.05 * kv.n))
            np.testing.assert_array_equal(sess.c2_list(0, h * 4 + g),
                                          lo.topk_oracle(kv, Q[0, h, g, 5], k, 4, "fp32"))
    sess.release_request(1)
    assert sess.kv_mapped_bytes() == 2 * 2 * 2 * page
    with pytest.raises(ValueError):
        sess.decode_step(q, gpu_drive.bf16(K[:, :, n0]).cuda(), gpu_drive.bf16(V[:, :, n0]).cuda(),
                         0.05)
    # reload request 1 from its prefill, bootstrap its sessions, decode on
    sess.load_prefill(1, gpu_drive.bf16(K[1, :, :n0]).cuda(), gpu_drive.bf16(V[1, :, :n0]).cuda())
    w = torch.as_tensor(np.ascontiguousarray(pair.weights[1], dtype=np.float32))
    sess.bootstrap_tables(8, w.reshape(8, pair.cfg.s, n0 - 4).cuda())
    finals = np.concatenate([pair.finals[0].reshape(8, 128), pair.finals[1].reshape(8, 128)])
    sess.bootstrap_stats(gpu_drive.bf16(finals.reshape(2, 8, 128)).cuda(), requests=(1, 1))
    torch.cuda.synchronize()
    sess.check_errors("reload")
    for h in range(2):
        pair.units[2 + h] = lo.bootstrap_unit(K[1, h, :n0], V[1, h, :n0], pair.weights[1, h],
                                              pair.finals[1, h], pair.cfg, lo.DevArith)
    # request 0 continues at step 6; request 1 restarts at step 0 (ragged contexts)
    for t in range(6, 9):
        qs = Q[:, :, :, t].copy()
        qs[1] = Q[1, :, :, t - 6]
        kn = np.stack([K[0, :, n0 + t], K[1, :, n0 + t - 6]])
        vn = np.stack([V[0, :, n0 + t], V[1, :, n0 + t - 6]])
        res, outs = pair.step(qs, kn, vn, 0.05)
        pair.compare_step(res, outs)


def test_two_threads_two_sessions_bit_exact():
    """Reentrancy across distinct sessions (SURVEY §8(b) threading): two host
    threads step two sessions concurrently, each on its own CUDA stream, with
    LFPS_FLAG_SPLIT set (256 sessions each: below the split threshold, so
    each runs its gate on its own workspace's internal stream, joined by
    event before the finish).  Each session's trajectory is identical
    to the oracle's, as if it had run alone."""
    import threading
    import gpu_drive
    steps = 10
    pairs = [gqa_pair_cached(seed) for seed in (41, 43)]
    results = [[], []]
    errors = []
    start = threading.Barrier(2)

    def drive(i):
        try:
            pair, K, V, Q = pairs[i]
            sess, n0 = pair.sess, pair.n0
            B, Hkv, G, d = pair.B, pair.Hkv, pair.G, pair.d
            inputs = [(gpu_drive.bf16(Q[:, :, :, t].reshape(B, Hkv * G, d)).cuda(),
                       gpu_drive.bf16(K[:, :, n0 + t]).cuda(), gpu_drive.bf16(V[:, :, n0 + t]).cuda())
                      for t in range(steps)]
            st = torch.cuda.Stream()
            torch.cuda.synchronize()
            start.wait()
            with torch.cuda.stream(st):
                for t in range(steps):
                    res = sess.decode_step(*inputs[t], 0.05)
                    results[i].append((res.counts.clone(), res.output.clone(), res.rho.clone(),
                                       res.bypassed.clone(), res.c2_idx.clone(),
                                       sess.probe_idx.clone()))
            st.synchronize()
            sess.check_errors("threaded steps")
        except BaseException as e:  # noqa: BLE001
            errors.append(e)

    th = [threading.Thread(target=drive, args=(i,)) for i in range(2)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    assert not errors, errors
    from paper_2506_15704_b200.session import BatchedStepResult
    for i, (pair, K, V, Q) in enumerate(pairs):
        n0 = pair.n0
        for t in range(steps):
            cnt, out, rho, byp, c2, probe = results[i][t]
            outs = []
            for b in range(pair.B):
                for h in range(pair.Hkv):
                    kv, trs, prs = pair.units[b * pair.Hkv + h]
                    outs.append(lo_step(kv, trs, prs, Q[b, h, :, t], K[b, h, n0 + t],
                                        V[b, h, n0 + t], pair.cfg))
            # replay the recorded device lists into the session views for compare_step
            pair.sess.counts.copy_(cnt)
            pair.sess.c2_idx.copy_(c2)
            pair.sess.probe_idx.copy_(probe)
            res = BatchedStepResult(output=out, rho=rho, bypassed=byp, counts=cnt, c2_idx=c2,
                                    c2_score=pair.sess.c2_score, err=pair.sess.err)
            pair.compare_step(res, outs, tables=(t == steps - 1), bitmaps=(t == steps - 1))


def lo_step(kv, trs, prs, qs, k_new, v_new, cfg):
    from oracle import lfps_oracle as lo
    return lo.unit_step(kv, trs, prs, qs, k_new, v_new, 0.05, cfg, lo.DevArith, "fp32")


def gqa_pair_cached(seed):
    pair, K, V, Q = _gqa_pair(batch=8, kv_heads=8, group=4, d=64, n0=700, steps=10, seed=seed)
    pair.sess.split = True
    return pair, K, V, Q


@pytest.mark.parametrize("block_rows,d", [(16, 128), (64, 64)])
def test_block_table_kv_bit_exact(block_rows, d):
    """N4, the serving caller with a block table (vLLM-style 16-row blocks
    in a random order, lfps_state.block_table): every kernel reads and the
    commit appends rows through the table.  Multi-step parity with the
    oracle (so identical to the contiguous cache), the exact path and full
    attention over block-table rows."""
    import math
    import gpu_drive
    from oracle import lfps_oracle as lo
    pair, K, V, Q = _gqa_pair(batch=2, kv_heads=2, n0=2500, steps=6, d=d, seed=59,
                              block_rows=block_rows)
    sess = pair.sess
    assert sess.block_table is not None and sess.block_rows == block_rows
    n0 = pair.n0
    for t in range(6):
        pair.host_io = t % 3 == 2
        res, outs = pair.step(Q[:, :, :, t], K[:, :, n0 + t], V[:, :, n0 + t], 0.05 if t % 2 else 0.01)
        pair.compare_step(res, outs)
    kr, vr = sess.kv_rows(1, 1, n0 + 6)                 # appended rows went through the table
    np.testing.assert_array_equal(kr.float().cpu().numpy(), K[1, 1, :n0 + 6])
    q = Q[:, :, :, 5]
    qd = gpu_drive.bf16(q.reshape(2, -1, d)).cuda()
    sess.exact_topk_step(qd, 0.05)
    torch.cuda.synchronize()
    for h in range(2):
        kv = pair.units[h][0]
        for g in range(4):
            k = max(1, round(0.05 * kv.n))
            np.testing.assert_array_equal(sess.c2_list(0, h * 4 + g),
                                          lo.topk_oracle(kv, q[0, h, g], k, 4, "fp32"))
    full = sess.full_attention(qd).cpu().numpy()
    kv = pair.units[0][0]
    z = kv.keys[:kv.n] @ q[0, 0, 0] / math.sqrt(d)
    w = np.exp(z - z.max())
    ref = (w / w.sum()) @ kv.values[:kv.n]
    assert np.linalg.norm(full[0, 0] - ref) / np.linalg.norm(ref) <= 1e-5


@pytest.mark.parametrize("host_io,split", [(False, False), (True, False), (False, True)])
def test_graph_replay_bit_exact(host_io, split):
    """LFPS_FLAG_GRAPH: the step is captured once and replayed (device inputs
    copied into the same buffers every step, or packed host inputs through
    the captured copy node, whose host pointer is updated per replay); the
    call stamp comes from the device.  Parity with the oracle every step,
    then a failing step (non-finite query) raises and commits nothing, and
    the following replays commit again."""
    import gpu_drive
    B, Hkv, G, d = (32, 8, 4, 64) if split else (2, 2, 4, 128)
    pair, K, V, Q = _gqa_pair(batch=B, kv_heads=Hkv, group=G, d=d, n0=900, steps=8, seed=83)
    sess = pair.sess
    sess.graph = sess.graph_device = True
    sess.split = split
    qd = torch.empty(B, Hkv * G, d, dtype=torch.bfloat16, device="cuda")
    kd = torch.empty(B, Hkv, d, dtype=torch.bfloat16, device="cuda")
    vd = torch.empty_like(kd)
    n0 = pair.n0

    def device_step(q, k, v, frac, check=True):
        qd.copy_(gpu_drive.bf16(q.reshape(B, Hkv * G, d)))
        kd.copy_(gpu_drive.bf16(k))
        vd.copy_(gpu_drive.bf16(v))
        return sess.decode_step(qd, kd, vd, frac, check=check)

    for t in range(8):
        if t == 5:                                     # a failing step in the middle
            qbad = Q[:, :, :, t].copy()
            qbad[0, 0, 1, 3] = np.inf
            before = [x.clone() for x in (sess.ver, sess.sla, sess.scale, sess.n_ctx)]
            with pytest.raises(ValueError):
                if host_io:
                    sess.decode_step_host(sess.pack_step_inputs(
                        gpu_drive.bf16(qbad.reshape(B, Hkv * G, d)), gpu_drive.bf16(K[:, :, n0 + t]),
                        gpu_drive.bf16(V[:, :, n0 + t])), 0.05, check=True)
                else:
                    device_step(qbad, K[:, :, n0 + t], V[:, :, n0 + t], 0.05)
            after = (sess.ver, sess.sla, sess.scale, sess.n_ctx)
            assert all(torch.equal(x, y) for x, y in zip(before, after))
        if host_io:
            pair.host_io = True
            res, outs = pair.step(Q[:, :, :, t], K[:, :, n0 + t], V[:, :, n0 + t], 0.05)
        else:
            res = device_step(Q[:, :, :, t], K[:, :, n0 + t], V[:, :, n0 + t], 0.05)
            outs = []
            from oracle import lfps_oracle as lo
            for b in range(B):
                for h in range(Hkv):
                    kv, trs, prs = pair.units[b * Hkv + h]
                    outs.append(lo.unit_step(kv, trs, prs, Q[b, h, :, t], K[b, h, n0 + t],
                                             V[b, h, n0 + t], 0.05, pair.cfg, lo.DevArith,
                                             "fp32"))
        pair.compare_step(res, outs, tables=(t % 3 == 2 or t == 7))




@pytest.mark.parametrize("epsilon,host_io,split,frac", [
    (1.0, False, True, 0.05), (1e-6, True, True, 0.05), (0.3, False, False, 0.01),
    (0.6, True, False, 0.05)])
def test_prefetched_steps_bit_exact(epsilon, host_io, split, frac):
    """lfps_decode_prefetch + a LFPS_FLAG_PREFETCHED step: the thresholds, C0,
    C1 and probe sets built ahead of the gate (they do not depend on q,
    engine.py:146-160) give the same step as the normal path -- sets,
    counts (bypassed sessions report none), tables and outputs against the
    oracle -- with gated sessions (epsilon), the stream split, host I/O and
    Top-k cuts (1%)."""
    pair, K, V, Q = _gqa_pair(batch=32 if split else 8, kv_heads=8, group=4, d=64, n0=900,
                              steps=6, seed=7, epsilon=epsilon)
    pair.sess.split = split
    pair.host_io = host_io
    pair.prefetch = True
    n0 = pair.n0
    for t in range(6):
        res, outs = pair.step(Q[:, :, :, t], K[:, :, n0 + t], V[:, :, n0 + t], frac)
        pair.compare_step(res, outs, tables=(t % 2 == 1))
        cnt = res.counts.cpu().numpy()
        byp = res.bypassed.cpu().numpy().astype(bool)
        assert (cnt[byp][:, :6] == 0).all()          # no candidates on a bypassed session


def test_prefetched_step_requires_a_prefetch():
    """A LFPS_FLAG_PREFETCHED step without a preceding lfps_decode_prefetch on
    the workspace is rejected before any launch; a prefetch serves one step
    only, and a full step in between makes it stale."""
    pair, K, V, Q = _gqa_pair(batch=1, kv_heads=2, n0=700, steps=2)
    B, Hkv, G, d = pair.B, pair.Hkv, pair.G, pair.d
    q = torch.zeros(B, Hkv * G, d, dtype=torch.bfloat16, device="cuda")
    kv = torch.zeros(B, Hkv, d, dtype=torch.bfloat16, device="cuda")
    with pytest.raises(ValueError, match="lfps_decode_prefetch"):
        pair.sess.decode_step(q, kv, kv, 0.05, prefetched=True)
    pair.prefetch = True
    res, outs = pair.step(Q[:, :, :, 0], K[:, :, pair.n0], V[:, :, pair.n0], 0.05)
    pair.compare_step(res, outs)
    with pytest.raises(ValueError, match="lfps_decode_prefetch"):
        pair.sess.decode_step(q, kv, kv, 0.05, prefetched=True)
    # a full step after a prefetch makes the prefetched sets stale
    pair.sess.prefetch()
    pair.prefetch = False
    res, outs = pair.step(Q[:, :, :, 1], K[:, :, pair.n0 + 1], V[:, :, pair.n0 + 1], 0.05)
    pair.compare_step(res, outs)
    with pytest.raises(ValueError, match="lfps_decode_prefetch"):
        pair.sess.decode_step(q, kv, kv, 0.05, prefetched=True)


def test_wait_output_returns_the_step_output():
    """lfps_wait_output: after decode_step_host with a pinned host output, the
    host waits for the output copy only (the commit may still run); the host
    buffer then holds the step's output, bit-identical to the device's once
    the stream is done -- through the stream-launched and the CUDA-graph
    step."""
    pair, K, V, Q = _gqa_pair(batch=1, kv_heads=2, n0=900, steps=4, seed=71)
    sess = pair.sess
    B, Hkv, G, d = pair.B, pair.Hkv, pair.G, pair.d
    import gpu_drive
    for t, graph in enumerate((False, True, True, False)):
        sess.graph = graph
        packed = sess.pack_step_inputs(gpu_drive.bf16(Q[:, :, :, t].reshape(B, Hkv * G, d)),
                                       gpu_drive.bf16(K[:, :, pair.n0 + t]),
                                       gpu_drive.bf16(V[:, :, pair.n0 + t]))
        host = torch.full(tuple(sess.out.shape), float("nan")).pin_memory()
        sess.decode_step_host(packed, 0.05, out_host=host)
        sess.wait_output()
        got = host.clone()
        torch.cuda.synchronize()
        assert torch.equal(got, sess.out.cpu())
        sess.check_errors("wait_output steps")
