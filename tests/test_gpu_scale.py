"""Device parity at the benchmarked sizes.

The persistent block summaries (csrc/tables.cuh) and the multi-round
candidate construction (csrc/select.cuh) only take their deep paths at large
contexts: a 128k window has 257 512-slot segments, so the canonical merge
tree runs across three of its four 128-leaf warp quarters, and the select
kernel needs several 256-word rounds once more than 8192 slots are active.
These tests drive those paths step by step against the devmath oracle
(bit-exact sets, tables, scale and rho; outputs within 1e-5 relative L2).
"""

import dataclasses

import numpy as np
import pytest

from gpu_drive import gqa_pair
from paper_2506_15704_b200.session import CNT_C0, CNT_PROBE

pytestmark = pytest.mark.gpu

KBLK = 512


def window_segments(sess, s):
    """512-slot segments of session s's slash window (tables.cuh make_window)."""
    b = s // sess.Hq
    m = sess.n_host[b] - sess.cfg.sink_count
    lo = int(sess.sla_base[s])
    return (lo + m - 1) // KBLK - lo // KBLK + 1


# 128k: realistic plants (band width ~n/650, slash offsets 300/301)
C4_SPEC = dict(slash_offsets=(300, 301), band_width=201)


@pytest.mark.parametrize("frac", [0.05, 0.01])
def test_c4_context_128k_bit_exact(frac):
    """B=1 x Hkv=2 x G=4 at n0 = 131072, 8 steps: every step's sets, rho,
    counts and outputs, the tables every 4th step.  Every window spans more
    than 128 segments (the cross-quarter merge of the 512-leaf tree)."""
    n0, steps = 131072, 8
    pair, K, V, Q = gqa_pair(batch=1, kv_heads=2, group=4, n0=n0, steps=steps, seed=3,
                             spec_kw=C4_SPEC)
    sess = pair.sess
    for t in range(steps):
        res, outs = pair.step(Q[:, :, :, t], K[:, :, n0 + t], V[:, :, n0 + t], frac)
        pair.compare_step(res, outs, tables=(t % 4 == 3))
        segs = [window_segments(sess, s) for s in range(sess.NS)]
        assert min(segs) > 128, segs
        # the sets are not trivial: C0 non-empty somewhere, probe > tail
        cnt = res.counts.cpu().numpy()
        assert cnt[..., CNT_C0].max() > 0
        assert cnt[..., CNT_PROBE].max() > 100


def test_c1_shape_16k_bit_exact():
    """The full C1 shape: B=1 x 8 KV heads x 4 q-heads at n0 = 16384
    (32 sessions), alternating 5% and 1% budgets."""
    n0, steps = 16384, 6
    pair, K, V, Q = gqa_pair(batch=1, kv_heads=8, group=4, n0=n0, steps=steps, seed=16,
                             spec_kw=dict(slash_offsets=(300, 301), band_width=25))
    for t in range(steps):
        frac = 0.05 if t % 2 == 0 else 0.01
        res, outs = pair.step(Q[:, :, :, t], K[:, :, n0 + t], V[:, :, n0 + t], frac)
        pair.compare_step(res, outs, tables=(t % 3 == 2))


@pytest.mark.parametrize("n0", [12000, 40000])
def test_exhaustive_fallback_multi_round_select(n0):
    """exhaustive_fallback at m > 8192: C0 is every slot, so the select
    kernel's candidate construction runs ceil(m / 8192) rounds of 256 active
    words (select.cuh); the probe list holds all m slots plus the tail and
    the Top-k selects among them (k < |probe|)."""
    steps = 3
    pair, K, V, Q = gqa_pair(batch=1, kv_heads=1, group=2, n0=n0, steps=steps, d=64, seed=7,
                             exhaustive_fallback=True, epsilon=1.0)
    m = n0 - pair.cfg.sink_count
    for t in range(steps):
        res, outs = pair.step(Q[:, :, :, t], K[:, :, n0 + t], V[:, :, n0 + t], 0.05)
        pair.compare_step(res, outs, tables=(t == steps - 1))
        cnt = res.counts.cpu().numpy()
        assert cnt[0, :, CNT_PROBE].min() == m + t        # every slot is a candidate
        assert (m + t + 31) // 32 > 256


def test_renormalisation_with_live_block_summaries():
    """The lazy scale crosses 1e-120 while the block summaries are live.

    A purely non-exhaustive trajectory cannot get there: the reference's own
    moments overflow first (s2 * s2 -> inf, kappa == 0, ZeroDivisionError at
    tables.py:315; see test_moment_overflow_raises_like_the_reference).  The
    reference's decode_step takes a config per call (engine.py:97), so this
    trajectory runs non-exhaustive steps (summaries built and maintained),
    then exhaustive steps through the renormalisation (tables.py:165-169),
    then non-exhaustive steps again: their thresholds come from summaries
    that must have been invalidated by the renormalisation.  r = 0.5
    renormalises on the 399th update."""
    n0, steps = 700, 520
    pair, K, V, Q = gqa_pair(batch=1, kv_heads=1, group=2, n0=n0, steps=steps, d=32, seed=33,
                             r=0.5, epsilon=1.0)
    exh = dataclasses.replace(pair.cfg, exhaustive_fallback=True)
    sess = pair.sess
    renormed_at = None
    for t in range(steps):
        cfg = exh if 200 <= t < 440 else None
        res, outs = pair.step(Q[:, :, :, t], K[:, :, n0 + t], V[:, :, n0 + t], 0.05, cfg=cfg)
        if renormed_at is None and float(sess.scale[0]) == 1.0 and t > 0:
            renormed_at = t
        near = renormed_at is not None and t - renormed_at < 4
        pair.compare_step(res, outs, tables=(t % 20 == 0 or near or t >= 440))
    assert renormed_at is not None and 200 <= renormed_at < 440, renormed_at


def _reference_fate(pair, K, V, Q, n0, steps):
    """Step at which the reference arithmetic (RefArith, fp64 scores) raises
    ZeroDivisionError on this trajectory, or None."""
    from oracle import lfps_oracle as lo
    cfg = pair.cfg
    kv, trs, prs = lo.bootstrap_unit(K[0, 0, :n0], V[0, 0, :n0], pair.weights[0, 0],
                                     pair.finals[0, 0], cfg, lo.RefArith)
    for t in range(steps):
        try:
            lo.unit_step(kv, trs, prs, Q[0, 0, :, t], K[0, 0, n0 + t], V[0, 0, n0 + t], 0.05,
                         cfg, lo.RefArith, "fp64")
        except ZeroDivisionError:
            return t
    return None


@pytest.mark.parametrize("group", [1, 2])
def test_moment_overflow_regime_matches_the_reference(group):
    """Non-exhaustive at r = 0.5 the phys values grow as 1 / scale until the
    fp64 moments overflow (scale ~1e-77, step ~256 here).  There the
    reference's kappa = s4 / (s2 * s2) is 0 when only s2 * s2 overflowed
    (ZeroDivisionError, tables.py:315) and NaN when s4 overflowed with it
    (empty C0 from then on).  With one q-head the trajectory raises, with
    two it continues; the device follows the canonical oracle step for step
    through the regime (same sets and tables, the raise on the same step
    with nothing committed), and the reference's own arithmetic meets the
    same fate on the same step."""
    import warnings
    import torch
    n0, steps = 700, 300
    pair, K, V, Q = gqa_pair(batch=1, kv_heads=1, group=group, n0=n0, steps=steps, d=32,
                             seed=33, r=0.5, epsilon=1.0)
    sess = pair.sess
    failed = None
    with warnings.catch_warnings():
        warnings.simplefilter("ignore", RuntimeWarning)       # numpy overflow in the oracle
        for t in range(steps):
            before = [x.clone() for x in (sess.ver, sess.sla, sess.scale, sess.n_ctx)]
            try:
                res, outs = pair.step(Q[:, :, :, t], K[:, :, n0 + t], V[:, :, n0 + t], 0.05)
            except ZeroDivisionError:
                failed = t
                after = (sess.ver, sess.sla, sess.scale, sess.n_ctx)
                assert all(torch.equal(x, y) for x, y in zip(before, after))
                break
            pair.compare_step(res, outs, tables=(t % 25 == 0 or 250 <= t <= 262))
        if failed is not None:
            # the device raised: so does the canonical oracle on this step
            from oracle import lfps_oracle as lo
            kv, trs, prs = pair.units[0]
            with pytest.raises(ZeroDivisionError):
                lo.unit_step(kv, trs, prs, Q[0, 0, :, failed], K[0, 0, n0 + failed],
                             V[0, 0, n0 + failed], 0.05, pair.cfg, lo.DevArith, "fp32")
        else:
            assert float(sess.scale[0]) < 1e-80              # deep in the overflow regime
        assert failed == _reference_fate(pair, K, V, Q, n0, steps)
    assert (failed is not None) == (group == 1)


def test_seeded_reference_golden_c1_16k():
    """The C1 shape against the reference's OWN outputs (tests/golden/seeded/
    c1_16k.npz, made by make_golden_seeded.py from the reference's
    prefill_bootstrap / decode_step): every device C0 / C1 / probe / C2 set
    equals the reference's, and the device matches the canonical oracle
    bit for bit on the way (tables after the last step)."""
    from gpu_drive import Pair
    from golden_io import load_seeded
    from paper_2506_15704_b200.config import LfpsConfig
    g = load_seeded("c1_16k")
    sp = g.spec
    n0, T, Hkv, G = sp.n_prefill, sp.steps, sp.kv_heads, sp.group
    pair = Pair(LfpsConfig(d=sp.d, **g.cfg), g.K[None], g.V[None], g.W[None], g.F[None], n0)
    ref = {k: g.sets(k) for k in ("c0", "c1", "probe", "c2")}
    for t in range(T):
        res, outs = pair.step(g.Q[None, :, :, t], g.K[None, :, n0 + t], g.V[None, :, n0 + t],
                              float(g.fracs[t]))
        pair.compare_step(res, outs, tables=(t == T - 1))
        byp = res.bypassed.cpu().numpy()
        for qh in range(Hkv * G):
            rec = t * Hkv * G + qh
            assert bool(byp[0, qh]) == bool(g.raw["bypassed"][rec])
            if byp[0, qh]:
                continue
            np.testing.assert_array_equal(pair.sess.c0_list(0, qh), ref["c0"][rec])
            np.testing.assert_array_equal(pair.sess.c1_list(0, qh), ref["c1"][rec])
            np.testing.assert_array_equal(pair.sess.probe_list(0, qh), ref["probe"][rec])
            np.testing.assert_array_equal(pair.sess.c2_list(0, qh), ref["c2"][rec])
        out = res.output.cpu().numpy()[0]
        want = g.raw["outputs"][t * Hkv * G:(t + 1) * Hkv * G]
        err = np.linalg.norm(out - want, axis=1) / np.linalg.norm(want, axis=1)
        assert err.max() <= 1e-5, err.max()
