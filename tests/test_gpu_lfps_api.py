"""The reference's per-head surface on the device (paper_2506_15704_b200.lfps,
csrc/k_stages.cu): the decode step and each stage against the reference's
own golden vectors and against numpy restatements of the reference's
expressions (its unit tests' oracles), at float64."""

import math

import numpy as np
import pytest

from golden_io import load
from oracle_run import golden_config

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def lfps():
    import paper_2506_15704_b200.lfps as m
    return m


def build_session(lfps, rng, n=64, d=16, s=4, sink=2, window=3, **cfg_kw):
    cfg = lfps.LfpsConfig(d=d, s=s, sink_count=sink, local_window=window, **cfg_kw)
    keys = rng.standard_normal((n, d))
    values = rng.standard_normal((n, d))
    m = n - sink
    w = np.zeros((s, m))
    for c in range(s):
        support = (n - s + c) - sink + 1
        row = rng.random(support) + 1e-3
        w[c, :support] = row / row.sum()
    return lfps.prefill_bootstrap(keys, values, w, rng.standard_normal(d), cfg), cfg


def random_step(rng, d):
    return tuple(rng.standard_normal(d) for _ in range(3))


@pytest.mark.parametrize("name", ["planted", "planted5", "gated", "gated_mean_only",
                                  "exhaustive_ties", "wide_offsets", "renorm"])
def test_golden_through_run_session(lfps, name):
    """The reference's own trajectories (tests/golden, made by the reference
    package): every set, bypass, budget, dot count and clamp count equal;
    rho, outputs and final tables within 1e-9 (fp64 on both sides)."""
    g = load(name)
    cfg = golden_config(g)
    for gi in range(g.G):
        ses = lfps.prefill_bootstrap(g.keys[: g.n0], g.values[: g.n0], g.weights[gi],
                                     g.finals[gi], cfg)
        np.testing.assert_array_equal(ses.tables.ver_values(), g.raw["init_ver"][gi])
        np.testing.assert_array_equal(ses.tables.sla_values(), g.raw["init_sla"][gi])
        steps = [(g.queries[t, gi], g.keys[g.n0 + t], g.values[g.n0 + t]) for t in range(g.steps)]
        res = lfps.run_session(ses, steps, g.frac)
        for t, r in enumerate(res):
            rec = t * g.G + gi
            assert r.bypassed == bool(g.raw["bypassed"][rec])
            assert r.dot_products == g.raw["dots"][rec]
            assert r.clamp_count == g.raw["clamps"][rec]
            assert r.candidate.budget_k == g.raw["budget_k"][rec]
            assert r.rho == pytest.approx(g.raw["rho"][rec], rel=1e-12)
            for key in ("c0", "c1", "probe", "c2"):
                np.testing.assert_array_equal(getattr(r.candidate, key), g.sets(key)[rec],
                                              err_msg=f"{name} step {t} {key}")
            np.testing.assert_allclose(r.output, g.raw["outputs"][rec], rtol=1e-9, atol=1e-12)
            if not r.bypassed:
                assert r.attention.weights.sum() == pytest.approx(1.0, abs=1e-9)
                assert set(r.timings_ns) >= {"gate", "thresholds", "topk", "update", "total"}
                assert r.sparsity.w_sink > 0 and math.isfinite(r.sparsity.w_global)
        np.testing.assert_allclose(ses.tables.ver_values(), g.raw["final_ver"][gi], rtol=1e-9,
                                   atol=1e-300)
        np.testing.assert_allclose(ses.tables.sla_values(), g.raw["final_sla"][gi], rtol=1e-9,
                                   atol=1e-300)
        assert ses.tables.clamp_count == g.raw["final_clamps"][gi]


def test_epsilon_zero_forces_bypass_everywhere(lfps):
    rng = np.random.default_rng(4)
    ses, cfg = build_session(lfps, rng, epsilon=1e-300)
    v0, s0 = ses.tables.ver_values(), ses.tables.sla_values()
    for _ in range(10):
        res = lfps.decode_step(ses, *random_step(rng, 16), 0.05, cfg)
        assert res.bypassed and res.candidate.c2.size == 0
        assert res.dot_products == cfg.sink_count + cfg.local_window + 1
    assert ses.store.n == 74 and ses.tables.m == 72
    np.testing.assert_array_equal(ses.tables.ver_values()[:62], v0)
    np.testing.assert_array_equal(ses.tables.sla_values()[:62], s0)
    assert np.all(ses.tables.ver_values()[62:] == 0.0)
    assert np.all(ses.tables.sla_values()[62:] == 0.0)


def test_exhaustive_fallback_matches_oracles(lfps):
    from paper_2506_15704_b200.lfps.bench import _snapshot, exact_topk_step
    rng = np.random.default_rng(6)
    ses, cfg = build_session(lfps, rng, n=128, exhaustive_fallback=True, epsilon=1.0)
    for _ in range(20):
        q, nk, nv = random_step(rng, 16)
        n_before = ses.store.n
        res = lfps.decode_step(ses, q, nk, nv, 0.05, cfg)
        assert not res.bypassed
        ref = _snapshot(ses.store, n_before)
        k = max(1, round(0.05 * n_before))
        want = lfps.topk_oracle(q, ref, k, cfg.sink_count)
        np.testing.assert_array_equal(res.candidate.c2, want)
        sel, out = exact_topk_step(q, ref, k, cfg.sink_count)
        np.testing.assert_array_equal(sel, want)
        np.testing.assert_allclose(res.output, out.output, rtol=1e-12)
        assert res.candidate.probe.size == n_before - cfg.sink_count
        # host restatement of topk_oracle (attention.py:100-113)
        keys = ref.keys
        z = keys[cfg.sink_count:] @ q / math.sqrt(16)
        idx = np.arange(cfg.sink_count, n_before)
        np.testing.assert_array_equal(want, np.sort(idx[np.lexsort((idx, -z))[:k]]))


def test_validation_leaves_state_unchanged_and_run_session_errors(lfps):
    rng = np.random.default_rng(8)
    ses, cfg = build_session(lfps, rng, n=256)
    for _ in range(20):
        res = lfps.decode_step(ses, *random_step(rng, 16), 0.02, cfg)
        if not res.bypassed:
            assert res.dot_products == (res.candidate.probe.size + cfg.local_window
                                        + cfg.sink_count + 1)
    n0 = ses.store.n
    v0 = ses.tables.ver_values()
    with pytest.raises(ValueError):
        lfps.decode_step(ses, np.ones(5), np.ones(16), np.ones(16), 0.05, cfg)
    with pytest.raises(ValueError):
        lfps.decode_step(ses, np.ones(16), np.ones(16), np.ones(16), 0.0, cfg)
    assert ses.store.n == n0
    np.testing.assert_array_equal(ses.tables.ver_values(), v0)
    steps = [random_step(rng, 16) for _ in range(150)]    # past the store's capacity
    res = lfps.run_session(ses, steps, 0.05, cfg)
    assert len(res) == 150 and ses.store.n == n0 + 150 and ses.tables.m == n0 + 150 - 2
    bad = [random_step(rng, 16) for _ in range(2)] + [(np.ones(3), np.ones(16), np.ones(16))]
    with pytest.raises(lfps.SessionRunError) as exc:
        lfps.run_session(ses, bad, 0.05, cfg)
    assert exc.value.step == 2 and len(exc.value.results) == 2


def _np_thresholds(ver, sla, a):
    out = []
    for x in (ver, sla):
        mean = float(x.mean())
        c = (x - mean) ** 2
        s2, s4 = float(c.sum()), float(np.dot(c, c))
        if s2 < 1e-12:
            out.append((float("nan"), mean, True))
        else:
            out.append((a * mean / (s4 / (s2 * s2)), mean, False))
    return out


def test_stage_functions_against_reference_expressions(lfps):
    """select_initial / expand / finalize_probe_set / compute_thresholds on
    the device against numpy restatements of candidates.py:45-100 and
    tables.py:295-331 (the oracles of the reference's test_candidates.py)."""
    rng = np.random.default_rng(0)
    cfg = lfps.LfpsConfig(d=4, s=1, sink_count=1, a=0.2)
    for trial in range(30):
        m = int(rng.integers(5, 3000))
        ver, sla = rng.random(m), rng.random(m)
        t = lfps.ScoreTablePair(ver, sla, 1)
        th = lfps.compute_thresholds(t, cfg)
        want = _np_thresholds(ver, sla, 0.2)
        assert th.tau_ver == pytest.approx(want[0][0], rel=1e-9)
        assert th.mean_sla == pytest.approx(want[1][1], rel=1e-12)
        from paper_2506_15704_b200.lfps.tables import thresholds_oracle
        orc = thresholds_oracle(t, cfg)
        assert orc.tau_ver == pytest.approx(th.tau_ver, rel=1e-9)
        c0 = lfps.select_initial(t, th)
        want0 = np.nonzero((ver > th.tau_ver) | (sla > th.tau_sla))[0] + 1
        np.testing.assert_array_equal(c0, want0)
        c1 = lfps.expand(c0, t, th, cfg)
        offs = cfg.expansion_offsets
        want1 = sorted({j + 1 for i in (c0 - 1) for dj in offs for j in [i + dj]
                        if 0 <= j < m and (ver[j] > th.mean_ver or sla[j] > th.mean_sla)})
        np.testing.assert_array_equal(c1, want1)
        store = lfps.KvStore.from_matrices(np.ones((m + 1, 4)), np.ones((m + 1, 4)))
        probe = lfps.finalize_probe_set(c1, store, cfg)
        tail = np.arange(max(1, m + 1 - cfg.local_window), m + 1)
        np.testing.assert_array_equal(probe, np.union1d(np.asarray(c1, dtype=np.int64), tail))
    # the reference's unit fixtures (test_candidates.py:23-101)
    t = lfps.ScoreTablePair([0.9, 0.1, 0.1], [0.3, 0.3, 0.3], 1)
    th = lfps.ThresholdPair(0.5, float("nan"), 0.37, 0.3, sla_degenerate=True)
    np.testing.assert_array_equal(lfps.select_initial(t, th), [1])
    ver = np.array([0.9, 0.05, 0.9, 0.9])
    t = lfps.ScoreTablePair(ver, ver, 1)
    th = lfps.ThresholdPair(0.0, 0.0, 0.5, 0.5)
    np.testing.assert_array_equal(lfps.expand(np.array([2]), t, th, cfg), [1, 3, 4])


def test_topk_and_attention_stages(lfps):
    """topk_from_scores with planted ties (attention.py:34-47, lower index
    wins, -0.0 == +0.0), exact_topk_restricted, attention_output and
    full_attention_oracle against numpy."""
    rng = np.random.default_rng(3)
    for p, k in ((50, 7), (3000, 150), (20000, 1000), (10, 10), (10, 30)):
        idx = np.sort(rng.choice(100000, size=p, replace=False)).astype(np.int64)
        sc = np.round(rng.standard_normal(p), 1)          # many exact ties
        sc[:3] = [0.0, -0.0, 0.0]
        got = lfps.topk_from_scores(idx, sc, k)
        order = np.lexsort((idx, -(sc + 0.0)))
        np.testing.assert_array_equal(got, np.sort(idx[order[: min(k, p)]]))
    n, d = 500, 24
    keys, values = rng.standard_normal((n, d)), rng.standard_normal((n, d))
    store = lfps.KvStore.from_matrices(keys, values)
    q = rng.standard_normal(d)
    probe = np.sort(rng.choice(np.arange(4, n), 120, replace=False))
    cnt = lfps.DotCounter()
    got = lfps.exact_topk_restricted(q, store, probe, 17, cnt)
    z = keys[probe] @ q / math.sqrt(d)
    np.testing.assert_array_equal(got, np.sort(probe[np.lexsort((probe, -z))[:17]]))
    assert cnt.count == 120
    att = lfps.attention_output(q, store, got, 4)
    idx = np.union1d(np.arange(4), got)
    lg = keys[idx] @ q / math.sqrt(d)
    w = np.exp(lg - lg.max())
    w /= w.sum()
    np.testing.assert_array_equal(att.indices, idx)
    np.testing.assert_allclose(att.weights, w, rtol=1e-12)
    np.testing.assert_allclose(att.output, w @ values[idx], rtol=1e-11, atol=1e-14)
    full = lfps.full_attention_oracle(q, store)
    lg = keys @ q / math.sqrt(d)
    w = np.exp(lg - lg.max())
    w /= w.sum()
    np.testing.assert_allclose(full.output, w @ values, rtol=1e-11, atol=1e-14)
    rep = lfps.overlap_ratio(got, got, got.size)
    assert (rep.eta, rep.k, rep.intersection) == (1.0, 17, 17)
    assert lfps.output_error(att, att) == 0.0


def test_tables_update_grow_and_seed_against_naive_mirror(lfps):
    """ScoreTablePair.update / grow on the device against an eager numpy
    mirror (the reference's NaiveTables, test_tables.py:19-45), through a
    renormalisation (r = 0.5 -> scale < 1e-120 after 399 updates), and
    init_tables bit-exact against the reference's seeding order."""
    from oracle import lfps_oracle as lo
    rng = np.random.default_rng(7)
    cfg = lfps.LfpsConfig(d=4, s=3, sink_count=1, r=0.5)
    m0 = 40
    w = rng.random((3, m0))
    w /= w.sum(axis=1, keepdims=True)
    t = lfps.init_tables(w, cfg)
    seed = lo.seed_tables(w, cfg)
    np.testing.assert_array_equal(t.ver_values(), seed.ver_view())
    np.testing.assert_array_equal(t.sla_values(), seed.sla_view())
    ver, sla = t.ver_values(), t.sla_values()
    clamps = 0
    for step in range(450):
        m = t.m
        k = int(rng.integers(1, min(m, 12) + 1))
        sel = np.sort(rng.choice(m, k, replace=False))
        u = rng.random(k) + 0.01
        u /= u.sum()
        got = t.update(sel, u, cfg.r)
        # eager mirror of tables.py:144-200 on values
        ver = ver * 0.5
        sla = np.concatenate([[0.0], sla * 0.5])
        add = u - 1.0 / (2.0 * k)
        ver[sel] += add
        sla[sel] += add
        neg = int((ver[sel] < 0).sum() + (sla[sel] < 0).sum())
        ver[sel] = np.maximum(ver[sel], 0.0)
        sla[sel] = np.maximum(sla[sel], 0.0)
        assert got == neg
        clamps += neg
        t.grow()
        ver = np.concatenate([ver, [0.0]])       # sla's top is the parked carry
        if step % 50 == 0 or step in (397, 398, 399, 449):
            np.testing.assert_allclose(t.ver_values(), ver, rtol=1e-9, atol=1e-12)
            np.testing.assert_allclose(t.sla_values(), sla, rtol=1e-9, atol=1e-12)
    assert t.clamp_count == clamps
    assert t.scale > 1e-120           # renormalised on the way
