"""The reference-named per-head API (compat.py) on the device: the
reference's own engine tests (pkg/tests/test_engine.py) restated, plus a
golden trajectory driven through prefill_bootstrap / run_session."""

import numpy as np
import pytest

from golden_io import load
from oracle_run import golden_config

pytestmark = pytest.mark.gpu


def _lfps():
    import paper_2506_15704_b200 as lfps
    return lfps


def bf16(x):
    import torch
    return torch.as_tensor(np.asarray(x, dtype=np.float32)).to(torch.bfloat16).float().numpy()


def build_session(rng, n=64, d=32, s=4, sink=2, window=3, **cfg_kw):
    lfps = _lfps()
    cfg = lfps.LfpsConfig(d=d, s=s, sink_count=sink, local_window=window, **cfg_kw)
    keys = bf16(rng.standard_normal((n, d)))
    values = bf16(rng.standard_normal((n, d)))
    m = n - sink
    w = np.zeros((s, m))
    for c in range(s):
        support = (n - s + c) - sink + 1
        row = rng.random(support) + 1e-3
        w[c, :support] = row / row.sum()
    return lfps.prefill_bootstrap(keys, values, w, bf16(rng.standard_normal(d)), cfg), cfg


def random_step(rng, d):
    return tuple(bf16(rng.standard_normal(d)) for _ in range(3))


def test_golden_through_run_session():
    lfps = _lfps()
    for name in ("planted", "gated"):
        g = load(name)
        cfg = golden_config(g)
        for gi in range(g.G):
            ses = lfps.prefill_bootstrap(g.keys[: g.n0], g.values[: g.n0], g.weights[gi],
                                         g.finals[gi], cfg)
            steps = [(g.queries[t, gi], g.keys[g.n0 + t], g.values[g.n0 + t])
                     for t in range(g.steps)]
            res = lfps.run_session(ses, steps, g.frac)
            for t, r in enumerate(res):
                rec = t * g.G + gi
                assert r.bypassed == bool(g.raw["bypassed"][rec])
                assert r.dot_products == g.raw["dots"][rec]
                for key in ("c0", "c1", "probe", "c2"):
                    np.testing.assert_array_equal(getattr(r.candidate, key), g.sets(key)[rec])
                ref = g.raw["outputs"][rec]
                assert np.linalg.norm(r.output - ref) / np.linalg.norm(ref) <= 1e-5


def test_epsilon_zero_forces_bypass_everywhere():
    lfps = _lfps()
    rng = np.random.default_rng(4)
    ses, cfg = build_session(rng, epsilon=1e-300)
    v0, s0 = ses.tables()
    for _ in range(10):
        res = lfps.decode_step(ses, *random_step(rng, 32), 0.05, cfg)
        assert res.bypassed and res.candidate.c2.size == 0
    assert ses.n == 74
    v1, s1 = ses.tables()
    np.testing.assert_array_equal(v1[:62], v0)
    np.testing.assert_array_equal(s1[:62], s0)
    assert np.all(v1[62:] == 0.0) and np.all(s1[62:] == 0.0)


def test_exhaustive_fallback_matches_exact_topk():
    lfps = _lfps()
    rng = np.random.default_rng(6)
    ses, cfg = build_session(rng, n=128, exhaustive_fallback=True, epsilon=1.0)
    for _ in range(10):
        q, nk, nv = random_step(rng, 32)
        n_before = ses.n
        exact, _ = lfps.exact_topk_step(ses, q, 0.05)
        res = lfps.decode_step(ses, q, nk, nv, 0.05, cfg)
        assert not res.bypassed
        np.testing.assert_array_equal(res.candidate.c2, exact)
        assert res.candidate.probe.size == n_before - cfg.sink_count


def test_work_bound_and_validation_leave_state_unchanged():
    lfps = _lfps()
    rng = np.random.default_rng(8)
    ses, cfg = build_session(rng, n=256)
    for _ in range(5):
        res = lfps.decode_step(ses, *random_step(rng, 32), 0.02, cfg)
        if not res.bypassed:
            assert res.dot_products == (res.candidate.probe.size + cfg.local_window
                                        + cfg.sink_count + 1)
    n0 = ses.n
    v0, _ = ses.tables()
    with pytest.raises(ValueError):
        lfps.decode_step(ses, np.ones(5), np.ones(32), np.ones(32), 0.05, cfg)
    with pytest.raises(ValueError):
        lfps.decode_step(ses, np.ones(32), np.ones(32), np.ones(32), 0.0, cfg)
    assert ses.n == n0
    np.testing.assert_array_equal(ses.tables()[0], v0)


def test_failure_carries_partial_results_and_regrow():
    lfps = _lfps()
    rng = np.random.default_rng(11)
    ses, cfg = build_session(rng, n=64)
    steps = [random_step(rng, 32) for _ in range(300)]   # beyond the initial capacity
    res = lfps.run_session(ses, steps, 0.05, cfg)
    assert len(res) == 300 and ses.n == 364
    bad = [random_step(rng, 32) for _ in range(2)] + [(np.ones(3), np.ones(32), np.ones(32))]
    with pytest.raises(lfps.SessionRunError) as exc:
        lfps.run_session(ses, bad, 0.05, cfg)
    assert exc.value.step == 2 and len(exc.value.results) == 2
