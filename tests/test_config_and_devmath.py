"""Host logic: LfpsConfig validation (config.py:44-66), the canonical
device arithmetic of oracle/devmath.py, and the GQA workload generator."""

import math

import numpy as np
import pytest

from oracle import devmath as dm
from paper_2506_15704_b200.config import LfpsConfig


class TestConfig:
    def test_defaults(self):
        c = LfpsConfig(d=64)
        assert (c.s, c.r, c.epsilon, c.a, c.sink_count, c.local_window) == (32, 0.95, 0.85, 0.2, 4, 6)
        assert c.expansion_offsets == (-1, 0, 1, 2)
        assert c.device_limits_error() is None

    @pytest.mark.parametrize("kw", [
        {"d": 0}, {"d": 8, "r": 1.0}, {"d": 8, "r": -0.1}, {"d": 8, "epsilon": 0.0},
        {"d": 8, "epsilon": 1.5}, {"d": 8, "a": 0.0}, {"d": 8, "s": 0},
        {"d": 8, "sink_count": 0}, {"d": 8, "local_window": 0},
        {"d": 8, "expansion_offsets": (1, 2)}, {"d": 8, "tie_break": "coin_flip"},
        {"d": 8, "bypass_mode": "nope"},
    ])
    def test_invalid_rejected(self, kw):
        with pytest.raises(ValueError):
            LfpsConfig(**kw)

    def test_device_limits(self):
        assert LfpsConfig(d=48).device_limits_error()
        assert LfpsConfig(d=64, expansion_offsets=(0, 40)).device_limits_error()
        assert LfpsConfig(d=64, sink_count=40).device_limits_error()


class TestDevmath:
    def test_cexp_within_one_ulp(self):
        x = -np.random.default_rng(0).random(200000) * 700
        got, want = dm.cexp(x), np.exp(x)
        assert (np.abs(got - want) / np.spacing(want)).max() <= 1.0
        assert dm.cexp(np.array([-709.0]))[0] == 0.0 and dm.cexp(np.array([0.0]))[0] == 1.0

    @pytest.mark.parametrize("n", [1, 7, 511, 512, 513, 5000, 70000])
    def test_table_moments_match_two_pass(self, n):
        x = np.random.default_rng(n).random(n) * np.exp(np.random.default_rng(n + 1).normal(0, 3, n))
        mean = x.mean()
        c2 = (x - mean) ** 2
        got = dm.table_moments(x)
        want = (mean, c2.sum(), np.dot(c2, c2))
        for g, w in zip(got, want):
            assert g == pytest.approx(w, rel=1e-13, abs=1e-300)

    def test_merge_with_empty_is_identity(self):
        a = (np.float64(512.0), np.float64(0.3), np.float64(2.0), np.float64(-0.1), np.float64(5.0))
        z = tuple(np.float64(0.0) for _ in range(5))
        assert all(x == y for x, y in zip(dm.merge_moments(a, z), a))
        assert all(x == y for x, y in zip(dm.merge_moments(z, a), a))

    def test_chunk_moments_exact_on_constant_chunk(self):
        cnt, mu, m2, m3, m4 = dm.chunk_moments(np.full(1024, 0.25))
        assert np.all(mu == 0.25) and np.all(m2 == 0.0) and np.all(m4 == 0.0)

    def test_block_and_table_sums_are_exact_reductions(self):
        x = np.random.default_rng(3).random(4097)
        assert dm.block_sum(x) == pytest.approx(math.fsum(x), rel=1e-14)
        assert dm.table_sum(x) == pytest.approx(math.fsum(x), rel=1e-14)

    def test_gdot_and_sdot(self):
        rng = np.random.default_rng(5)
        a = rng.standard_normal((9, 128))
        q = rng.standard_normal(128)
        np.testing.assert_allclose(dm.gdot(a, q), a @ q, rtol=1e-12)
        kb = a.astype(np.float32)
        z = dm.sdot32(kb, q.astype(np.float32), dm.rsd_f32(128))
        np.testing.assert_allclose(z, (kb.astype(np.float64) @ q.astype(np.float32)) / math.sqrt(128),
                                   rtol=1e-5, atol=1e-6)

    def test_axis0_sum_is_sequential(self):
        x = np.random.default_rng(2).standard_normal((3000, 64))
        seq = np.zeros(64)
        for row in x:
            seq = seq + row
        np.testing.assert_array_equal(dm.stats_sum_rows(x), seq)


class TestWorkload:
    def test_gqa_unit_shapes_and_weights(self):
        from paper_2506_15704_b200.workload import GqaSpec, gen_unit
        spec = GqaSpec(batch=1, kv_heads=1, group=4, d=64, n_prefill=600, steps=5, seed=3,
                       slash_offsets=(40, 41), band_width=3)
        u = gen_unit(spec, 0, 0)
        assert u.keys.shape == (605, 64) and u.queries.shape == (4, 5, 64)
        w = u.weights.double()
        assert w.shape == (4, 32, 596)
        np.testing.assert_allclose(w.sum(-1).numpy(), 1.0, atol=1e-5)
        # causal: the oldest of the trailing s queries sees rows [0, n0 - s]
        assert float(w[0, 0, 600 - 32 - 4 + 1:].abs().max()) == 0.0

    def test_deterministic(self):
        from paper_2506_15704_b200.workload import GqaSpec, gen_unit
        spec = GqaSpec(batch=2, kv_heads=2, group=2, d=64, n_prefill=300, steps=2, seed=9,
                       slash_offsets=(20, 21), band_width=2)
        a, b = gen_unit(spec, 1, 1), gen_unit(spec, 1, 1)
        assert bool((a.keys == b.keys).all()) and bool((a.queries == b.queries).all())
