"""The oracle at survey scale (CPU): pinned against the reference's own
outputs at 16k (the C1 shape, tests/golden/seeded/) and the two arithmetic
modes against each other at 128k (the C4 context).

The GPU tests at these sizes (tests/test_gpu_scale.py) compare the device
with DevArith; these tests are why DevArith is trusted there: it selects the
reference's sets step for step.
"""

import numpy as np
import pytest

from golden_io import load_seeded, seeded_names
from oracle import lfps_oracle as lo
from paper_2506_15704_b200.config import LfpsConfig


def run_seeded(g, arith, score):
    """The oracle over a seeded golden; records in the fixture's order
    (step, KV head, q-head)."""
    cfg = LfpsConfig(d=g.spec.d, **g.cfg)
    n0, T, Hkv = g.spec.n_prefill, g.spec.steps, g.spec.kv_heads
    units = [lo.bootstrap_unit(g.K[h, :n0], g.V[h, :n0], g.W[h], g.F[h], cfg, arith)
             for h in range(Hkv)]
    recs = []
    for t in range(T):
        for h, (kv, trs, prs) in enumerate(units):
            recs += lo.unit_step(kv, trs, prs, g.Q[h, :, t], g.K[h, n0 + t], g.V[h, n0 + t],
                                 float(g.fracs[t]), cfg, arith, score)
    return recs, units


def _check(g, recs):
    for key in ("c0", "c1", "probe", "c2"):
        want = g.sets(key)
        assert len(want) == len(recs)
        for i, (o, w) in enumerate(zip(recs, want)):
            np.testing.assert_array_equal(getattr(o, key), w, err_msg=f"{key} record {i}")
    for key, attr in (("bypassed", "bypassed"), ("budget_k", "budget_k"), ("clamps", "clamps"),
                      ("dots", "dot_products"), ("c0_dropped", "c0_dropped")):
        np.testing.assert_array_equal([getattr(o, attr) for o in recs], g.raw[key], err_msg=key)


@pytest.mark.parametrize("name", seeded_names())
def test_seeded_reference_arithmetic_reproduces_reference(name):
    g = load_seeded(name)
    recs, units = run_seeded(g, lo.RefArith, "fp64")
    _check(g, recs)
    np.testing.assert_allclose([o.rho for o in recs], g.raw["rho"], rtol=1e-12, atol=0)
    np.testing.assert_allclose(np.stack([o.output for o in recs]), g.raw["outputs"],
                               rtol=1e-10, atol=1e-12)
    trs = [tr for _, t, _ in units for tr in t]
    np.testing.assert_allclose([tr.values()[0].sum() for tr in trs], g.raw["final_ver_sum"],
                               rtol=1e-12)
    np.testing.assert_array_equal([tr.clamp_count for tr in trs], g.raw["final_clamps"])


@pytest.mark.parametrize("name", seeded_names())
def test_seeded_device_arithmetic_selects_reference_sets(name):
    g = load_seeded(name)
    recs, units = run_seeded(g, lo.DevArith, "fp32")
    _check(g, recs)
    np.testing.assert_allclose([o.rho for o in recs], g.raw["rho"], rtol=1e-12)
    got = np.stack([o.output for o in recs])
    ref = g.raw["outputs"]
    err = np.linalg.norm(got - ref, axis=1) / np.linalg.norm(ref, axis=1)
    assert err.max() <= 1e-5, err.max()
    trs = [tr for _, t, _ in units for tr in t]
    np.testing.assert_allclose([tr.values()[1].sum() for tr in trs], g.raw["final_sla_sum"],
                               rtol=1e-6)


def test_device_and_reference_arithmetic_agree_at_128k():
    """C4 context: one unit (G = 4 sessions) at n0 = 131072, 6 steps at 5%
    and 1%: the canonical device arithmetic (fp32 scores) and the
    reference's numpy arithmetic (fp64 scores) select identical C0, C1,
    probe and C2 sets on every session-step; the 257-segment merge tree
    changes no threshold decision."""
    import torch
    from paper_2506_15704_b200.workload import GqaSpec, gen_unit
    n0, T = 131072, 6
    spec = GqaSpec(batch=1, kv_heads=1, group=4, d=128, n_prefill=n0, steps=T, seed=5,
                   slash_offsets=(300, 301), band_width=201)
    u = gen_unit(spec, 0, 0, device="cpu")
    K, V = u.keys.float().numpy(), u.values.float().numpy()
    W, F, Q = u.weights.numpy(), u.final_query.float().numpy(), u.queries.float().numpy()
    cfg = LfpsConfig(d=128)
    runs = []
    for arith, score in ((lo.RefArith, "fp64"), (lo.DevArith, "fp32")):
        kv, trs, prs = lo.bootstrap_unit(K[:n0], V[:n0], W, F, cfg, arith)
        steps = []
        for t in range(T):
            steps.append(lo.unit_step(kv, trs, prs, Q[:, t], K[n0 + t], V[n0 + t],
                                      0.05 if t % 2 == 0 else 0.01, cfg, arith, score))
        runs.append(steps)
    del torch
    nonempty = 0
    for t in range(T):
        for g in range(4):
            a, b = runs[0][t][g], runs[1][t][g]
            assert a.bypassed == b.bypassed
            for key in ("c0", "c1", "probe", "c2"):
                np.testing.assert_array_equal(getattr(a, key), getattr(b, key),
                                              err_msg=f"step {t} head {g} {key}")
            nonempty += a.c0.size > 0
    assert nonempty > 0
