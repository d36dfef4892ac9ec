"""Generate golden vectors by running the reference package itself.

Run in the build container only (it imports /root/reference/pkg/src, which
does not exist on the GPU box):

    OPENBLAS_NUM_THREADS=1 python tests/golden/make_golden.py

For every case it builds bf16-representable inputs, runs the reference's own
prefill_bootstrap / decode_step once per q-head (the reference has no GQA, so
the G q-heads of a unit are G independent reference sessions over identical
K/V rows), and records every observable of every step plus the
final tables.  The committed ``*.npz`` files are what tests/ compare against;
this script is kept so they can be regenerated.
"""

from __future__ import annotations

import os
import sys

import numpy as np

REF_SRC = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))


def bf16_bits(x: np.ndarray) -> np.ndarray:
    return (np.ascontiguousarray(x, dtype=np.float32).view(np.uint32) >> 16).astype(np.uint16)


CASES = {
    # planted vertical bands + slash offsets; Top-k 2% so |probe| > k occurs
    "planted": dict(spec=dict(n_prefill=1100, steps=40, d=64, group=2, seed=42,
                              slash_offsets=(48, 49), band_width=6),
                    frac=0.02, cfg=dict()),
    # 5% budget: C2 == probe pass-through regime of the survey configs
    "planted5": dict(spec=dict(n_prefill=900, steps=30, d=128, group=2, seed=7,
                               slash_offsets=(40, 41), band_width=5),
                     frac=0.05, cfg=dict()),
    # sink-dominated queries: the gate bypasses some steps
    "gated": dict(spec=dict(n_prefill=400, steps=30, d=64, group=2, seed=11,
                            signal_gain=0.0, sink_gain=14.0, query_correlation=0.9),
                  frac=0.05, cfg=dict(epsilon=0.85)),
    "gated_mean_only": dict(spec=dict(n_prefill=400, steps=20, d=64, group=2, seed=12,
                                      signal_gain=0.0, sink_gain=14.0,
                                      query_correlation=0.9),
                            frac=0.05, cfg=dict(epsilon=0.85, bypass_mode="mean_only")),
    # oracle-equivalence mode with planted exact ties (test_acceptance.py:94-144)
    "exhaustive_ties": dict(spec=dict(n_prefill=300, steps=12, d=64, group=2, seed=3,
                                      signal_gain=0.0, noise_scale=1.0,
                                      query_correlation=0.5),
                            frac=0.03, cfg=dict(exhaustive_fallback=True, epsilon=1.0),
                            ties=True),
    # fast decay: the lazy scale crosses 1e-120 and renormalises (tables.py:240).
    # Exhaustive mode, because the reference's moments overflow (kappa -> 0,
    # ZeroDivisionError at tables.py:315) long before the scale reaches 1e-120.
    "renorm": dict(spec=dict(n_prefill=160, steps=420, d=32, group=1, seed=5,
                             slash_offsets=(20, 21), band_width=2, band_fracs=(0.4,),
                             signal_gain=4.0, query_correlation=0.99),
                   frac=0.1, cfg=dict(r=0.5, epsilon=1.0, exhaustive_fallback=True)),
    # wide expansion offsets
    "wide_offsets": dict(spec=dict(n_prefill=700, steps=20, d=64, group=2, seed=19,
                                   slash_offsets=(30, 31), band_width=4, plant_jitter=3),
                         frac=0.02, cfg=dict(expansion_offsets=(-3, -2, -1, 0, 1, 2, 3),
                                             a=0.3)),
}


def build_inputs(case):
    """Unit inputs from the GQA workload recipe, bf16-representable."""
    import torch
    from paper_2506_15704_b200.workload import GqaSpec, gen_unit
    spec = GqaSpec(batch=1, kv_heads=1, **case["spec"])
    u = gen_unit(spec, 0, 0, device="cpu")
    keys = u.keys.float().numpy()
    values = u.values.float().numpy()
    if case.get("ties"):
        n0 = spec.n_prefill
        keys[n0 // 2: n0] = keys[: n0 - n0 // 2]
        from paper_2506_15704_b200.workload import prefill_weights
        pq = torch.stack([u.final_query] * spec.s, dim=1)
        u.weights = prefill_weights(torch.from_numpy(keys[:n0]).to(torch.bfloat16), pq,
                                    spec.sink_count)
    queries = u.queries.float().numpy().transpose(1, 0, 2)      # [steps, G, d]
    return (spec, keys, values, u.weights.numpy(), u.final_query.float().numpy(),
            np.ascontiguousarray(queries))


def run_case(name, case):
    sys.path.insert(0, REF_SRC)
    import lfps  # the reference package
    spec, keys, values, weights, finals, queries = build_inputs(case)
    n0, steps, d, G = spec.n_prefill, spec.steps, spec.d, spec.group
    cfg = lfps.LfpsConfig(d=d, **case["cfg"])
    sessions = [lfps.prefill_bootstrap(keys[:n0], values[:n0], weights[g], finals[g], cfg)
                for g in range(G)]
    rec = {k: [] for k in ("bypassed", "rho", "budget_k", "clamps", "dots", "c0_dropped")}
    sets = {k: [] for k in ("c0", "c1", "probe", "c2")}
    outputs = []
    init_tables = [np.stack([s.tables.ver_values() for s in sessions]),
                   np.stack([s.tables.sla_values() for s in sessions])]
    stats = dict(mean_key=np.stack([s.stats.mean_key for s in sessions]),
                 mean_value=np.stack([s.stats.mean_value for s in sessions]),
                 sigma_hat_sq=np.array([s.stats.sigma_hat_sq for s in sessions]))
    for t in range(steps):
        for g in range(G):
            res = lfps.decode_step(sessions[g], queries[t, g], keys[n0 + t], values[n0 + t],
                                   case["frac"], cfg)
            rec["bypassed"].append(res.bypassed)
            rec["rho"].append(res.rho)
            rec["budget_k"].append(res.candidate.budget_k)
            rec["clamps"].append(res.clamp_count)
            rec["dots"].append(res.dot_products)
            rec["c0_dropped"].append(res.c0_dropped)
            for k in sets:
                sets[k].append(np.asarray(getattr(res.candidate, k), dtype=np.int64))
            outputs.append(res.output)
    out = dict(
        keys=bf16_bits(keys), values=bf16_bits(values), weights=weights,
        finals=bf16_bits(finals), queries=bf16_bits(queries),
        meta=np.array([n0, steps, d, G, spec.sink_count, spec.s], dtype=np.int64),
        frac=np.float64(case["frac"]),
        cfg_json=np.array(repr(case["cfg"])),
        init_ver=init_tables[0], init_sla=init_tables[1],
        final_ver=np.stack([s.tables.ver_values() for s in sessions]),
        final_sla=np.stack([s.tables.sla_values() for s in sessions]),
        final_clamps=np.array([s.tables.clamp_count for s in sessions]),
        outputs=np.stack(outputs), **stats,
    )
    for k, v in rec.items():
        out[k] = np.array(v)
    for k, lists in sets.items():
        out[k + "_len"] = np.array([a.size for a in lists], dtype=np.int64)
        out[k + "_cat"] = np.concatenate(lists) if lists else np.empty(0, np.int64)
    path = os.path.join(HERE, f"{name}.npz")
    np.savez_compressed(path, **out)
    byp = np.mean(rec["bypassed"])
    print(f"{name}: {steps} steps x {G} heads, bypass rate {byp:.2f}, "
          f"mean |probe| {np.mean(out['probe_len']):.1f}, "
          f"mean |c2| {np.mean(out['c2_len']):.1f} -> {os.path.getsize(path) / 1e3:.0f} kB")


if __name__ == "__main__":
    names = sys.argv[1:] or list(CASES)
    for nm in names:
        run_case(nm, CASES[nm])
