"""Reference-generated golden outputs at survey scale, with seeded inputs.

Run in the build container only (it imports /root/reference/pkg/src, which
does not exist on the GPU box):

    OPENBLAS_NUM_THREADS=1 python tests/golden/make_golden_seeded.py [name ...]

At 16k context the inputs of a C1-shaped case (8 KV heads x 4 q-heads) are
~50 MB, too large to commit.  So the inputs are NOT stored: they are
regenerated from the workload spec (paper_2506_15704_b200/workload.py
gen_unit on the CPU, a fixed torch.Generator seed per unit) and the fixture
keeps a SHA-256 of them; a test whose regenerated inputs hash differently
fails loudly instead of comparing against the wrong trajectory.  The
fixture stores what the reference's own prefill_bootstrap / decode_step
produced for them (engine.py:67-201): every step's C0 / C1 / probe / C2 set,
bypass, rho, budget, clamps, dot count and output, plus the final tables'
sums (one reference session per q-head: the reference has no GQA,
SPEC.md:8).
"""

from __future__ import annotations

import hashlib
import os
import sys

import numpy as np

REF_SRC = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))
OUT_DIR = os.path.join(HERE, "seeded")
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

CASES = {
    # BASELINE config 1: batch 1 x 16k context, Llama-3.1-8B shapes (8 KV heads
    # x 4 q-heads, d=128), Top-k 5% (and 1% on odd steps: k < |probe| there)
    "c1_16k": dict(spec=dict(batch=1, kv_heads=8, group=4, d=128, n_prefill=16384, steps=6,
                             seed=16, slash_offsets=(300, 301), band_width=25),
                   fracs=(0.05, 0.01, 0.05, 0.01, 0.05, 0.01), cfg=dict()),
}


def case_inputs(case):
    """Per-unit inputs regenerated from the spec (CPU), as float32 arrays of
    bf16 values: keys/values [Hkv, n0 + T, d], weights [Hkv, G, s, m0],
    finals [Hkv, G, d], queries [Hkv, G, T, d]; and their SHA-256."""
    import torch
    from paper_2506_15704_b200.workload import GqaSpec, gen_unit
    threads = torch.get_num_threads()
    torch.set_num_threads(1)                   # one reduction order for the weights
    spec = GqaSpec(**case["spec"])
    K, V, W, F, Q = [], [], [], [], []
    h = hashlib.sha256()
    for kv in range(spec.kv_heads):
        u = gen_unit(spec, 0, kv, device="cpu")
        for t in (u.keys, u.values, u.final_query, u.queries):
            h.update(t.contiguous().view(torch.int16).numpy().tobytes())
        h.update(u.weights.contiguous().numpy().tobytes())
        K.append(u.keys.float().numpy())
        V.append(u.values.float().numpy())
        W.append(u.weights.numpy())
        F.append(u.final_query.float().numpy())
        Q.append(u.queries.float().numpy())
    torch.set_num_threads(threads)
    return spec, (np.stack(K), np.stack(V), np.stack(W), np.stack(F), np.stack(Q)), h.hexdigest()


def run_case(name, case):
    sys.path.insert(0, REF_SRC)
    import lfps  # the reference package
    spec, (K, V, W, F, Q), digest = case_inputs(case)
    n0, T, d, G, Hkv = spec.n_prefill, spec.steps, spec.d, spec.group, spec.kv_heads
    cfg = lfps.LfpsConfig(d=d, **case["cfg"])
    sessions = [[lfps.prefill_bootstrap(K[h, :n0], V[h, :n0], W[h, g], F[h, g], cfg)
                 for g in range(G)] for h in range(Hkv)]
    rec = {k: [] for k in ("bypassed", "rho", "budget_k", "clamps", "dots", "c0_dropped")}
    sets = {k: [] for k in ("c0", "c1", "probe", "c2")}
    outputs = []
    for t in range(T):                      # record order: step, KV head, q-head
        for h in range(Hkv):
            for g in range(G):
                res = lfps.decode_step(sessions[h][g], Q[h, g, t], K[h, n0 + t], V[h, n0 + t],
                                       case["fracs"][t], cfg)
                rec["bypassed"].append(res.bypassed)
                rec["rho"].append(res.rho)
                rec["budget_k"].append(res.candidate.budget_k)
                rec["clamps"].append(res.clamp_count)
                rec["dots"].append(res.dot_products)
                rec["c0_dropped"].append(res.c0_dropped)
                for k in sets:
                    sets[k].append(np.asarray(getattr(res.candidate, k), dtype=np.int64))
                outputs.append(res.output)
    flat = [s for row in sessions for s in row]
    out = dict(
        spec=np.array(repr(case["spec"])), cfg_json=np.array(repr(case["cfg"])),
        fracs=np.asarray(case["fracs"], dtype=np.float64), sha256=np.array(digest),
        outputs=np.stack(outputs),
        final_ver_sum=np.array([s.tables.ver_values().sum() for s in flat]),
        final_sla_sum=np.array([s.tables.sla_values().sum() for s in flat]),
        final_clamps=np.array([s.tables.clamp_count for s in flat]),
    )
    for k, v in rec.items():
        out[k] = np.array(v)
    for k, lists in sets.items():
        out[k + "_len"] = np.array([a.size for a in lists], dtype=np.int64)
        out[k + "_cat"] = np.concatenate(lists).astype(np.int32)
    os.makedirs(OUT_DIR, exist_ok=True)
    path = os.path.join(OUT_DIR, f"{name}.npz")
    np.savez_compressed(path, **out)
    print(f"{name}: {T} steps x {Hkv * G} sessions at n0={n0}, bypass rate "
          f"{np.mean(rec['bypassed']):.2f}, mean |probe| {np.mean(out['probe_len']):.1f}, "
          f"mean |c2| {np.mean(out['c2_len']):.1f} -> {os.path.getsize(path) / 1e3:.0f} kB")


if __name__ == "__main__":
    for nm in sys.argv[1:] or list(CASES):
        run_case(nm, CASES[nm])
