"""BASELINE.json config 5 on one B200: context x batch x Top-k budget (and
expansion width at one point) -> LFPS us per layer-step, exact full-scan us
per layer-step, recall eta against the exact Top-k, and output error against
full attention.  One JSON line per point.

    python tools/sweep.py [--contexts 8192,32768,131072] [--batches 1,16,64]
                          [--fracs 0.01,0.05,0.1] [--out gpurun_out/sweep.jsonl]

Llama-3.1-8B attention shapes (8 KV heads x 4 q-heads, d = 128), synthetic
planted inputs (paper_2506_15704_b200/workload.py).  Each (context, batch)
session is populated once; every budget then runs warm-up, timed steps and
scoring steps on it (the tables keep evolving between points, as in a long
decode).  Times are device times from CUDA events around single steps.
"""

from __future__ import annotations

import argparse
import dataclasses
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--contexts", default="8192,32768,131072")
    ap.add_argument("--batches", default="1,16,64")
    ap.add_argument("--fracs", default="0.01,0.05,0.1")
    ap.add_argument("--widths", default="0,1,4,7", help="expansion offsets -w..w at the width point")
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--out", default=os.path.join(ROOT, "gpurun_out", "sweep.jsonl"))
    args = ap.parse_args()
    import torch
    from paper_2506_15704_b200.config import LfpsConfig
    from paper_2506_15704_b200.session import CNT_C2, CNT_PROBE, BatchedSession
    from paper_2506_15704_b200.workload import GqaSpec, populate

    dev = torch.device("cuda", 0)
    torch.cuda.set_device(dev)
    contexts = [int(x) for x in args.contexts.split(",")]
    batches = [int(x) for x in args.batches.split(",")]
    fracs = [float(x) for x in args.fracs.split(",")]
    widths = [int(x) for x in args.widths.split(",")]
    os.makedirs(os.path.dirname(args.out), exist_ok=True)
    out = open(args.out, "w")

    def timed(fn):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize(dev)
        return a.elapsed_time(b) * 1e3

    for ctx in contexts:
        for B in batches:
            free = torch.cuda.mem_get_info(dev)[0]
            need = B * 8 * ctx * 128 * 2 * 2 * 1.25 + B * 32 * ctx * 8 * 3.2
            if need > free * 0.9:
                out.write(json.dumps({"context": ctx, "batch": B, "skipped": "does not fit"}) + "\n")
                continue
            points = [(f, None) for f in fracs]
            if ctx == contexts[len(contexts) // 2] and B == batches[len(batches) // 2]:
                points += [(0.05, w) for w in widths]
            T_in = 32
            spec = GqaSpec(batch=B, kv_heads=8, group=4, d=128, n_prefill=ctx, steps=T_in, seed=5)
            cfg0 = LfpsConfig(d=128)
            total_steps = len(points) * (3 + args.steps + 3) + 8
            t0 = time.time()
            sess = BatchedSession(cfg0, B, 8, 4, n_max=ctx + total_steps + 8, device=dev)
            stream = populate(sess, spec)
            setup = time.time() - t0
            t = 0

            def step(frac):
                nonlocal t
                i = t % T_in
                sess.decode_step(stream.q[i], stream.k_new[i], stream.v_new[i], frac)
                t += 1

            for frac, w in points:
                sess.cfg = cfg0 if w is None else dataclasses.replace(
                    cfg0, expansion_offsets=tuple(range(-w, w + 1)))
                for _ in range(3):
                    step(frac)
                torch.cuda.synchronize(dev)
                lf = sorted(timed(lambda: step(frac)) for _ in range(args.steps))
                etas, errs, ex = [], [], []
                for _ in range(3):
                    q = stream.q[t % T_in]
                    full = sess.full_attention(q)
                    ex.append(timed(lambda: sess.exact_topk_step(q, frac)))
                    ex_idx, ex_cnt = sess.c2_idx.clone(), sess.counts.clone()
                    step(frac)
                    keep = sess.bypass.flatten() == 0
                    eta = sess.overlap(sess.c2_idx, sess.counts, ex_idx, ex_cnt).flatten()
                    etas.append(eta[keep])
                    fn = full.double().norm(dim=-1).clamp_min(1e-12)
                    errs.append(((sess.out.double() - full.double()).norm(dim=-1) / fn).flatten())
                sess.check_errors("sweep")
                counts = sess.counts
                rec = {"context": ctx, "batch": B, "topk_fraction": frac,
                       "expansion_offsets": list(sess.cfg.expansion_offsets),
                       "lfps_us_per_layer_step": lf[len(lf) // 2],
                       "exact_us_per_layer_step": sorted(ex)[1],
                       "speedup_vs_exact": sorted(ex)[1] / lf[len(lf) // 2],
                       "eta_mean": float(torch.cat(etas).mean()),
                       "output_error_vs_full_mean": float(torch.cat(errs).mean()),
                       "probe_mean": float(counts[..., CNT_PROBE].float().mean()),
                       "c2_mean": float(counts[..., CNT_C2].float().mean()),
                       "setup_s": setup}
                out.write(json.dumps(rec) + "\n")
                out.flush()
                print(json.dumps(rec), flush=True)
            del sess, stream
            torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
