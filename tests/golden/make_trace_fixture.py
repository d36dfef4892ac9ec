"""Generate the trace / report fixtures by running the reference itself.

Run in the build container only (imports /root/reference/pkg/src):

    OPENBLAS_NUM_THREADS=1 python tests/golden/make_trace_fixture.py

* ``small.lfps``: a 1-layer x 3-head trace from the reference generator
  (gen_synthetic, planted verticals + slashes, one sink-dominated head so the
  gate bypasses some steps), every value rounded to bf16 so the device path
  (bf16 KV cache) sees exactly the reference's numbers, written by the
  reference's own writer;
* ``small_report.json``: the reference's ``run_trace`` on that trace (lfps
  mode, 5% budget, oracle scoring), canonical JSON from its own emitter.
"""

from __future__ import annotations

import os
import sys

import numpy as np

REF_SRC = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))


def bf16(x):
    import torch
    return torch.as_tensor(np.asarray(x, dtype=np.float32)).to(torch.bfloat16).float().numpy()


def main():
    sys.path.insert(0, REF_SRC)
    from lfps import bench, report, synth, tracefile
    spec = synth.SyntheticSpec(n_prefill=600, steps=12, d=32, vertical_positions=(90, 300, 470),
                               slash_offsets=(40, 41), signal_gain=5.0, noise_scale=0.5, seed=7,
                               layers=1, heads=3, plant_band_width=3, plant_jitter=1,
                               sink_gain=0.0, query_correlation=0.99)
    tr = synth.gen_synthetic(spec)
    heads = []
    for h in tr.heads_data:
        w = np.asarray(h.prefill_weights, dtype=np.float64)
        w = w / w.sum(axis=1, keepdims=True)
        heads.append(tracefile.HeadTrace(
            prefill_keys=bf16(h.prefill_keys), prefill_values=bf16(h.prefill_values),
            prefill_weights=w.astype(np.float32), final_query=bf16(h.final_query),
            step_queries=bf16(h.step_queries), step_keys=bf16(h.step_keys),
            step_values=bf16(h.step_values)))
    tr = tracefile.TraceFile(layers=tr.layers, heads=tr.heads, d=tr.d, n_prefill=tr.n_prefill,
                             steps=tr.steps, s=tr.s, sink_count=tr.sink_count, heads_data=heads)
    path = os.path.join(HERE, "small.lfps")
    tracefile.save_trace(tr, path)
    rep = bench.run_trace(tracefile.load_trace(path), mode="lfps", budget=0.05,
                          score_oracle=True, trace_path="small.lfps")
    with open(os.path.join(HERE, "small_report.json"), "wb") as f:
        f.write(report.emit_json(rep))
    print("wrote", path, os.path.getsize(path), "bytes")


if __name__ == "__main__":
    main()
