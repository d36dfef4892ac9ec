"""Trace replay on the GPU with reference-schema reports (next-row N3).

``run_trace`` restates bench.run_trace (pkg/src/lfps/bench.py:125-218) on the
device: the trace (tracefile.upload) is ONE batched session whose units are
the trace's (layer, head) pairs, so every decode step of every head is a
single ``lfps_decode_step`` call.  Modes:

* ``"lfps"``        -- the LFPS pipeline; with ``score_oracle`` each step is
  also scored, on the device, against the exact Top-k of the same pre-append
  context (eta, attention.py:116-124) and against full attention
  (output_error, attention.py:88-134);
* ``"topk_oracle"`` -- the exact full-scan path (bench.py:73-80);
* ``"full"``        -- full softmax attention over every row.

Records follow report_schema.md.  Timings are device times (CUDA events) of
the batched step divided evenly over its heads: ``total`` per record, and
``oracle_ns`` for the exact-path scoring step.  Per-stage fields other than
``total`` are 0 (the stages are fused kernels here; per-kernel times come from
``_lib.profile_collect``).
"""

from __future__ import annotations

import torch

from .config import LfpsConfig
from .report import RunReport, StepRecord
from .session import (CNT_C0, CNT_C1, CNT_C2, CNT_CLAMP, CNT_DROP, CNT_K, CNT_PROBE)
from .tracefile import TraceFile, upload

MODES = ("lfps", "topk_oracle", "full")


def config_for_trace(trace: TraceFile, *, r: float = 0.95, epsilon: float = 0.85,
                     a: float = 0.2, local_window: int = 6, expansion_offsets=(-1, 0, 1, 2),
                     bypass_mode: str = "sink_average",
                     exhaustive_fallback: bool = False) -> LfpsConfig:
    """Config whose structural fields (d, s, sink_count) come from the trace
    (bench.py:25-35)."""
    return LfpsConfig(d=trace.d, s=trace.s, r=r, epsilon=epsilon, a=a,
                      expansion_offsets=tuple(expansion_offsets), sink_count=trace.sink_count,
                      local_window=local_window, bypass_mode=bypass_mode,
                      exhaustive_fallback=exhaustive_fallback)


def _timed(fn, dev):
    a = torch.cuda.Event(enable_timing=True)
    b = torch.cuda.Event(enable_timing=True)
    s = torch.cuda.current_stream(dev)
    a.record(s)
    out = fn()
    b.record(s)
    torch.cuda.synchronize(dev)
    return out, int(a.elapsed_time(b) * 1e6)


def _rel_err(out, ref):
    o = out.double()
    r = ref.double()
    return ((o - r).norm(dim=-1) / r.norm(dim=-1).clamp_min(1e-12)).flatten().cpu().tolist()


def run_trace(trace: TraceFile, mode: str = "lfps", budget: float = 0.02,
              config: LfpsConfig | None = None, score_oracle: bool = True,
              snapshot_tables: bool = False, trace_path: str | None = None,
              device=None) -> RunReport:
    """Replay a trace on the GPU and assemble a reference-schema report."""
    if mode not in MODES:
        raise ValueError(f"mode must be one of {MODES}, got {mode!r}")
    if trace.steps < 1:
        raise ValueError("trace has no decode steps")
    if config is None:
        config = config_for_trace(trace)
    if (config.d, config.s, config.sink_count) != (trace.d, trace.s, trace.sink_count):
        raise ValueError("config d / s / sink_count must match the trace")
    dt = upload(trace, config, device)
    sess = dt.session
    dev = sess.device
    U, H, S, L = trace.head_count, trace.heads, config.sink_count, config.local_window
    per_head: list[list[StepRecord]] = [[] for _ in range(U)]
    for t in range(trace.steps):
        n = sess.n_host[0]
        q, kn, vn = dt.q[t], dt.k_new[t], dt.v_new[t]
        full = None
        if score_oracle:
            full = sess.full_attention(q)
        if mode == "lfps":
            exact_idx = exact_cnt = None
            oracle_ns = None
            if score_oracle:
                k = max(1, round(budget * n))
                _, ons = _timed(lambda: sess.exact_topk_step(q, budget), dev)
                exact_idx, exact_cnt = sess.c2_idx.clone(), sess.counts.clone()
                oracle_ns = ons // U
                assert int(exact_cnt[0, 0, CNT_C2]) == min(k, n - S)
            res, ns = _timed(lambda: sess.decode_step(q, kn, vn, budget), dev)
            sess.check_errors(f"trace step {t}")
            counts = res.counts[0].cpu().tolist()
            rho = res.rho[0].cpu().tolist()
            byp = res.bypassed[0].cpu().tolist()
            etas = errs = [None] * U
            if score_oracle:
                etas = sess.overlap(res.c2_idx, res.counts, exact_idx, exact_cnt)[0].cpu().tolist()
                errs = _rel_err(res.output[0], full[0])
            for i in range(U):
                c = counts[i]
                bypassed = bool(byp[i])
                probe = 0 if bypassed else c[CNT_PROBE]
                per_head[i].append(StepRecord(
                    layer=i // H, head=i % H, step=t, n=n, bypassed=bypassed, rho=float(rho[i]),
                    eta=None if (bypassed or not score_oracle) else float(etas[i]),
                    c0_size=0 if bypassed else c[CNT_C0], c1_size=0 if bypassed else c[CNT_C1],
                    probe_size=probe, c2_size=0 if bypassed else c[CNT_C2],
                    budget_k=0 if bypassed else c[CNT_K],
                    candidate_fraction=(0 if bypassed else c[CNT_C1]) / n,
                    probe_fraction=probe / n,
                    output_error=None if not score_oracle else float(errs[i]),
                    clamp_count=0 if bypassed else c[CNT_CLAMP],
                    c0_dropped=0 if bypassed else c[CNT_DROP],
                    dot_products=S + L + 1 + probe,
                    timings_ns={"total": ns // U}, oracle_ns=oracle_ns))
        else:
            if mode == "topk_oracle":
                res, ns = _timed(lambda: sess.exact_topk_step(q, budget), dev)
                sizes = res.counts[0, :, CNT_C2].cpu().tolist()
                out = res.output.clone()
                k = max(1, round(budget * n))
            else:
                out, ns = _timed(lambda: sess.full_attention(q), dev)
                sizes = [0] * U
                k = 0
            errs = _rel_err(out[0], full[0]) if score_oracle else [None] * U
            oracle_ns = None
            if score_oracle:
                _, ons = _timed(lambda: sess.full_attention(q), dev)
                oracle_ns = ons // U
            sess.append_rows(kn, vn)
            for i in range(U):
                probe = sizes[i] if mode == "topk_oracle" else n - S
                per_head[i].append(StepRecord(
                    layer=i // H, head=i % H, step=t, n=n, bypassed=False, rho=0.0, eta=None,
                    c0_size=0, c1_size=0, probe_size=probe, c2_size=sizes[i], budget_k=k,
                    candidate_fraction=probe / n, probe_fraction=probe / n,
                    output_error=None if errs[i] is None else float(errs[i]),
                    clamp_count=0, c0_dropped=0, dot_products=n - S,
                    timings_ns={"total": ns // U}, oracle_ns=oracle_ns))
    records = [r for recs in per_head for r in recs]
    snapshots = None
    if snapshot_tables and mode == "lfps":
        snapshots = {}
        for i in range(U):
            ver, sla, sc = sess.session_tables(i)
            snapshots[str(i)] = {"ver": (ver * sc).tolist(), "sla": (sla * sc).tolist()}
    return RunReport(
        config=config.as_dict(),
        run={"mode": mode, "budget_fraction": budget, "threads": 1, "oracle": score_oracle,
             "trace_path": trace_path, "layers": trace.layers, "heads": trace.heads,
             "d": trace.d, "n_prefill": trace.n_prefill, "steps": trace.steps},
        records=records,
        instrumentation={"oracle_steps": sum(1 for r in records if r.oracle_ns is not None),
                         "probe_dot_products": sum(r.dot_products for r in records)},
        table_snapshot=snapshots)
