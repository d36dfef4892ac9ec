"""Run reports in the reference's schema (next-row N3).

Restates pkg/docs/report_schema.md (pkg/src/lfps/report.py:29-222): one
``StepRecord`` per (layer, head, step), aggregates recomputable from the
records, canonical JSON (insertion-ordered fields, floats at 17 significant
digits, integral floats as ``x.0``, no NaN / Inf) and CSV.  GPU runs
(``replay.run_trace``) emit documents the reference's tooling reads
unchanged.
"""

from __future__ import annotations

import json
import math
from dataclasses import dataclass, field

SCHEMA_VERSION = 1
TIMING_KEYS = ("gate", "thresholds", "select", "expand", "finalize", "topk", "output",
               "update", "append", "total")
CSV_COLUMNS = ("layer", "head", "step", "n", "bypassed", "rho", "eta", "c0_size", "c1_size",
               "probe_size", "c2_size", "budget_k", "candidate_fraction", "probe_fraction",
               "output_error", "clamp_count", "c0_dropped", "dot_products",
               *(f"{k}_ns" for k in TIMING_KEYS), "oracle_ns")


@dataclass
class StepRecord:
    """Metrics of one (layer, head, step) (report_schema.md "Records")."""

    layer: int
    head: int
    step: int
    n: int
    bypassed: bool
    rho: float
    eta: float | None
    c0_size: int
    c1_size: int
    probe_size: int
    c2_size: int
    budget_k: int
    candidate_fraction: float
    probe_fraction: float
    output_error: float | None
    clamp_count: int
    c0_dropped: int
    dot_products: int
    timings_ns: dict
    oracle_ns: int | None = None

    def as_dict(self) -> dict:
        out = {}
        for name in ("layer", "head", "step", "n", "bypassed", "rho", "eta", "c0_size",
                     "c1_size", "probe_size", "c2_size", "budget_k", "candidate_fraction",
                     "probe_fraction", "output_error", "clamp_count", "c0_dropped",
                     "dot_products"):
            out[name] = getattr(self, name)
        out["timings_ns"] = {k: int(self.timings_ns.get(k, 0)) for k in TIMING_KEYS}
        out["oracle_ns"] = self.oracle_ns
        return out


def compute_aggregates(records: list) -> dict:
    """Aggregates of report_schema.md, all derived from the records."""
    total = len(records)
    etas = sorted(r.eta for r in records if r.eta is not None)
    fracs = [r.candidate_fraction for r in records if not r.bypassed]
    errs = [r.output_error for r in records if r.output_error is not None]
    lfps_ns = sum(r.timings_ns.get("total", 0) for r in records)
    oracle = [r.oracle_ns for r in records if r.oracle_ns is not None]
    oracle_ns = sum(oracle)
    steps = max((r.step for r in records), default=-1) + 1

    def mean(xs):
        return sum(xs) / len(xs) if xs else 0.0

    def median(xs):
        if not xs:
            return 0.0
        h = len(xs) // 2
        return xs[h] if len(xs) % 2 else (xs[h - 1] + xs[h]) / 2.0

    secs = lfps_ns / 1e9
    osecs = oracle_ns / 1e9
    return {
        "records": total,
        "steps": steps,
        "mean_eta": mean(etas),
        "median_eta": median(etas),
        "mean_candidate_fraction": mean(fracs),
        "bypass_rate": sum(1 for r in records if r.bypassed) / total if total else 0.0,
        "mean_output_error": mean(errs),
        "clamp_count": sum(r.clamp_count for r in records),
        "c0_dropped": sum(r.c0_dropped for r in records),
        "dot_products": sum(r.dot_products for r in records),
        "lfps_seconds": secs,
        "steps_per_sec_per_head": total / secs if lfps_ns else 0.0,
        "tokens_per_sec": steps / secs if lfps_ns else 0.0,
        "reference_seconds": osecs,
        "reference_tokens_per_sec": (steps * len(oracle) / total / osecs
                                     if oracle_ns and total else 0.0),
    }


@dataclass
class RunReport:
    """Config echo, run description, records, instrumentation, snapshot."""

    config: dict
    run: dict
    records: list
    instrumentation: dict = field(default_factory=dict)
    table_snapshot: dict | None = None

    def aggregates(self) -> dict:
        return compute_aggregates(self.records)

    def as_dict(self) -> dict:
        return {
            "schema_version": SCHEMA_VERSION,
            "kind": "lfps-run-report",
            "config": self.config,
            "run": self.run,
            "aggregates": self.aggregates(),
            "instrumentation": self.instrumentation,
            "records": [r.as_dict() for r in self.records],
            "table_snapshot": self.table_snapshot,
        }


def _fmt_float(x: float) -> str:
    if not math.isfinite(x):
        raise ValueError(f"non-finite value {x!r} cannot be serialized")
    if x == int(x) and abs(x) < 1e16:
        return f"{x:.1f}"
    return format(x, ".17g")


def _emit(x, out: list) -> None:
    if x is None:
        out.append("null")
    elif x is True or x is False:
        out.append("true" if x else "false")
    elif isinstance(x, int):
        out.append(str(x))
    elif isinstance(x, float):
        out.append(_fmt_float(x))
    elif isinstance(x, str):
        out.append(json.dumps(x))
    elif isinstance(x, dict):
        out.append("{")
        for i, (k, v) in enumerate(x.items()):
            if i:
                out.append(",")
            out.append(json.dumps(str(k)))
            out.append(":")
            _emit(v, out)
        out.append("}")
    elif isinstance(x, (list, tuple)):
        out.append("[")
        for i, v in enumerate(x):
            if i:
                out.append(",")
            _emit(v, out)
        out.append("]")
    else:
        raise TypeError(f"cannot serialize {type(x)!r}")


def emit_json(report) -> bytes:
    """Canonical JSON bytes (parse + re-emit is byte-identical)."""
    doc = report.as_dict() if isinstance(report, RunReport) else report
    out: list = []
    _emit(doc, out)
    out.append("\n")
    return "".join(out).encode("utf-8")


def emit_csv(report: RunReport) -> bytes:
    """One CSV row per record; booleans 0/1, missing values empty."""
    lines = [",".join(CSV_COLUMNS)]
    for r in report.records:
        row = r.as_dict()
        flat = dict(row)
        flat.update({f"{k}_ns": v for k, v in row["timings_ns"].items()})
        cells = []
        for col in CSV_COLUMNS:
            v = flat.get(col)
            if v is None:
                cells.append("")
            elif v is True or v is False:
                cells.append("1" if v else "0")
            elif isinstance(v, float):
                cells.append(format(v, ".17g"))
            else:
                cells.append(str(v))
        lines.append(",".join(cells))
    return ("\n".join(lines) + "\n").encode("utf-8")
