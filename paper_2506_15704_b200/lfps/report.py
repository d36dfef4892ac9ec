"""Run reports (pkg/src/lfps/report.py:29-222)."""
from ..report import *  # noqa: F401,F403
from ..report import RunReport, StepRecord, compute_aggregates, emit_csv, emit_json  # noqa: F401
