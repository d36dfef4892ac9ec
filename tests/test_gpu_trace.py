"""N2 + N3 on the device: a trace written by the reference replays through
the batched GPU path (tracefile.upload, replay.run_trace) and reproduces the
reference's own run report (tests/golden/small_report.json): every set
size, budget, clamp and dot count exact, eta exact, rho and the output error
against full attention within fp32-score tolerance."""

import json
import os

import pytest

from paper_2506_15704_b200 import replay
from paper_2506_15704_b200 import report as rp
from paper_2506_15704_b200 import tracefile as tf

pytestmark = pytest.mark.gpu

HERE = os.path.dirname(os.path.abspath(__file__))


def test_lfps_replay_matches_reference_report():
    tr = tf.load_trace(os.path.join(HERE, "golden", "small.lfps"))
    with open(os.path.join(HERE, "golden", "small_report.json")) as f:
        ref = json.load(f)
    rep = replay.run_trace(tr, mode="lfps", budget=0.05, trace_path="small.lfps",
                           snapshot_tables=True)
    got = rep.as_dict()
    assert got["config"] == ref["config"]
    assert len(got["records"]) == len(ref["records"])
    for a, b in zip(got["records"], ref["records"]):
        tag = (a["layer"], a["head"], a["step"])
        for key in ("layer", "head", "step", "n", "bypassed", "c0_size", "c1_size", "probe_size",
                    "c2_size", "budget_k", "clamp_count", "c0_dropped", "dot_products"):
            assert a[key] == b[key], (tag, key, a[key], b[key])
        assert a["rho"] == pytest.approx(b["rho"], rel=1e-9, abs=1e-12), tag
        if b["eta"] is not None:
            assert a["eta"] == pytest.approx(b["eta"], abs=1e-12), tag
        assert a["output_error"] == pytest.approx(b["output_error"], rel=1e-3, abs=1e-5), tag
    assert rp.emit_json(rep).startswith(b'{"schema_version":1,"kind":"lfps-run-report"')
    assert set(got["table_snapshot"]) == {"0", "1", "2"}


@pytest.mark.parametrize("mode", ["topk_oracle", "full"])
def test_reference_modes_replay(mode):
    tr = tf.load_trace(os.path.join(HERE, "golden", "small.lfps"))
    rep = replay.run_trace(tr, mode=mode, budget=0.05)
    recs = rep.records
    assert len(recs) == 36
    for r in recs:
        assert r.dot_products == r.n - 4
        if mode == "full":
            assert r.output_error < 1e-5 and r.probe_size == r.n - 4
        else:
            assert r.c2_size == max(1, round(0.05 * r.n))
    assert rep.aggregates()["records"] == 36
