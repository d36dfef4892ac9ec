"""N2 / N3 on the CPU: the LFPS v1 trace container and the run-report schema
against artefacts produced by the reference itself (tests/golden/
small.lfps and small_report.json, made by tests/golden/make_trace_fixture.py
with the reference's own writer, run_trace and emitter)."""

import json
import os
import struct
import zlib

import numpy as np
import pytest

from paper_2506_15704_b200 import errors
from paper_2506_15704_b200 import report as rp
from paper_2506_15704_b200 import tracefile as tf

HERE = os.path.dirname(os.path.abspath(__file__))
TRACE = os.path.join(HERE, "golden", "small.lfps")
REPORT = os.path.join(HERE, "golden", "small_report.json")


def raw():
    with open(TRACE, "rb") as f:
        return f.read()


def test_reads_reference_trace_and_rewrites_it_byte_identically():
    data = raw()
    tr = tf.read_trace(data)
    assert (tr.layers, tr.heads, tr.d, tr.n_prefill, tr.steps, tr.s, tr.sink_count) == \
        (1, 3, 32, 600, 12, 32, 4)
    h = tr.heads_data[1]
    assert h.prefill_keys.shape == (600, 32) and h.prefill_weights.shape == (32, 596)
    assert h.step_queries.shape == (12, 32)
    np.testing.assert_allclose(h.prefill_weights.sum(axis=1), 1.0, atol=1e-5)
    assert tf.write_trace(tr) == data
    assert "3 head(s)" in tf.describe(tr)


def _patch(data, off, b):
    return data[:off] + b + data[off + len(b):]


def _recrc(data):
    payload = data[tf.HEADER_BYTES:-4]
    return data[:-4] + struct.pack("<I", zlib.crc32(payload) & 0xFFFFFFFF)


@pytest.mark.parametrize("case,exc", [
    ("magic", errors.BadMagicError),
    ("version", errors.UnsupportedVersionError),
    ("encoding", errors.LayoutError),
    ("zero_heads", errors.LayoutError),
    ("short_prefill", errors.LayoutError),
    ("truncated", errors.TruncatedFileError),
    ("header_only", errors.TruncatedFileError),
    ("payload_flip", errors.ChecksumError),
    ("crc_flip", errors.ChecksumError),
])
def test_validation_order_and_errors(case, exc):
    """Validation order of trace_format.md: magic, version, header
    constraints, total length, checksum."""
    data = raw()
    if case == "magic":
        data = _patch(data, 0, b"LFPX")
    elif case == "version":
        data = _patch(data, 4, bytes([2]))
    elif case == "encoding":
        data = _patch(data, 61, struct.pack("<Q", 2))
    elif case == "zero_heads":
        data = _patch(data, 13, struct.pack("<Q", 0))
    elif case == "short_prefill":
        data = _patch(data, 29, struct.pack("<Q", 10))
    elif case == "truncated":
        data = data[:-9]
    elif case == "header_only":
        data = data[:40]
    elif case == "payload_flip":
        data = _patch(data, 5000, bytes([data[5000] ^ 0x10]))
    elif case == "crc_flip":
        data = _patch(data, len(data) - 1, bytes([data[-1] ^ 1]))
    with pytest.raises(exc):
        tf.read_trace(data)


def test_writer_checks_shapes():
    tr = tf.read_trace(raw())
    bad = tf.HeadTrace(*(np.asarray(x) for x in (tr.heads_data[0].prefill_keys[:-1],) +
                         tuple(getattr(tr.heads_data[0], f) for f in
                               ("prefill_values", "prefill_weights", "final_query",
                                "step_queries", "step_keys", "step_values"))))
    broken = tf.TraceFile(tr.layers, tr.heads, tr.d, tr.n_prefill, tr.steps, tr.s, tr.sink_count,
                          (bad,) + tr.heads_data[1:])
    with pytest.raises(ValueError):
        tf.write_trace(broken)


def _report_from_doc(doc):
    recs = [rp.StepRecord(**{k: v for k, v in r.items()}) for r in doc["records"]]
    return rp.RunReport(config=doc["config"], run=doc["run"], records=recs,
                        instrumentation=doc["instrumentation"], table_snapshot=doc["table_snapshot"])


def test_report_schema_reemits_reference_bytes():
    """The reference's canonical JSON, parsed into this package's records and
    re-emitted, is byte-identical (field order, 17-digit floats, x.0 ints),
    and the aggregates recompute to the reference's."""
    with open(REPORT, "rb") as f:
        ref = f.read()
    doc = json.loads(ref)
    rep = _report_from_doc(doc)
    assert rp.emit_json(rep) == ref
    assert rep.aggregates() == doc["aggregates"]


def test_report_csv_and_non_finite_rejection():
    with open(REPORT, "rb") as f:
        doc = json.loads(f.read())
    rep = _report_from_doc(doc)
    lines = rp.emit_csv(rep).decode().strip().split("\n")
    assert lines[0].split(",") == list(rp.CSV_COLUMNS)
    assert len(lines) == 1 + len(doc["records"])
    first = dict(zip(rp.CSV_COLUMNS, lines[1].split(",")))
    assert first["bypassed"] in ("0", "1") and int(first["n"]) == doc["records"][0]["n"]
    with pytest.raises(ValueError):
        rp.emit_json({"x": float("nan")})
