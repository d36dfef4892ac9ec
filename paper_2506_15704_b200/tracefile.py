"""LFPS v1 trace container (next-row N2): read, write, and upload to the GPU.

The on-disk format is the reference's (pkg/docs/trace_format.md;
pkg/src/lfps/tracefile.py:1-31), so traces written by ``lfps gen`` or the
reference's exporter replay here unchanged, and traces written here load in
the reference:

* header, 69 bytes: ``"LFPS"``, version byte 1, then eight u64 LE -- layers
  L, heads H, head dim d, prefill length n, decode steps T, prefill weight
  window s, sink count, value encoding (1 = float32);
* payload: per (layer, head), layer-major -- prefill keys [n, d], prefill
  values [n, d], prefill weights [s, n - sink], final prefill query [d];
  then per step, per (layer, head) -- query, new key, new value ([d] each);
  all float32 LE, row-major;
* trailer: zlib CRC-32 of the payload bytes, u32 LE.

Validation order on read (the reference's): magic, version, header
constraints, total length, checksum -- each failure raises its
``TraceFormatError`` subclass before any payload is interpreted.

``upload`` places a trace on the device: every (layer, head) becomes a
(request 0, KV-head) unit with one query head (the trace heads are
independent MHA heads), so the whole trace steps as ONE batched
decode call per step.  Values are rounded to bf16 on the way in (the device
KV cache is bf16); traces of bf16-representable values replay exactly.
"""

from __future__ import annotations

import struct
import zlib
from dataclasses import dataclass

import numpy as np

from .errors import (BadMagicError, ChecksumError, LayoutError, TruncatedFileError,
                     UnsupportedVersionError)

MAGIC = b"LFPS"
VERSION = 1
ENCODING_F32 = 1
HEADER_BYTES = 69
_HEAD = struct.Struct("<4sB8Q")
assert _HEAD.size == HEADER_BYTES


@dataclass(frozen=True)
class HeadTrace:
    """One (layer, head)'s share of a trace, float32 arrays."""

    prefill_keys: np.ndarray      # [n, d]
    prefill_values: np.ndarray    # [n, d]
    prefill_weights: np.ndarray   # [s, n - sink]
    final_query: np.ndarray       # [d]
    step_queries: np.ndarray      # [T, d]
    step_keys: np.ndarray         # [T, d]
    step_values: np.ndarray       # [T, d]


@dataclass(frozen=True)
class TraceFile:
    """A decoded trace: dimensions plus one ``HeadTrace`` per (layer, head)
    in layer-major order (index = layer * heads + head)."""

    layers: int
    heads: int
    d: int
    n_prefill: int
    steps: int
    s: int
    sink_count: int
    heads_data: tuple
    value_encoding: int = ENCODING_F32

    @property
    def head_count(self) -> int:
        return self.layers * self.heads


def _payload_bytes(L, H, d, n, T, s, sink) -> int:
    m0 = n - sink
    return L * H * 4 * (2 * n * d + s * m0 + d) + T * L * H * 12 * d


def write_trace(trace: TraceFile) -> bytes:
    """Serialise a trace (shapes are checked; arrays cast to float32 LE)."""
    L, H, d, n, T = trace.layers, trace.heads, trace.d, trace.n_prefill, trace.steps
    s, sink = trace.s, trace.sink_count
    if trace.value_encoding != ENCODING_F32:
        raise ValueError(f"unsupported value encoding {trace.value_encoding}")
    if len(trace.heads_data) != L * H:
        raise ValueError(f"expected {L * H} head blocks, got {len(trace.heads_data)}")
    if n <= sink:
        raise ValueError("n_prefill must exceed sink_count")
    m0 = n - sink

    def f32(a, shape, what):
        a = np.asarray(a)
        if a.shape != shape:
            raise ValueError(f"{what} must have shape {shape}, got {a.shape}")
        return np.ascontiguousarray(a, dtype="<f4").tobytes()

    parts = []
    for h in trace.heads_data:
        parts += [f32(h.prefill_keys, (n, d), "prefill_keys"),
                  f32(h.prefill_values, (n, d), "prefill_values"),
                  f32(h.prefill_weights, (s, m0), "prefill_weights"),
                  f32(h.final_query, (d,), "final_query")]
        for name in ("step_queries", "step_keys", "step_values"):
            if np.asarray(getattr(h, name)).shape != (T, d):
                raise ValueError(f"{name} must have shape {(T, d)}")
    for t in range(T):
        for h in trace.heads_data:
            parts += [f32(h.step_queries[t], (d,), "query"), f32(h.step_keys[t], (d,), "key"),
                      f32(h.step_values[t], (d,), "value")]
    payload = b"".join(parts)
    header = _HEAD.pack(MAGIC, VERSION, L, H, d, n, T, s, sink, ENCODING_F32)
    return header + payload + struct.pack("<I", zlib.crc32(payload) & 0xFFFFFFFF)


def read_trace(data: bytes) -> TraceFile:
    """Decode and validate a trace byte stream (magic, version, header,
    length, checksum -- in that order)."""
    data = bytes(data)
    if len(data) < HEADER_BYTES:
        raise TruncatedFileError(f"stream of {len(data)} bytes is shorter than the header")
    magic, version, L, H, d, n, T, s, sink, enc = _HEAD.unpack_from(data, 0)
    if magic != MAGIC:
        raise BadMagicError(f"bad magic {magic!r}")
    if version != VERSION:
        raise UnsupportedVersionError(f"unsupported version {version}")
    if enc != ENCODING_F32:
        raise LayoutError(f"unknown value encoding {enc}")
    if min(L, H, d, s, sink) < 1:
        raise LayoutError("layer/head/d/s/sink counts must all be >= 1")
    if n < sink + s:
        raise LayoutError(f"n_prefill {n} too small for sink_count {sink} and s {s}")
    want = HEADER_BYTES + _payload_bytes(L, H, d, n, T, s, sink) + 4
    if len(data) != want:
        raise TruncatedFileError(f"stream is {len(data)} bytes, header implies {want}")
    payload = memoryview(data)[HEADER_BYTES:-4]
    (crc,) = struct.unpack_from("<I", data, len(data) - 4)
    if zlib.crc32(payload) & 0xFFFFFFFF != crc:
        raise ChecksumError("payload checksum mismatch")
    flat = np.frombuffer(payload, dtype="<f4")
    m0 = n - sink
    off = 0

    def take(count, shape):
        nonlocal off
        a = flat[off: off + count].reshape(shape).astype(np.float32)
        off += count
        return a

    blocks = []
    for _ in range(L * H):
        blocks.append([take(n * d, (n, d)), take(n * d, (n, d)), take(s * m0, (s, m0)),
                       take(d, (d,))])
    steps = flat[off:].reshape(T, L * H, 3, d).astype(np.float32)
    heads = tuple(HeadTrace(k, v, w, f, steps[:, i, 0].copy(), steps[:, i, 1].copy(),
                            steps[:, i, 2].copy())
                  for i, (k, v, w, f) in enumerate(blocks))
    return TraceFile(layers=L, heads=H, d=d, n_prefill=n, steps=T, s=s, sink_count=sink,
                     heads_data=heads)


def save_trace(trace: TraceFile, path) -> None:
    with open(path, "wb") as f:
        f.write(write_trace(trace))


def load_trace(path) -> TraceFile:
    with open(path, "rb") as f:
        return read_trace(f.read())


def describe(trace: TraceFile) -> str:
    return (f"LFPS v{VERSION} trace: {trace.layers} layer(s) x {trace.heads} head(s), d={trace.d}, "
            f"prefill {trace.n_prefill}, {trace.steps} step(s), s={trace.s}, "
            f"sink={trace.sink_count}")


# --------------------------------------------------------------------------
# device upload
# --------------------------------------------------------------------------

@dataclass
class DeviceTrace:
    """A trace resident on the GPU: the batched session (bootstrapped) and
    the per-step inputs q [T, 1, L*H, d], k_new / v_new [T, 1, L*H, d]."""

    session: object
    q: object
    k_new: object
    v_new: object


def upload(trace: TraceFile, config, device=None, headroom: int = 8) -> DeviceTrace:
    """Bootstrap a ``BatchedSession`` with every (layer, head) of the trace
    as a one-query-head unit of request 0 and stage the step inputs."""
    import torch

    from .session import BatchedSession
    if config.d != trace.d or config.s != trace.s or config.sink_count != trace.sink_count:
        raise ValueError("config d / s / sink_count must match the trace")
    U, T, d, n = trace.head_count, trace.steps, trace.d, trace.n_prefill
    sess = BatchedSession(config, 1, U, 1, n_max=n + T + headroom, device=device)
    dev = sess.device
    bf = torch.bfloat16
    keys = torch.stack([torch.as_tensor(h.prefill_keys) for h in trace.heads_data])
    values = torch.stack([torch.as_tensor(h.prefill_values) for h in trace.heads_data])
    sess.load_prefill(0, keys.to(dev, bf), values.to(dev, bf))
    w = torch.stack([torch.as_tensor(h.prefill_weights) for h in trace.heads_data])
    sess.bootstrap_tables(0, w.to(dev, torch.float32))
    fq = torch.stack([torch.as_tensor(h.final_query) for h in trace.heads_data])
    sess.bootstrap_stats(fq.reshape(1, U, d).to(dev, bf))
    torch.cuda.synchronize(dev)
    sess.check_errors("trace bootstrap")

    def steps(name):
        a = np.stack([getattr(h, name) for h in trace.heads_data], axis=1)   # [T, U, d]
        return torch.as_tensor(a).reshape(T, 1, U, d).to(dev, bf)

    return DeviceTrace(session=sess, q=steps("step_queries"), k_new=steps("step_keys"),
                       v_new=steps("step_values"))
