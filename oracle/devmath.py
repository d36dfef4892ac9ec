"""Canonical device arithmetic ("devmath"), restated in numpy.

TEST INFRASTRUCTURE ONLY.  Nothing in the product package imports this
module; only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg
may use it, and only as the checker.

The reference (pkg/src/lfps) computes with numpy's pairwise sums, BLAS ddot
and libm exp.  Those orders are machine-specific, so a GPU cannot reproduce
them bit for bit.  The B200 kernels instead follow the fixed orders defined
here; every function below is the exact IEEE-754 op sequence the CUDA code
performs (`paper_2506_15704_b200/csrc/canon.cuh`), so GPU results can be
compared with this oracle bit for bit.  The reference's own tests pin these
quantities to tolerances only (moments 1e-12: pkg/tests/test_core.py:145-154,
thresholds 1e-9: pkg/tests/test_tables.py:258-273), and tests/ check that the
devmath oracle and the reference-arithmetic oracle select identical index
sets on the golden trajectories.

Definitions (DESIGN.md §3 "Canonical arithmetic"):

* ``table_sum``   -- chunks of 512 elements; lane l of a warp holds
  x[c*512 + e*32 + l], e = 0..15, and reduces them by an adjacent-pair tree
  over e, the 32 lane sums fold halves (16, 8, 4, 2, 1); chunk partials then
  reduce by a pairwise tree (zero-padded to a power of two).  Used for the
  head-stats variance.
* ``table_moments`` -- per *segment* the segment mean (table_sum order /
  count) and the segment's centred power sums M2, M3, M4 (same lane/fold
  order), then a pairwise tree of exact pairwise-update merges (Chan et al.;
  Pebay 2008) over the segments in logical order.  A segment is a maximal run
  of logical slots i whose *virtual slot* off + i lies in one 512-aligned
  block: off = 0 for the vertical table (segments = logical chunks of 512);
  for the slash table off is the tracker's virtual base (TrackerState.vbase,
  -m0 at bootstrap, minus one per slash shift), so a slash value keeps its
  block while its logical index moves.  Block summaries are therefore
  stable across steps and the device recomputes only the blocks a step
  touched.  Same quantities as the reference's two-pass _phys_moments
  (tables.py:127-140), different rounding; the golden tests pin identical
  selections.
* ``gdot``        -- fp64 dot: lane l (of 32) accumulates j = l, l+32, ...
  in order, then folds 16..1.  Gate logits, head stats (gate.py:77-98).
* ``sdot32``      -- fp32 probe score: 16 lanes each own d/16 contiguous
  elements, sequential fused accumulate (exact: bf16*bf16 products are exact
  in fp32), fold 8, 4, 2, 1, then IEEE division by fp32(sqrt(d))
  (numerics.py:33-49, engine.py:169).
* ``cexp``        -- fp64 exp from +,-,*,rint and an exact power-of-two
  scale; arguments below -708 give 0.
* ``block_sum``   -- 256 threads: thread t accumulates e[t + 256 i] in order,
  warps fold 16..1, the 8 warp sums fold 4, 2, 1.  Update softmax
  (engine.py:184, numerics.py:52-66).
"""

from __future__ import annotations

import math

import numpy as np

TABLE_CHUNK = 512  # elements per warp chunk in table_sum
TABLE_LANES = 32
BLOCK_THREADS = 256

# fdlibm split of ln 2: LN2_HI has 21 trailing zero bits so k*LN2_HI is exact.
LN2_HI = 6.93147180369123816490e-01
LN2_LO = 1.90821492927058770002e-10
INV_LN2 = 1.44269504088896338700e+00
EXP_LOW = -708.0
# Taylor coefficients 1/i!, i = 0..13, rounded to double.
EXP_COEF = tuple(1.0 / math.factorial(i) for i in range(14))


def _fold_halves(v: np.ndarray) -> np.ndarray:
    """Butterfly fold over the last axis (length a power of two):
    v[i] + v[i + h] for h = len/2, ..., 1.  Equals __shfl_xor reduction."""
    while v.shape[-1] > 1:
        h = v.shape[-1] // 2
        v = v[..., :h] + v[..., h:]
    return v[..., 0]


def _pairwise_tree(p: np.ndarray) -> float:
    """Adjacent-pair tree over a 1-D array zero-padded to a power of two."""
    n = p.shape[0]
    if n == 0:
        return 0.0
    size = 1
    while size < n:
        size *= 2
    buf = np.zeros(size, dtype=np.float64)
    buf[:n] = p
    while buf.shape[0] > 1:
        buf = buf[0::2] + buf[1::2]
    return float(buf[0])


def table_chunk_partials(x: np.ndarray) -> np.ndarray:
    """Per-chunk partial sums of ``x`` (fp64, any length)."""
    x = np.asarray(x, dtype=np.float64)
    n = x.shape[0]
    nch = max(1, -(-n // TABLE_CHUNK))
    buf = np.zeros(nch * TABLE_CHUNK, dtype=np.float64)
    buf[:n] = x
    buf = buf.reshape(nch, TABLE_CHUNK // TABLE_LANES, TABLE_LANES)
    while buf.shape[1] > 1:                 # per-lane adjacent-pair tree over e
        buf = buf[:, 0::2, :] + buf[:, 1::2, :]
    return _fold_halves(buf[:, 0, :])


def table_sum(x: np.ndarray) -> float:
    """Canonical sum used by the table-moment kernel."""
    return _pairwise_tree(table_chunk_partials(x))


def _lane_tree(buf: np.ndarray) -> np.ndarray:
    """[nch, 16, 32] -> per-chunk fold of per-lane adjacent-pair trees."""
    while buf.shape[1] > 1:
        buf = buf[:, 0::2, :] + buf[:, 1::2, :]
    return _fold_halves(buf[:, 0, :])


def segment_bounds(n: int, off: int = 0) -> list[tuple[int, int]]:
    """(start, length) of the segments of a table of n logical slots whose
    logical slot 0 sits at virtual slot ``off`` (see table_moments)."""
    out = []
    i = 0
    while i < n:
        first = TABLE_CHUNK - ((off + i) % TABLE_CHUNK)
        ln = min(first, n - i)
        out.append((i, ln))
        i += ln
    return out


def chunk_moments(x: np.ndarray, off: int = 0):
    """Per-segment (count, mean, M2, M3, M4) of a table, device order.

    Element j of a segment is held by lane j % 32 at position j // 32."""
    x = np.asarray(x, dtype=np.float64)
    segs = segment_bounds(x.shape[0], off) or [(0, 0)]
    nch = len(segs)
    buf = np.zeros((nch, TABLE_CHUNK), dtype=np.float64)
    valid = np.zeros((nch, TABLE_CHUNK), dtype=bool)
    cnt = np.zeros(nch, dtype=np.float64)
    for k, (a, ln) in enumerate(segs):
        buf[k, :ln] = x[a: a + ln]
        valid[k, :ln] = True
        cnt[k] = ln
    shape = (nch, TABLE_CHUNK // TABLE_LANES, TABLE_LANES)
    buf = buf.reshape(shape)
    valid = valid.reshape(shape)
    with np.errstate(invalid="ignore", divide="ignore"):
        mu = _lane_tree(buf) / cnt
    d = np.where(valid, buf - mu[:, None, None], 0.0)
    d2 = d * d
    d3 = d2 * d
    d4 = d2 * d2
    return cnt, mu, _lane_tree(d2), _lane_tree(d3), _lane_tree(d4)


def merge_moments(a, b):
    """Exact pairwise update of (n, mean, M2, M3, M4), device op order.

    Arrays broadcast; an empty side (n == 0) returns the other unchanged."""
    na, ma, a2, a3, a4 = a
    nb, mb, b2, b3, b4 = b
    with np.errstate(invalid="ignore", divide="ignore"):
        n = na + nb
        delta = mb - ma
        dn = delta / n
        dn2 = dn * dn
        t = ((delta * dn) * na) * nb
        mean = ma + nb * dn
        m2 = (a2 + b2) + t
        m3 = ((a3 + b3) + (t * dn) * (na - nb)) + (3.0 * dn) * (na * b2 - nb * a2)
        m4 = (((a4 + b4) + (t * dn2) * ((na * na - na * nb) + nb * nb))
              + (6.0 * dn2) * ((na * na) * b2 + (nb * nb) * a2)) + (4.0 * dn) * (na * b3 - nb * a3)
    out = []
    for merged, av, bv in zip((n, mean, m2, m3, m4), a, b):
        merged = np.where(nb == 0, av, merged)
        merged = np.where(na == 0, bv, merged)
        out.append(merged)
    return tuple(out)


def table_moments(x: np.ndarray, off: int = 0) -> tuple[float, float, float]:
    """(mean_p, sum c^2, sum c^4) of a phys table view.

    Restates ScoreTablePair._phys_moments (tables.py:127-140) as segment
    moments merged by a pairwise tree over the segments (zero-count padding
    to a power of two); ``off`` is the virtual slot of logical slot 0."""
    st = chunk_moments(x, off)
    nch = st[0].shape[0]
    size = 1
    while size < nch:
        size *= 2
    st = [np.concatenate([v, np.zeros(size - nch)]) for v in st]
    while st[0].shape[0] > 1:
        st = list(merge_moments(tuple(v[0::2] for v in st), tuple(v[1::2] for v in st)))
    return float(st[1][0]), float(st[2][0]), float(st[4][0])


def gdot(a: np.ndarray, b: np.ndarray) -> np.ndarray:
    """Canonical fp64 dot over the last axis (broadcasting).

    Lane l accumulates products a[j]*b[j] for j = l (mod 32) in increasing j
    (separate multiply and add; no fused op), then lanes fold 16..1."""
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    a, b = np.broadcast_arrays(a, b)
    d = a.shape[-1]
    steps = -(-d // 32)
    pad = steps * 32 - d
    if pad:
        widths = [(0, 0)] * (a.ndim - 1) + [(0, pad)]
        a = np.pad(a, widths)
        b = np.pad(b, widths)
    a = a.reshape(a.shape[:-1] + (steps, 32))
    b = b.reshape(b.shape[:-1] + (steps, 32))
    acc = np.zeros(a.shape[:-2] + (32,), dtype=np.float64)
    for e in range(steps):
        acc = acc + a[..., e, :] * b[..., e, :]
    return _fold_halves(acc)


def sdot32(keys: np.ndarray, q: np.ndarray, rsd: np.float32) -> np.ndarray:
    """Canonical fp32 probe score (keys[..., d] . q) / fp32(sqrt d).

    ``keys`` and ``q`` hold bf16-representable values.  Each of 16 lanes owns
    d/16 contiguous elements and accumulates k*q (exact in fp32) in order;
    the lane sums fold 8, 4, 2, 1; the result is divided (IEEE) by rsd."""
    keys = np.asarray(keys, dtype=np.float32)
    q = np.asarray(q, dtype=np.float32)
    d = keys.shape[-1]
    assert d % 16 == 0, "score kernels require d % 16 == 0"
    per = d // 16
    prod = (keys * q).reshape(keys.shape[:-1] + (16, per))
    acc = np.zeros(keys.shape[:-1] + (16,), dtype=np.float32)
    for e in range(per):
        acc = acc + prod[..., e]
    dot = _fold_halves(acc)
    return (dot / np.float32(rsd)).astype(np.float32)


def rsd_f32(d: int) -> np.float32:
    """fp32 sqrt(d) constant handed to the score kernels."""
    return np.float32(math.sqrt(d))


def cexp(x) -> np.ndarray:
    """Canonical fp64 exp (accurate to ~1 ulp), elementwise.

    k = rint(x / ln2); r = (x - k*LN2_HI) - k*LN2_LO; Horner Taylor degree 13
    on r; times 2^k.  Arguments below -708 return 0.0."""
    x = np.asarray(x, dtype=np.float64)
    k = np.rint(x * INV_LN2)
    r = (x - k * LN2_HI) - k * LN2_LO
    p = np.full_like(x, EXP_COEF[13])
    for i in range(12, -1, -1):
        p = p * r + EXP_COEF[i]
    out = np.ldexp(p, k.astype(np.int64))
    return np.where(x < EXP_LOW, 0.0, out)


def block_sum(e: np.ndarray) -> float:
    """Canonical 256-thread block reduction of a 1-D fp64 array."""
    e = np.asarray(e, dtype=np.float64)
    n = e.shape[0]
    rows = max(1, -(-n // BLOCK_THREADS))
    buf = np.zeros(rows * BLOCK_THREADS, dtype=np.float64)
    buf[:n] = e
    buf = buf.reshape(rows, BLOCK_THREADS)
    acc = np.zeros(BLOCK_THREADS, dtype=np.float64)
    for i in range(rows):
        acc = acc + buf[i]
    warp = _fold_halves(acc.reshape(BLOCK_THREADS // 32, 32))
    return float(_fold_halves(warp))


def softmax_update(z: np.ndarray) -> np.ndarray:
    """Canonical fp64 softmax over the selected scores (engine.py:184)."""
    z = np.asarray(z, dtype=np.float64)
    e = cexp(z - z.max())
    return e / block_sum(e)


def seq_sum(x) -> float:
    """Left-to-right fp64 sum from 0.0 (gate terms, gate.py:108-109)."""
    acc = 0.0
    for v in np.asarray(x, dtype=np.float64).tolist():
        acc = acc + v
    return acc


def stats_sum_rows(x: np.ndarray) -> np.ndarray:
    """Column sums of an (n, d) matrix, rows accumulated in order.

    This is numpy's own axis-0 reduction order, so K-bar / V-bar match the
    reference's keys_ns.mean(axis=0) bit for bit (gate.py:71-72)."""
    x = np.asarray(x, dtype=np.float64)
    acc = np.zeros(x.shape[1], dtype=np.float64)
    for i in range(x.shape[0]):
        acc = acc + x[i]
    return acc


def chunked_sum(x: np.ndarray) -> float:
    """Canonical long 1-D sum (head-stats logits): same as table_sum."""
    return table_sum(x)
