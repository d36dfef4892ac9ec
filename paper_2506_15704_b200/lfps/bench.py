"""The exact comparison step and trace replay (pkg/src/lfps/bench.py:48-218).

``exact_topk_step`` is the reference's "fair baseline" step (bench.py:73-80)
for one head, on the device: scaled dots over every non-sink row, bounded
Top-k with lower-index ties, joint sink + selection output.  ``run_trace``
and ``config_for_trace`` are the batched GPU replay (replay.py)."""

from __future__ import annotations

import numpy as np
import torch

from ..replay import config_for_trace, run_trace  # noqa: F401  (re-exported)
from . import _dev
from .attention import AttentionOutput, _attend_dev, _logits_dev, _topk_dev
from .store import KvStore


def _snapshot(store: KvStore, n: int) -> KvStore:
    """A copy of the first n rows (the pre-append context of a step)."""
    return KvStore._from_device(store._kt, store._vt, n)


def exact_topk_step(q, store: KvStore, k: int, sink: int):
    """(selected absolute indices, AttentionOutput) of one exact Top-k step."""
    q = np.asarray(q, dtype=np.float64)
    if q.shape != (store.d,):
        raise ValueError(f"q must have shape ({store.d},), got {q.shape}")
    n = store.n
    qd = _dev.f64(q)
    idx = torch.arange(sink, n, dtype=_dev.I64, device=qd.device)
    scores = _logits_dev(store, qd, idx, n - sink)
    sel = _topk_dev(idx, scores, k)
    att = torch.cat([torch.arange(sink, dtype=_dev.I64, device=qd.device), sel])
    out, w = _attend_dev(store, qd, att, int(att.shape[0]))
    return _dev.host(sel), AttentionOutput(_dev.host(out), _dev.host(att), _dev.host(w))
