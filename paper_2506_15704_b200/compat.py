"""Reference-facing per-head API on the B200 path.

Same names, arguments, return types and exceptions as the reference's
decode-step entry points (pkg/src/lfps/engine.py:38-219): a user of
``lfps.prefill_bootstrap`` / ``lfps.decode_step`` / ``lfps.run_session``
switches by importing them from ``paper_2506_15704_b200`` instead.  Each
HeadSession is a batch-of-one BatchedSession (one request, one KV head, one
query head) on the current CUDA device; every stage runs in
liblfps_b200.so.  Differences, by design of the device path:

* inputs are rounded to bf16 on the way in (the reference upcasts to fp64);
  for bf16-representable inputs candidate sets, Top-k sets, bypass decisions
  and tables match the reference arithmetic, outputs to 1e-5 relative;
* probe scores are fp32, the tables and the gate fp64;
* ``timings_ns`` carries the device-synchronised wall time under "total"
  (per-stage device times come from ``_lib.profile_collect``);
* ``StepResult.attention.weights`` is None (the weights stay on the device).
"""

from __future__ import annotations

import math
import time
from dataclasses import dataclass, field

import numpy as np
import torch

from .config import LfpsConfig
from .errors import SessionRunError
from .session import CNT_C2, CNT_CLAMP, CNT_DROP, CNT_K, CNT_PROBE, BatchedSession

_EMPTY = np.empty(0, dtype=np.int64)
_STAGES = ("gate", "thresholds", "select", "expand", "finalize", "topk", "output", "update",
           "append")


@dataclass(frozen=True)
class CandidateSet:
    """Index sets of one decode step (candidates.py:17-42)."""

    c0: np.ndarray = field(default_factory=lambda: _EMPTY)
    c1: np.ndarray = field(default_factory=lambda: _EMPTY)
    probe: np.ndarray = field(default_factory=lambda: _EMPTY)
    c2: np.ndarray = field(default_factory=lambda: _EMPTY)
    budget_k: int = 0

    @property
    def c0_dropped(self) -> int:
        if self.c0.size == 0:
            return 0
        return int(self.c0.size - np.isin(self.c0, self.c1).sum())


@dataclass(frozen=True)
class SparsityEstimate:
    """Sink share of the gate (gate.py:37-48); only rho leaves the device."""

    w_sink: float
    w_global: float
    w_local: float
    rho: float


@dataclass(frozen=True)
class AttentionOutput:
    """Output plus the attended indices (attention.py:21-31)."""

    output: np.ndarray
    indices: np.ndarray
    weights: np.ndarray | None = None


@dataclass
class HeadSession:
    """Per-head decode state (engine.py:38-47), resident on the GPU."""

    device_session: BatchedSession
    config: LfpsConfig
    step: int = 0

    @property
    def n(self) -> int:
        return self.device_session.n_host[0]

    def tables(self):
        """(ver values, sla values) = phys * scale in logical order (host copy)."""
        ver, sla, sc = self.device_session.session_tables(0)
        return ver * sc, sla * sc


@dataclass(frozen=True)
class StepResult:
    """Everything observable about one decode step (engine.py:50-64)."""

    output: np.ndarray
    candidate: CandidateSet
    bypassed: bool
    rho: float
    sparsity: SparsityEstimate
    timings_ns: dict
    dot_products: int
    clamp_count: int
    c0_dropped: int
    n_context: int
    attention: AttentionOutput | None = field(default=None, repr=False)


def _bf16(x, shape, name) -> torch.Tensor:
    a = np.asarray(x, dtype=np.float64)
    if a.shape != shape:
        raise ValueError(f"{name} must have shape {shape}, got {a.shape}")
    return torch.as_tensor(a, dtype=torch.float32).to(torch.bfloat16)


def prefill_bootstrap(keys, values, prefill_weights, last_query, config: LfpsConfig,
                      capacity: int | None = None) -> HeadSession:
    """Build a decode session from offloaded prefill state (engine.py:67-94)."""
    keys = np.asarray(keys, dtype=np.float64)
    values = np.asarray(values, dtype=np.float64)
    if keys.ndim != 2 or keys.shape[1] != config.d:
        raise ValueError(f"keys must be (n, {config.d})")
    n = keys.shape[0]
    if values.shape != keys.shape:
        raise ValueError(f"keys shape {keys.shape} != values shape {values.shape}")
    if n <= config.sink_count + config.s:
        raise ValueError(
            f"prefill needs more than sink_count + s = {config.sink_count + config.s} rows, got {n}")
    w = np.asarray(prefill_weights, dtype=np.float64)
    if w.shape != (config.s, n - config.sink_count):
        raise ValueError(
            f"prefill weights must be ({config.s}, {n - config.sink_count}), got {w.shape}")
    if np.any(np.abs(w.sum(axis=1) - 1.0) > 1e-4):
        raise ValueError("each prefill weight vector must sum to 1 over its non-sink range")
    d = config.d
    cap = capacity or (n + max(256, n // 4))
    dev = torch.device("cuda", torch.cuda.current_device())
    sess = BatchedSession(config, 1, 1, 1, n_max=cap, device=dev, export_sets=True)
    sess.load_unit(0, 0, _bf16(keys, (n, d), "keys").to(dev), _bf16(values, (n, d), "values").to(dev))
    sess.bootstrap_tables(0, torch.as_tensor(w, dtype=torch.float32)[None].to(dev))
    sess.bootstrap_stats(_bf16(last_query, (d,), "last_query").reshape(1, 1, d).to(dev))
    torch.cuda.synchronize(dev)
    sess.check_errors("prefill_bootstrap")
    return HeadSession(device_session=sess, config=config)


def _regrow(session: HeadSession) -> None:
    """Double the KV / table capacity (the reference's KvStore doubles too,
    store.py:79-87): a larger session with the logical state copied over."""
    old = session.device_session
    cfg = old.cfg
    n = old.n_host[0]
    new = BatchedSession(cfg, 1, 1, 1, n_max=2 * old.n_max, device=old.device,
                         export_sets=old.export_sets)
    new.k_cache[0, 0, :n].copy_(old.k_cache[0, 0, :n])
    new.v_cache[0, 0, :n].copy_(old.v_cache[0, 0, :n])
    m = n - cfg.sink_count
    new.ver[0, : m + 1].copy_(old.ver[0, : m + 1])
    # slash window (logical [0, m] incl. the parked slot) moved by a multiple
    # of 512 slots so its block alignment -- hence the canonical moment
    # order -- is unchanged; the fresh workspace rebuilds the block summaries
    base = int(old.sla_base[0])
    home = new.sla_cap // 2
    new_base = home - (m + 1) - ((home - (m + 1) - base) % 512)
    new.sla[0, new_base: new_base + m + 1].copy_(old.sla[0, base: base + m + 1])
    new.sla_base.fill_(new_base)
    for name in ("scale", "clamp_count", "mean_key", "mean_value", "sigma_hat_sq", "n_ctx"):
        getattr(new, name).copy_(getattr(old, name))
    new.n_host = list(old.n_host)
    session.device_session = new


def decode_step(session: HeadSession, q, new_key, new_value, k_fraction: float,
                config: LfpsConfig | None = None) -> StepResult:
    """Run one decode step and append the step's new KV row (engine.py:97-201)."""
    cfg = config if config is not None else session.config
    d = cfg.d
    qt = _bf16(q, (d,), "q")
    kt = _bf16(new_key, (d,), "new_key")
    vt = _bf16(new_value, (d,), "new_value")
    if not 0.0 < k_fraction <= 1.0:
        raise ValueError(f"k_fraction must be in (0, 1], got {k_fraction}")
    sess = session.device_session
    if sess.cfg is not cfg:
        sess.cfg = cfg
    n = sess.n_host[0]
    if n <= cfg.sink_count + cfg.local_window:
        raise ValueError("context shorter than sink_count + local_window")
    if n + 1 >= sess.n_max or n - cfg.sink_count + 2 > sess.m_cap:
        _regrow(session)
        sess = session.device_session
    dev = sess.device
    t0 = time.perf_counter_ns()
    res = sess.decode_step(qt.reshape(1, 1, d).to(dev), kt.reshape(1, 1, d).to(dev),
                           vt.reshape(1, 1, d).to(dev), k_fraction, check=True)
    counts = res.counts[0, 0].cpu().numpy()
    total_ns = time.perf_counter_ns() - t0
    out = res.output[0, 0].double().cpu().numpy()
    bypassed = bool(int(res.bypassed[0, 0]))
    rho = float(res.rho[0, 0])
    timings = dict.fromkeys(_STAGES, 0)
    timings["total"] = total_ns
    session.step += 1
    est = SparsityEstimate(math.nan, math.nan, math.nan, rho)
    dots = cfg.sink_count + cfg.local_window + 1
    if bypassed:
        return StepResult(output=out, candidate=CandidateSet(budget_k=0), bypassed=True, rho=rho,
                          sparsity=est, timings_ns=timings, dot_products=dots, clamp_count=0,
                          c0_dropped=0, n_context=n)
    c2 = sess.c2_list(0, 0).astype(np.int64)
    cand = CandidateSet(c0=sess.c0_list(0, 0), c1=sess.c1_list(0, 0),
                        probe=sess.probe_list(0, 0).astype(np.int64), c2=c2,
                        budget_k=int(counts[CNT_K]))
    att_idx = np.concatenate([np.arange(cfg.sink_count, dtype=np.int64), c2])
    return StepResult(output=out, candidate=cand, bypassed=False, rho=rho, sparsity=est,
                      timings_ns=timings, dot_products=dots + int(counts[CNT_PROBE]),
                      clamp_count=int(counts[CNT_CLAMP]), c0_dropped=int(counts[CNT_DROP]),
                      n_context=n, attention=AttentionOutput(out, att_idx, None))


def run_session(session: HeadSession, steps, k_fraction: float,
                config: LfpsConfig | None = None) -> list:
    """Apply decode_step over a (q, new_key, new_value) stream (engine.py:204-219)."""
    results: list = []
    for i, (q, new_key, new_value) in enumerate(steps):
        try:
            results.append(decode_step(session, q, new_key, new_value, k_fraction, config))
        except Exception as e:  # noqa: BLE001 - context preserved on the error
            raise SessionRunError(i, results, e) from e
    if not results:
        raise ValueError("decode stream is empty")
    return results


def exact_topk_step(session: HeadSession, q, k_fraction: float):
    """Exact full-scan Top-k step over the session's rows (bench.py:73-80):
    returns (selected absolute indices, output)."""
    sess = session.device_session
    d = session.config.d
    res = sess.exact_topk_step(_bf16(q, (d,), "q").reshape(1, 1, d).to(sess.device), k_fraction)
    torch.cuda.synchronize(sess.device)
    return sess.c2_list(0, 0).astype(np.int64), res.output[0, 0].double().cpu().numpy()


def full_attention_oracle(q, session: HeadSession) -> AttentionOutput:
    """Exact softmax attention over every stored position (attention.py:88-97),
    on the device; q is a d-vector, the session supplies the rows."""
    sess = session.device_session
    d = session.config.d
    out = sess.full_attention(_bf16(q, (d,), "q").reshape(1, 1, d).to(sess.device))
    torch.cuda.synchronize(sess.device)
    n = sess.n_host[0]
    return AttentionOutput(out[0, 0].double().cpu().numpy(), np.arange(n, dtype=np.int64), None)


def overlap_ratio(c, i_exact, k: int) -> float:
    """eta = |C2 cap I| / k (attention.py:116-124); a host metric."""
    if k < 1:
        raise ValueError("k must be >= 1")
    i_exact = np.asarray(i_exact, dtype=np.int64)
    if i_exact.size != k:
        raise ValueError(f"exact set has {i_exact.size} indices, expected k={k}")
    return int(np.intersect1d(np.asarray(c, dtype=np.int64), i_exact).size) / k


def output_error(approx, exact) -> float:
    """Relative L2 error (attention.py:127-134); a host metric."""
    a = approx.output if isinstance(approx, AttentionOutput) else np.asarray(approx)
    e = exact.output if isinstance(exact, AttentionOutput) else np.asarray(exact)
    if np.shape(a) != np.shape(e):
        raise ValueError(f"shape mismatch: {np.shape(a)} vs {np.shape(e)}")
    return float(np.linalg.norm(np.asarray(a) - np.asarray(e))) / max(
        float(np.linalg.norm(np.asarray(e))), 1e-12)
