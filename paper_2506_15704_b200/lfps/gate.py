"""Head priors and the sparsity gate on the device
(restates pkg/src/lfps/gate.py:21-147).

compute_head_stats, gate_logits, estimate_sparsity run as k_stages.cu
kernels over the store's device rows.  global_exponent,
sparsity_from_logits and bypass_output take HOST arrays in the reference
(logits and priors already computed) and stay host numeric helpers; the
decode step (engine.py) computes its bypass output on the device."""

from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np
import torch

from ..config import LfpsConfig
from . import _dev
from .numerics import DotCounter, softmax_weights
from .store import KvStore


@dataclass(frozen=True)
class HeadStats:
    """Priors frozen at the end of prefill (gate.py:21-34); host arrays,
    with their device copies kept for the decode kernels."""

    sink_keys: np.ndarray
    sink_values: np.ndarray
    mean_key: np.ndarray
    mean_value: np.ndarray
    sigma_hat_sq: float
    _dev_mean_key: torch.Tensor | None = field(default=None, repr=False, compare=False)
    _dev_mean_value: torch.Tensor | None = field(default=None, repr=False, compare=False)

    def _device(self):
        mk = self._dev_mean_key if self._dev_mean_key is not None else _dev.f64(self.mean_key)
        mv = self._dev_mean_value if self._dev_mean_value is not None else _dev.f64(self.mean_value)
        return mk, mv


@dataclass(frozen=True)
class SparsityEstimate:
    """Sink / global / local mass split and the sink share rho (gate.py:37-48)."""

    w_sink: float
    w_global: float
    w_local: float
    rho: float


def compute_head_stats(store: KvStore, last_prefill_query, config: LfpsConfig) -> HeadStats:
    """Freeze the per-head priors from the final prefill step (gate.py:51-74)."""
    n, d = store.n, store.d
    sink = config.sink_count
    if n <= sink + 1:
        raise ValueError(f"need more than sink_count + 1 = {sink + 1} rows, have {n}")
    q = np.asarray(last_prefill_query, dtype=np.float64)
    if q.shape != (d,):
        raise ValueError(f"query must have shape ({d},), got {q.shape}")
    if not np.any(q):
        raise ValueError("zero-norm prefill query")
    dev = _dev.device()
    mk = torch.empty(d, dtype=_dev.F64, device=dev)
    mv = torch.empty(d, dtype=_dev.F64, device=dev)
    sig = torch.empty(1, dtype=_dev.F64, device=dev)
    tmp = torch.empty(n, dtype=_dev.F64, device=dev)
    err = torch.zeros(1, dtype=torch.int32, device=dev)
    _dev.call("lfps_stage_head_stats", _dev.ptr(store._kt), _dev.ptr(store._vt), n, d, sink,
              _dev.ptr(_dev.f64(q)), _dev.ptr(mk), _dev.ptr(mv), _dev.ptr(sig), _dev.ptr(tmp),
              _dev.ptr(err), _dev.stream())
    _dev.raise_code(int(err.item()))
    return HeadStats(sink_keys=_dev.host(store._kt[:sink]).copy(),
                     sink_values=_dev.host(store._vt[:sink]).copy(),
                     mean_key=_dev.host(mk), mean_value=_dev.host(mv),
                     sigma_hat_sq=float(sig.item()), _dev_mean_key=mk, _dev_mean_value=mv)


def global_exponent(q, stats: HeadStats, d: int) -> float:
    """Log of the mean non-sink weight under the log-normal model (host helper)."""
    q = np.asarray(q, dtype=np.float64)
    return float(q @ stats.mean_key) / math.sqrt(d) + float(q @ q) * stats.sigma_hat_sq / 2.0


def _gate_dev(q, store: KvStore, stats: HeadStats, config: LfpsConfig):
    """The gate kernel: host copy of [sink logits | local logits | gexp |
    w_sink | w_global | w_local | rho | bypass output]."""
    n, d = store.n, store.d
    if n <= config.sink_count + config.local_window:
        raise ValueError("context shorter than sink_count + local_window")
    q = np.asarray(q, dtype=np.float64)
    if q.shape != (d,):
        raise ValueError(f"q must have shape ({d},), got {q.shape}")
    S, L = config.sink_count, config.local_window
    dev = _dev.device()
    out = torch.empty(S + L + 5 + d, dtype=_dev.F64, device=dev)
    err = torch.zeros(1, dtype=torch.int32, device=dev)
    mk, mv = stats._device()
    _dev.call("lfps_stage_gate", _dev.ptr(store._kt), _dev.ptr(store._vt), n, d, S, L,
              _dev.ptr(_dev.f64(q)), _dev.ptr(mk), _dev.ptr(mv), float(stats.sigma_hat_sq),
              1 if config.bypass_mode == "mean_only" else 0, _dev.ptr(out), _dev.ptr(err),
              _dev.stream())
    o = _dev.host(out)
    return o, int(err.item())


def gate_logits(q, store: KvStore, stats: HeadStats, config: LfpsConfig,
                counter: DotCounter | None = None):
    """Sink logits, trailing-window logits and the global exponent against
    the pre-append store (gate.py:84-98)."""
    o, _ = _gate_dev(q, store, stats, config)
    S, L = config.sink_count, config.local_window
    if counter is not None:
        counter.add(S + L + 1)
    return o[:S].copy(), o[S:S + L].copy(), float(o[S + L])


def sparsity_from_logits(sink_logits, local_logits, global_exp: float,
                         n_nonsink: int) -> SparsityEstimate:
    """Combine the three mass terms with a shared max shift (host helper,
    gate.py:101-114)."""
    sink_logits = np.asarray(sink_logits, dtype=np.float64)
    local_logits = np.asarray(local_logits, dtype=np.float64)
    if not (np.all(np.isfinite(sink_logits)) and np.all(np.isfinite(local_logits))
            and math.isfinite(global_exp)):
        raise ValueError("non-finite logits in sparsity estimate")
    shift = max(float(sink_logits.max()), float(local_logits.max()), global_exp)
    w_sink = float(np.exp(sink_logits - shift).sum())
    w_local = float(np.exp(local_logits - shift).sum())
    w_global = math.exp(global_exp - shift) * n_nonsink
    rho = w_sink / (w_sink + w_global + w_local)
    if not math.isfinite(rho):
        raise ValueError("non-finite sparsity ratio")
    return SparsityEstimate(w_sink=w_sink, w_global=w_global, w_local=w_local, rho=rho)


def _estimate(o, err, config) -> SparsityEstimate:
    S, L = config.sink_count, config.local_window
    if err == 1:
        raise ValueError("non-finite logits in sparsity estimate")
    if err == 2:
        raise ValueError("non-finite sparsity ratio")
    return SparsityEstimate(w_sink=float(o[S + L + 1]), w_global=float(o[S + L + 2]),
                            w_local=float(o[S + L + 3]), rho=float(o[S + L + 4]))


def estimate_sparsity(q, store: KvStore, stats: HeadStats, config: LfpsConfig,
                      counter: DotCounter | None = None) -> SparsityEstimate:
    """Sink share of the head's attention mass for this step, on the device
    (S + L + 1 dot products, gate.py:117-128)."""
    o, err = _gate_dev(q, store, stats, config)
    if counter is not None:
        counter.add(config.sink_count + config.local_window + 1)
    return _estimate(o, err, config)


def bypass_output(q, stats: HeadStats, config: LfpsConfig, sink_logits=None) -> np.ndarray:
    """Output of a gated head (host helper over the frozen priors,
    gate.py:131-147)."""
    if config.bypass_mode == "mean_only":
        return stats.mean_value.copy()
    q = np.asarray(q, dtype=np.float64)
    d = stats.mean_key.shape[0]
    if sink_logits is None:
        sink_logits = stats.sink_keys @ q / math.sqrt(d)
    logits = np.concatenate([np.asarray(sink_logits, dtype=np.float64),
                             [global_exponent(q, stats, d)]])
    w = softmax_weights(logits)
    return w[:-1] @ stats.sink_values + w[-1] * stats.mean_value
