"""Candidate construction on the device (restates pkg/src/lfps/candidates.py).

select_initial (Eq. 7), expand (Eq. 9) and finalize_probe_set run as
k_stages.cu kernels over the device tables / store; results are sorted
unique int64 absolute indices (host arrays), as in the reference."""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np
import torch

from ..config import LfpsConfig
from . import _dev
from .store import KvStore
from .tables import ScoreTablePair, ThresholdPair

_EMPTY = np.empty(0, dtype=np.int64)


@dataclass(frozen=True)
class CandidateSet:
    """Index sets produced for one decode step (candidates.py:17-42)."""

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


def _run(mode, tables, thr, in_idx, cfg, n, cap):
    """One stage_candidates launch; returns (device indices [count], count)."""
    dev = _dev.device()
    out = torch.empty(max(cap, 1), dtype=_dev.I64, device=dev)
    cnt = torch.zeros(1, dtype=torch.int32, device=dev)
    if tables is not None:
        ver, sla, scale = tables._phys()
        m = tables.m
        base = tables.base_index
    else:
        ver = sla = None
        scale, m, base = 1.0, 0, 0
    offs = torch.tensor(sorted(set(cfg.expansion_offsets)) if cfg else [0], dtype=torch.int32,
                        device=dev)
    n_in = 0 if in_idx is None else int(in_idx.shape[0])
    _dev.call("lfps_stage_candidates", mode, _dev.ptr(ver), _dev.ptr(sla), m, float(scale),
              _dev.ptr(thr), _dev.ptr(in_idx), n_in, _dev.ptr(offs), int(offs.shape[0]),
              int(base), int(n), int(cfg.sink_count) if cfg else 0,
              int(cfg.local_window) if cfg else 0, _dev.ptr(out), _dev.ptr(cnt), _dev.stream())
    c = int(cnt.item())
    return out[:c], c


def _select_initial_dev(tables: ScoreTablePair, thresholds: ThresholdPair):
    return _run(0, tables, thresholds._device(), None, None, 0, tables.m)[0]


def _expand_dev(c0: torch.Tensor, tables: ScoreTablePair, thresholds: ThresholdPair,
                config: LfpsConfig):
    if c0.shape[0] == 0:
        return c0
    return _run(1, tables, thresholds._device(), c0, config, 0, tables.m)[0]


def _finalize_dev(c1: torch.Tensor, store: KvStore, config: LfpsConfig):
    n = store.n
    if n <= config.sink_count:
        raise ValueError("store holds only sink positions")
    return _run(2, None, None, c1, config, n, n)[0]


def select_initial(tables: ScoreTablePair, thresholds: ThresholdPair) -> np.ndarray:
    """Slots whose vertical or slash score strictly exceeds its threshold
    (a degenerate table contributes nothing); absolute indices."""
    return _dev.host(_select_initial_dev(tables, thresholds))


def expand(c0, tables: ScoreTablePair, thresholds: ThresholdPair,
           config: LfpsConfig) -> np.ndarray:
    """c0 widened by the offsets, kept where a score exceeds its table mean
    (the zero offset is filtered too: c0 members can drop out)."""
    c0 = np.asarray(c0, dtype=np.int64)
    if c0.size == 0:
        return _EMPTY.copy()
    return _dev.host(_expand_dev(_dev.i64(c0), tables, thresholds, config))


def finalize_probe_set(c1, store: KvStore, config: LfpsConfig) -> np.ndarray:
    """c1 united with the trailing window [max(S, n - L), n)."""
    c1 = np.asarray(c1, dtype=np.int64)
    return _dev.host(_finalize_dev(_dev.i64(c1), store, config))
