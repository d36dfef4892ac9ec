"""Score tables on the device (restates pkg/src/lfps/tables.py:33-331).

``ScoreTablePair`` keeps the reference's representation -- phys values
behind a lazy decay scale, a slash window with headroom on both sides whose
base moves down one slot per update, the parked carry slot, the clamp
counter -- in fp64 device memory.  The update, growth, Eq. 4 seeding and the
threshold moments run in csrc/k_stages.cu; the host keeps the scalars
(scale, base, m) and the buffer management (recentre / capacity doubling
copy values only, as in the reference)."""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np
import torch

from ..config import LfpsConfig
from . import _dev

_RENORM_FLOOR = 1e-120
_DEGENERATE_S2 = 1e-12
_MAX_M = 512 * 512          # stage_thresholds: 512 segments of 512 slots


@dataclass(frozen=True)
class ThresholdPair:
    """Selection thresholds and table means for one step (tables.py:33-46)."""

    tau_ver: float
    tau_sla: float
    mean_ver: float
    mean_sla: float
    ver_degenerate: bool = False
    sla_degenerate: bool = False

    def _device(self) -> torch.Tensor:
        """[tau_v, mean_v, deg_v, tau_s, mean_s, deg_s] (the stage layout)."""
        return _dev.f64([self.tau_ver, self.mean_ver, float(self.ver_degenerate),
                         self.tau_sla, self.mean_sla, float(self.sla_degenerate)])


class ScoreTablePair:
    """Paired vertical/slash score tables for one head, in device memory.

    Logical slot i covers absolute position base_index + i; value(i) =
    scale * phys(i).  Single writer: one update()/grow() per decode step."""

    __slots__ = ("_ver", "_sla", "_sla_base", "_m", "_scale", "_shift_count", "_carry_ready",
                 "base_index", "clamp_count")

    def __init__(self, ver, sla, base_index: int):
        ver = np.asarray(ver, dtype=np.float64)
        sla = np.asarray(sla, dtype=np.float64)
        if ver.shape != sla.shape or ver.ndim != 1:
            raise ValueError("vertical and slash tables must be 1-D and equal length")
        self._init(_dev.f64(ver), _dev.f64(sla), int(base_index))

    def _init(self, ver: torch.Tensor, sla: torch.Tensor, base_index: int):
        m = ver.shape[0]
        cap = max(4 * m, m + 64)
        self._ver = torch.zeros(cap, dtype=_dev.F64, device=ver.device)
        self._ver[:m] = ver
        self._sla = torch.zeros(cap, dtype=_dev.F64, device=ver.device)
        base = (cap - m) // 2
        self._sla[base: base + m] = sla
        self._sla_base = base
        self._m = m
        self._scale = 1.0
        self._shift_count = 0
        self._carry_ready = False
        self.base_index = base_index
        self.clamp_count = 0

    @classmethod
    def _from_device(cls, ver: torch.Tensor, sla: torch.Tensor, base_index: int):
        t = object.__new__(cls)
        t._init(ver, sla, base_index)
        return t

    # -- read side ---------------------------------------------------------
    @property
    def m(self) -> int:
        return self._m

    @property
    def shift(self) -> int:
        return self._shift_count

    @property
    def scale(self) -> float:
        return self._scale

    def ver_values(self) -> np.ndarray:
        """Vertical scores in logical order (fresh host array)."""
        return _dev.host(self._ver[: self._m]) * self._scale

    def sla_values(self) -> np.ndarray:
        b = self._sla_base
        return _dev.host(self._sla[b: b + self._m]) * self._scale

    def ver_at(self, i: int) -> float:
        self._check_index(i)
        return float(self._ver[i]) * self._scale

    def sla_at(self, i: int) -> float:
        self._check_index(i)
        return float(self._sla[self._sla_base + i]) * self._scale

    def sums(self) -> tuple[float, float]:
        b = self._sla_base
        return (float(_dev.host(self._ver[: self._m]).sum() * self._scale),
                float(_dev.host(self._sla[b: b + self._m]).sum() * self._scale))

    def _check_index(self, i: int) -> None:
        if not 0 <= i < self._m:
            raise IndexError(f"logical index {i} out of range [0, {self._m})")

    def _phys(self):
        """(ver phys, sla phys, scale): device views in logical order."""
        b = self._sla_base
        return self._ver[: self._m], self._sla[b: b + self._m], self._scale

    # -- write side ----------------------------------------------------------
    def update(self, selected, weights, r: float) -> int:
        """Decay, slash shift and residual fold at the selected logical
        slots (tables.py:144-200); returns the clamp count."""
        selected = np.asarray(selected, dtype=np.int64)
        weights = np.asarray(weights, dtype=np.float64)
        if selected.size == 0:
            raise ValueError("update requires a non-empty selected set")
        if selected.shape != weights.shape:
            raise ValueError("selected and weights must align")
        if selected.min() < 0 or selected.max() >= self._m:
            raise ValueError("selected logical index out of table range")
        total = float(weights.sum())
        if abs(total - 1.0) > 1e-6:
            raise ValueError(f"selection weights must sum to 1, got {total!r}")
        return self._update_dev(_dev.i64(selected), _dev.f64(weights), r)

    def _update_dev(self, sel: torch.Tensor, w: torch.Tensor, r: float) -> int:
        if self._sla_base == 0:
            self._recenter()
        scale = self._scale * r
        rf, renorm = 1.0, 0
        if scale < _RENORM_FLOOR:
            rf, scale, renorm = scale, 1.0, 1      # _renormalize (tables.py:240-244)
        k = sel.shape[0]
        clamps = torch.zeros(1, dtype=_dev.I64, device=sel.device)
        tmp = torch.empty(k, dtype=_dev.F64, device=sel.device)
        _dev.call("lfps_stage_update", _dev.ptr(self._ver), _dev.ptr(self._sla), self._sla_base,
                  self._m, _dev.ptr(sel), _dev.ptr(w), k, renorm, rf, scale, _dev.ptr(clamps),
                  _dev.ptr(tmp), _dev.stream())
        self._scale = scale
        self._sla_base -= 1
        self._shift_count += 1
        self._carry_ready = True
        n = int(clamps.item())
        self.clamp_count += n
        return n

    def grow(self) -> None:
        """Expose one new logical slot after a KV append (tables.py:202-220)."""
        m = self._m
        if m == self._ver.shape[0]:
            new = torch.zeros(2 * m, dtype=_dev.F64, device=self._ver.device)
            new[:m] = self._ver[:m]
            self._ver = new
        if self._sla_base + m >= self._sla.shape[0]:
            self._recenter()
        _dev.call("lfps_stage_grow", _dev.ptr(self._ver), _dev.ptr(self._sla), self._sla_base, m,
                  1 if self._carry_ready else 0, _dev.stream())
        self._carry_ready = False
        self._m = m + 1

    def _recenter(self) -> None:
        m = self._m
        extent = m + 1                         # keep a parked carry slot if present
        cap = max(self._sla.shape[0] * 2, 4 * extent)
        new = torch.zeros(cap, dtype=_dev.F64, device=self._sla.device)
        base = (cap - extent) // 2
        old = self._sla[self._sla_base: self._sla_base + extent]
        new[base: base + old.shape[0]] = old
        self._sla = new
        self._sla_base = base


def init_tables(prefill_weights, config: LfpsConfig) -> ScoreTablePair:
    """Eq. 4 seeding from the trailing prefill weights (tables.py:247-281)."""
    if isinstance(prefill_weights, torch.Tensor):
        w = prefill_weights.to(_dev.device(), _dev.F64).contiguous()
    else:
        w = np.asarray(prefill_weights, dtype=np.float64)
        if w.ndim != 2:
            raise ValueError("prefill weights must be a (s, m) matrix")
        w = _dev.f64(w)
    if w.dim() != 2:
        raise ValueError("prefill weights must be a (s, m) matrix")
    s, m = w.shape
    if s != config.s:
        raise ValueError(f"expected {config.s} prefill weight vectors, got {s}")
    if m < 1:
        raise ValueError("prefill weight vectors are empty")
    ver = torch.empty(m, dtype=_dev.F64, device=w.device)
    sla = torch.empty(m, dtype=_dev.F64, device=w.device)
    _dev.call("lfps_stage_init_tables", _dev.ptr(w), s, m, float(config.r), _dev.ptr(ver),
              _dev.ptr(sla), _dev.stream())
    return ScoreTablePair._from_device(ver, sla, config.sink_count)


def update_tables(tables: ScoreTablePair, selected_abs, weights, config: LfpsConfig) -> int:
    """Fold one step's selection weights into the tables (absolute indices)."""
    selected_abs = np.asarray(selected_abs, dtype=np.int64)
    return tables.update(selected_abs - tables.base_index, weights, config.r)


def grow_tables(tables: ScoreTablePair, config: LfpsConfig) -> None:
    """Extend the tables by one slot after a KV append."""
    tables.grow()


def _thresholds(tables: ScoreTablePair, config: LfpsConfig, materialize: int) -> ThresholdPair:
    if tables.m < 2:
        raise ValueError("thresholds require at least 2 table slots")
    if tables.m > _MAX_M:
        raise ValueError(f"thresholds on the device support m <= {_MAX_M}")
    ver, sla, scale = tables._phys()
    out = torch.zeros(7, dtype=_dev.F64, device=ver.device)
    scratch = torch.empty(4096, dtype=_dev.F64, device=ver.device)
    _dev.call("lfps_stage_thresholds", _dev.ptr(ver), _dev.ptr(sla), tables.m, float(scale),
              float(config.a), materialize, _dev.ptr(out), _dev.ptr(scratch), _dev.stream())
    o = _dev.host(out)
    if o[6] == 3.0:
        raise ZeroDivisionError("float division by zero")
    return ThresholdPair(float(o[0]), float(o[3]), float(o[1]), float(o[4]), bool(o[2]),
                         bool(o[5]))


def compute_thresholds(tables: ScoreTablePair, config: LfpsConfig) -> ThresholdPair:
    """Peakedness-adaptive thresholds (tables.py:295-317): per table
    kappa = sum c^4 / (sum c^2)^2, tau = a * mean / kappa, degenerate when the
    centred spread is below 1e-12; canonical fp64 moments on the device."""
    return _thresholds(tables, config, 0)


def thresholds_oracle(tables: ScoreTablePair, config: LfpsConfig) -> ThresholdPair:
    """The same on materialised values (tables.py:320-331)."""
    return _thresholds(tables, config, 1)


del math
