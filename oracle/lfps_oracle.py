"""CPU restatement of the LFPS decode step (arXiv 2506.15704) for GQA units.

TEST INFRASTRUCTURE ONLY.  This module is the checker for the B200 kernels.
Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / reference
arm may import it; the product package never does.

It restates the reference path pkg/src/lfps (engine.py:97-201 and the stage
functions it calls) with the state laid out exactly like the device state:

* a (request, KV-head) *unit* owns one K/V row store shared by its G query
  heads (the reference has no GQA; every q-head is an independent
  reference session that happens to see identical K/V rows);
* every q-head *session* owns a TrackerState: the vertical phys table, the
  slash table as a ring buffer (phys slot of logical i = (base + i) mod C),
  the lazy decay scale, the parked-carry flag and the clamp counter
  (tables.py:49-244; the ring reproduces _recenter / base decrement bit for
  bit because recentring never does arithmetic).

Two arithmetic modes share all control flow:

* ``RefArith``  -- the reference's own numpy expressions (x.mean(), c.sum(),
  np.dot, BLAS gemv, np.exp, math.exp).  With ``score="fp64"`` it reproduces
  the reference package bit for bit on the same machine; pinned against
  golden vectors produced by the reference itself (tests/golden/).
* ``DevArith``  -- the canonical device arithmetic of oracle/devmath.py, with
  fp32 probe scores (``score="fp32"``).  The CUDA kernels match it bit for bit
  on every index set, table entry and scalar; outputs match to a stated
  tolerance.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

from . import devmath as dm

RENORM_FLOOR = 1e-120       # tables.py:29
DEGENERATE_S2 = 1e-12       # tables.py:30
_EMPTY = np.empty(0, dtype=np.int64)


# --------------------------------------------------------------------------
# arithmetic modes
# --------------------------------------------------------------------------

class RefArith:
    """numpy arithmetic exactly as the reference evaluates it."""

    name = "ref"

    @staticmethod
    def moments(x, off=0):
        # tables.py:135-140 (mean, subtract, square, sum, dot); off unused
        x = np.ascontiguousarray(x, dtype=np.float64)
        mean = float(x.mean())
        c = x - mean
        c = c * c
        return mean, float(c.sum()), float(np.dot(c, c))

    @staticmethod
    def logits64(rows, q, d):
        # numerics.py:41-49: dot first, then divide by sqrt(d)
        out = rows @ q
        out /= math.sqrt(d)
        return out

    @staticmethod
    def gate_terms(q, sink_keys, local_rows, mean_key, sigma_hat_sq, d):
        sl = RefArith.logits64(sink_keys, q, d)
        ll = RefArith.logits64(local_rows, q, d)
        g = float(q @ mean_key) / math.sqrt(d) + float(q @ q) * sigma_hat_sq / 2.0
        return sl, ll, g

    @staticmethod
    def gate_mass(sl, ll, g, n_nonsink):
        # gate.py:101-114
        shift = max(float(sl.max()), float(ll.max()), g)
        w_sink = float(np.exp(sl - shift).sum())
        w_local = float(np.exp(ll - shift).sum())
        w_global = math.exp(g - shift) * n_nonsink
        return w_sink, w_global, w_local

    @staticmethod
    def softmax(z):
        z = np.asarray(z, dtype=np.float64)
        w = np.exp(z - z.max())
        w /= w.sum()
        return w

    @staticmethod
    def weight_total(u):
        return float(u.sum())

    @staticmethod
    def head_sigma(keys_ns, q, d):
        # gate.py:61-67
        qq = float(q @ q)
        logits = keys_ns @ q / math.sqrt(d)
        return float(np.var(logits)) / qq, qq

    @staticmethod
    def exp_scalar(x):
        return math.exp(x)


class DevArith:
    """Canonical device arithmetic (oracle/devmath.py)."""

    name = "dev"

    @staticmethod
    def moments(x, off=0):
        return dm.table_moments(x, off)

    @staticmethod
    def logits64(rows, q, d):
        return dm.gdot(rows, q) / math.sqrt(d)

    @staticmethod
    def gate_terms(q, sink_keys, local_rows, mean_key, sigma_hat_sq, d):
        sd = math.sqrt(d)
        sl = dm.gdot(sink_keys, q) / sd
        ll = dm.gdot(local_rows, q) / sd
        qk = float(dm.gdot(q, mean_key))
        qq = float(dm.gdot(q, q))
        g = qk / sd + qq * sigma_hat_sq / 2.0
        return sl, ll, g

    @staticmethod
    def gate_mass(sl, ll, g, n_nonsink):
        shift = max(float(sl.max()), float(ll.max()), g)
        w_sink = dm.seq_sum(dm.cexp(sl - shift))
        w_local = dm.seq_sum(dm.cexp(ll - shift))
        w_global = float(dm.cexp(np.float64(g - shift))) * n_nonsink
        return w_sink, w_global, w_local

    @staticmethod
    def softmax(z):
        return dm.softmax_update(z)

    @staticmethod
    def weight_total(u):
        return dm.block_sum(u)

    @staticmethod
    def head_sigma(keys_ns, q, d):
        qq = float(dm.gdot(q, q))
        logits = dm.gdot(keys_ns, q) / math.sqrt(d)
        cnt = logits.shape[0]
        mu = dm.table_sum(logits) / cnt
        dev = logits - mu
        var = dm.table_sum(dev * dev) / cnt
        return var / qq, qq

    @staticmethod
    def exp_scalar(x):
        return float(dm.cexp(np.float64(x)))


ARITH = {"ref": RefArith, "dev": DevArith}


# --------------------------------------------------------------------------
# state
# --------------------------------------------------------------------------

@dataclass
class TrackerState:
    """One session's score tables in device layout (tables.py:49-81)."""

    ver: np.ndarray          # [Mcap] phys vertical table, logical i at i
    ring: np.ndarray         # [C] phys slash ring, logical i at (base+i) % C
    base: int
    m: int
    scale: float = 1.0
    carry: bool = False
    clamp_count: int = 0
    vbase: int = 0           # virtual slot of slash logical 0 (devmath.table_moments)

    def ver_view(self) -> np.ndarray:
        return self.ver[: self.m]

    def sla_slots(self, logical) -> np.ndarray:
        return (self.base + np.asarray(logical, dtype=np.int64)) % self.ring.shape[0]

    def sla_view(self) -> np.ndarray:
        return self.ring[self.sla_slots(np.arange(self.m))]

    def values(self) -> tuple[np.ndarray, np.ndarray]:
        """Materialised table values phys * scale (tables.py:94-101)."""
        return self.ver_view() * self.scale, self.sla_view() * self.scale

    def copy(self) -> "TrackerState":
        return TrackerState(self.ver.copy(), self.ring.copy(), self.base, self.m,
                            self.scale, self.carry, self.clamp_count, self.vbase)


@dataclass
class HeadPriors:
    """Frozen per-session priors (gate.py:21-34)."""

    mean_key: np.ndarray
    mean_value: np.ndarray
    sigma_hat_sq: float


@dataclass
class UnitKV:
    """K/V rows of one (request, KV-head), fp64 upcast of the bf16 cache."""

    keys: np.ndarray         # [cap, d]
    values: np.ndarray       # [cap, d]
    n: int

    def append(self, k, v):
        if self.n >= self.keys.shape[0]:
            grow = max(64, self.keys.shape[0])
            self.keys = np.concatenate([self.keys, np.zeros((grow, self.keys.shape[1]))])
            self.values = np.concatenate([self.values, np.zeros((grow, self.values.shape[1]))])
        self.keys[self.n] = k
        self.values[self.n] = v
        self.n += 1


@dataclass
class StepOut:
    """Observable result of one session-step (engine.py:50-64)."""

    output: np.ndarray
    bypassed: bool
    rho: float
    c0: np.ndarray = field(default_factory=lambda: _EMPTY)
    c1: np.ndarray = field(default_factory=lambda: _EMPTY)
    probe: np.ndarray = field(default_factory=lambda: _EMPTY)
    c2: np.ndarray = field(default_factory=lambda: _EMPTY)
    probe_scores: np.ndarray = field(default_factory=lambda: np.empty(0))
    budget_k: int = 0
    clamps: int = 0
    dot_products: int = 0
    thresholds: tuple = ()
    weights: np.ndarray | None = None

    @property
    def c0_dropped(self) -> int:
        if self.c0.size == 0:
            return 0
        return int(self.c0.size - np.isin(self.c0, self.c1).sum())


# --------------------------------------------------------------------------
# bootstrap (engine.py:67-94, tables.py:247-281, gate.py:51-74)
# --------------------------------------------------------------------------

def seed_tables(weights: np.ndarray, cfg, mcap: int | None = None,
                ring_cap: int | None = None) -> TrackerState:
    """Eq. 4 seeding: column sums for vertical, diagonal sums for slash.

    Rows are accumulated oldest first, matching numpy's axis-0 order, so the
    result is bit-identical to the reference's init_tables."""
    w = np.asarray(weights, dtype=np.float64)
    if w.ndim != 2:
        raise ValueError("prefill weights must be a (s, m) matrix")
    s, m = w.shape
    if s != cfg.s:
        raise ValueError(f"expected {cfg.s} prefill weight vectors, got {s}")
    if m < 1:
        raise ValueError("prefill weight vectors are empty")
    coeff = 1.0 / (2.0 * s * (1.0 - cfg.r))
    col = np.zeros(m)
    diag = np.zeros(m)
    for c in range(s):
        col = col + w[c]
        lag = s - 1 - c                 # distance of row c from the newest step
        if lag < m:
            diag[lag:] = diag[lag:] + w[c, : m - lag]
    mcap = mcap or (m + 64)
    ring_cap = ring_cap or (mcap + 2)
    ver = np.zeros(mcap)
    ver[:m] = col * coeff
    ring = np.zeros(ring_cap)
    ring[:m] = diag * coeff
    return TrackerState(ver=ver, ring=ring, base=0, m=m, vbase=-m)


def head_priors(keys, values, last_query, cfg, arith) -> HeadPriors:
    keys = np.asarray(keys, dtype=np.float64)
    values = np.asarray(values, dtype=np.float64)
    n, d = keys.shape
    S = cfg.sink_count
    if n <= S + 1:
        raise ValueError(f"need more than sink_count + 1 = {S + 1} rows, have {n}")
    q = np.asarray(last_query, dtype=np.float64)
    kns = keys[S:]
    sig, qq = arith.head_sigma(kns, q, d)
    if qq == 0.0:
        raise ValueError("zero-norm prefill query")
    cnt = kns.shape[0]
    return HeadPriors(mean_key=kns.sum(axis=0) / cnt,
                      mean_value=values[S:].sum(axis=0) / cnt,
                      sigma_hat_sq=sig)


def bootstrap_unit(keys, values, prefill_weights, last_queries, cfg, arith,
                   headroom: int = 64):
    """Build one unit: shared KV plus G (tracker, priors) sessions."""
    keys = np.asarray(keys, dtype=np.float64)
    values = np.asarray(values, dtype=np.float64)
    n, d = keys.shape
    if d != cfg.d:
        raise ValueError(f"keys must be (n, {cfg.d})")
    if n <= cfg.sink_count + cfg.s:
        raise ValueError("prefill needs more than sink_count + s rows")
    cap = n + headroom
    kv = UnitKV(np.zeros((cap, d)), np.zeros((cap, d)), n)
    kv.keys[:n] = keys
    kv.values[:n] = values
    trackers, priors = [], []
    for w, q in zip(prefill_weights, last_queries):
        w = np.asarray(w, dtype=np.float64)
        if w.shape != (cfg.s, n - cfg.sink_count):
            raise ValueError("prefill weights have the wrong shape")
        if np.any(np.abs(w.sum(axis=1) - 1.0) > 1e-4):
            raise ValueError("each prefill weight vector must sum to 1")
        trackers.append(seed_tables(w, cfg, mcap=cap))
        priors.append(head_priors(keys, values, q, cfg, arith))
    return kv, trackers, priors


# --------------------------------------------------------------------------
# decode-step stages
# --------------------------------------------------------------------------

def thresholds(tr: TrackerState, cfg, arith):
    """(tau_v, tau_s, mean_v, mean_s, deg_v, deg_s) -- tables.py:295-317."""
    if cfg.exhaustive_fallback:
        ninf = float("-inf")
        return (ninf, ninf, ninf, ninf, False, False)
    if tr.m < 2:
        raise ValueError("thresholds require at least 2 table slots")
    res = []
    for x, off in ((tr.ver_view(), 0), (tr.sla_view(), tr.vbase)):
        mean_p, s2_p, s4_p = arith.moments(x, off)
        mean = mean_p * tr.scale
        s2 = s2_p * tr.scale * tr.scale
        if s2 < DEGENERATE_S2:
            res.append((float("nan"), mean, True))
        else:
            kappa = s4_p / (s2_p * s2_p)
            res.append((cfg.a * mean / kappa, mean, False))
    (tv, mv, dv), (ts, ms, ds) = res
    return (tv, ts, mv, ms, dv, ds)


def candidates(tr: TrackerState, th, cfg, n: int):
    """C0, C1 and probe as sorted absolute indices (candidates.py:45-100)."""
    tv, ts, mv, ms, dv, ds = th
    S = cfg.sink_count
    ver, sla, sc = tr.ver_view(), tr.sla_view(), tr.scale
    hit = np.zeros(tr.m, dtype=bool)
    if not dv:
        hit |= ver > (tv / sc)
    if not ds:
        hit |= sla > (ts / sc)
    c0_log = np.nonzero(hit)[0].astype(np.int64)
    if c0_log.size:
        offs = np.asarray(cfg.expansion_offsets, dtype=np.int64)
        cand = (c0_log[:, None] + offs[None, :]).ravel()
        cand = np.unique(cand[(cand >= 0) & (cand < tr.m)])
        above = (ver[cand] > mv / sc) | (sla[cand] > ms / sc)
        c1_log = cand[above]
    else:
        c1_log = _EMPTY
    if n <= S:
        raise ValueError("store holds only sink positions")
    tail = np.arange(max(S, n - cfg.local_window), n, dtype=np.int64)
    c1 = c1_log + S
    probe = np.union1d(c1, tail) if c1.size else tail
    return c0_log + S, c1, probe


def budget_k(frac: float, n: int) -> int:
    """k = max(1, round(frac * n)), Python round-half-even (engine.py:167)."""
    return max(1, round(frac * n))


def topk_lower_index(idx: np.ndarray, scores: np.ndarray, k: int) -> np.ndarray:
    """Top-k with lower-index tie-break over sorted idx (attention.py:34-47)."""
    p = idx.shape[0]
    if k >= p:
        return idx.copy()
    kth = np.partition(scores, p - k)[p - k]
    keep = idx[scores > kth]
    short = k - keep.shape[0]
    if short > 0:
        keep = np.concatenate([keep, idx[scores == kth][:short]])
    return np.sort(keep)


def probe_scores(kv: UnitKV, probe, q, d, score: str):
    if score == "fp64":
        rows = kv.keys[: kv.n][probe]
        return RefArith.logits64(rows, q, d)
    rows = kv.keys[: kv.n][probe].astype(np.float32)
    return dm.sdot32(rows, q.astype(np.float32), dm.rsd_f32(d)).astype(np.float64)


def apply_update(tr: TrackerState, c2_log: np.ndarray, u: np.ndarray, r: float,
                 total: float) -> int:
    """Decay, slash shift and residual fold (tables.py:144-200), ring form."""
    if c2_log.size == 0:
        raise ValueError("update requires a non-empty selected set")
    if abs(total - 1.0) > 1e-6:
        raise ValueError(f"selection weights must sum to 1, got {total!r}")
    C = tr.ring.shape[0]
    tr.scale *= r
    if tr.scale < RENORM_FLOOR:
        tr.ver[: tr.m] *= tr.scale
        slots = tr.sla_slots(np.arange(tr.m + 1))
        tr.ring[slots] *= tr.scale
        tr.scale = 1.0
    tr.base = (tr.base - 1) % C
    tr.vbase -= 1
    tr.ring[tr.base] = 0.0
    tr.carry = True
    k = c2_log.size
    add = (u - 1.0 / (2.0 * k)) / tr.scale
    tr.ver[c2_log] += add
    slots = tr.sla_slots(c2_log)
    tr.ring[slots] += add
    clamps = 0
    v = tr.ver[c2_log]
    neg = v < 0.0
    if neg.any():
        clamps += int(neg.sum())
        v[neg] = 0.0
        tr.ver[c2_log] = v
    sv = tr.ring[slots]
    neg = sv < 0.0
    if neg.any():
        clamps += int(neg.sum())
        sv[neg] = 0.0
        tr.ring[slots] = sv
    tr.clamp_count += clamps
    return clamps


def grow(tr: TrackerState):
    """Expose one slot after the KV append (tables.py:202-220)."""
    if tr.m + 2 > tr.ring.shape[0] or tr.m + 1 > tr.ver.shape[0]:
        nv = np.zeros(max(tr.ver.shape[0] * 2, tr.m + 2))
        nv[: tr.m] = tr.ver[: tr.m]
        slots = tr.sla_slots(np.arange(tr.m + 1))
        nr = np.zeros(nv.shape[0] + 2)
        nr[: tr.m + 1] = tr.ring[slots]
        tr.ver, tr.ring, tr.base = nv, nr, 0
    tr.ver[tr.m] = 0.0
    if not tr.carry:
        tr.ring[(tr.base + tr.m) % tr.ring.shape[0]] = 0.0
    tr.carry = False
    tr.m += 1


def session_step(kv: UnitKV, tr: TrackerState, pri: HeadPriors, q, frac, cfg,
                 arith, score: str = "fp64") -> StepOut:
    """One session's decode step against the pre-append rows [0, n).

    Mutates ``tr`` (update + grow); the caller appends the unit's KV row once
    for all of its sessions.  engine.py:97-201."""
    d = cfg.d
    S, L = cfg.sink_count, cfg.local_window
    q = np.asarray(q, dtype=np.float64)
    n = kv.n
    if q.shape != (d,):
        raise ValueError(f"q must have shape ({d},)")
    if not 0.0 < frac <= 1.0:
        raise ValueError(f"k_fraction must be in (0, 1], got {frac}")
    if tr.m != n - S:
        raise ValueError("tables out of sync with the KV store")
    if n <= S + L:
        raise ValueError("context shorter than sink_count + local_window")
    keys = kv.keys[:n]
    sink_keys = keys[:S]
    local_rows = keys[np.arange(n - L, n, dtype=np.int64)]
    sl, ll, g = arith.gate_terms(q, sink_keys, local_rows, pri.mean_key,
                                 pri.sigma_hat_sq, d)
    if not (np.all(np.isfinite(sl)) and np.all(np.isfinite(ll)) and math.isfinite(g)):
        raise ValueError("non-finite logits in sparsity estimate")
    w_s, w_g, w_l = arith.gate_mass(sl, ll, g, n - S)
    rho = w_s / (w_s + w_g + w_l)
    if not math.isfinite(rho):
        raise ValueError("non-finite sparsity ratio")
    dots = S + L + 1
    if rho > cfg.epsilon:
        # gate.py:131-147
        if cfg.bypass_mode == "mean_only":
            out = pri.mean_value.copy()
        else:
            w = arith.softmax(np.concatenate([sl, [g]]))
            if arith is RefArith:
                out = w[:-1] @ kv.values[:S] + w[-1] * pri.mean_value
            else:
                out = np.zeros(d)
                for i in range(S):
                    out = out + w[i] * kv.values[i]
                out = out + w[S] * pri.mean_value
        grow(tr)
        return StepOut(output=out, bypassed=True, rho=rho, dot_products=dots)

    th = thresholds(tr, cfg, arith)
    c0, c1, probe = candidates(tr, th, cfg, n)
    k = budget_k(frac, n)
    z = probe_scores(kv, probe, q, d, score)
    dots += probe.size
    c2 = topk_lower_index(probe, z, k)
    zc2 = z[np.searchsorted(probe, c2)]
    att_idx = np.concatenate([np.arange(S, dtype=np.int64), c2])
    if score == "fp64":
        sink_z = sl
    else:
        sink_z = dm.sdot32(keys[:S].astype(np.float32), q.astype(np.float32),
                           dm.rsd_f32(d)).astype(np.float64)
    att_w = RefArith.softmax(np.concatenate([sink_z, zc2]))
    out = att_w @ kv.values[att_idx]
    u = arith.softmax(zc2)
    total = arith.weight_total(u)
    clamps = apply_update(tr, c2 - S, u, cfg.r, total)
    grow(tr)
    return StepOut(output=out, bypassed=False, rho=rho, c0=c0, c1=c1, probe=probe,
                   c2=c2, probe_scores=z, budget_k=k, clamps=clamps,
                   dot_products=dots, thresholds=th, weights=att_w)


def unit_step(kv: UnitKV, trackers, priors, qs, k_new, v_new, frac, cfg, arith,
              score="fp64") -> list[StepOut]:
    """All G sessions of a unit step against the same pre-append rows, then
    the unit appends its new K/V row (engine.py:188-191)."""
    outs = [session_step(kv, tr, pri, q, frac, cfg, arith, score)
            for tr, pri, q in zip(trackers, priors, qs)]
    kv.append(np.asarray(k_new, dtype=np.float64), np.asarray(v_new, dtype=np.float64))
    return outs


# --------------------------------------------------------------------------
# exact comparison path and metrics (bench.py:73-80, attention.py:66-134)
# --------------------------------------------------------------------------

def exact_topk_step(kv: UnitKV, q, k: int, cfg, score: str = "fp64"):
    """Full-range scores, bounded Top-k, joint sink+selection output."""
    d = cfg.d
    S = cfg.sink_count
    n = kv.n
    q = np.asarray(q, dtype=np.float64)
    idx = np.arange(S, n, dtype=np.int64)
    z = probe_scores(kv, idx, q, d, score)
    sel = topk_lower_index(idx, z, k)
    att = np.union1d(np.arange(S, dtype=np.int64), sel)
    if score == "fp64":
        logits = RefArith.logits64(kv.keys[:n][att], q, d)
    else:
        logits = dm.sdot32(kv.keys[:n][att].astype(np.float32), q.astype(np.float32),
                           dm.rsd_f32(d)).astype(np.float64)
    w = RefArith.softmax(logits)
    return sel, w @ kv.values[:n][att]


def topk_oracle(kv: UnitKV, q, k: int, sink: int, score: str = "fp64"):
    """Exact Top-k via a full stable sort (attention.py:100-113)."""
    d = kv.keys.shape[1]
    idx = np.arange(sink, kv.n, dtype=np.int64)
    z = probe_scores(kv, idx, np.asarray(q, dtype=np.float64), d, score)
    order = np.lexsort((idx, -z))
    return np.sort(idx[order[: min(k, idx.size)]])


def overlap_ratio(c, exact, k: int) -> float:
    """eta = |C2 cap I| / k (attention.py:116-124)."""
    return int(np.intersect1d(np.asarray(c), np.asarray(exact)).size) / k


def output_error(approx, exact) -> float:
    """Relative L2 error (attention.py:127-134)."""
    a, e = np.asarray(approx, dtype=np.float64), np.asarray(exact, dtype=np.float64)
    return float(np.linalg.norm(a - e)) / max(float(np.linalg.norm(e)), 1e-12)
