"""Drive the CPU oracle over a golden case (shared by several tests)."""

from __future__ import annotations

import numpy as np

from oracle import lfps_oracle as lo
from paper_2506_15704_b200.config import LfpsConfig


def golden_config(g) -> LfpsConfig:
    return LfpsConfig(d=g.d, s=g.s, sink_count=g.sink, **g.cfg)


def run_oracle(g, arith: str = "ref", score: str = "fp64", steps: int | None = None):
    """Run the oracle over golden case ``g``; returns (per-step outs [t][g],
    trackers, priors, unit kv)."""
    cfg = golden_config(g)
    ar = lo.ARITH[arith]
    n0 = g.n0
    kv, trackers, priors = lo.bootstrap_unit(g.keys[:n0], g.values[:n0], g.weights,
                                             g.finals, cfg, ar)
    outs = []
    for t in range(steps if steps is not None else g.steps):
        outs.append(lo.unit_step(kv, trackers, priors, g.queries[t], g.keys[n0 + t],
                                 g.values[n0 + t], g.frac, cfg, ar, score))
    return outs, trackers, priors, kv


def flatten(outs):
    return [o for step in outs for o in step]
