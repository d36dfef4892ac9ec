"""Load the committed golden vectors (tests/golden/*.npz) made by the
reference package itself (tests/golden/make_golden.py)."""

from __future__ import annotations

import ast
import glob
import os
from dataclasses import dataclass

import numpy as np

GOLDEN_DIR = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def bits_to_f32(bits: np.ndarray) -> np.ndarray:
    return (bits.astype(np.uint32) << 16).view(np.float32)


@dataclass
class Golden:
    name: str
    n0: int
    steps: int
    d: int
    G: int
    sink: int
    s: int
    frac: float
    cfg: dict
    keys: np.ndarray       # f32 (bf16 values) [n0 + steps, d]
    values: np.ndarray
    weights: np.ndarray    # f32 [G, s, n0 - sink]
    finals: np.ndarray     # [G, d]
    queries: np.ndarray    # [steps, G, d]
    raw: dict

    def sets(self, key: str):
        lens = self.raw[key + "_len"]
        cat = self.raw[key + "_cat"]
        offs = np.concatenate([[0], np.cumsum(lens)])
        return [cat[offs[i]: offs[i + 1]] for i in range(lens.size)]

    def per_step(self, key: str):
        return self.raw[key].reshape(self.steps, self.G, *self.raw[key].shape[1:])


def load(name: str) -> Golden:
    z = dict(np.load(os.path.join(GOLDEN_DIR, name + ".npz")))
    n0, steps, d, G, sink, s = (int(v) for v in z["meta"])
    return Golden(name=name, n0=n0, steps=steps, d=d, G=G, sink=sink, s=s,
                  frac=float(z["frac"]), cfg=ast.literal_eval(str(z["cfg_json"])),
                  keys=bits_to_f32(z["keys"]), values=bits_to_f32(z["values"]),
                  weights=z["weights"], finals=bits_to_f32(z["finals"]),
                  queries=bits_to_f32(z["queries"]), raw=z)


def names():
    return sorted(os.path.splitext(os.path.basename(p))[0]
                  for p in glob.glob(os.path.join(GOLDEN_DIR, "*.npz")))


# ---------------------------------------------------------------------------
# seeded goldens (tests/golden/make_golden_seeded.py): reference outputs for
# inputs regenerated from a workload spec, pinned by a SHA-256
# ---------------------------------------------------------------------------

SEEDED_DIR = os.path.join(GOLDEN_DIR, "seeded")


@dataclass
class Seeded:
    name: str
    spec: object           # workload.GqaSpec
    cfg: dict
    fracs: np.ndarray      # per step
    K: np.ndarray          # f32 [Hkv, n0 + T, d]
    V: np.ndarray
    W: np.ndarray          # f32 [Hkv, G, s, m0]
    F: np.ndarray          # [Hkv, G, d]
    Q: np.ndarray          # [Hkv, G, T, d]
    raw: dict

    def sets(self, key: str):
        lens = self.raw[key + "_len"]
        cat = self.raw[key + "_cat"].astype(np.int64)
        offs = np.concatenate([[0], np.cumsum(lens)])
        return [cat[offs[i]: offs[i + 1]] for i in range(lens.size)]


def seeded_names():
    return sorted(os.path.splitext(os.path.basename(p))[0]
                  for p in glob.glob(os.path.join(SEEDED_DIR, "*.npz")))


def load_seeded(name: str) -> Seeded:
    import sys
    sys.path.insert(0, GOLDEN_DIR)
    from make_golden_seeded import case_inputs
    z = dict(np.load(os.path.join(SEEDED_DIR, name + ".npz")))
    case = {"spec": ast.literal_eval(str(z["spec"]))}
    spec, (K, V, W, F, Q), digest = case_inputs(case)
    if digest != str(z["sha256"]):
        raise AssertionError(
            f"seeded golden {name}: the regenerated inputs hash to {digest}, the fixture "
            f"was made from {z['sha256']} (torch CPU RNG / BLAS differ on this host)")
    return Seeded(name=name, spec=spec, cfg=ast.literal_eval(str(z["cfg_json"])),
                  fracs=z["fracs"], K=K, V=V, W=W, F=F, Q=Q, raw=z)
