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
