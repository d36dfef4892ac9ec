"""pytest plugin: make `import lfps` (and its submodules) resolve to this
repo's device-backed mirror paper_2506_15704_b200.lfps, so the reference's
own test files run against it (tests/test_gpu_reference_suite.py)."""

import importlib
import sys

import paper_2506_15704_b200.lfps as _pkg

sys.modules["lfps"] = _pkg
for _sub in ("attention", "bench", "candidates", "config", "engine", "errors", "gate",
             "numerics", "report", "store", "synth", "tables", "tracefile"):
    sys.modules["lfps." + _sub] = importlib.import_module("paper_2506_15704_b200.lfps." + _sub)
