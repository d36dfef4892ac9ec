"""B200-native LFPS sparse-index prediction for decode-step attention
(arXiv 2506.15704), drop-in for the reference package ``lfps``
(pkg/src/lfps/__init__.py:13-58).

The decode path runs in hand-written sm_100a kernels (csrc/, built into
lib/liblfps_b200.so) behind a C-ABI (include/lfps_b200.h); this package is
the host side.  ``BatchedSession`` is the batched GPU API (``ShardedSession``
over several GPUs); the reference's whole per-head surface -- the decode
step and every stage, state type and oracle, with the same names, arguments
and errors -- is ``paper_2506_15704_b200.lfps`` (re-exported here), running
on the device at the reference's float64 precision.
"""

from .config import LfpsConfig
from .errors import (BadMagicError, ChecksumError, DeviceError, LayoutError, LfpsError,
                     SessionRunError, TraceFormatError, TruncatedFileError,
                     UnsupportedVersionError)

__version__ = "0.1.0"


_LAZY = {"BatchedSession": "session", "BatchedStepResult": "session",
         "ShardedSession": "sharded", "plan_shards": "sharded",
         # trace container (N2), reports (N3), GPU replay
         "RunReport": "report", "StepRecord": "report", "emit_json": "report",
         "emit_csv": "report", "compute_aggregates": "report",
         "run_trace": "replay", "config_for_trace": "replay"}


def __getattr__(name):
    # device-backed names load lazily so that importing the package (configs,
    # errors, the C-ABI loader) works on machines without a GPU; every name
    # of the reference's surface (pkg/src/lfps/__init__.py:13-58) resolves to
    # the device-backed mirror in .lfps
    import importlib
    if name.startswith("__") or name in ("session", "workload", "_lib", "tracefile", "report",
                                         "replay", "sharded", "lfps", "kv_pool"):
        raise AttributeError(name)
    mod = importlib.import_module(__name__ + "." + _LAZY.get(name, "lfps"))
    if hasattr(mod, name):
        return getattr(mod, name)
    raise AttributeError(name)
