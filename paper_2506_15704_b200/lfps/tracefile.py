"""LFPS v1 trace container (pkg/src/lfps/tracefile.py:92-197)."""
from ..tracefile import (HeadTrace, TraceFile, load_trace, read_trace,  # noqa: F401
                         save_trace, write_trace)
