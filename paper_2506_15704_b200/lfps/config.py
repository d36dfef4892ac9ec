"""LfpsConfig (pkg/src/lfps/config.py:11-82)."""
from ..config import LfpsConfig  # noqa: F401
