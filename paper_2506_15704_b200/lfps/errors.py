"""Exception tree (pkg/src/lfps/errors.py:4-43)."""
from ..errors import (BadMagicError, ChecksumError, LayoutError, LfpsError,  # noqa: F401
                      SessionRunError, TraceFormatError, TruncatedFileError,
                      UnsupportedVersionError)
