"""B200-native KIFMM evaluate (drop-in for the evaluate section of SPEC.md `run`)."""
from .errors import (CacheMismatch, CorruptArchive, DeviceError, InvalidArgument, IoError,  # noqa: F401
                     KifmmError, NumericalError)

__version__ = "0.1.0"
