"""Error taxonomy of the reference (proj/src/common.hpp:19-49) on the Python side.

Every C-ABI status code (include/kifmm.h) maps to exactly one class here.
"""


class KifmmError(Exception):
    """Base class of all library errors."""


class InvalidArgument(KifmmError, ValueError):
    """Bad caller input (common.hpp:19-25)."""


class IoError(KifmmError, OSError):
    """Filesystem failure on particle files or caches (common.hpp:26-31)."""


class NumericalError(KifmmError, ArithmeticError):
    """Numerical breakdown, e.g. an unusable pseudo-inverse (common.hpp:32-37)."""


class CacheMismatch(KifmmError):
    """Cache archive built for another configuration/version (common.hpp:38-43)."""


class CorruptArchive(KifmmError):
    """Cache archive that cannot be parsed (common.hpp:44-49)."""


class DeviceError(KifmmError, RuntimeError):
    """CUDA / NCCL / device-memory failure (new: the reference has no device)."""


STATUS_TO_ERROR = {
    1: InvalidArgument,
    2: IoError,
    3: NumericalError,
    4: DeviceError,
    5: DeviceError,
    6: DeviceError,
    7: CacheMismatch,
    8: CorruptArchive,
    9: KifmmError,
}
