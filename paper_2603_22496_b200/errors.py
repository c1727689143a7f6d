"""Error types of the drop-in boundary.

Mirrors the exception hierarchy of the reference (``kkbeam/errors.py:8-41``)
so callers that catch ``GeometryError`` / ``GuardBandError`` / ``DataError``
keep working.  Kernels never raise: all validation happens on the host
before a launch, and a non-zero status from the C ABI is mapped here.
"""

from __future__ import annotations


class KKBeamError(Exception):
    """Root of every error this package raises (errors.py:8)."""


class ConfigError(KKBeamError):
    """A parameter or configuration value is invalid (errors.py:12)."""


class DataError(KKBeamError):
    """Data is malformed or outside the contract (errors.py:16)."""


class WindowOverflowError(DataError):
    """An echo would land past the acquisition window (errors.py:20)."""


class GuardBandError(DataError):
    """The window leaves too few trailing samples for the shear (errors.py:24)."""


class GeometryError(DataError):
    """Data geometry disagrees with the delay tables or grid (errors.py:28)."""


class RoiError(DataError):
    """Region of interest is unusable (errors.py:32)."""


class MetricError(DataError):
    """A quality metric cannot be evaluated on this image (errors.py:36)."""


class FileFormatError(DataError):
    """A container file violates the binary format (errors.py:40)."""


class DeviceError(KKBeamError):
    """The CUDA library reported a failure (no reference counterpart: the
    reference never leaves the host)."""


# C-ABI status codes (include/kkb.h) -> exception type
_STATUS = {
    -1: ConfigError,      # KKB_ERR_ARG
    -2: GeometryError,    # KKB_ERR_SHAPE
    -3: DeviceError,      # KKB_ERR_CUDA
    -4: DeviceError,      # KKB_ERR_NOMEM
    -5: ConfigError,      # KKB_ERR_UNSUPPORTED
    -6: FileFormatError,  # KKB_ERR_FORMAT
    -7: OSError,          # KKB_ERR_IO
}


def raise_for_status(status: int, what: str, detail: str = "") -> None:
    if status == 0:
        return
    exc = _STATUS.get(status, DeviceError)
    msg = f"{what} failed with status {status}"
    if detail:
        msg += f": {detail}"
    raise exc(msg)
