"""Exception taxonomy of the reference (proj/core/include/cpd/errors.hpp:8-35),
mapped 1:1 from C-ABI status codes (include/cpdgpu.h)."""
import builtins


class CpdError(Exception):
    """Base of every error raised by this package."""


class ShapeError(CpdError, ValueError):
    """Invalid dimensions or incompatible shapes (errors.hpp:9-11)."""


class IndexError(CpdError, builtins.IndexError):  # noqa: A001 - mirrors cpd::IndexError
    """Out-of-range index; the message names the offending mode (errors.hpp:14-16)."""


class ArgumentError(CpdError, ValueError):
    """Bad argument values (ranks, modes, options) (errors.hpp:19-21)."""


class DomainError(CpdError, ValueError):
    """Input violates a mathematical domain requirement (errors.hpp:24-26)."""


class NumericError(CpdError, ArithmeticError):
    """Numerical failure, e.g. non-finite values (errors.hpp:29-31)."""


class ParseError(CpdError, RuntimeError):
    """Malformed tensor file; the message carries the byte offset (errors.hpp:33-36)."""


class DeviceError(CpdError, RuntimeError):
    """CUDA/device failure or a missing device library (no reference counterpart)."""


_BY_STATUS = {1: ShapeError, 2: IndexError, 3: ArgumentError, 4: NumericError, 5: DomainError,
              6: DeviceError, 7: DeviceError, 8: ParseError}


def from_status(status: int, msg: str) -> CpdError:
    return _BY_STATUS.get(status, DeviceError)(msg or f"cpdgpu status {status}")
