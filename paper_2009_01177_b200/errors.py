"""Error taxonomy mirroring the reference (errors.hpp:13-78).

Every error carries a stable machine-readable ``code`` of the form
"module/kind".  The C ABI returns the status numbers below and fills a
``tor_error`` struct; ``raise_for_status`` maps them back onto these classes.
Like the reference's pybind module (bindings.cpp:108) the base class is a
RuntimeError subclass named ``TorfpError``.
"""
from __future__ import annotations

# tor_capi.h status codes
TOR_OK = 0
TOR_E_INVALID = 1
TOR_E_BREAKDOWN = 2
TOR_E_PRECISION = 3
TOR_E_PARSE = 4
TOR_E_RESOURCE = 5
TOR_E_DEVICE = 6
TOR_E_ERROR = 7


class TorfpError(RuntimeError):
    """Base error: code "module/kind" + message (errors.hpp:13-24)."""

    status = TOR_E_ERROR

    def __init__(self, code: str, message: str = ""):
        super().__init__(message or code)
        self.code = code
        self.message = message


class InvalidArgument(TorfpError):  # errors.hpp:27-31
    status = TOR_E_INVALID


class BreakdownError(TorfpError):  # errors.hpp:34-50
    status = TOR_E_BREAKDOWN

    def __init__(self, code: str, message: str = "", pivot_row: int = -1, subset_mask: int = 0):
        super().__init__(code, message)
        self.pivot_row = pivot_row
        self.subset_mask = subset_mask


class ParseError(TorfpError):  # errors.hpp:54-62
    status = TOR_E_PARSE

    def __init__(self, code: str, message: str = "", position: int = 0):
        super().__init__(code, message)
        self.position = position


class PrecisionError(TorfpError):  # errors.hpp:66-70
    status = TOR_E_PRECISION


class ResourceError(TorfpError):  # errors.hpp:73-77
    status = TOR_E_RESOURCE


class DeviceError(TorfpError):
    """CUDA / NCCL failure (no reference counterpart: the reference is CPU-only)."""

    status = TOR_E_DEVICE


_BY_STATUS = {
    TOR_E_INVALID: InvalidArgument,
    TOR_E_PRECISION: PrecisionError,
    TOR_E_PARSE: ParseError,
    TOR_E_RESOURCE: ResourceError,
    TOR_E_DEVICE: DeviceError,
    TOR_E_ERROR: TorfpError,
}


def raise_for_status(status: int, code: str, message: str, pivot_row: int = -1,
                     subset_mask: int = 0) -> None:
    if status == TOR_OK:
        return
    if status == TOR_E_BREAKDOWN:
        raise BreakdownError(code, message, pivot_row, subset_mask)
    if status == TOR_E_PARSE:  # the C ABI reports ParseError::position() in pivot_row
        raise ParseError(code, message, max(pivot_row, 0))
    raise _BY_STATUS.get(status, TorfpError)(code, message)
