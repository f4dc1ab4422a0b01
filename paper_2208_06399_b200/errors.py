"""Exception taxonomy mirroring autoshard/common.hpp:15-50, mapped from as_status."""
from __future__ import annotations


class Error(RuntimeError):
    """Base of every error raised by the library (autoshard::Error)."""


class ConfigError(Error):
    pass


class ParseError(Error):
    pass


class OffsetError(ParseError):
    pass


class IndexError_(ParseError):
    """autoshard::IndexError (renamed to avoid shadowing the Python builtin)."""


class InfeasibleError(Error):
    pass


class ShapeError(Error):
    pass


class LookupError_(Error):
    """autoshard::LookupError."""


class GuardError(Error):
    pass


class StateError(Error):
    pass


class CudaError(Error):
    pass


class NcclError(Error):
    pass


_BY_STATUS = {
    1: ConfigError,
    2: ParseError,
    3: OffsetError,
    4: IndexError_,
    5: InfeasibleError,
    6: ShapeError,
    7: LookupError_,
    8: GuardError,
    9: StateError,
    10: CudaError,
    11: NcclError,
}


def check(status: int) -> None:
    """Raise the exception class matching a non-zero as_status."""
    if status:
        from ._capi import lib

        msg = lib().as_last_error().decode(errors="replace")
        raise _BY_STATUS.get(status, Error)(msg)
