"""Exception hierarchy mirroring proj/include/hcc/errors.hpp:10-60.

Each C ABI status code (include/hccx.h) maps onto exactly one class, so a
caller of the reference's API sees the same exception types.
"""
from __future__ import annotations


class Error(RuntimeError):
    """hcc::Error (errors.hpp:10-13): base of all library errors."""


class NonFiniteInputError(Error):
    """Lossy codec handed NaN/Inf (errors.hpp:15-19)."""


class CorruptPayloadError(Error):
    """Truncated payload / bad block count / bad header (errors.hpp:21-25)."""


class DataDependentSizeError(Error):
    """wire_size_bytes() on a data-dependent codec (errors.hpp:27-31)."""


class BadChunkingError(Error):
    """Collective length does not fit the communicator (errors.hpp:33-37)."""


class BadLayoutError(Error):
    """dp*pp*tp does not factor the world (errors.hpp:39-43)."""


class InvalidSchemeError(Error):
    """Scheme/codec parameters violate a precondition (errors.hpp:45-49)."""


class ConfigError(Error):
    """Invalid configuration; ``field`` names the entry (errors.hpp:51-60)."""

    def __init__(self, field: str, msg: str):
        super().__init__(f"config field '{field}': {msg}")
        self.field = field


class CudaError(Error):
    """A CUDA runtime call or kernel launch failed (device-side addition)."""


class PeerTimeoutError(Error):
    """A peer rank did not answer within the spin budget (device-side addition)."""


class UnsupportedError(Error):
    """The requested codec/operation has no device implementation."""


_BY_STATUS = {
    1: NonFiniteInputError,
    2: CorruptPayloadError,
    3: DataDependentSizeError,
    4: BadChunkingError,
    5: BadLayoutError,
    6: InvalidSchemeError,
    8: CudaError,
    9: ValueError,
    10: PeerTimeoutError,
    11: UnsupportedError,
}


def check(status: int, what: str = "") -> None:
    """Raise the exception the reference would throw for a C ABI status."""
    if status == 0:
        return
    from . import _lib

    msg = _lib.hccx_status_string(status).decode()
    if what:
        msg = f"{what}: {msg}"
    if status == 7:
        raise ConfigError("codec", msg)
    raise _BY_STATUS.get(status, Error)(msg)
