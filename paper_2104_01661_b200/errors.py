"""gblite::ErrCode (include/gblite/error.hpp:13-41) + the device codes of gbx.h."""
from enum import IntEnum


class ErrCode(IntEnum):
    Success = 0
    NoValue = 1
    DimensionMismatch = -1
    DomainMismatch = -2
    IndexOutOfBounds = -3
    InvalidMatrix = -4
    InvalidGraph = -5
    MissingProperty = -6
    SourceOutOfRange = -7
    EmptyBatch = -8
    NonPositiveDamping = -9
    NonPositiveDelta = -10
    NonPositiveWeight = -11
    PreconditionViolated = -12
    ParseError = -13
    DuplicateEntry = -14
    IoFailure = -15
    BadMagic = -16
    UnsupportedVersion = -17
    TruncatedStream = -18
    LengthMismatch = -19
    AliasedOutput = -20
    InvalidValue = -21
    CudaError = -30
    OutOfMemory = -31
    Unsupported = -32
    NullArgument = -33
    CommError = -34


class Error(RuntimeError):
    """gblite::Error (error.hpp:45-55): `ErrCodeName: message`, with .code."""

    def __init__(self, code: int, message: str):
        try:
            self.code = ErrCode(code)
            name = self.code.name
        except ValueError:
            self.code = code
            name = str(code)
        super().__init__(f"{name}: {message}")
        self.message = message
