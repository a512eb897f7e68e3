"""The reference's exception hierarchy (proj/core/include/pegrad/common.hpp:56-114),
raised from pgb_status codes returned by the C ABI."""


class Error(RuntimeError):
    pass


class ShapeError(Error):
    pass


class DomainError(Error):
    pass


class IndexError_(Error):  # pegrad::IndexError; trailing _ avoids the builtin
    pass


class ConfigError(Error):
    pass


class ContractError(Error):
    pass


class UnsupportedError(Error):
    pass


class TraceError(Error):
    pass


class FormatError(Error):
    pass


class IoError(Error):
    pass


class CudaError(Error):
    pass


class NcclError(Error):
    pass


class OutOfMemoryError(Error):
    pass


IndexError = IndexError_  # noqa: A001  (reference name, module-scoped)

_BY_STATUS = {1: ShapeError, 2: DomainError, 3: IndexError_, 4: ConfigError, 5: ContractError,
              6: UnsupportedError, 7: TraceError, 8: FormatError, 9: IoError, 10: CudaError,
              11: NcclError, 12: OutOfMemoryError}


def from_status(status: int, message: str) -> Error:
    return _BY_STATUS.get(status, Error)(message)
