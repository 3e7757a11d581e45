"""Exception taxonomy of the reference (include/ttstream/errors.hpp:9-55).

The C ABI returns status codes (include/ttg.h ``ttg_status``); the host
mirror raises the matching class, so callers see the reference's errors.
"""


class Error(RuntimeError):
    """ttstream::Error (errors.hpp:9-12)."""


class DimensionError(Error):
    """errors.hpp:15-18."""


class NumericError(Error):
    """errors.hpp:21-24."""


class StateError(Error):
    """errors.hpp:28-31."""


class FormatError(Error):
    """errors.hpp:34-37."""


class IndexError_(Error):
    """errors.hpp:40-43 (trailing underscore avoids shadowing the builtin)."""


class ConfigError(Error):
    """errors.hpp:46-49."""


class ResourceError(Error):
    """errors.hpp:52-55."""


class CudaError(Error):
    """TTG_E_CUDA: a CUDA runtime failure (no reference analogue)."""


class NcclError(Error):
    """TTG_E_NCCL: an NCCL failure (no reference analogue)."""


class ArgumentError(Error):
    """TTG_E_ARGUMENT: bad pointer / enum at the ABI."""


STATUS_TO_ERROR = {
    1: DimensionError,
    2: NumericError,
    3: StateError,
    4: FormatError,
    5: IndexError_,
    6: ConfigError,
    7: ResourceError,
    8: CudaError,
    9: NcclError,
    10: ArgumentError,
}
