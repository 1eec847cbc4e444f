"""Exception types mirroring the reference's (include/sxen/errors.hpp:8-15) and the status -> exception map."""
from __future__ import annotations

from . import _abi


class IoError(RuntimeError):
    """sxen::IoError"""


class TrainingError(RuntimeError):
    """sxen::TrainingError: non-finite loss or gradient"""


class CudaError(RuntimeError):
    """Device/runtime failure (no reference analogue)."""


def raise_for(lib, status: int) -> None:
    """Re-raise a C-ABI status as the exception type the reference would have thrown."""
    if status == _abi.OK:
        return
    msg = lib.sxen_last_error().decode()
    if status == _abi.INVALID_ARGUMENT:
        raise ValueError(msg)  # std::invalid_argument
    if status == _abi.LOGIC_ERROR:
        raise RuntimeError(msg)  # std::logic_error
    if status == _abi.TRAINING_ERROR:
        raise TrainingError(msg)
    if status == _abi.IO_ERROR:
        raise IoError(msg)
    raise CudaError(msg)
