"""Counter RNG mirror (include/sxen/rng.hpp:9-54).  Scalars are computed by the library's host entry points;
bulk fills run on the device (sxen_rng_fill_dev) and are bit-identical to CounterRng::next_double."""
from __future__ import annotations

import ctypes as C

from . import _abi
from .errors import raise_for

_MASK = (1 << 64) - 1


def _lib():
    from . import lib
    return lib


def mix64(z: int) -> int:
    return _lib().sxen_mix64(z & _MASK)


def hash_combine(a: int, b: int) -> int:
    return _lib().sxen_hash_combine(a & _MASK, b & _MASK)


class CounterRng:
    """CounterRng(seed[, stream]); draws are addressed by a 1-based counter, so fills can start anywhere."""

    def __init__(self, seed: int, stream: int | None = None):
        self.seed, self.stream = seed & _MASK, stream
        self.counter = 0

    def fill_device(self, tensor, lo: float = 0.0, hi: float = 1.0, cuda_stream: int = 0):
        """Fill a contiguous CUDA tensor (float64 or float32) with next_double(lo, hi) draws and advance."""
        import torch
        assert tensor.is_cuda and tensor.is_contiguous()
        typ = {torch.float64: _abi.COORD_F64, torch.float32: _abi.COORD_F32}[tensor.dtype]
        n = tensor.numel()
        lib = _lib()
        raise_for(lib, lib.sxen_rng_fill_dev(self.seed, 0 if self.stream is None else 1, self.stream or 0,
                                             self.counter + 1, lo, hi, C.c_void_p(tensor.data_ptr()), n, typ,
                                             C.c_void_p(cuda_stream)))
        self.counter += n
        return tensor
