"""Adam mirrors (include/sxen/optimizer.hpp:13-59) over sxen_adam_* / sxen_sparse_adam_*."""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import _abi
from .errors import raise_for


def _lib():
    from . import lib
    return lib


@dataclass
class AdamConfig:
    """sxen::AdamConfig, same defaults (include/sxen/optimizer.hpp:13-18)."""

    lr: float = 1e-3
    beta1: float = 0.9
    beta2: float = 0.99
    epsilon: float = 1e-15

    def c(self) -> _abi.AdamConfigC:
        return _abi.AdamConfigC(self.lr, self.beta1, self.beta2, self.epsilon)


class SparseAdamState:
    """sxen::SparseAdamState: lazy Adam over the hash tables, visits only rows the accumulator touched."""

    def __init__(self, encoder):
        self._lib = _lib()
        self._h = C.c_void_p()
        raise_for(self._lib, self._lib.sxen_sparse_adam_create(encoder._h, C.byref(self._h)))
        self._cfg = encoder.config

    def __del__(self):
        if getattr(self, "_h", None):
            self._lib.sxen_sparse_adam_destroy(self._h)
            self._h = None

    def step_count(self) -> int:
        out = C.c_int64()
        raise_for(self._lib, self._lib.sxen_sparse_adam_step_count(self._h, C.byref(out)))
        return out.value

    def step(self, encoder, grads, cfg: AdamConfig, clear_grad: bool = False, stream: int = 0, check: bool = True):
        c = cfg.c()
        raise_for(self._lib, self._lib.sxen_sparse_adam_step(self._h, encoder._h, grads._h, C.byref(c),
                                                             1 if clear_grad else 0, C.c_void_p(stream)))
        if check:  # the reference throws TrainingError from inside step (src/optimizer.cpp:73-76)
            raise_for(self._lib, self._lib.sxen_sparse_adam_check(self._h, C.c_void_p(stream)))

    def moments(self, level: int):
        per = self._cfg.table_size * self._cfg.features
        m, v = np.empty(per), np.empty(per)
        raise_for(self._lib, self._lib.sxen_sparse_adam_download(self._h, level, m.ctypes.data_as(C.POINTER(C.c_double)),
                                                                 v.ctypes.data_as(C.POINTER(C.c_double))))
        return m, v


class AdamState:
    """sxen::AdamState over a dense f32 parameter vector living on the device."""

    def __init__(self, size: int, device: int = 0):
        self._lib = _lib()
        self._h = C.c_void_p()
        self.size = size
        raise_for(self._lib, self._lib.sxen_adam_create(size, device, C.byref(self._h)))

    def __del__(self):
        if getattr(self, "_h", None):
            self._lib.sxen_adam_destroy(self._h)
            self._h = None

    def step_count(self) -> int:
        out = C.c_int64()
        raise_for(self._lib, self._lib.sxen_adam_step_count(self._h, C.byref(out)))
        return out.value

    def step(self, params, grads, cfg: AdamConfig, stream: int = 0, check: bool = True):
        """params: CUDA float32 tensor; grads: CUDA float64 or float32 tensor of the same length."""
        import torch
        if params.numel() != self.size or grads.numel() != self.size:
            raise ValueError("adam step: parameter/gradient size mismatch")
        typ = {torch.float64: _abi.COORD_F64, torch.float32: _abi.COORD_F32}[grads.dtype]
        c = cfg.c()
        raise_for(self._lib, self._lib.sxen_adam_step(self._h, C.c_void_p(params.data_ptr()), C.c_void_p(grads.data_ptr()),
                                                      typ, self.size, C.byref(c), C.c_void_p(stream)))
        if check:
            raise_for(self._lib, self._lib.sxen_adam_check(self._h, C.c_void_p(stream)))
