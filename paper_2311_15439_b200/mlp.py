"""MLP head mirror (include/sxen/mlp.hpp) over sxen_mlp_*: MlpConfig, Mlp (parameters + gradient + batched workspace)."""
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
class MlpConfig:
    """sxen::MlpConfig, same defaults (include/sxen/mlp.hpp:11-25). Hidden activation ReLU, output identity."""

    input_width: int = 32
    hidden_width: int = 64
    hidden_layers: int = 2
    output_width: int = 3

    def layer_count(self) -> int:
        return self.hidden_layers + 1

    def layer_input_width(self, layer: int) -> int:
        return self.input_width if layer == 0 else self.hidden_width

    def layer_output_width(self, layer: int) -> int:
        return self.output_width if layer == self.layer_count() - 1 else self.hidden_width

    def c(self) -> _abi.MlpConfigC:
        return _abi.MlpConfigC(int(self.input_width), int(self.hidden_width), int(self.hidden_layers),
                               int(self.output_width))

    def validate(self) -> None:
        lib = _lib()
        c = self.c()
        raise_for(lib, lib.sxen_mlp_validate(C.byref(c)))


class Mlp:
    """sxen::Mlp on one B200.  forward() keeps the batch's activations (the reference's MlpWorkspace) inside the handle;
    backward() consumes them and accumulates into the handle's fp64 MlpGradient."""

    def __init__(self, cfg: MlpConfig, device: int = 0):
        self._lib = _lib()
        self._h = C.c_void_p()
        self._cfg = MlpConfig(**cfg.__dict__)
        c = cfg.c()
        raise_for(self._lib, self._lib.sxen_mlp_create(C.byref(c), device, C.byref(self._h)))
        self.device = device

    def __del__(self):
        if getattr(self, "_h", None):
            self._lib.sxen_mlp_destroy(self._h)
            self._h = None

    @property
    def config(self) -> MlpConfig:
        return self._cfg

    def layer_count(self) -> int:
        return self._cfg.layer_count()

    def parameter_count(self) -> int:
        out = C.c_uint64()
        raise_for(self._lib, self._lib.sxen_mlp_parameter_count(self._h, C.byref(out)))
        return out.value

    def init_params(self, seed: int, stream=0) -> None:
        raise_for(self._lib, self._lib.sxen_mlp_init_params(self._h, seed & ((1 << 64) - 1), C.c_void_p(stream)))

    def parameters(self) -> np.ndarray:
        out = np.empty(self.parameter_count(), dtype=np.float32)
        raise_for(self._lib, self._lib.sxen_mlp_download_params(self._h, out.ctypes.data_as(C.POINTER(C.c_float))))
        return out

    def set_parameters(self, values) -> None:
        v = np.ascontiguousarray(values, dtype=np.float32).reshape(-1)
        if v.size != self.parameter_count():
            raise ValueError("mlp: parameter vector has the wrong length")
        raise_for(self._lib, self._lib.sxen_mlp_upload_params(self._h, v.ctypes.data_as(C.POINTER(C.c_float))))

    def _offsets(self, layer: int):
        off = 0
        for l in range(layer):
            off += self._cfg.layer_input_width(l) * self._cfg.layer_output_width(l) + self._cfg.layer_output_width(l)
        nw = self._cfg.layer_input_width(layer) * self._cfg.layer_output_width(layer)
        return off, nw, self._cfg.layer_output_width(layer)

    def weights(self, layer: int) -> np.ndarray:
        off, nw, _ = self._offsets(layer)
        return self.parameters()[off:off + nw]

    def biases(self, layer: int) -> np.ndarray:
        off, nw, nb = self._offsets(layer)
        return self.parameters()[off + nw:off + nw + nb]

    def gradient(self) -> np.ndarray:
        """MlpGradient::values(): fp64, laid out like parameters()."""
        out = np.empty(self.parameter_count(), dtype=np.float64)
        raise_for(self._lib, self._lib.sxen_mlp_grad_download(self._h, out.ctypes.data_as(C.POINTER(C.c_double))))
        return out

    def clear_gradient(self, stream=0) -> None:
        raise_for(self._lib, self._lib.sxen_mlp_grad_clear(self._h, C.c_void_p(stream)))

    def parameters_device(self):
        import torch
        from .encoding import _wrap_device
        p = C.c_void_p()
        raise_for(self._lib, self._lib.sxen_mlp_params_dev(self._h, C.byref(p)))
        return _wrap_device(p.value, self.parameter_count(), torch.float32, self)

    def gradient_device(self):
        import torch
        from .encoding import _wrap_device
        p = C.c_void_p()
        raise_for(self._lib, self._lib.sxen_mlp_grads_dev(self._h, C.byref(p)))
        return _wrap_device(p.value, self.parameter_count(), torch.float64, self)

    def set_precision(self, mode: int) -> None:
        """0 = exact fp64-accumulate (default), 1 = tcgen05 split-bf16, three products (within 1.5e-5), 2 = tcgen05 single bf16
        (~4e-3), 3 = split-bf16 with the fourth (lo x lo) product (within 1e-5, +15 % kernel time)."""
        raise_for(self._lib, self._lib.sxen_mlp_set_precision(self._h, int(mode)))

    def set_reproducible(self, on: bool = True) -> None:
        """sxen_mlp_set_reproducible: the kernels' partial parameter gradients (and the tensor-core head's loss) meet in
        64-bit fixed point, so they do not depend on block scheduling (src/mlp.cpp:83-88's fixed-order merge)."""
        raise_for(self._lib, self._lib.sxen_mlp_set_reproducible(self._h, 1 if on else 0))

    def precision(self) -> int:
        out = C.c_int32()
        raise_for(self._lib, self._lib.sxen_mlp_get_precision(self._h, C.byref(out)))
        return out.value

    def forward_backward(self, inputs, targets, global_batch=None, want_pred=False, stream=None):
        """Fused forward + MSE + backward of one batch (run_chunk per sample, src/trainer.cpp:36-46).
        Returns (input_grad [N, in] float32, loss_sum 1-element float64 tensor, pred or None)."""
        import torch
        from .encoding import _stream_ptr
        x = inputs.to(torch.float32).contiguous()
        tg = targets.contiguous()
        n = x.shape[0]
        typ = {torch.float64: _abi.COORD_F64, torch.float32: _abi.COORD_F32}[tg.dtype]
        ig = torch.empty((n, self._cfg.input_width), dtype=torch.float32, device=x.device)
        loss = torch.zeros(1, dtype=torch.float64, device=x.device)
        pred = torch.empty((n, self._cfg.output_width), dtype=torch.float32, device=x.device) if want_pred else None
        raise_for(self._lib, self._lib.sxen_mlp_forward_backward(
            self._h, C.c_void_p(x.data_ptr()), C.c_void_p(tg.data_ptr()), typ, n, global_batch or n,
            C.c_void_p(pred.data_ptr()) if want_pred else None, C.c_void_p(ig.data_ptr()), C.c_void_p(loss.data_ptr()),
            _stream_ptr(stream, self.device)))
        return ig, loss, pred

    def forward(self, inputs, stream=None):
        """Batched Mlp::forward.  inputs: CUDA float32 [N, input_width] -> CUDA float32 [N, output_width]; a numpy array takes
        the host-buffer entry point and returns numpy."""
        if isinstance(inputs, np.ndarray):
            # the reference's host spans (Mlp::forward(span<const float>, ws) + ws.output()), N samples per call
            x = np.ascontiguousarray(inputs, dtype=np.float32)
            if x.ndim != 2 or x.shape[1] != self._cfg.input_width:
                raise ValueError("mlp forward: input width mismatch")
            out = np.empty((x.shape[0], self._cfg.output_width), dtype=np.float32)
            raise_for(self._lib, self._lib.sxen_mlp_forward_host(self._h, C.c_void_p(x.ctypes.data), x.shape[0],
                                                                 C.c_void_p(out.ctypes.data)))
            return out
        import torch
        from .encoding import _stream_ptr
        if inputs.ndim != 2 or inputs.shape[1] != self._cfg.input_width:  # src/mlp.cpp:138-140
            raise ValueError("mlp forward: input width mismatch")
        x = inputs.to(torch.float32).contiguous()
        out = torch.empty((x.shape[0], self._cfg.output_width), dtype=torch.float32, device=x.device)
        raise_for(self._lib, self._lib.sxen_mlp_forward(self._h, C.c_void_p(x.data_ptr()), x.shape[0],
                                                        C.c_void_p(out.data_ptr()), _stream_ptr(stream, self.device)))
        return out

    def backward(self, upstream, stream=None, dtype=None):
        """Batched Mlp::backward.  upstream: CUDA float64 [N, output_width]; returns d(loss)/d(input) [N, input_width]
        (float64 by default, the reference's type; float32 when dtype=torch.float32)."""
        if isinstance(upstream, np.ndarray):
            # host spans: Mlp::backward(span<const double>, ws, grad) + ws.input_grad()
            up = np.ascontiguousarray(upstream, dtype=np.float64)
            if up.ndim != 2 or up.shape[1] != self._cfg.output_width:
                raise ValueError("mlp backward: upstream width mismatch")
            ig = np.empty((up.shape[0], self._cfg.input_width), dtype=np.float64)
            raise_for(self._lib, self._lib.sxen_mlp_backward_host(self._h, C.c_void_p(up.ctypes.data), up.shape[0],
                                                                  C.c_void_p(ig.ctypes.data)))
            return ig
        import torch
        from .encoding import _stream_ptr
        if upstream.ndim != 2 or upstream.shape[1] != self._cfg.output_width:  # src/mlp.cpp:168-170
            raise ValueError("mlp backward: upstream width mismatch")
        up = upstream.to(torch.float64).contiguous()
        n = up.shape[0]
        want32 = dtype == torch.float32
        ig = torch.empty((n, self._cfg.input_width), dtype=torch.float32 if want32 else torch.float64, device=up.device)
        raise_for(self._lib, self._lib.sxen_mlp_backward(
            self._h, C.c_void_p(up.data_ptr()), n, C.c_void_p(ig.data_ptr()) if want32 else None,
            None if want32 else C.c_void_p(ig.data_ptr()), _stream_ptr(stream, self.device)))
        return ig
