"""Host-side mirror of the reference's encoder interface (include/sxen/encoding.hpp) over the C ABI.

Names, argument meaning and error behaviour follow the reference: EncoderConfig / HashEncoder / EncoderGradient /
LookupCounters.  Calls are the BATCHED form of the reference's per-sample methods.  numpy inputs take the host-buffer
entry points (synchronous, errors raised directly, like the reference); torch CUDA tensors take the asynchronous
device entry points -- call ``HashEncoder.check()`` to surface what the reference would have thrown.
"""
from __future__ import annotations

import ctypes as C
import enum
from dataclasses import dataclass, field

import numpy as np

from . import _abi
from .errors import raise_for


def _lib():
    from . import lib
    return lib


class Backend(enum.IntEnum):  # include/sxen/encoding.hpp:12
    simplex = 0
    grid = 1


class LevelScale(enum.IntEnum):  # include/sxen/encoding.hpp:13
    raw = 0
    equal_memory = 1


@dataclass
class EncoderConfig:
    """sxen::EncoderConfig, same fields and defaults (include/sxen/encoding.hpp:18-33)."""

    dim: int = 2
    levels: int = 8
    table_size: int = 1 << 16
    features: int = 2
    base_resolution: int = 16
    growth: float = 2.0
    backend: int = Backend.simplex
    level_scale: int = LevelScale.raw

    def encoded_width(self) -> int:
        return self.levels * self.features

    def c(self) -> _abi.EncoderConfigC:
        # table_size is validated by the library; keep the ctypes conversion from masking garbage
        if not (0 <= int(self.table_size) < 2**32):
            raise ValueError(f"encoder table_size must be a power of two, got {self.table_size}")
        return _abi.EncoderConfigC(int(self.dim), int(self.levels), int(self.table_size), int(self.features),
                                   int(self.base_resolution), float(self.growth), int(self.backend),
                                   int(self.level_scale))

    def validate(self) -> None:
        """Raises ValueError (std::invalid_argument) exactly where EncoderConfig::validate throws."""
        lib = _lib()
        c = self.c()
        raise_for(lib, lib.sxen_encoder_validate(C.byref(c)))

    @property
    def vertices(self) -> int:
        return self.dim + 1 if self.backend == Backend.simplex else 1 << self.dim


@dataclass
class LookupCounters:  # include/sxen/encoding.hpp:44-47
    touched_vertices: int = 0
    out_of_bounds: int = 0


@dataclass
class Tuning:
    """Launch-shape knobs (sxen_tuning). 0 keeps the library default."""

    levels_per_thread: int = 0
    block_threads: int = 0
    level_major: int = -1  # -1 auto, 0 sample-major, 1 level-major
    exact_blend: int = 1
    warp_aggregate: int = 0
    merge_pairs: int = 0  # 1 on, -1 off, 0 library default (on)
    cache_hints: int = -1  # F == 2: gather L2 policy + 4 * red L2 policy (0 none, 1 evict_last, 2 evict_first, 3 evict_unchanged); -1 auto
    coarse_replicas: int = 0  # 0 library default (on from 2^16 samples per launch), 1 always, -1 off
    level_chunk: int = 0  # sample-major launches: levels per grid slice; 0 library default, -1 off

    def c(self) -> _abi.TuningC:
        return _abi.TuningC(self.levels_per_thread, self.block_threads, self.level_major, self.exact_blend,
                            self.warp_aggregate, self.merge_pairs, self.cache_hints, self.coarse_replicas, self.level_chunk)


def equal_memory_multiplier(n: int) -> float:
    lib = _lib()
    out = C.c_double()
    raise_for(lib, lib.sxen_equal_memory_multiplier(n, C.byref(out)))
    return out.value


def level_resolution(cfg: EncoderConfig, level: int) -> int:
    lib = _lib()
    out = C.c_uint32()
    c = cfg.c()
    raise_for(lib, lib.sxen_level_resolution(C.byref(c), level, C.byref(out)))
    return out.value


def skew_constants(n: int):
    """(F_n, G_n, S_n) = SkewConstants::make(n) (src/lattice.cpp:21-30)."""
    lib = _lib()
    out = (C.c_double * 3)()
    raise_for(lib, lib.sxen_skew_constants(n, out))
    return tuple(out)


def hash_coords(coords) -> int:
    lib = _lib()
    c = np.ascontiguousarray(coords, dtype=np.int64)
    out = C.c_uint32()
    raise_for(lib, lib.sxen_hash_coords(c.ctypes.data_as(C.POINTER(C.c_int64)), c.size, C.byref(out)))
    return out.value


def _is_torch(x) -> bool:
    return type(x).__module__.startswith("torch")


def _coord_type(t):
    import torch
    if t.dtype == torch.float64:
        return _abi.COORD_F64
    if t.dtype == torch.float32:
        return _abi.COORD_F32
    raise ValueError("coordinates must be float64 or float32")


def _stream_ptr(stream, device=None) -> C.c_void_p:
    """`stream` as a cudaStream_t; None = torch's current stream ON `device` (a handle's device index or a torch.device;
    default: the current device) -- never another device's stream for a handle that lives elsewhere."""
    if stream is None:
        import torch
        return C.c_void_p(torch.cuda.current_stream(device).cuda_stream)
    return C.c_void_p(int(stream))


def _owner_device(owner) -> int:
    """Device index of the library handle behind `owner` (encoder / gradient / MLP / trainer mirrors)."""
    for path in (("device",), ("encoder", "device"), ("mlp", "device")):
        o = owner
        for name in path:
            o = getattr(o, name, None)
            if o is None:
                break
        if isinstance(o, int):
            return o
    import torch
    return torch.cuda.current_device()


class EncoderGradient:
    """sxen::EncoderGradient (include/sxen/encoding.hpp:53-86): dense device accumulator, f32, touched in-band."""

    def __init__(self, encoder: "HashEncoder"):
        self._lib = _lib()
        self._h = C.c_void_p()
        self._cfg = encoder.config
        self.device = encoder.device
        raise_for(self._lib, self._lib.sxen_grad_create(encoder._h, C.byref(self._h)))

    def __del__(self):
        if getattr(self, "_h", None):
            self._lib.sxen_grad_destroy(self._h)
            self._h = None

    def levels(self) -> int:
        return self._cfg.levels

    def features(self) -> int:
        return self._cfg.features

    def clear(self, stream=0) -> None:
        raise_for(self._lib, self._lib.sxen_grad_clear(self._h, C.c_void_p(stream)))

    def merge(self, other: "EncoderGradient", stream=0) -> None:
        raise_for(self._lib, self._lib.sxen_grad_merge(self._h, other._h, C.c_void_p(stream)))

    def touched_total(self) -> int:
        out = C.c_uint64()
        raise_for(self._lib, self._lib.sxen_grad_touched_total(self._h, C.byref(out)))
        return out.value

    def level(self, level: int):
        """(values[T, F] float32, touched[T] uint8) of one level -- slice() and touched() of the reference."""
        T, F = self._cfg.table_size, self._cfg.features
        vals = np.empty((T, F), dtype=np.float32)
        touched = np.empty(T, dtype=np.uint8)
        raise_for(self._lib, self._lib.sxen_grad_download(self._h, level, vals.ctypes.data_as(C.POINTER(C.c_float)),
                                                          touched.ctypes.data_as(C.POINTER(C.c_uint8))))
        return vals, touched

    def set_reproducible(self, on: bool = True) -> None:
        """sxen_grad_set_reproducible: every backward also keeps order-free 64-bit fixed-point sums (units of 2^-52) that
        the optimizers and ``level`` / ``level_f64`` then use -- the reference's bit-reproducible merge
        (src/trainer.cpp:125-128) instead of fp32-atomic order."""
        raise_for(self._lib, self._lib.sxen_grad_set_reproducible(self._h, 1 if on else 0))

    def reproducible(self) -> bool:
        out = C.c_int32()
        raise_for(self._lib, self._lib.sxen_grad_is_reproducible(self._h, C.byref(out)))
        return bool(out.value)

    def level_f64(self, level: int) -> np.ndarray:
        """values[T, F] of one level as doubles: the exact fixed-point sums in reproducible mode, else the f32 values."""
        T, F = self._cfg.table_size, self._cfg.features
        vals = np.empty((T, F), dtype=np.float64)
        raise_for(self._lib, self._lib.sxen_grad_download_f64(self._h, level, vals.ctypes.data_as(C.POINTER(C.c_double))))
        return vals

    def fixed_device_view(self):
        """The fixed-point words as a flat int64 CUDA tensor (reproducible mode), for an exchange or a bit comparison."""
        import torch
        ptr, cnt = C.c_void_p(), C.c_size_t()
        raise_for(self._lib, self._lib.sxen_grad_fixed_dev(self._h, C.byref(ptr), C.byref(cnt)))
        if not ptr.value:
            raise RuntimeError("gradient accumulator is not in reproducible mode")
        t = torch.as_tensor(_DevArray(ptr.value, cnt.value, "<i8", self), device=f"cuda:{self.device}")
        assert t.data_ptr() == ptr.value
        return t

    def set_level(self, level: int, values, touched) -> None:
        vals = np.ascontiguousarray(values, dtype=np.float32)
        tch = np.ascontiguousarray(touched, dtype=np.uint8)
        if vals.size != self._cfg.table_size * self._cfg.features or tch.size != self._cfg.table_size:
            raise ValueError("EncoderGradient.set_level: shape mismatch")
        raise_for(self._lib, self._lib.sxen_grad_upload(self._h, level, vals.ctypes.data_as(C.POINTER(C.c_float)),
                                                        tch.ctypes.data_as(C.POINTER(C.c_uint8))))

    def device_view(self):
        """The whole accumulator as a flat CUDA float32 tensor (zero-copy) -- what multi-GPU all-reduces."""
        import torch
        ptr, cnt = C.c_void_p(), C.c_size_t()
        raise_for(self._lib, self._lib.sxen_grad_values_dev(self._h, C.byref(ptr), C.byref(cnt)))
        return _wrap_device(ptr.value, cnt.value, torch.float32, self)


class _DevArray:
    """__cuda_array_interface__ carrier so torch can wrap library-owned device memory without copying."""

    def __init__(self, ptr: int, count: int, typestr: str, owner):
        self.__cuda_array_interface__ = {"shape": (count,), "typestr": typestr, "data": (ptr, False), "version": 2}
        self._owner = owner


def _wrap_device(ptr: int, count: int, dtype, owner):
    import torch
    typestr = {torch.float32: "<f4", torch.float64: "<f8"}[dtype]
    # the handle's device, not the current one: on another device torch would silently hand back a COPY, and a gradient
    # exchange over that copy would exchange nothing
    t = torch.as_tensor(_DevArray(ptr, count, typestr, owner), device=f"cuda:{_owner_device(owner)}")
    if count and t.data_ptr() != ptr:
        raise RuntimeError("device view: torch copied library-owned memory instead of wrapping it")
    return t


class HashEncoder:
    """sxen::HashEncoder (include/sxen/encoding.hpp:92-148) on one B200."""

    def __init__(self, cfg: EncoderConfig, device: int = 0):
        self._lib = _lib()
        self._h = C.c_void_p()
        self._cfg = EncoderConfig(**cfg.__dict__)
        c = cfg.c()
        raise_for(self._lib, self._lib.sxen_encoder_create(C.byref(c), device, C.byref(self._h)))
        self.device = device

    def __del__(self):
        if getattr(self, "_h", None):
            self._lib.sxen_encoder_destroy(self._h)
            self._h = None

    # ---- reference accessors
    @property
    def config(self) -> EncoderConfig:
        return self._cfg

    def resolution(self, level: int) -> int:
        out = C.c_uint32()
        raise_for(self._lib, self._lib.sxen_encoder_resolution(self._h, level, C.byref(out)))
        return out.value

    def parameter_count(self) -> int:
        out = C.c_uint64()
        raise_for(self._lib, self._lib.sxen_encoder_parameter_count(self._h, C.byref(out)))
        return out.value

    def init_tables(self, seed: int, stream=0) -> None:
        raise_for(self._lib, self._lib.sxen_encoder_init_tables(self._h, seed & ((1 << 64) - 1), C.c_void_p(stream)))

    def table(self, level: int) -> np.ndarray:
        """Host copy of one level's table, T*F float32 (reference: table(level) span)."""
        out = np.empty(self._cfg.table_size * self._cfg.features, dtype=np.float32)
        raise_for(self._lib, self._lib.sxen_encoder_download_table(self._h, level, out.ctypes.data_as(C.POINTER(C.c_float))))
        return out

    def set_table(self, level: int, values) -> None:
        v = np.ascontiguousarray(values, dtype=np.float32).reshape(-1)
        if v.size != self._cfg.table_size * self._cfg.features:
            raise ValueError("table: wrong element count")
        raise_for(self._lib, self._lib.sxen_encoder_upload_table(self._h, level, v.ctypes.data_as(C.POINTER(C.c_float))))

    def tables_device(self):
        import torch
        ptr = C.c_void_p()
        raise_for(self._lib, self._lib.sxen_encoder_tables_dev(self._h, C.byref(ptr)))
        return _wrap_device(ptr.value, self.parameter_count(), torch.float32, self)

    def counters(self) -> LookupCounters:
        c = _abi.LookupCountersC()
        raise_for(self._lib, self._lib.sxen_encoder_counters(self._h, C.byref(c)))
        return LookupCounters(c.touched_vertices, c.out_of_bounds)

    def reset_counters(self) -> None:
        raise_for(self._lib, self._lib.sxen_encoder_reset_counters(self._h))

    # ---- tuning (no reference analogue)
    def set_tuning(self, t: Tuning) -> None:
        c = t.c()
        raise_for(self._lib, self._lib.sxen_encoder_set_tuning(self._h, C.byref(c)))

    def tuning(self) -> Tuning:
        c = _abi.TuningC()
        raise_for(self._lib, self._lib.sxen_encoder_get_tuning(self._h, C.byref(c)))
        return Tuning(c.levels_per_thread, c.block_threads, c.level_major, c.exact_blend, c.warp_aggregate,
                      c.merge_pairs, c.cache_hints, c.coarse_replicas, c.level_chunk)

    # ---- the hot path
    def _check_x(self, x):
        if x.ndim != 2 or x.shape[1] != self._cfg.dim:  # src/encoding.cpp:184-187
            raise ValueError(f"encode: expected {self._cfg.dim} coordinates, got {x.shape[-1] if x.ndim else 0}")

    def encode(self, x, out=None, stream=None):
        """Batched HashEncoder::encode.  x: [N, dim]; returns [N, L*F] float32 (numpy in -> numpy out)."""
        LF = self._cfg.encoded_width()
        if _is_torch(x):
            import torch
            self._check_x(x)
            x = x.contiguous()
            n = x.shape[0]
            if out is None:
                out = torch.empty((n, LF), dtype=torch.float32, device=x.device)
            elif tuple(out.shape) != (n, LF):  # src/encoding.cpp:297-299
                raise ValueError("encode: output span has wrong width")
            raise_for(self._lib, self._lib.sxen_encoder_encode(self._h, C.c_void_p(x.data_ptr()), _coord_type(x), n,
                                                               C.c_void_p(out.data_ptr()), _stream_ptr(stream, self.device)))
            return out
        x = np.ascontiguousarray(x, dtype=np.float64)
        self._check_x(x)
        n = x.shape[0]
        if out is None:
            out = np.empty((n, LF), dtype=np.float32)
        elif out.shape != (n, LF) or out.dtype != np.float32:
            raise ValueError("encode: output span has wrong width")
        raise_for(self._lib, self._lib.sxen_encoder_encode_host(self._h, x.ctypes.data_as(C.POINTER(C.c_double)), n,
                                                                out.ctypes.data_as(C.POINTER(C.c_float))))
        return out

    def encode_backward(self, x, upstream, grad: EncoderGradient, stream=None, levels=None) -> None:
        """Batched HashEncoder::encode_backward: grad[l][idx] += w * upstream[l*F:(l+1)*F] for every vertex.
        ``levels=(first, count)`` (device tensors only) restricts the launch to that range of encoder levels."""
        LF = self._cfg.encoded_width()
        if _is_torch(x):
            import torch
            self._check_x(x)
            x = x.contiguous()
            if tuple(upstream.shape) != (x.shape[0], LF):  # src/encoding.cpp:320-322
                raise ValueError("encode_backward: upstream span has wrong width")
            upstream = upstream.to(torch.float32).contiguous()
            if levels is not None:
                raise_for(self._lib, self._lib.sxen_encoder_encode_backward_levels(
                    self._h, C.c_void_p(x.data_ptr()), _coord_type(x), C.c_void_p(upstream.data_ptr()), x.shape[0],
                    grad._h, int(levels[0]), int(levels[1]), _stream_ptr(stream, self.device)))
                return
            raise_for(self._lib, self._lib.sxen_encoder_encode_backward(
                self._h, C.c_void_p(x.data_ptr()), _coord_type(x), C.c_void_p(upstream.data_ptr()), x.shape[0],
                grad._h, _stream_ptr(stream, self.device)))
            return
        if levels is not None:
            raise ValueError("encode_backward: a level range needs device tensors")
        x = np.ascontiguousarray(x, dtype=np.float64)
        self._check_x(x)
        up = np.ascontiguousarray(upstream, dtype=np.float64)
        if up.shape != (x.shape[0], LF):
            raise ValueError("encode_backward: upstream span has wrong width")
        raise_for(self._lib, self._lib.sxen_encoder_encode_backward_host(
            self._h, x.ctypes.data_as(C.POINTER(C.c_double)), up.ctypes.data_as(C.POINTER(C.c_double)), x.shape[0],
            grad._h))

    def encode_forward_backward(self, x, upstream, grad: EncoderGradient, out=None, stream=None, levels=None):
        """encode + encode_backward of one batch off a single lattice walk.  numpy inputs (x float64; upstream float64
        or float32) take the pipelined host entry point; torch CUDA tensors the asynchronous device one.
        ``levels=(first, count)`` (device tensors only) restricts the launch to that range of encoder levels: only that
        slice of every feature row is written."""
        if not _is_torch(x):
            if levels is not None:
                raise ValueError("encode_forward_backward: a level range needs device tensors")
            x = np.ascontiguousarray(x, dtype=np.float64)
            self._check_x(x)
            n, LF = x.shape[0], self._cfg.encoded_width()
            up = np.ascontiguousarray(upstream)
            if up.dtype not in (np.float32, np.float64):
                up = up.astype(np.float64)
            if up.shape != (n, LF):
                raise ValueError("encode_backward: upstream span has wrong width")
            if out is None:
                out = np.empty((n, LF), dtype=np.float32)
            typ = _abi.COORD_F32 if up.dtype == np.float32 else _abi.COORD_F64
            raise_for(self._lib, self._lib.sxen_encoder_encode_forward_backward_host(
                self._h, x.ctypes.data_as(C.POINTER(C.c_double)), C.c_void_p(up.ctypes.data), typ, n,
                out.ctypes.data_as(C.POINTER(C.c_float)), grad._h))
            return out
        import torch
        self._check_x(x)
        LF = self._cfg.encoded_width()
        x = x.contiguous()
        n = x.shape[0]
        if tuple(upstream.shape) != (n, LF):
            raise ValueError("encode_backward: upstream span has wrong width")
        if out is None:
            out = torch.empty((n, LF), dtype=torch.float32, device=x.device)
        upstream = upstream.to(torch.float32).contiguous()
        if levels is not None:
            raise_for(self._lib, self._lib.sxen_encoder_encode_forward_backward_levels(
                self._h, C.c_void_p(x.data_ptr()), _coord_type(x), C.c_void_p(upstream.data_ptr()), n,
                C.c_void_p(out.data_ptr()), grad._h, int(levels[0]), int(levels[1]), _stream_ptr(stream, self.device)))
            return out
        raise_for(self._lib, self._lib.sxen_encoder_encode_forward_backward(
            self._h, C.c_void_p(x.data_ptr()), _coord_type(x), C.c_void_p(upstream.data_ptr()), n,
            C.c_void_p(out.data_ptr()), grad._h, _stream_ptr(stream, self.device)))
        return out

    def encode_debug(self, x, stream=None):
        """(idx[N, L, V] int64-safe uint32, w[N, L, V] float64): the vertex chains the kernels use (parity probe)."""
        import torch
        if not _is_torch(x):
            x = torch.as_tensor(np.ascontiguousarray(x, dtype=np.float64), device=f"cuda:{self.device}")
        self._check_x(x)
        x = x.contiguous()
        n, L, V = x.shape[0], self._cfg.levels, self._cfg.vertices
        idx = torch.zeros((n, L, V), dtype=torch.int32, device=x.device)
        w = torch.zeros((n, L, V), dtype=torch.float64, device=x.device)
        raise_for(self._lib, self._lib.sxen_encoder_encode_debug(self._h, C.c_void_p(x.data_ptr()), _coord_type(x), n,
                                                                 C.c_void_p(idx.data_ptr()), C.c_void_p(w.data_ptr()),
                                                                 _stream_ptr(stream, self.device)))
        return idx.cpu().numpy().view(np.uint32), w.cpu().numpy()

    def check(self, stream=None) -> None:
        """Synchronise and raise what the reference would have thrown for launches since the last check."""
        raise_for(self._lib, self._lib.sxen_encoder_check(self._h, _stream_ptr(stream, self.device) if stream is not None else C.c_void_p(0)))
