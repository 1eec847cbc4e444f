"""ctypes front-end for the CPU checker libraries (TEST INFRASTRUCTURE ONLY).

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / ``--impl reference`` legs may
import this package.  The product package (paper_2311_15439_b200) never does.

Two libraries, same semantics:
  * ``Oracle``  -> oracle/_build/libsxen_oracle.so : our plain-C restatement (sxen_oracle.c)
  * ``Ref``     -> oracle/_ref/libsxen_ref.so      : the unmodified reference + extern-C shim
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "_build", "libsxen_oracle.so")
REF_SO = os.path.join(HERE, "_ref", "libsxen_ref.so")
REF_ROOT = os.environ.get("SXEN_REF", "/root/reference/proj")

BACKEND_SIMPLEX, BACKEND_GRID = 0, 1
SCALE_RAW, SCALE_EQUAL_MEMORY = 0, 1


class CConfig(C.Structure):
    _fields_ = [
        ("dim", C.c_int32),
        ("levels", C.c_int32),
        ("table_size", C.c_uint32),
        ("features", C.c_int32),
        ("base_resolution", C.c_int32),
        ("growth", C.c_double),
        ("backend", C.c_int32),
        ("level_scale", C.c_int32),
    ]


class CMlpConfig(C.Structure):
    _fields_ = [
        ("input_width", C.c_int32),
        ("hidden_width", C.c_int32),
        ("hidden_layers", C.c_int32),
        ("output_width", C.c_int32),
    ]


class CAdamConfig(C.Structure):
    _fields_ = [("lr", C.c_double), ("beta1", C.c_double), ("beta2", C.c_double), ("epsilon", C.c_double)]


@dataclass
class Config:
    """Mirror of sxen::EncoderConfig (include/sxen/encoding.hpp:18-33), same defaults."""

    dim: int = 2
    levels: int = 8
    table_size: int = 1 << 16
    features: int = 2
    base_resolution: int = 16
    growth: float = 2.0
    backend: int = BACKEND_SIMPLEX
    level_scale: int = SCALE_RAW

    def c(self) -> CConfig:
        return CConfig(self.dim, self.levels, self.table_size, self.features, self.base_resolution,
                       self.growth, self.backend, self.level_scale)

    @property
    def encoded_width(self) -> int:
        return self.levels * self.features

    @property
    def vertices(self) -> int:
        return self.dim + 1 if self.backend == BACKEND_SIMPLEX else 1 << self.dim


@dataclass
class MlpConfig:
    input_width: int = 32
    hidden_width: int = 64
    hidden_layers: int = 2
    output_width: int = 3

    def c(self) -> CMlpConfig:
        return CMlpConfig(self.input_width, self.hidden_width, self.hidden_layers, self.output_width)

    @property
    def layer_count(self) -> int:
        return self.hidden_layers + 1

    def layer_in(self, l: int) -> int:
        return self.input_width if l == 0 else self.hidden_width

    def layer_out(self, l: int) -> int:
        return self.output_width if l == self.layer_count - 1 else self.hidden_width

    @property
    def param_count(self) -> int:
        return sum(self.layer_in(l) * self.layer_out(l) + self.layer_out(l) for l in range(self.layer_count))


@dataclass
class AdamConfig:
    lr: float = 1e-3
    beta1: float = 0.9
    beta2: float = 0.99
    epsilon: float = 1e-15

    def c(self) -> CAdamConfig:
        return CAdamConfig(self.lr, self.beta1, self.beta2, self.epsilon)


def build(ref: bool = True) -> None:
    """Compile the checker libraries (idempotent). The reference arm is only built when its tree exists."""
    targets = ["liboracle"]
    if ref and os.path.isdir(os.path.join(REF_ROOT, "src")):
        targets.append("ref")
    subprocess.run(["make", "-C", HERE, f"SXEN_REF={REF_ROOT}"] + targets, check=True,
                   stdout=subprocess.DEVNULL, stderr=subprocess.PIPE)


def _ptr(a, ct):
    return a.ctypes.data_as(C.POINTER(ct)) if a is not None else None


def _f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


def _f32(a):
    return np.ascontiguousarray(a, dtype=np.float32)


class Oracle:
    """Plain-C restatement. Every method names the reference lines it follows in sxen_oracle.c."""

    def __init__(self, path: str = ORACLE_SO):
        if not os.path.exists(path):
            build(ref=False)
        L = self.lib = C.CDLL(path)
        u64, dbl, i64 = C.c_uint64, C.c_double, C.c_int64
        P = C.POINTER
        L.sxo_mix64.restype = u64
        L.sxo_mix64.argtypes = [u64]
        L.sxo_hash_combine.restype = u64
        L.sxo_hash_combine.argtypes = [u64, u64]
        L.sxo_rng_key.restype = u64
        L.sxo_rng_key.argtypes = [u64, C.c_int, u64]
        L.sxo_rng_u64.restype = u64
        L.sxo_rng_u64.argtypes = [u64, u64]
        L.sxo_rng_double.restype = dbl
        L.sxo_rng_double.argtypes = [u64, u64]
        L.sxo_rng_fill_double.restype = None
        L.sxo_rng_fill_double.argtypes = [u64, u64, C.c_size_t, dbl, dbl, P(dbl)]
        L.sxo_validate.restype = C.c_int
        L.sxo_validate.argtypes = [P(CConfig)]
        L.sxo_equal_memory_multiplier.restype = dbl
        L.sxo_equal_memory_multiplier.argtypes = [C.c_int]
        L.sxo_level_resolution.restype = C.c_uint32
        L.sxo_level_resolution.argtypes = [P(CConfig), C.c_int]
        L.sxo_skew_constants.restype = None
        L.sxo_skew_constants.argtypes = [C.c_int, P(dbl)]
        L.sxo_subdivide.restype = None
        L.sxo_subdivide.argtypes = [C.c_int, P(dbl), P(C.c_uint8), P(dbl)]
        L.sxo_barycentric.restype = None
        L.sxo_barycentric.argtypes = [C.c_int, P(dbl), P(dbl)]
        L.sxo_hash_coords.restype = C.c_uint32
        L.sxo_hash_coords.argtypes = [C.c_int, P(i64)]
        L.sxo_init_tables.restype = None
        L.sxo_init_tables.argtypes = [P(CConfig), u64, P(C.c_float)]
        L.sxo_encode.restype = C.c_long
        L.sxo_encode.argtypes = [P(CConfig), P(C.c_float), P(dbl), C.c_size_t, P(C.c_float), P(u64)]
        L.sxo_encode_debug.restype = C.c_long
        L.sxo_encode_debug.argtypes = [P(CConfig), P(dbl), C.c_size_t, P(C.c_uint32), P(dbl), P(i64), P(C.c_uint8)]
        L.sxo_encode_backward.restype = C.c_long
        L.sxo_encode_backward.argtypes = [P(CConfig), P(dbl), P(dbl), C.c_size_t, P(dbl), P(C.c_uint8)]
        L.sxo_mlp_param_count.restype = C.c_size_t
        L.sxo_mlp_param_count.argtypes = [P(CMlpConfig)]
        L.sxo_mlp_validate.restype = C.c_int
        L.sxo_mlp_validate.argtypes = [P(CMlpConfig)]
        L.sxo_mlp_act_width.restype = C.c_size_t
        L.sxo_mlp_act_width.argtypes = [P(CMlpConfig)]
        L.sxo_mlp_init.restype = None
        L.sxo_mlp_init.argtypes = [P(CMlpConfig), u64, P(C.c_float)]
        L.sxo_mlp_forward.restype = None
        L.sxo_mlp_forward.argtypes = [P(CMlpConfig), P(C.c_float), P(C.c_float), C.c_size_t, P(C.c_float), P(C.c_float)]
        L.sxo_mlp_backward.restype = None
        L.sxo_mlp_backward.argtypes = [P(CMlpConfig), P(C.c_float), P(C.c_float), P(dbl), C.c_size_t, P(dbl), P(dbl)]
        L.sxo_adam_step.restype = C.c_long
        L.sxo_adam_step.argtypes = [P(C.c_float), P(dbl), P(dbl), P(dbl), C.c_size_t, i64, P(CAdamConfig)]
        L.sxo_sparse_adam_step.restype = C.c_long
        L.sxo_sparse_adam_step.argtypes = [P(CConfig), P(C.c_float), P(dbl), P(C.c_uint8), P(dbl), P(dbl), i64, P(CAdamConfig)]
        L.sxo_train_grads.restype = dbl
        L.sxo_train_grads.argtypes = [P(CConfig), P(CMlpConfig), P(C.c_float), P(C.c_float), P(dbl), P(dbl),
                                      C.c_size_t, C.c_size_t, P(dbl), P(C.c_uint8), P(dbl), P(dbl)]
        L.sxo_bench_fwd_bwd.restype = dbl
        L.sxo_bench_fwd_bwd.argtypes = [P(CConfig), P(C.c_float), P(dbl), P(dbl), C.c_size_t, C.c_int]

    # -- rng
    def mix64(self, z):
        return self.lib.sxo_mix64(z & (2**64 - 1))

    def hash_combine(self, a, b):
        return self.lib.sxo_hash_combine(a & (2**64 - 1), b & (2**64 - 1))

    def rng_key(self, seed, stream=None):
        return self.lib.sxo_rng_key(seed, 0 if stream is None else 1, 0 if stream is None else stream)

    def rng_u64(self, seed, stream, n):
        key = self.rng_key(seed, stream)
        return np.array([self.lib.sxo_rng_u64(key, i + 1) for i in range(n)], dtype=np.uint64)

    def rng_doubles(self, seed, stream, n, lo=0.0, hi=1.0, first=1):
        """next_double(lo,hi) draws first..first+n-1 of CounterRng(seed[, stream]). lo=0,hi=1 is exact next_double()."""
        out = np.empty(n, dtype=np.float64)
        self.lib.sxo_rng_fill_double(self.rng_key(seed, stream), first, n, lo, hi, _ptr(out, C.c_double))
        return out

    # -- config
    def validate(self, cfg: Config) -> int:
        return self.lib.sxo_validate(C.byref(cfg.c()))

    def level_resolution(self, cfg: Config, level: int) -> int:
        return self.lib.sxo_level_resolution(C.byref(cfg.c()), level)

    def resolutions(self, cfg: Config):
        return [self.level_resolution(cfg, l) for l in range(cfg.levels)]

    def equal_memory_multiplier(self, n):
        return self.lib.sxo_equal_memory_multiplier(n)

    def skew_constants(self, n):
        out = np.empty(3)
        self.lib.sxo_skew_constants(n, _ptr(out, C.c_double))
        return out

    def subdivide(self, fracs):
        fr = _f64(fracs)
        n = fr.size
        perm = np.empty(n, dtype=np.uint8)
        srt = np.empty(n)
        self.lib.sxo_subdivide(n, _ptr(fr, C.c_double), _ptr(perm, C.c_uint8), _ptr(srt, C.c_double))
        return perm, srt

    def barycentric(self, sorted_fracs):
        s = _f64(sorted_fracs)
        w = np.empty(s.size + 1)
        self.lib.sxo_barycentric(s.size, _ptr(s, C.c_double), _ptr(w, C.c_double))
        return w

    def hash_coords(self, coords):
        c = np.ascontiguousarray(coords, dtype=np.int64)
        return self.lib.sxo_hash_coords(c.size, _ptr(c, C.c_int64))

    # -- encoder
    def init_tables(self, cfg: Config, seed: int):
        t = np.empty((cfg.levels, cfg.table_size * cfg.features), dtype=np.float32)
        self.lib.sxo_init_tables(C.byref(cfg.c()), seed, _ptr(t, C.c_float))
        return t

    def encode(self, cfg: Config, tables, x, counters=None):
        x = _f64(x).reshape(-1, cfg.dim)
        tables = _f32(tables)
        out = np.zeros((x.shape[0], cfg.encoded_width), dtype=np.float32)
        bad = self.lib.sxo_encode(C.byref(cfg.c()), _ptr(tables, C.c_float), _ptr(x, C.c_double), x.shape[0],
                                  _ptr(out, C.c_float), _ptr(counters, C.c_uint64))
        return out, bad

    def encode_debug(self, cfg: Config, x):
        x = _f64(x).reshape(-1, cfg.dim)
        n, V = x.shape[0], cfg.vertices
        idx = np.zeros((n, cfg.levels, V), dtype=np.uint32)
        w = np.zeros((n, cfg.levels, V), dtype=np.float64)
        base = np.zeros((n, cfg.levels, cfg.dim), dtype=np.int64)
        perm = np.zeros((n, cfg.levels, cfg.dim), dtype=np.uint8)
        bad = self.lib.sxo_encode_debug(C.byref(cfg.c()), _ptr(x, C.c_double), n, _ptr(idx, C.c_uint32),
                                        _ptr(w, C.c_double), _ptr(base, C.c_int64), _ptr(perm, C.c_uint8))
        return idx, w, base, perm, bad

    def encode_backward(self, cfg: Config, x, upstream, grad=None, touched=None):
        x = _f64(x).reshape(-1, cfg.dim)
        up = _f64(upstream).reshape(-1, cfg.encoded_width)
        if grad is None:
            grad = np.zeros((cfg.levels, cfg.table_size, cfg.features), dtype=np.float64)
        if touched is None:
            touched = np.zeros((cfg.levels, cfg.table_size), dtype=np.uint8)
        bad = self.lib.sxo_encode_backward(C.byref(cfg.c()), _ptr(x, C.c_double), _ptr(up, C.c_double), x.shape[0],
                                           _ptr(grad, C.c_double), _ptr(touched, C.c_uint8))
        return grad, touched, bad

    # -- mlp
    def mlp_init(self, mc: MlpConfig, seed: int):
        p = np.empty(mc.param_count, dtype=np.float32)
        self.lib.sxo_mlp_init(C.byref(mc.c()), seed, _ptr(p, C.c_float))
        return p

    def mlp_forward(self, mc: MlpConfig, params, inputs):
        inputs = _f32(inputs).reshape(-1, mc.input_width)
        params = _f32(params)
        n = inputs.shape[0]
        aw = self.lib.sxo_mlp_act_width(C.byref(mc.c()))
        acts = np.empty((n, aw), dtype=np.float32)
        out = np.empty((n, mc.output_width), dtype=np.float32)
        self.lib.sxo_mlp_forward(C.byref(mc.c()), _ptr(params, C.c_float), _ptr(inputs, C.c_float), n,
                                 _ptr(acts, C.c_float), _ptr(out, C.c_float))
        return out, acts

    def mlp_backward(self, mc: MlpConfig, params, acts, upstream, grad=None):
        params = _f32(params)
        acts = _f32(acts)
        up = _f64(upstream).reshape(-1, mc.output_width)
        n = up.shape[0]
        if grad is None:
            grad = np.zeros(mc.param_count, dtype=np.float64)
        ig = np.empty((n, mc.input_width), dtype=np.float64)
        self.lib.sxo_mlp_backward(C.byref(mc.c()), _ptr(params, C.c_float), _ptr(acts, C.c_float),
                                  _ptr(up, C.c_double), n, _ptr(grad, C.c_double), _ptr(ig, C.c_double))
        return grad, ig

    # -- optimizers (in place on params/m/v)
    def adam_step(self, params, grads, m, v, t, ac: AdamConfig):
        return self.lib.sxo_adam_step(_ptr(params, C.c_float), _ptr(_f64(grads), C.c_double), _ptr(m, C.c_double),
                                      _ptr(v, C.c_double), params.size, t, C.byref(ac.c()))

    def sparse_adam_step(self, cfg: Config, tables, grad, touched, m, v, t, ac: AdamConfig):
        return self.lib.sxo_sparse_adam_step(C.byref(cfg.c()), _ptr(tables, C.c_float), _ptr(_f64(grad), C.c_double),
                                             _ptr(np.ascontiguousarray(touched, dtype=np.uint8), C.c_uint8),
                                             _ptr(m, C.c_double), _ptr(v, C.c_double), t, C.byref(ac.c()))

    def train_grads(self, cfg: Config, mc: MlpConfig, tables, mlp_params, coords, targets, global_batch=None):
        coords = _f64(coords).reshape(-1, cfg.dim)
        targets = _f64(targets).reshape(-1, mc.output_width)
        n = coords.shape[0]
        tg = np.zeros((cfg.levels, cfg.table_size, cfg.features), dtype=np.float64)
        touched = np.zeros((cfg.levels, cfg.table_size), dtype=np.uint8)
        mg = np.zeros(mc.param_count, dtype=np.float64)
        sl = np.zeros(n, dtype=np.float64)
        loss = self.lib.sxo_train_grads(C.byref(cfg.c()), C.byref(mc.c()), _ptr(_f32(tables), C.c_float),
                                        _ptr(_f32(mlp_params), C.c_float), _ptr(coords, C.c_double),
                                        _ptr(targets, C.c_double), n, global_batch or n, _ptr(tg, C.c_double),
                                        _ptr(touched, C.c_uint8), _ptr(mg, C.c_double), _ptr(sl, C.c_double))
        return loss, tg, touched, mg, sl

    def bench_fwd_bwd(self, cfg: Config, tables, x, upstream, threads: int) -> float:
        x = _f64(x).reshape(-1, cfg.dim)
        up = _f64(upstream).reshape(-1, cfg.encoded_width)
        return self.lib.sxo_bench_fwd_bwd(C.byref(cfg.c()), _ptr(_f32(tables), C.c_float), _ptr(x, C.c_double),
                                          _ptr(up, C.c_double), x.shape[0], threads)


class RefError(Exception):
    def __init__(self, status, msg):
        super().__init__(f"reference raised status={status}: {msg}")
        self.status = status


class Ref:
    """The unmodified reference library behind oracle/ref_shim.cpp."""

    @staticmethod
    def available() -> bool:
        return os.path.exists(REF_SO)

    def __init__(self, path: str = REF_SO):
        if not os.path.exists(path):
            build(ref=True)
        L = self.lib = C.CDLL(path)
        u64, dbl, vp = C.c_uint64, C.c_double, C.c_void_p
        P = C.POINTER
        L.sxr_last_error.restype = C.c_char_p
        L.sxr_mix64.restype = u64
        L.sxr_mix64.argtypes = [u64]
        L.sxr_hash_combine.restype = u64
        L.sxr_hash_combine.argtypes = [u64, u64]
        L.sxr_rng_u64.argtypes = [u64, C.c_int, u64, C.c_size_t, P(u64)]
        L.sxr_rng_double.argtypes = [u64, C.c_int, u64, C.c_size_t, dbl, dbl, C.c_int, P(dbl)]
        L.sxr_hash_coords.restype = C.c_uint32
        L.sxr_hash_coords.argtypes = [C.c_int, P(C.c_int64)]
        L.sxr_skew_constants.argtypes = [C.c_int, P(dbl)]
        L.sxr_subdivide.argtypes = [C.c_int, P(dbl), P(C.c_uint8), P(dbl)]
        L.sxr_barycentric.argtypes = [C.c_int, P(dbl), P(dbl)]
        L.sxr_validate.argtypes = [P(CConfig)]
        L.sxr_level_resolution.argtypes = [P(CConfig), C.c_int, P(C.c_uint32)]
        L.sxr_equal_memory_multiplier.restype = dbl
        L.sxr_equal_memory_multiplier.argtypes = [C.c_int]
        L.sxr_encoder_create.restype = vp
        L.sxr_encoder_create.argtypes = [P(CConfig)]
        L.sxr_encoder_destroy.argtypes = [vp]
        L.sxr_encoder_init_tables.argtypes = [vp, u64]
        L.sxr_encoder_table.restype = P(C.c_float)
        L.sxr_encoder_table.argtypes = [vp, C.c_int]
        L.sxr_encoder_resolution.restype = C.c_uint32
        L.sxr_encoder_resolution.argtypes = [vp, C.c_int]
        L.sxr_encoder_counters.argtypes = [vp, P(u64)]
        L.sxr_encoder_reset_counters.argtypes = [vp]
        L.sxr_encode.argtypes = [vp, P(dbl), C.c_size_t, P(C.c_float), P(C.c_long)]
        L.sxr_grad_create.restype = vp
        L.sxr_grad_create.argtypes = [C.c_int, C.c_uint32, C.c_int]
        L.sxr_grad_destroy.argtypes = [vp]
        L.sxr_grad_clear.argtypes = [vp]
        L.sxr_grad_touched_count.restype = C.c_size_t
        L.sxr_grad_touched_count.argtypes = [vp, C.c_int]
        L.sxr_grad_read.argtypes = [vp, C.c_int, P(C.c_uint32), P(dbl)]
        L.sxr_grad_merge.argtypes = [vp, vp]
        L.sxr_encode_backward.argtypes = [vp, P(dbl), P(dbl), C.c_size_t, vp, P(C.c_long)]
        L.sxr_mlp_create.restype = vp
        L.sxr_mlp_create.argtypes = [P(CMlpConfig)]
        L.sxr_mlp_destroy.argtypes = [vp]
        L.sxr_mlp_param_count.restype = C.c_size_t
        L.sxr_mlp_param_count.argtypes = [vp]
        L.sxr_mlp_params.restype = P(C.c_float)
        L.sxr_mlp_params.argtypes = [vp]
        L.sxr_mlp_init.argtypes = [vp, u64]
        L.sxr_mlp_forward_backward.argtypes = [vp, P(C.c_float), C.c_size_t, P(C.c_float), P(dbl), P(dbl), P(dbl)]
        L.sxr_adam_create.restype = vp
        L.sxr_adam_create.argtypes = [C.c_size_t]
        L.sxr_adam_destroy.argtypes = [vp]
        L.sxr_adam_step.argtypes = [vp, P(C.c_float), P(dbl), C.c_size_t, P(CAdamConfig)]
        L.sxr_sparse_adam_create.restype = vp
        L.sxr_sparse_adam_create.argtypes = [C.c_int, C.c_uint32, C.c_int]
        L.sxr_sparse_adam_destroy.argtypes = [vp]
        L.sxr_sparse_adam_step.argtypes = [vp, vp, vp, P(CAdamConfig)]
        L.sxr_train_field.argtypes = [vp, vp, P(dbl), P(dbl), C.c_int, C.c_int, C.c_int, P(CAdamConfig),
                                      P(CAdamConfig), P(dbl)]
        L.sxr_bench_fwd_bwd.restype = dbl
        L.sxr_bench_fwd_bwd.argtypes = [vp, P(dbl), P(dbl), C.c_size_t, C.c_int]
        L.sxr_hardware_concurrency.restype = C.c_int
        L.sxr_make_test_image.argtypes = [C.c_int, C.c_int, u64, P(dbl)]
        L.sxr_fit_image.argtypes = [P(dbl), C.c_int, C.c_int, P(CConfig), C.c_int, C.c_int, u64, C.c_int, u64, C.c_int,
                                    C.c_int, P(CAdamConfig), P(CAdamConfig), P(dbl), P(dbl), P(C.c_float), P(C.c_float)]
        L.sxr_psnr_from_mse.restype = dbl
        L.sxr_psnr_from_mse.argtypes = [dbl]
        if hasattr(L, "sxr_noise_field"):  # a libsxen_ref.so built before the noise shim lacks these two
            L.sxr_noise_field.argtypes = [C.c_int, u64, C.c_int, C.c_int, dbl, P(dbl), C.c_size_t, P(dbl)]
            L.sxr_fit_field.argtypes = [C.c_int, u64, C.c_int, C.c_int, dbl, P(CConfig), C.c_int, C.c_int, u64, C.c_int, u64,
                                        C.c_int, C.c_int, C.c_int, P(dbl), P(dbl), P(dbl)]
        L.sxr_save_checkpoint.argtypes = [C.c_char_p, vp, vp]
        L.sxr_load_checkpoint.argtypes = [C.c_char_p, P(CConfig), P(C.c_float), C.c_size_t, P(C.c_int), P(CMlpConfig),
                                          P(C.c_float), C.c_size_t]

    def _check(self, st):
        if st != 0:
            raise RefError(st, self.lib.sxr_last_error().decode())

    def mix64(self, z):
        return self.lib.sxr_mix64(z)

    def hash_combine(self, a, b):
        return self.lib.sxr_hash_combine(a, b)

    def rng_u64(self, seed, stream, n):
        out = np.empty(n, dtype=np.uint64)
        self.lib.sxr_rng_u64(seed, 0 if stream is None else 1, stream or 0, n, _ptr(out, C.c_uint64))
        return out

    def rng_doubles(self, seed, stream, n, lo=None, hi=None):
        out = np.empty(n, dtype=np.float64)
        ranged = lo is not None
        self.lib.sxr_rng_double(seed, 0 if stream is None else 1, stream or 0, n, lo or 0.0, hi or 0.0,
                                1 if ranged else 0, _ptr(out, C.c_double))
        return out

    def hash_coords(self, coords):
        c = np.ascontiguousarray(coords, dtype=np.int64)
        return self.lib.sxr_hash_coords(c.size, _ptr(c, C.c_int64))

    def skew_constants(self, n):
        out = np.empty(3)
        self._check(self.lib.sxr_skew_constants(n, _ptr(out, C.c_double)))
        return out

    def subdivide(self, fracs):
        fr = _f64(fracs)
        perm = np.empty(fr.size, dtype=np.uint8)
        srt = np.empty(fr.size)
        self._check(self.lib.sxr_subdivide(fr.size, _ptr(fr, C.c_double), _ptr(perm, C.c_uint8), _ptr(srt, C.c_double)))
        return perm, srt

    def barycentric(self, sorted_fracs):
        s = _f64(sorted_fracs)
        w = np.empty(s.size + 1)
        self._check(self.lib.sxr_barycentric(s.size, _ptr(s, C.c_double), _ptr(w, C.c_double)))
        return w

    def validate(self, cfg: Config) -> int:
        return self.lib.sxr_validate(C.byref(cfg.c()))

    def level_resolution(self, cfg: Config, level: int) -> int:
        out = C.c_uint32(0)
        self._check(self.lib.sxr_level_resolution(C.byref(cfg.c()), level, C.byref(out)))
        return out.value

    def equal_memory_multiplier(self, n):
        return self.lib.sxr_equal_memory_multiplier(n)

    def encoder(self, cfg: Config) -> "RefEncoder":
        return RefEncoder(self, cfg)

    def mlp(self, mc: MlpConfig) -> "RefMlp":
        return RefMlp(self, mc)

    def hardware_concurrency(self) -> int:
        return self.lib.sxr_hardware_concurrency()

    def make_test_image(self, width: int, height: int, seed: int):
        """sxen::make_test_image (src/image.cpp:68-96): [h, w, 3] doubles in [0, 1]."""
        out = np.empty((height, width, 3), dtype=np.float64)
        self._check(self.lib.sxr_make_test_image(width, height, seed, _ptr(out, C.c_double)))
        return out

    def fit_image(self, pixels, cfg: Config, batch: int, steps: int, train_seed: int = 1234, threads: int = 1,
                  init_seed: int = 42, hidden_width: int = 64, hidden_layers: int = 2, table_adam: AdamConfig = None,
                  mlp_adam: AdamConfig = None):
        """sxen::fit_image (src/tasks.cpp:98-137). Returns (final_psnr, loss[steps], tables[L, T*F], mlp_params)."""
        px = _f64(pixels)
        h, w = px.shape[0], px.shape[1]
        ta = (table_adam or AdamConfig(lr=1e-2)).c()
        ma = (mlp_adam or AdamConfig(lr=1e-3)).c()
        mc = MlpConfig(cfg.encoded_width, hidden_width, hidden_layers, 3)
        psnr = C.c_double()
        loss = np.zeros(steps, dtype=np.float64)
        tables = np.zeros((cfg.levels, cfg.table_size * cfg.features), dtype=np.float32)
        params = np.zeros(mc.param_count, dtype=np.float32)
        self._check(self.lib.sxr_fit_image(_ptr(px, C.c_double), w, h, C.byref(cfg.c()), batch, steps, train_seed, threads,
                                           init_seed, hidden_width, hidden_layers, C.byref(ta), C.byref(ma), C.byref(psnr),
                                           _ptr(loss, C.c_double), _ptr(tables, C.c_float), _ptr(params, C.c_float)))
        return psnr.value, loss, tables, params

    def psnr_from_mse(self, mse: float) -> float:
        return self.lib.sxr_psnr_from_mse(mse)

    def noise_field(self, dim: int, seed: int, kind: int, octaves: int, frequency: float, x) -> np.ndarray:
        """sxen::noise_field_value (src/noise.cpp:167-188) at every row of x [N, dim]; kind 0 perlin, 1 simplex."""
        xs = _f64(x)
        out = np.zeros(xs.shape[0], dtype=np.float64)
        self._check(self.lib.sxr_noise_field(dim, C.c_uint64(seed), kind, octaves, C.c_double(frequency), _ptr(xs, C.c_double),
                                             C.c_size_t(xs.shape[0]), _ptr(out, C.c_double)))
        return out

    def fit_field(self, dim: int, seed: int, kind: int, octaves: int, frequency: float, cfg: Config, batch: int, steps: int,
                  train_seed: int = 1234, threads: int = 1, init_seed: int = 42, hidden_width: int = 64,
                  hidden_layers: int = 2, holdout_samples: int = 1 << 14):
        """sxen::fit_field (src/tasks.cpp:139-194). Returns (loss[steps], holdout_mse, field_variance)."""
        loss = np.zeros(steps, dtype=np.float64)
        mse, var = C.c_double(), C.c_double()
        self._check(self.lib.sxr_fit_field(dim, C.c_uint64(seed), kind, octaves, C.c_double(frequency), C.byref(cfg.c()), batch,
                                           steps, C.c_uint64(train_seed), threads, C.c_uint64(init_seed), hidden_width,
                                           hidden_layers, holdout_samples, _ptr(loss, C.c_double), C.byref(mse), C.byref(var)))
        return loss, mse.value, var.value

    def save_checkpoint(self, path: str, encoder: "RefEncoder", mlp: "RefMlp" = None) -> None:
        self._check(self.lib.sxr_save_checkpoint(path.encode(), encoder.h, mlp.h if mlp is not None else None))

    def load_checkpoint(self, path: str, max_table_floats: int = 1 << 24, max_mlp_floats: int = 1 << 20):
        """Returns (Config, tables[L, T*F], MlpConfig or None, mlp params or None) as read by the reference."""
        cfg, mcfg, has = CConfig(), CMlpConfig(), C.c_int(0)
        tables = np.zeros(max_table_floats, dtype=np.float32)
        params = np.zeros(max_mlp_floats, dtype=np.float32)
        self._check(self.lib.sxr_load_checkpoint(path.encode(), C.byref(cfg), _ptr(tables, C.c_float), tables.size,
                                                 C.byref(has), C.byref(mcfg), _ptr(params, C.c_float), params.size))
        c = Config(cfg.dim, cfg.levels, cfg.table_size, cfg.features, cfg.base_resolution, cfg.growth, cfg.backend, 0)
        t = tables[:c.levels * c.table_size * c.features].reshape(c.levels, -1).copy()
        if not has.value:
            return c, t, None, None
        m = MlpConfig(mcfg.input_width, mcfg.hidden_width, mcfg.hidden_layers, mcfg.output_width)
        return c, t, m, params[:m.param_count].copy()


class RefEncoder:
    def __init__(self, ref: Ref, cfg: Config):
        self.ref, self.cfg = ref, cfg
        self.h = ref.lib.sxr_encoder_create(C.byref(cfg.c()))
        if not self.h:
            raise RefError(1, ref.lib.sxr_last_error().decode())

    def __del__(self):
        if getattr(self, "h", None):
            self.ref.lib.sxr_encoder_destroy(self.h)
            self.h = None

    def init_tables(self, seed):
        self.ref.lib.sxr_encoder_init_tables(self.h, seed)

    def table(self, level):
        """numpy view (no copy) of the reference's own table storage."""
        p = self.ref.lib.sxr_encoder_table(self.h, level)
        return np.ctypeslib.as_array(p, shape=(self.cfg.table_size * self.cfg.features,))

    def tables(self):
        return np.stack([self.table(l).copy() for l in range(self.cfg.levels)])

    def set_tables(self, tables):
        for l in range(self.cfg.levels):
            self.table(l)[:] = np.asarray(tables[l], dtype=np.float32).reshape(-1)

    def resolution(self, level):
        return self.ref.lib.sxr_encoder_resolution(self.h, level)

    def counters(self):
        out = np.zeros(2, dtype=np.uint64)
        self.ref.lib.sxr_encoder_counters(self.h, _ptr(out, C.c_uint64))
        return int(out[0]), int(out[1])

    def reset_counters(self):
        self.ref.lib.sxr_encoder_reset_counters(self.h)

    def encode(self, x):
        x = _f64(x).reshape(-1, self.cfg.dim)
        out = np.zeros((x.shape[0], self.cfg.encoded_width), dtype=np.float32)
        bad = C.c_long(-1)
        st = self.ref.lib.sxr_encode(self.h, _ptr(x, C.c_double), x.shape[0], _ptr(out, C.c_float), C.byref(bad))
        return out, bad.value, st

    def encode_backward(self, x, upstream):
        """Returns dense (grad[L,T,F] float64, touched[L,T] uint8, bad, status) from a fresh EncoderGradient."""
        cfg = self.cfg
        x = _f64(x).reshape(-1, cfg.dim)
        up = _f64(upstream).reshape(-1, cfg.encoded_width)
        lib = self.ref.lib
        g = lib.sxr_grad_create(cfg.levels, cfg.table_size, cfg.features)
        bad = C.c_long(-1)
        st = lib.sxr_encode_backward(self.h, _ptr(x, C.c_double), _ptr(up, C.c_double), x.shape[0], g, C.byref(bad))
        grad = np.zeros((cfg.levels, cfg.table_size, cfg.features), dtype=np.float64)
        touched = np.zeros((cfg.levels, cfg.table_size), dtype=np.uint8)
        order = []
        for l in range(cfg.levels):
            cnt = lib.sxr_grad_touched_count(g, l)
            idx = np.empty(cnt, dtype=np.uint32)
            vals = np.empty((cnt, cfg.features), dtype=np.float64)
            lib.sxr_grad_read(g, l, _ptr(idx, C.c_uint32), _ptr(vals, C.c_double))
            grad[l, idx] = vals
            touched[l, idx] = 1
            order.append(idx)
        lib.sxr_grad_destroy(g)
        return grad, touched, order, bad.value, st

    def bench_fwd_bwd(self, x, upstream, threads: int) -> float:
        x = _f64(x).reshape(-1, self.cfg.dim)
        up = _f64(upstream).reshape(-1, self.cfg.encoded_width)
        return self.ref.lib.sxr_bench_fwd_bwd(self.h, _ptr(x, C.c_double), _ptr(up, C.c_double), x.shape[0], threads)


class RefMlp:
    def __init__(self, ref: Ref, mc: MlpConfig):
        self.ref, self.mc = ref, mc
        self.h = ref.lib.sxr_mlp_create(C.byref(mc.c()))
        if not self.h:
            raise RefError(1, ref.lib.sxr_last_error().decode())

    def __del__(self):
        if getattr(self, "h", None):
            self.ref.lib.sxr_mlp_destroy(self.h)
            self.h = None

    def params(self):
        n = self.ref.lib.sxr_mlp_param_count(self.h)
        return np.ctypeslib.as_array(self.ref.lib.sxr_mlp_params(self.h), shape=(n,))

    def init(self, seed):
        self.ref.lib.sxr_mlp_init(self.h, seed)

    def forward_backward(self, inputs, upstream=None):
        mc = self.mc
        inputs = _f32(inputs).reshape(-1, mc.input_width)
        n = inputs.shape[0]
        out = np.empty((n, mc.output_width), dtype=np.float32)
        grad = np.zeros(mc.param_count, dtype=np.float64)
        ig = np.zeros((n, mc.input_width), dtype=np.float64)
        up = _f64(upstream).reshape(-1, mc.output_width) if upstream is not None else None
        st = self.ref.lib.sxr_mlp_forward_backward(self.h, _ptr(inputs, C.c_float), n, _ptr(out, C.c_float),
                                                   _ptr(up, C.c_double), _ptr(grad, C.c_double), _ptr(ig, C.c_double))
        self.ref._check(st)
        return out, grad, ig
