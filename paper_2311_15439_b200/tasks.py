"""Image-fitting task mirror (include/sxen/tasks.hpp, src/tasks.cpp): psnr_from_mse, render_image, fit_image.

Host logic only; sampling, encode, MLP, loss, updates and the rendered-image error all run in libsxen_b200."""
from __future__ import annotations

import ctypes as C
import enum
import math
from dataclasses import dataclass, field
from typing import List, Tuple

import numpy as np

from .encoding import EncoderConfig, HashEncoder
from .errors import raise_for
from .mlp import Mlp, MlpConfig
from .rng import hash_combine
from .trainer import TrainConfig, TrainResult, train_field

K_PSNR_CAP = 99.0  # include/sxen/tasks.hpp:15


def _lib():
    from . import lib
    return lib


def psnr_from_mse(mse: float) -> float:
    """src/tasks.cpp:30-33"""
    if not (mse > 0.0):
        return K_PSNR_CAP
    return min(K_PSNR_CAP, 10.0 * math.log10(1.0 / mse))


@dataclass
class FitImageOptions:  # include/sxen/tasks.hpp:30-34
    init_seed: int = 42
    mlp_hidden_width: int = 64
    mlp_hidden_layers: int = 2
    mlp_precision: int = 0  # 0 exact, 1 tcgen05 split-bf16, 2 tcgen05 bf16 (no reference analogue)


@dataclass
class FitImageResult:  # include/sxen/tasks.hpp:36-42
    encoder: HashEncoder
    mlp: Mlp
    train: TrainResult
    final_psnr: float = 0.0
    psnr_curve: List[Tuple[int, float]] = field(default_factory=list)


def _image_to_device(image, device: int):
    import torch
    px = np.ascontiguousarray(image, dtype=np.float64)
    if px.ndim != 3 or px.shape[2] != 3 or px.shape[0] < 1 or px.shape[1] < 1:  # ImageDataset::validate, src/image.cpp:16-29
        raise ValueError("image: pixel buffer size != width*height*3")
    if not ((px >= 0.0) & (px <= 1.0)).all():
        raise ValueError("image: pixel values must lie in [0, 1]")
    return torch.as_tensor(px, device=f"cuda:{device}"), px.shape[1], px.shape[0]


def image_sampler(image_dev, width: int, height: int, seed: int):
    """fit_image's BatchSampler (src/tasks.cpp:112-126) evaluated on the device."""
    import torch
    lib = _lib()

    def sampler(step: int, batch: int):
        coords = torch.empty((batch, 2), dtype=torch.float64, device=image_dev.device)
        targets = torch.empty((batch, 3), dtype=torch.float64, device=image_dev.device)
        raise_for(lib, lib.sxen_sample_image_batch(seed & ((1 << 64) - 1), step, C.c_void_p(image_dev.data_ptr()), width,
                                                   height, batch, C.c_void_p(coords.data_ptr()),
                                                   C.c_void_p(targets.data_ptr()),
                                                   C.c_void_p(torch.cuda.current_stream(image_dev.device).cuda_stream)))
        return coords, targets

    return sampler


def test_image_sampler(width: int, height: int, image_seed: int, train_seed: int, device: int = 0, first: int = 0,
                       count: int = None):
    """fit_image's BatchSampler over make_test_image(width, height, image_seed) without the image in memory
    (sxen_sample_test_image_batch; BASELINE configs[2]: a 32768 x 32768 image is 26 GB as doubles).  ``first`` / ``count``
    restrict every batch to that slice of its samples (a rank's chunk of a sharded batch)."""
    import torch
    lib = _lib()
    dev = torch.device(f"cuda:{device}")
    m64 = (1 << 64) - 1

    def sampler(step: int, batch: int):
        n = batch - first if count is None else count
        coords = torch.empty((n, 2), dtype=torch.float64, device=dev)
        targets = torch.empty((n, 3), dtype=torch.float64, device=dev)
        raise_for(lib, lib.sxen_sample_test_image_batch(image_seed & m64, width, height, train_seed & m64, step, first, n,
                                                        C.c_void_p(coords.data_ptr()), C.c_void_p(targets.data_ptr()),
                                                        C.c_void_p(torch.cuda.current_stream(dev).cuda_stream)))
        return coords, targets

    return sampler


def test_image_mse(encoder: HashEncoder, mlp: Mlp, width: int, height: int, image_seed: int, first_pixel: int = 0,
                   count: int = None, chunk: int = 1 << 20) -> float:
    """render_image's MSE (src/tasks.cpp:51-96, 35-46) against the never-materialised test image over pixels
    [first_pixel, first_pixel + count) in row-major order (default: the whole image)."""
    import torch
    lib = _lib()
    dev = torch.device(f"cuda:{encoder.device}")
    total = width * height - first_pixel if count is None else count
    acc = torch.zeros(1, dtype=torch.float64, device=dev)
    stream = C.c_void_p(torch.cuda.current_stream(dev).cuda_stream)
    coords = torch.empty((min(chunk, total), 2), dtype=torch.float64, device=dev)
    for off in range(0, total, chunk):
        n = min(chunk, total - off)
        raise_for(lib, lib.sxen_pixel_centers(width, height, first_pixel + off, n, C.c_void_p(coords.data_ptr()), stream))
        pred = mlp.forward(encoder.encode(coords[:n]))
        raise_for(lib, lib.sxen_test_image_sq_error(image_seed & ((1 << 64) - 1), width, height, C.c_void_p(pred.data_ptr()),
                                                    first_pixel + off, n, C.c_void_p(acc.data_ptr()), stream))
    return float(acc.item()) / (3.0 * total)


def fit_test_image(width: int, height: int, image_seed: int, encoder_cfg: EncoderConfig, train_cfg: TrainConfig,
                   opt: FitImageOptions = None, device: int = 0, psnr_pixels: int = 1 << 24) -> FitImageResult:
    """fit_image (src/tasks.cpp:98-137) on make_test_image(width, height, image_seed) evaluated on the fly -- the gigapixel
    workload (BASELINE configs[2]).  The final PSNR is measured over the first ``psnr_pixels`` pixels in row-major order
    (the whole image when it has no more than that)."""
    opt = opt or FitImageOptions()
    if encoder_cfg.dim != 2:
        raise ValueError("fit_image: encoder dim must be 2")
    encoder = HashEncoder(encoder_cfg, device=device)
    encoder.init_tables(opt.init_seed)
    mlp = Mlp(MlpConfig(encoder_cfg.encoded_width(), opt.mlp_hidden_width, opt.mlp_hidden_layers, 3), device=device)
    mlp.init_params(hash_combine(opt.init_seed, 1))
    if opt.mlp_precision:
        mlp.set_precision(opt.mlp_precision)
    train = train_field(encoder, mlp, test_image_sampler(width, height, image_seed, train_cfg.seed, device), train_cfg)
    result = FitImageResult(encoder, mlp, train)
    result.psnr_curve = [(s, psnr_from_mse(l)) for s, l in train.loss_curve]
    result.final_psnr = psnr_from_mse(test_image_mse(encoder, mlp, width, height, image_seed, 0,
                                                     min(psnr_pixels, width * height)))
    return result


def render_mse(encoder: HashEncoder, mlp: Mlp, image_dev, width: int, height: int, chunk: int = 1 << 20) -> float:
    """MSE of render_image(encoder, mlp) against the image over all channels (src/tasks.cpp:51-96, 35-46), without
    materialising the rendered image on the host."""
    import torch
    if encoder.config.dim != 2:
        raise ValueError("render_image: encoder dim must be 2")
    if mlp.config.input_width != encoder.config.encoded_width() or mlp.config.output_width != 3:
        raise ValueError("render_image: model widths do not form a 2D->RGB map")
    lib = _lib()
    dev = image_dev.device
    total = width * height
    acc = torch.zeros(1, dtype=torch.float64, device=dev)
    stream = C.c_void_p(torch.cuda.current_stream(dev).cuda_stream)
    coords = torch.empty((min(chunk, total), 2), dtype=torch.float64, device=dev)
    for first in range(0, total, chunk):
        n = min(chunk, total - first)
        raise_for(lib, lib.sxen_pixel_centers(width, height, first, n, C.c_void_p(coords.data_ptr()), stream))
        feats = encoder.encode(coords[:n])
        pred = mlp.forward(feats)
        raise_for(lib, lib.sxen_render_sq_error(C.c_void_p(pred.data_ptr()), C.c_void_p(image_dev.data_ptr()), first, n,
                                                C.c_void_p(acc.data_ptr()), stream))
    encoder.check()
    return float(acc.item()) / (3.0 * total)


def render_image(encoder: HashEncoder, mlp: Mlp, width: int, height: int, threads: int = 0, chunk: int = 1 << 20) -> np.ndarray:
    """sxen::render_image (src/tasks.cpp:51-96): the fitted model at every pixel centre, clamped to [0, 1], as a
    [height, width, 3] float64 array (ImageDataset::pixels order).  `threads` has no device meaning."""
    import torch
    if encoder.config.dim != 2:
        raise ValueError("render_image: encoder dim must be 2")
    if mlp.config.input_width != encoder.config.encoded_width() or mlp.config.output_width != 3:
        raise ValueError("render_image: model widths do not form a 2D->RGB map")
    if width < 1 or height < 1:
        raise ValueError("image: width and height must be >= 1")
    lib = _lib()
    dev = torch.device(f"cuda:{encoder.device}")
    total = width * height
    out = np.empty((total, 3), dtype=np.float64)
    stream = C.c_void_p(torch.cuda.current_stream(dev).cuda_stream)
    coords = torch.empty((min(chunk, total), 2), dtype=torch.float64, device=dev)
    for first in range(0, total, chunk):
        n = min(chunk, total - first)
        raise_for(lib, lib.sxen_pixel_centers(width, height, first, n, C.c_void_p(coords.data_ptr()), stream))
        pred = mlp.forward(encoder.encode(coords[:n]))
        out[first:first + n] = pred.double().clamp_(0.0, 1.0).cpu().numpy()
    encoder.check()
    return out.reshape(height, width, 3)


def image_mse(a: np.ndarray, b: np.ndarray) -> float:
    """src/tasks.cpp:35-45"""
    a, b = np.asarray(a, dtype=np.float64), np.asarray(b, dtype=np.float64)
    if a.shape != b.shape:
        raise ValueError("image_mse: shape mismatch")
    e = (a - b).ravel()
    return float(np.dot(e, e)) / e.size


def image_psnr(a: np.ndarray, b: np.ndarray) -> float:
    return psnr_from_mse(image_mse(a, b))


def fit_image(image, encoder_cfg: EncoderConfig, train_cfg: TrainConfig, opt: FitImageOptions = None,
              device: int = 0) -> FitImageResult:
    """sxen::fit_image (src/tasks.cpp:98-137): image is [h, w, 3] in [0, 1]."""
    opt = opt or FitImageOptions()
    image_dev, w, h = _image_to_device(image, device)
    if encoder_cfg.dim != 2:
        raise ValueError("fit_image: encoder dim must be 2")
    encoder = HashEncoder(encoder_cfg, device=device)
    encoder.init_tables(opt.init_seed)
    mlp = Mlp(MlpConfig(encoder_cfg.encoded_width(), opt.mlp_hidden_width, opt.mlp_hidden_layers, 3), device=device)
    mlp.init_params(hash_combine(opt.init_seed, 1))
    if opt.mlp_precision:
        mlp.set_precision(opt.mlp_precision)
    train = train_field(encoder, mlp, image_sampler(image_dev, w, h, train_cfg.seed), train_cfg)
    result = FitImageResult(encoder, mlp, train)
    result.psnr_curve = [(s, psnr_from_mse(l)) for s, l in train.loss_curve]
    result.final_psnr = psnr_from_mse(render_mse(encoder, mlp, image_dev, w, h))
    return result


# ------------------------------------------------------------------------------------------------ noise-field task
class NoiseKind(enum.IntEnum):  # include/sxen/noise.hpp:38; .name is to_string(NoiseKind)
    perlin = 0
    simplex = 1


@dataclass
class NoiseFieldSpec:  # include/sxen/noise.hpp:42-50, same defaults
    dim: int = 2
    seed: int = 7
    kind: int = NoiseKind.perlin
    octaves: int = 1
    frequency: float = 4.0

    def c(self):
        from . import _abi
        return _abi.NoiseSpecC(int(self.dim), int(self.kind), int(self.octaves), 0, int(self.seed) & ((1 << 64) - 1),
                               float(self.frequency))

    def validate(self) -> None:
        lib = _lib()
        spec = self.c()
        raise_for(lib, lib.sxen_noise_spec_validate(C.byref(spec)))


def noise_field_value(spec: NoiseFieldSpec, x, device: int = 0):
    """sxen::noise_field_value (src/noise.cpp:167-188), batched: x [N, dim] float64 (numpy or CUDA tensor) -> [N] float64
    of the same kind."""
    import torch
    lib = _lib()
    as_numpy = not isinstance(x, torch.Tensor)
    xd = torch.as_tensor(np.ascontiguousarray(x, dtype=np.float64), device=f"cuda:{device}") if as_numpy else x.contiguous()
    if xd.ndim != 2 or xd.shape[1] != spec.dim:  # src/noise.cpp:169-171
        raise ValueError("noise field: coordinate count != dim")
    if xd.dtype != torch.float64:
        raise ValueError("noise field: coordinates must be float64")
    if not bool(torch.isfinite(xd).all()):  # check_coords, src/noise.cpp:15-23
        raise ValueError("noise: coordinates must be finite")
    out = torch.empty((xd.shape[0],), dtype=torch.float64, device=xd.device)
    c = spec.c()
    raise_for(lib, lib.sxen_noise_field(C.byref(c), C.c_void_p(xd.data_ptr()), xd.shape[0], C.c_void_p(out.data_ptr()),
                                        C.c_void_p(torch.cuda.current_stream(xd.device).cuda_stream)))
    return out.cpu().numpy() if as_numpy else out


def field_sampler(spec: NoiseFieldSpec, seed: int, device: int = 0):
    """fit_field's BatchSampler (src/tasks.cpp:156-166) evaluated on the device."""
    import torch
    lib = _lib()
    c = spec.c()
    dev = torch.device(f"cuda:{device}")

    def sampler(step: int, batch: int):
        coords = torch.empty((batch, spec.dim), dtype=torch.float64, device=dev)
        targets = torch.empty((batch, 1), dtype=torch.float64, device=dev)
        raise_for(lib, lib.sxen_sample_field_batch(C.byref(c), seed & ((1 << 64) - 1), 1, step, batch,
                                                   C.c_void_p(coords.data_ptr()), C.c_void_p(targets.data_ptr()),
                                                   C.c_void_p(torch.cuda.current_stream(dev).cuda_stream)))
        return coords, targets

    return sampler


@dataclass
class FitFieldOptions:  # include/sxen/tasks.hpp:49-54
    init_seed: int = 42
    mlp_hidden_width: int = 64
    mlp_hidden_layers: int = 2
    holdout_samples: int = 1 << 14
    mlp_precision: int = 0  # as FitImageOptions


@dataclass
class FitFieldResult:  # include/sxen/tasks.hpp:56-62
    encoder: HashEncoder
    mlp: Mlp
    train: TrainResult
    holdout_mse: float = 0.0
    field_variance: float = 0.0


def fit_field(spec: NoiseFieldSpec, encoder_cfg: EncoderConfig, train_cfg: TrainConfig, opt: FitFieldOptions = None,
              device: int = 0) -> FitFieldResult:
    """sxen::fit_field (src/tasks.cpp:139-194): regress the scalar noise field over the unit cube, then evaluate on a
    hold-out stream training never sees."""
    import torch
    opt = opt or FitFieldOptions()
    spec.validate()
    if encoder_cfg.dim != spec.dim:
        raise ValueError(f"fit_field: encoder dim {encoder_cfg.dim} != field dim {spec.dim}")
    if opt.holdout_samples < 2:
        raise ValueError("fit_field: holdout_samples must be >= 2")
    lib = _lib()
    encoder = HashEncoder(encoder_cfg, device=device)
    encoder.init_tables(opt.init_seed)
    mlp = Mlp(MlpConfig(encoder_cfg.encoded_width(), opt.mlp_hidden_width, opt.mlp_hidden_layers, 1), device=device)
    mlp.init_params(hash_combine(opt.init_seed, 1))
    if opt.mlp_precision:
        mlp.set_precision(opt.mlp_precision)
    train = train_field(encoder, mlp, field_sampler(spec, train_cfg.seed, device), train_cfg)
    # hold-out: CounterRng(hash_combine(seed, 'HOLD')) without a stream id (src/tasks.cpp:172-173)
    dev = torch.device(f"cuda:{device}")
    n = opt.holdout_samples
    coords = torch.empty((n, spec.dim), dtype=torch.float64, device=dev)
    targets = torch.empty((n, 1), dtype=torch.float64, device=dev)
    c = spec.c()
    raise_for(lib, lib.sxen_sample_field_batch(C.byref(c), hash_combine(train_cfg.seed & ((1 << 64) - 1), 0x484f4c44), 0, 0, n,
                                               C.c_void_p(coords.data_ptr()), C.c_void_p(targets.data_ptr()),
                                               C.c_void_p(torch.cuda.current_stream(dev).cuda_stream)))
    pred = mlp.forward(encoder.encode(coords)).double()
    encoder.check()
    t = targets[:, 0]
    e = pred[:, 0] - t
    mse = float((e * e).sum().item()) / n
    mean = float(t.sum().item()) / n
    var = max(0.0, float((t * t).sum().item()) / n - mean * mean)  # src/tasks.cpp:189-192
    return FitFieldResult(encoder, mlp, train, holdout_mse=mse, field_variance=var)


def make_test_image(width: int, height: int, seed: int, device: int = 0) -> np.ndarray:
    """sxen::make_test_image (src/image.cpp:68-96): the reference's procedural RGB test image -- a shared 4-octave Perlin
    field plus one 5-octave field per channel at the pixel centres -- evaluated with the device noise kernels.
    Returns [height, width, 3] float64 in [0, 1]; agrees with the reference's image to rounding (libm), not to the bit."""
    import torch
    if width < 1 or height < 1:
        raise ValueError("test image: width and height must be >= 1")
    lib = _lib()
    dev = torch.device(f"cuda:{device}")
    total = width * height
    coords = torch.empty((total, 2), dtype=torch.float64, device=dev)
    raise_for(lib, lib.sxen_pixel_centers(width, height, 0, total, C.c_void_p(coords.data_ptr()),
                                          C.c_void_p(torch.cuda.current_stream(dev).cuda_stream)))
    m64 = (1 << 64) - 1
    shared = NoiseFieldSpec(dim=2, seed=hash_combine(seed & m64, 0xAB), kind=NoiseKind.perlin, octaves=4, frequency=4.0)
    base = noise_field_value(shared, coords)
    out = torch.empty((total, 3), dtype=torch.float64, device=dev)
    for c in range(3):
        ch = NoiseFieldSpec(dim=2, seed=hash_combine(seed & m64, c + 1), kind=NoiseKind.perlin, octaves=5, frequency=8.0)
        v = 0.45 * base + 0.55 * noise_field_value(ch, coords)
        out[:, c] = torch.clamp(0.5 + 0.62 * v, 0.0, 1.0)
    return out.cpu().numpy().reshape(height, width, 3)
