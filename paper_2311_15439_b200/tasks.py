"""Image-fitting task mirror (include/sxen/tasks.hpp, src/tasks.cpp): psnr_from_mse, render_image, fit_image.

Host logic only; sampling, encode, MLP, loss, updates and the rendered-image error all run in libsxen_b200."""
from __future__ import annotations

import ctypes as C
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
                                                   C.c_void_p(torch.cuda.current_stream().cuda_stream)))
        return coords, targets

    return sampler


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
    stream = C.c_void_p(torch.cuda.current_stream().cuda_stream)
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
