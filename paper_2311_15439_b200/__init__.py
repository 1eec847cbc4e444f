"""paper_2311_15439_b200 -- B200-native simplex multiresolution hash encoding (hot path of arXiv 2311.15439).

Host-side mirror of the reference's C++ interface for the encode path (names follow
/root/reference/proj/include/sxen/*.hpp) over the C ABI in include/sxen_cuda.h.  All compute happens in
lib/libsxen_b200.so (hand-written sm_100a kernels); importing the package without it raises ImportError.
"""
from . import _abi

lib = _abi.load()  # raises ImportError when the CUDA extension has not been built

from .errors import CudaError, IoError, TrainingError  # noqa: E402
from .encoding import (Backend, EncoderConfig, EncoderGradient, HashEncoder, LevelScale, LookupCounters,  # noqa: E402
                       Tuning, equal_memory_multiplier, hash_coords, level_resolution, skew_constants)
from .optimizer import AdamConfig, AdamState, SparseAdamState  # noqa: E402
from .mlp import Mlp, MlpConfig  # noqa: E402
from .trainer import TrainConfig, Trainer, TrainResult, chunk_bounds, level_ranges, train_field  # noqa: E402
from .checkpoint import load_checkpoint, save_checkpoint  # noqa: E402
from .tasks import (FitFieldOptions, FitFieldResult, FitImageOptions, FitImageResult, NoiseFieldSpec, NoiseKind,  # noqa: E402
                    field_sampler, fit_field, fit_image, image_mse, image_psnr, image_sampler, make_test_image,
                    noise_field_value, psnr_from_mse, render_image, render_mse, fit_test_image, test_image_mse,
                    test_image_sampler)
from .rng import CounterRng, hash_combine, mix64  # noqa: E402
from .comm import Comm, CommError  # noqa: E402
from .analysis import (KernelBenchConfig, KernelBenchReport, bench_kernel, bench_side, read_kernel_csv,  # noqa: E402
                       write_kernel_csv)

__all__ = ["lib", "CudaError", "IoError", "TrainingError", "Backend", "LevelScale", "EncoderConfig", "HashEncoder",
           "EncoderGradient", "LookupCounters", "Tuning", "equal_memory_multiplier", "level_resolution",
           "skew_constants", "hash_coords", "AdamConfig", "AdamState", "SparseAdamState", "CounterRng", "mix64",
           "hash_combine", "Mlp", "MlpConfig", "TrainConfig", "Trainer", "TrainResult", "chunk_bounds", "level_ranges", "train_field",
           "FitImageOptions", "FitImageResult", "fit_image", "image_sampler", "psnr_from_mse", "render_mse", "render_image", "image_mse", "image_psnr",
           "save_checkpoint", "load_checkpoint", "KernelBenchConfig", "KernelBenchReport", "bench_kernel", "bench_side",
           "read_kernel_csv", "write_kernel_csv", "NoiseKind", "NoiseFieldSpec", "noise_field_value", "field_sampler",
           "FitFieldOptions", "FitFieldResult", "fit_field", "make_test_image", "Comm", "CommError", "fit_test_image", "test_image_sampler",
           "test_image_mse"]


def device_count() -> int:
    """Visible sm_100 devices."""
    return lib.sxen_device_count()


def launch_count() -> int:
    """Kernels this library has launched since load."""
    return lib.sxen_launch_count()
