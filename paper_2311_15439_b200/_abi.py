"""ctypes declarations for libsxen_b200.so -- one entry per function in include/sxen_cuda.h.

The library is the product; there is no fallback.  Importing this module without the built .so raises.
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "lib", "libsxen_b200.so")

OK, INVALID_ARGUMENT, LOGIC_ERROR, TRAINING_ERROR, CUDA_ERROR, IO_ERROR, NCCL_ERROR = range(7)
BACKEND_SIMPLEX, BACKEND_GRID = 0, 1
SCALE_RAW, SCALE_EQUAL_MEMORY = 0, 1
COORD_F64, COORD_F32 = 0, 1
MLP_EXACT, MLP_TENSOR_BF16X3, MLP_TENSOR_BF16, MLP_TENSOR_BF16X4 = 0, 1, 2, 3


class EncoderConfigC(C.Structure):
    _fields_ = [("dim", C.c_int32), ("levels", C.c_int32), ("table_size", C.c_uint32), ("features", C.c_int32),
                ("base_resolution", C.c_int32), ("growth", C.c_double), ("backend", C.c_int32),
                ("level_scale", C.c_int32)]


class MlpConfigC(C.Structure):
    _fields_ = [("input_width", C.c_int32), ("hidden_width", C.c_int32), ("hidden_layers", C.c_int32),
                ("output_width", C.c_int32)]


class AdamConfigC(C.Structure):
    _fields_ = [("lr", C.c_double), ("beta1", C.c_double), ("beta2", C.c_double), ("epsilon", C.c_double)]


class LookupCountersC(C.Structure):
    _fields_ = [("touched_vertices", C.c_uint64), ("out_of_bounds", C.c_uint64)]


class NoiseSpecC(C.Structure):  # sxen_noise_spec
    _fields_ = [("dim", C.c_int32), ("kind", C.c_int32), ("octaves", C.c_int32), ("reserved", C.c_int32),
                ("seed", C.c_uint64), ("frequency", C.c_double)]


class TuningC(C.Structure):
    _fields_ = [("levels_per_thread", C.c_int32), ("block_threads", C.c_int32), ("level_major", C.c_int32),
                ("exact_blend", C.c_int32), ("warp_aggregate", C.c_int32), ("merge_pairs", C.c_int32),
                ("cache_hints", C.c_int32), ("coarse_replicas", C.c_int32), ("level_chunk", C.c_int32)]


_P = C.POINTER
_vp, _u64, _i32, _u32, _sz, _dbl = C.c_void_p, C.c_uint64, C.c_int32, C.c_uint32, C.c_size_t, C.c_double

# name -> (restype, argtypes).  Status-returning functions use c_int.
SIGNATURES = {
    "sxen_last_error": (C.c_char_p, []),
    "sxen_version": (C.c_char_p, []),
    "sxen_device_count": (_i32, []),
    "sxen_launch_count": (_u64, []),
    "sxen_host_alloc": (C.c_int, [_sz, _P(_vp)]),
    "sxen_host_free": (C.c_int, [_vp]),
    "sxen_mix64": (_u64, [_u64]),
    "sxen_hash_combine": (_u64, [_u64, _u64]),
    "sxen_rng_fill_dev": (C.c_int, [_u64, _i32, _u64, _u64, _dbl, _dbl, _vp, _sz, C.c_int, _vp]),
    "sxen_encoder_config_default": (C.c_int, [_P(EncoderConfigC)]),
    "sxen_encoder_validate": (C.c_int, [_P(EncoderConfigC)]),
    "sxen_level_resolution": (C.c_int, [_P(EncoderConfigC), _i32, _P(_u32)]),
    "sxen_equal_memory_multiplier": (C.c_int, [_i32, _P(_dbl)]),
    "sxen_skew_constants": (C.c_int, [_i32, _P(_dbl)]),
    "sxen_hash_coords": (C.c_int, [_P(C.c_int64), _i32, _P(_u32)]),
    "sxen_encoder_create": (C.c_int, [_P(EncoderConfigC), _i32, _P(_vp)]),
    "sxen_encoder_destroy": (C.c_int, [_vp]),
    "sxen_encoder_get_config": (C.c_int, [_vp, _P(EncoderConfigC)]),
    "sxen_encoder_resolution": (C.c_int, [_vp, _i32, _P(_u32)]),
    "sxen_encoder_parameter_count": (C.c_int, [_vp, _P(_u64)]),
    "sxen_encoder_set_tuning": (C.c_int, [_vp, _P(TuningC)]),
    "sxen_encoder_get_tuning": (C.c_int, [_vp, _P(TuningC)]),
    "sxen_encoder_init_tables": (C.c_int, [_vp, _u64, _vp]),
    "sxen_encoder_upload_table": (C.c_int, [_vp, _i32, _P(C.c_float)]),
    "sxen_encoder_download_table": (C.c_int, [_vp, _i32, _P(C.c_float)]),
    "sxen_encoder_tables_dev": (C.c_int, [_vp, _P(_vp)]),
    "sxen_encoder_encode": (C.c_int, [_vp, _vp, C.c_int, _sz, _vp, _vp]),
    "sxen_encoder_encode_debug": (C.c_int, [_vp, _vp, C.c_int, _sz, _vp, _vp, _vp]),
    "sxen_encoder_encode_backward": (C.c_int, [_vp, _vp, C.c_int, _vp, _sz, _vp, _vp]),
    "sxen_encoder_encode_forward_backward": (C.c_int, [_vp, _vp, C.c_int, _vp, _sz, _vp, _vp, _vp]),
    "sxen_encoder_encode_backward_levels": (C.c_int, [_vp, _vp, C.c_int, _vp, _sz, _vp, C.c_int32, C.c_int32, _vp]),
    "sxen_encoder_encode_forward_backward_levels": (C.c_int, [_vp, _vp, C.c_int, _vp, _sz, _vp, _vp, C.c_int32, C.c_int32, _vp]),
    "sxen_encoder_check": (C.c_int, [_vp, _vp]),
    "sxen_encoder_counters": (C.c_int, [_vp, _P(LookupCountersC)]),
    "sxen_encoder_reset_counters": (C.c_int, [_vp]),
    "sxen_encoder_encode_host": (C.c_int, [_vp, _P(_dbl), _sz, _P(C.c_float)]),
    "sxen_encoder_encode_backward_host": (C.c_int, [_vp, _P(_dbl), _P(_dbl), _sz, _vp]),
    "sxen_encoder_encode_forward_backward_host": (C.c_int, [_vp, _P(_dbl), _vp, C.c_int, _sz, _P(C.c_float), _vp]),
    "sxen_grad_create": (C.c_int, [_vp, _P(_vp)]),
    "sxen_grad_destroy": (C.c_int, [_vp]),
    "sxen_grad_clear": (C.c_int, [_vp, _vp]),
    "sxen_grad_values_dev": (C.c_int, [_vp, _P(_vp), _P(_sz)]),
    "sxen_grad_download": (C.c_int, [_vp, _i32, _P(C.c_float), _P(C.c_uint8)]),
    "sxen_grad_upload": (C.c_int, [_vp, _i32, _P(C.c_float), _P(C.c_uint8)]),
    "sxen_grad_touched_total": (C.c_int, [_vp, _P(_u64)]),
    "sxen_grad_merge": (C.c_int, [_vp, _vp, _vp]),
    "sxen_adam_config_default": (C.c_int, [_P(AdamConfigC)]),
    "sxen_sparse_adam_create": (C.c_int, [_vp, _P(_vp)]),
    "sxen_sparse_adam_destroy": (C.c_int, [_vp]),
    "sxen_sparse_adam_step_count": (C.c_int, [_vp, _P(C.c_int64)]),
    "sxen_sparse_adam_step": (C.c_int, [_vp, _vp, _vp, _P(AdamConfigC), _i32, _vp]),
    "sxen_sparse_adam_check": (C.c_int, [_vp, _vp]),
    "sxen_sparse_adam_download": (C.c_int, [_vp, _i32, _P(_dbl), _P(_dbl)]),
    "sxen_adam_create": (C.c_int, [_sz, _i32, _P(_vp)]),
    "sxen_adam_destroy": (C.c_int, [_vp]),
    "sxen_adam_step_count": (C.c_int, [_vp, _P(C.c_int64)]),
    "sxen_adam_step": (C.c_int, [_vp, _vp, _vp, C.c_int, _sz, _P(AdamConfigC), _vp]),
    "sxen_adam_check": (C.c_int, [_vp, _vp]),
    "sxen_mlp_config_default": (C.c_int, [_P(MlpConfigC)]),
    "sxen_mlp_validate": (C.c_int, [_P(MlpConfigC)]),
    "sxen_mlp_create": (C.c_int, [_P(MlpConfigC), _i32, _P(_vp)]),
    "sxen_mlp_destroy": (C.c_int, [_vp]),
    "sxen_mlp_get_config": (C.c_int, [_vp, _P(MlpConfigC)]),
    "sxen_mlp_parameter_count": (C.c_int, [_vp, _P(_u64)]),
    "sxen_mlp_init_params": (C.c_int, [_vp, _u64, _vp]),
    "sxen_mlp_upload_params": (C.c_int, [_vp, _P(C.c_float)]),
    "sxen_mlp_download_params": (C.c_int, [_vp, _P(C.c_float)]),
    "sxen_mlp_params_dev": (C.c_int, [_vp, _P(_vp)]),
    "sxen_mlp_grads_dev": (C.c_int, [_vp, _P(_vp)]),
    "sxen_mlp_grad_clear": (C.c_int, [_vp, _vp]),
    "sxen_mlp_grad_download": (C.c_int, [_vp, _P(_dbl)]),
    "sxen_mlp_forward": (C.c_int, [_vp, _vp, _sz, _vp, _vp]),
    "sxen_mlp_backward": (C.c_int, [_vp, _vp, _sz, _vp, _vp, _vp]),
    "sxen_mlp_forward_host": (C.c_int, [_vp, _vp, _sz, _vp]),
    "sxen_mlp_backward_host": (C.c_int, [_vp, _vp, _sz, _vp]),
    "sxen_mlp_set_precision": (C.c_int, [_vp, _i32]),
    "sxen_mlp_get_precision": (C.c_int, [_vp, _P(_i32)]),
    "sxen_mlp_forward_backward": (C.c_int, [_vp, _vp, _vp, C.c_int, _sz, _sz, _vp, _vp, _vp, _vp]),
    "sxen_mlp_activations_dev": (C.c_int, [_vp, _P(_vp), _P(_sz), _P(_sz)]),
    "sxen_mse_loss": (C.c_int, [_vp, _sz, _vp, C.c_int, _i32, _sz, _sz, _vp, _vp, _vp, _vp]),
    "sxen_sample_image_batch": (C.c_int, [_u64, _u64, _vp, _i32, _i32, _sz, _vp, _vp, _vp]),
    "sxen_pixel_centers": (C.c_int, [_i32, _i32, _sz, _sz, _vp, _vp]),
    "sxen_render_sq_error": (C.c_int, [_vp, _vp, _sz, _sz, _vp, _vp]),
    "sxen_noise_spec_default": (C.c_int, [_P(NoiseSpecC)]),
    "sxen_noise_spec_validate": (C.c_int, [_P(NoiseSpecC)]),
    "sxen_noise_field": (C.c_int, [_P(NoiseSpecC), _vp, _sz, _vp, _vp]),
    "sxen_sample_field_batch": (C.c_int, [_P(NoiseSpecC), C.c_uint64, C.c_int32, C.c_uint64, _sz, _vp, _vp, _vp]),
    "sxen_trainer_create": (C.c_int, [_vp, _vp, _P(_vp)]),
    "sxen_trainer_destroy": (C.c_int, [_vp]),
    "sxen_trainer_accumulate": (C.c_int, [_vp, _vp, C.c_int, _vp, C.c_int, _sz, _sz, _vp]),
    "sxen_trainer_accumulate_head": (C.c_int, [_vp, _vp, C.c_int, _vp, C.c_int, _sz, _sz, _vp]),
    "sxen_trainer_accumulate_tables": (C.c_int, [_vp, _vp, C.c_int, _sz, C.c_int32, C.c_int32, _vp]),
    "sxen_trainer_table_grad": (C.c_int, [_vp, _P(_vp)]),
    "sxen_trainer_loss_dev": (C.c_int, [_vp, _P(_vp)]),
    "sxen_trainer_loss": (C.c_int, [_vp, _sz, _P(_dbl), _vp]),
    "sxen_trainer_update": (C.c_int, [_vp, _P(AdamConfigC), _P(AdamConfigC), _vp]),
    "sxen_trainer_check": (C.c_int, [_vp, _vp]),
    "sxen_trainer_step": (C.c_int, [_vp, _vp, C.c_int, _vp, C.c_int, _sz, _P(AdamConfigC), _P(AdamConfigC), _P(_dbl), _vp]),
    "sxen_trainer_step_enqueue": (C.c_int, [_vp, _vp, C.c_int, _vp, C.c_int, _sz, _P(AdamConfigC), _P(AdamConfigC), _vp]),
    "sxen_device_alloc": (C.c_int, [_i32, _sz, _P(_vp)]),
    "sxen_device_free": (C.c_int, [_i32, _vp]),
    "sxen_device_upload": (C.c_int, [_i32, _vp, _vp, _sz, _vp]),
    "sxen_device_download": (C.c_int, [_i32, _vp, _vp, _sz, _vp]),
    "sxen_device_zero": (C.c_int, [_i32, _vp, _sz, _vp]),
    "sxen_trainer_create_aux": (C.c_int, [_vp, _vp, _i32, _P(_vp)]),
    "sxen_trainer_set_aux": (C.c_int, [_vp, _vp, C.c_int]),
    "sxen_trainer_pending": (C.c_int, [_vp, _P(_sz)]),
    "sxen_trainer_collect": (C.c_int, [_vp, _P(_dbl), _sz, _P(_sz), _P(C.c_int64), _vp]),
    "sxen_grad_set_reproducible": (C.c_int, [_vp, _i32]),
    "sxen_grad_is_reproducible": (C.c_int, [_vp, _P(_i32)]),
    "sxen_grad_fixed_dev": (C.c_int, [_vp, _P(_vp), _P(_sz)]),
    "sxen_grad_download_f64": (C.c_int, [_vp, _i32, _P(_dbl)]),
    "sxen_mlp_set_reproducible": (C.c_int, [_vp, _i32]),
    "sxen_trainer_set_reproducible": (C.c_int, [_vp, _i32]),
    "sxen_trainer_set_fused": (C.c_int, [_vp, _i32]),
    "sxen_sample_test_image_batch": (C.c_int, [_u64, _i32, _i32, _u64, _u64, _sz, _sz, _vp, _vp, _vp]),
    "sxen_test_image_sq_error": (C.c_int, [_u64, _i32, _i32, _vp, _sz, _sz, _vp, _vp]),
    "sxen_debug_tc_progress": (C.c_int, [_vp]),
    "sxen_debug_fused_timing": (C.c_int, [_vp]),
    "sxen_debug_tc_timing": (C.c_int, [_vp]),
    "sxen_debug_tc_variant": (C.c_int, [_i32]),
    "sxen_comm_unique_id": (C.c_int, [_vp]),
    "sxen_comm_create": (C.c_int, [_vp, _i32, _i32, _i32, _P(_vp)]),
    "sxen_comm_create_local": (C.c_int, [_i32, _P(_i32), _P(_vp)]),
    "sxen_comm_destroy": (C.c_int, [_vp]),
    "sxen_comm_abort": (C.c_int, [_vp]),
    "sxen_comm_info": (C.c_int, [_vp, _P(_i32), _P(_i32), _P(_i32), _P(_i32)]),
    "sxen_comm_allreduce": (C.c_int, [_vp, _vp, _sz, C.c_int, _vp]),
    "sxen_trainer_set_comm": (C.c_int, [_vp, _vp]),
    "sxen_trainer_allreduce_head": (C.c_int, [_vp, _vp]),
    "sxen_trainer_allreduce_levels": (C.c_int, [_vp, _i32, _i32, _vp]),
    "sxen_trainer_step_sharded": (C.c_int, [_vp, _vp, C.c_int, _vp, C.c_int, _sz, _P(AdamConfigC), _P(AdamConfigC), _i32,
                                            _P(_dbl), _vp]),
}


def load(path: str = LIB_PATH) -> C.CDLL:
    if not os.path.exists(path):
        raise ImportError(
            f"{path} is missing: the CUDA extension is the product and there is no fallback. "
            "Build it with `python -c 'import __graft_entry__ as g; g.build()'` or `make -C paper_2311_15439_b200/csrc`.")
    lib = C.CDLL(path)
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)  # AttributeError here = header/library drift
        fn.restype = res
        fn.argtypes = args
    return lib
