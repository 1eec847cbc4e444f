"""CPU: the C-ABI library loads and exports every symbol include/sxen_cuda.h declares; host-only entry points
(config validation, resolutions, rng scalars, hash) behave like the reference.  No device work here."""
import ctypes as C
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "sxen_cuda.h")


@pytest.fixture(scope="module")
def sx():
    if not os.path.exists(os.path.join(ROOT, "paper_2311_15439_b200", "lib", "libsxen_b200.so")):
        import __graft_entry__
        __graft_entry__.build()
    import paper_2311_15439_b200 as pkg
    return pkg


def declared_symbols():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"SXEN_API\s+[\w\s\*]+?\b(sxen_\w+)\s*\(", text)))


def test_header_declares_expected_surface():
    syms = declared_symbols()
    assert len(syms) >= 50
    for must in ("sxen_encoder_encode", "sxen_encoder_encode_backward", "sxen_encoder_encode_forward_backward",
                 "sxen_grad_create", "sxen_sparse_adam_step", "sxen_adam_step", "sxen_last_error"):
        assert must in syms


def test_library_exports_every_declared_symbol(sx):
    lib = C.CDLL(sx._abi.LIB_PATH)
    missing = [s for s in declared_symbols() if not hasattr(lib, s)]
    assert not missing, f"declared in sxen_cuda.h but not exported: {missing}"
    # and the Python binding covers the whole header
    unbound = [s for s in declared_symbols() if s not in sx._abi.SIGNATURES]
    assert not unbound, f"declared but not bound in _abi.py: {unbound}"


def test_missing_library_fails_loudly(sx):
    with pytest.raises(ImportError, match="no fallback"):
        sx._abi.load("/nonexistent/libsxen_b200.so")


def test_no_product_code_touches_the_oracle():
    """oracle/ is test infrastructure: the package, the public headers and the measurement tools never import, link or
    execute it.  Only tests/, __graft_entry__.py (build of the checker, smoke's check) and bench.py's CPU legs may."""
    for top in ("paper_2311_15439_b200", "include", "tools"):
        for dirpath, _, files in os.walk(os.path.join(ROOT, top)):
            for f in files:
                if f.endswith((".py", ".cu", ".cuh", ".hpp", ".h", ".sh")):
                    src = open(os.path.join(dirpath, f)).read()
                    for needle in ("import oracle", "from oracle", "sxen_oracle", "libsxen_ref", "oracle/_ref/lib"):
                        assert needle not in src, (top, f, needle)


def test_config_defaults_and_validation(sx):
    c = sx._abi.EncoderConfigC()
    assert sx.lib.sxen_encoder_config_default(C.byref(c)) == 0
    assert (c.dim, c.levels, c.table_size, c.features, c.base_resolution, c.growth, c.backend, c.level_scale) == \
        (2, 8, 1 << 16, 2, 16, 2.0, 0, 0)  # include/sxen/encoding.hpp:18-27
    ok = sx.EncoderConfig(dim=2, levels=2, table_size=1 << 10, features=2, base_resolution=4, growth=2.0)
    ok.validate()
    # reference tests/test_encoding.cpp:108-138
    for field, value in [("dim", 0), ("dim", 9), ("levels", 0), ("table_size", 1000), ("features", 0), ("features", 65),
                         ("base_resolution", 0), ("growth", 1.0), ("growth", float("nan")), ("growth", float("inf")),
                         ("levels", 40)]:
        bad = sx.EncoderConfig(**{**ok.__dict__, field: value})
        with pytest.raises(ValueError):
            bad.validate()
    a = sx._abi.AdamConfigC()
    assert sx.lib.sxen_adam_config_default(C.byref(a)) == 0
    assert (a.lr, a.beta1, a.beta2, a.epsilon) == (1e-3, 0.9, 0.99, 1e-15)


def test_host_scalars_match_golden(sx, golden_scalar):
    g = golden_scalar
    assert [sx.mix64(int(z)) for z in g["mix64_in"]] == g["mix64_out"].tolist()
    zs = g["mix64_in"]
    assert [sx.hash_combine(int(a), int(b)) for a in zs for b in zs[:4]] == g["hash_combine_out"].tolist()
    assert np.array_equal(np.array([sx.skew_constants(n) for n in range(1, 9)]), g["skew"])
    assert [sx.equal_memory_multiplier(n) for n in range(1, 9)] == g["eqmem"].tolist()
    for c, n, h in zip(g["hash_coords_in"], g["hash_coords_n"], g["hash_coords_out"]):
        assert sx.hash_coords(c[:n]) == h
    ladders = {
        "res_b16_g1.5": sx.EncoderConfig(dim=3, levels=16, base_resolution=16, growth=1.5, table_size=1 << 19),
        "res_b16_g2": sx.EncoderConfig(dim=2, levels=16, base_resolution=16, growth=2.0, table_size=1 << 19),
        "res_eqmem_n2": sx.EncoderConfig(dim=2, levels=10, base_resolution=16, growth=1.6, level_scale=1),
        "res_eqmem_n5": sx.EncoderConfig(dim=5, levels=10, base_resolution=7, growth=1.37, level_scale=1),
        "res_grid_eqmem": sx.EncoderConfig(dim=3, levels=6, base_resolution=16, growth=1.5, backend=1, level_scale=1),
    }
    for k, cfg in ladders.items():
        assert [sx.level_resolution(cfg, l) for l in range(cfg.levels)] == g[k].tolist()
    with pytest.raises(ValueError):
        sx.level_resolution(ladders["res_b16_g2"], 16)
    with pytest.raises(ValueError):
        sx.equal_memory_multiplier(0)
    with pytest.raises(ValueError):
        sx.skew_constants(9)


def test_no_device_means_loud_failure(sx):
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    assert sx.device_count() == 0
    with pytest.raises(sx.CudaError):
        sx.HashEncoder(sx.EncoderConfig())
