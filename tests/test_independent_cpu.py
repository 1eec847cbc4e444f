"""CPU: the numpy first-principles pipelines of tests/independent.py against the C oracle -- the reference's own
"both backends match the independent pipeline at random points and levels" (tests/test_encoding.cpp:224-251), its hash
cross-check (:47-59), the dense-matrix skew check (tests/test_lattice.cpp:87-115) and the dense matrix-product MLP check
(tests/test_neural.cpp:68-81), with the oracle in the library's seat.  The device suites then use the same pipelines."""
import numpy as np
import pytest

import oracle
from independent import (encode_grid_level, encode_simplex_level, mlp_forward, simplex_vertices, skew_matrix, spatial_hash,
                         unskew_matrix)


def small_config(backend, dim, levels=2):      # tests/test_encoding.cpp:16-27
    return oracle.Config(dim=dim, levels=levels, table_size=1 << 10, features=2, base_resolution=4, growth=2.0,
                         backend=backend, level_scale=oracle.SCALE_RAW)


def test_hash_agrees_with_the_independent_reimplementation(oracle_lib):     # :47-59
    rng = np.random.default_rng(21)
    for n in range(1, 9):
        coords = rng.integers(-(1 << 20), 1 << 20, size=(200, n), dtype=np.int64)
        want = spatial_hash(coords)
        for c, w in zip(coords, want):
            assert oracle_lib.hash_coords(c) == int(w)
    assert spatial_hash(np.zeros((1, 5), dtype=np.int64))[0] == 0           # :39-45


def test_skew_matrices_are_exact_inverses_and_match_the_constants(oracle_lib):   # tests/test_lattice.cpp:39-45, 87-115
    for n in range(1, 9):
        f, g = oracle_lib.skew_constants(n)[:2]
        assert np.allclose(skew_matrix(n) @ unskew_matrix(n), np.eye(n), atol=1e-14)
        assert abs((skew_matrix(n) - np.eye(n))[0, 0] - f) < 1e-15 and abs((np.eye(n) - unskew_matrix(n))[0, 0] - g) < 1e-15


@pytest.mark.parametrize("backend", [oracle.BACKEND_SIMPLEX, oracle.BACKEND_GRID])
def test_oracle_matches_the_independent_pipeline(oracle_lib, backend):      # :224-251
    for n in range(1, 8):
        cfg = small_config(backend, n, 3)
        tables = oracle_lib.init_tables(cfg, 77)
        x = oracle_lib.rng_doubles(24 + n, None, 200 * n).reshape(200, n)
        got, _ = oracle_lib.encode(cfg, tables, x)
        for l in range(cfg.levels):
            res = oracle_lib.level_resolution(cfg, l)
            fn = encode_simplex_level if backend == oracle.BACKEND_SIMPLEX else encode_grid_level
            want = fn(n, res, cfg.table_size, cfg.features, tables[l], x)
            assert np.abs(got[:, l * 2:(l + 1) * 2].astype(np.float64) - want).max() < 1e-9


def test_simplex_weights_reconstruct_the_point():       # tests/test_lattice.cpp:186-225 (barycentric reconstructs)
    rng = np.random.default_rng(5)
    for n in range(1, 8):
        x = rng.random((100, n))
        res = 8
        verts, w = simplex_vertices(n, res, x)
        assert np.all(w >= 0) and np.allclose(w.sum(1), 1.0, atol=1e-14)
        y = (np.minimum(x, np.nextafter(1.0, 0.0)) * (res / np.sqrt(n + 1.0))) @ skew_matrix(n).T
        assert np.allclose((w[:, :, None] * verts).sum(1), y, atol=1e-12)


def test_oracle_mlp_matches_the_dense_matrix_product(oracle_lib):           # tests/test_neural.cpp:68-81
    mc = oracle.MlpConfig(8, 16, 2, 3)
    params = oracle_lib.mlp_init(mc, 41)
    ws, bs, off = [], [], 0
    for l in range(mc.layer_count):
        i, o = mc.layer_in(l), mc.layer_out(l)
        ws.append(params[off:off + i * o].reshape(o, i)); off += i * o
        bs.append(params[off:off + o]); off += o
    x = np.stack([oracle_lib.rng_doubles(1000 + it, None, 8, -1.0, 1.0) for it in range(200)]).astype(np.float32)
    got = oracle_lib.mlp_forward(mc, params, x)
    got = got[0] if isinstance(got, tuple) else got
    want = mlp_forward(mc, ws, bs, x)
    assert np.all(np.abs(got.astype(np.float64) - want) <= 1e-5 * np.maximum(1.0, np.abs(want)))
