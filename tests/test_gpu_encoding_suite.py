"""GPU (-m gpu): the reference's own `encoding` test suite (/root/reference/proj/tests/test_encoding.cpp), case by case,
against the device path -- same configurations (small_config: T = 2^10, F = 2, base 4, growth 2, raw level scale), same
random streams (CounterRng seeds 23..29), same assertions and tolerances.  Where the reference compares with its
"independent pipeline" (tests/oracles.hpp) this suite compares with tests/independent.py, a numpy restatement from first
principles that shares no code with the library or with oracle/ (checked against the C oracle in test_independent_cpu.py).
Single points go through the host-buffer entry points, like the reference's span calls."""
import numpy as np
import pytest

from independent import encode_grid_level, encode_simplex_level, spatial_hash

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def sx():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2311_15439_b200 as pkg
    return pkg


def small_config(sx, backend, dim, levels=2, **kw):      # tests/test_encoding.cpp:16-27
    base = dict(dim=dim, levels=levels, table_size=1 << 10, features=2, base_resolution=4, growth=2.0, backend=backend,
                level_scale=sx.LevelScale.raw)
    base.update(kw)
    return sx.EncoderConfig(**base)


def draws(sx, seed, count, lo=0.0, hi=1.0):
    """The first `count` next_double(lo, hi) draws of CounterRng(seed), from the device generator (bit-identical to the
    reference's, tests/test_gpu_parity.py pins that)."""
    t = torch.empty(count, dtype=torch.float64, device="cuda:0")
    sx.CounterRng(seed).fill_device(t, lo, hi)
    torch.cuda.synchronize()
    return t.cpu().numpy()


def backends(sx):
    return (sx.Backend.simplex, sx.Backend.grid)


def hash_index(coords, table_size):
    return int(spatial_hash(np.asarray([coords], dtype=np.int64))[0]) & (table_size - 1)


def test_hash_all_zero_and_independent_reimplementation(sx):                # :39-59
    for n in range(1, 9):
        assert sx.hash_coords([0] * n) == 0
    rng = np.random.default_rng(21)
    for n in range(1, 9):
        for c in rng.integers(-(1 << 20), 1 << 20, size=(100, n), dtype=np.int64):
            assert sx.hash_coords(c) == int(spatial_hash(c[None, :])[0])


def test_hash_index_validation(sx):                                         # :61-65
    with pytest.raises(ValueError):
        sx.hash_coords([])                                # an empty coordinate span
    with pytest.raises(ValueError):
        sx.HashEncoder(small_config(sx, sx.Backend.simplex, 2, table_size=1000))   # not a power of two


def test_level_resolution_growth_table_and_equal_memory_multipliers(sx):    # :88-106
    cfg = small_config(sx, sx.Backend.simplex, 2, 4, base_resolution=16)
    assert [sx.level_resolution(cfg, l) for l in (0, 1, 3)] == [16, 32, 128]
    assert abs(sx.equal_memory_multiplier(2) - 3.0 ** 0.25) <= 1e-12 * 3.0 ** 0.25
    assert abs(sx.equal_memory_multiplier(2) - 1.3161) <= 1e-4 * 1.3161
    assert abs(sx.equal_memory_multiplier(3) - np.cbrt(4.0)) <= 1e-12 * np.cbrt(4.0)
    assert abs(sx.equal_memory_multiplier(3) - 1.5874) <= 1e-4 * 1.5874
    cfg.level_scale = sx.LevelScale.equal_memory
    assert sx.level_resolution(cfg, 0) == int(np.floor(16.0 * 3.0 ** 0.25))
    enc = sx.HashEncoder(cfg)
    assert enc.resolution(0) == sx.level_resolution(cfg, 0)                  # the handle agrees with the free function
    cfg.backend = sx.Backend.grid                         # the multiplier only applies to the simplex lattice
    assert sx.level_resolution(cfg, 0) == 16


def test_config_validation_rejects_out_of_range_fields(sx):                 # :108-136
    small_config(sx, sx.Backend.simplex, 2).validate()
    for field, value in (("dim", 0), ("dim", 9), ("levels", 0), ("table_size", 1000), ("features", 0),
                         ("base_resolution", 0), ("growth", 1.0), ("levels", 40)):
        broken = small_config(sx, sx.Backend.simplex, 2)
        setattr(broken, field, value)
        with pytest.raises(ValueError):
            broken.validate()
        with pytest.raises(ValueError):
            sx.HashEncoder(broken)                        # and no handle is created from it


def test_zero_initialized_tables_encode_to_zero_everywhere(sx):             # :138-147
    x = draws(sx, 23, 2 * 50 * 3).reshape(2, 50, 3)
    for b, backend in enumerate(backends(sx)):
        enc = sx.HashEncoder(small_config(sx, backend, 3))
        assert not enc.encode(x[b]).any()


def test_a_point_at_a_lattice_vertex_reads_back_that_entry_exactly(sx):     # :149-174
    for backend in backends(sx):
        cfg = small_config(sx, backend, 2, 1)
        enc = sx.HashEncoder(cfg)
        t = enc.table(0)
        t[0], t[1] = 0.25, -0.75
        enc.set_table(0, t)
        out = enc.encode(np.array([[0.0, 0.0]]))[0]
        assert out[0] == np.float32(0.25) and out[1] == np.float32(-0.75)
    cfg = small_config(sx, sx.Backend.grid, 2, 1)
    enc = sx.HashEncoder(cfg)
    idx = hash_index([2, 1], cfg.table_size)
    t = enc.table(0)
    t[idx * 2], t[idx * 2 + 1] = 1.5, 2.5
    enc.set_table(0, t)
    out = enc.encode(np.array([[0.5, 0.25]]))[0]          # times resolution 4 -> (2, 1)
    assert out[0] == np.float32(1.5) and out[1] == np.float32(2.5)


def test_grid_backend_frozen_blends(sx):                                    # :176-206
    cfg = small_config(sx, sx.Backend.grid, 1, 1, base_resolution=1, features=1)
    enc = sx.HashEncoder(cfg)
    t = enc.table(0)
    t[hash_index([0], cfg.table_size)] = 2.0
    t[hash_index([1], cfg.table_size)] = 6.0
    enc.set_table(0, t)
    for s in (0.0, 0.25, 0.5, 0.75):
        assert abs(float(enc.encode(np.array([[s]]))[0, 0]) - (2.0 + 4.0 * s)) <= 1e-6 * (2.0 + 4.0 * s)
    cfg = small_config(sx, sx.Backend.grid, 2, 1, base_resolution=1, features=1)
    enc = sx.HashEncoder(cfg)
    t = enc.table(0)
    for m in range(4):
        t[hash_index([m & 1, (m >> 1) & 1], cfg.table_size)] = float(m)
    enc.set_table(0, t)
    assert abs(float(enc.encode(np.array([[0.5, 0.5]]))[0, 0]) - 1.5) <= 1.5e-7


def test_simplex_frozen_three_vertex_blend(sx):                             # :208-222
    cfg = small_config(sx, sx.Backend.simplex, 2, 1)
    enc = sx.HashEncoder(cfg)
    enc.init_tables(123)
    x = np.array([[0.25, 0.5]])
    got = enc.encode(x)[0].astype(np.float64)
    want = encode_simplex_level(2, enc.resolution(0), cfg.table_size, cfg.features, enc.table(0), x)[0]
    assert np.abs(got - want).max() < 1e-9


def test_both_backends_match_the_independent_pipeline(sx):                  # :224-251
    stream = draws(sx, 24, 2 * sum(200 * n for n in range(1, 8)))
    pos = 0
    for backend in backends(sx):
        for n in range(1, 8):
            cfg = small_config(sx, backend, n, 3)
            enc = sx.HashEncoder(cfg)
            enc.init_tables(77)
            x = stream[pos:pos + 200 * n].reshape(200, n)
            pos += 200 * n
            got = enc.encode(x).astype(np.float64)
            fn = encode_simplex_level if backend == sx.Backend.simplex else encode_grid_level
            for l in range(cfg.levels):
                want = fn(n, enc.resolution(l), cfg.table_size, cfg.features, enc.table(l), x)
                assert np.abs(got[:, l * 2:(l + 1) * 2] - want).max() < 1e-9, (backend, n, l)
            # and the asynchronous device entry point says the same, bit for bit
            dev_out = enc.encode(torch.as_tensor(x, device="cuda:0")).cpu().numpy()
            assert np.array_equal(dev_out.view(np.uint32), enc.encode(x).view(np.uint32))


def test_encoding_is_linear_in_the_table_entries(sx):                       # :253-268
    for backend in backends(sx):
        enc = sx.HashEncoder(small_config(sx, backend, 3))
        enc.init_tables(5)
        x = np.array([[0.31, 0.77, 0.12]])
        once = enc.encode(x)[0].astype(np.float64)
        for l in range(enc.config.levels):
            enc.set_table(l, enc.table(l) * np.float32(2.0))
        twice = enc.encode(x)[0].astype(np.float64)
        assert np.abs(twice - 2.0 * once).max() < 1e-9


def test_constant_tables_encode_to_the_constant(sx):                        # :270-288
    stream = draws(sx, 26, 2 * sum(100 * n for n in range(1, 8)))
    pos = 0
    for backend in backends(sx):
        for n in range(1, 8):
            cfg = small_config(sx, backend, n)
            enc = sx.HashEncoder(cfg)
            for l in range(cfg.levels):
                enc.set_table(l, np.full(cfg.table_size * cfg.features, 0.5, dtype=np.float32))
            x = stream[pos:pos + 100 * n].reshape(100, n)
            pos += 100 * n
            assert np.abs(enc.encode(x).astype(np.float64) - 0.5).max() < 1e-7, (backend, n)


def test_identical_config_and_seed_are_bit_identical(sx):                   # :290-306
    cfg = small_config(sx, sx.Backend.simplex, 4)
    a, b = sx.HashEncoder(cfg), sx.HashEncoder(cfg)
    a.init_tables(999)
    b.init_tables(999)
    for l in range(cfg.levels):
        assert np.array_equal(a.table(l).view(np.uint32), b.table(l).view(np.uint32))
    x = np.array([[0.1, 0.9, 0.4, 0.6]])
    assert np.array_equal(a.encode(x).view(np.uint32), b.encode(x).view(np.uint32))


def test_touched_vertex_counters_are_exact(sx):                             # :308-334
    stream = draws(sx, 27, sum(100 * n for n in range(2, 6)))
    pos = 0
    for n in range(2, 6):
        simplex = sx.HashEncoder(small_config(sx, sx.Backend.simplex, n))
        grid = sx.HashEncoder(small_config(sx, sx.Backend.grid, n))
        k = 100
        x = stream[pos:pos + k * n].reshape(k, n)
        pos += k * n
        for row in x:                                    # one encode call per point, like the reference's loop
            simplex.encode(row[None, :])
            grid.encode(row[None, :])
        levels = simplex.config.levels
        assert simplex.counters().touched_vertices == k * levels * (n + 1)
        assert grid.counters().touched_vertices == k * levels * (1 << n)
        assert simplex.counters().out_of_bounds == 0 and grid.counters().out_of_bounds == 0
        simplex.reset_counters()
        assert simplex.counters().touched_vertices == 0


def test_unit_cube_boundary_points_are_accepted(sx):                        # :336-346
    for backend in backends(sx):
        enc = sx.HashEncoder(small_config(sx, backend, 2))
        for p in ([0.0, 0.0], [1.0, 1.0], [1.0, 0.0], [0.999999999, 1.0]):
            enc.encode(np.array([p]))
        assert enc.counters().out_of_bounds == 0


def test_encode_input_and_shape_validation(sx):                             # :348-358
    enc = sx.HashEncoder(small_config(sx, sx.Backend.simplex, 2))
    for bad in ([0.5, 0.5, 0.5], [1.5, 0.5], [-0.1, 0.5], [float("nan"), 0.5]):
        with pytest.raises(ValueError):
            enc.encode(np.array([bad]))
    with pytest.raises(ValueError):
        enc.encode(np.array([[0.5, 0.5]]), out=np.empty((1, enc.config.encoded_width() + 1), dtype=np.float32))
    enc.encode(np.array([[0.5, 0.5]]))                   # and the handle is still usable afterwards


def test_gradient_accumulator_add_merge_clear(sx):                          # :360-387
    # the device accumulator has no scalar add(); rows are placed with set_level (values + touched marks)
    cfg = small_config(sx, sx.Backend.simplex, 2, 2, table_size=1 << 4)
    enc = sx.HashEncoder(cfg)
    T, F = cfg.table_size, cfg.features
    up = np.array([1.0, -2.0])

    def rows(entries):
        v, t = np.zeros((T, F), dtype=np.float32), np.zeros(T, dtype=np.uint8)
        for idx, w in entries:
            v[idx] += (w * up).astype(np.float32)
            t[idx] = 1
        return v, t

    g = sx.EncoderGradient(enc)
    g.set_level(0, *rows([(3, 0.5), (3, 0.5)]))          # same slot accumulates
    g.set_level(1, *rows([(7, 1.0)]))
    assert g.level(0)[1].sum() == 1 and g.level(1)[1].sum() == 1 and g.touched_total() == 2
    assert np.allclose(g.level(0)[0][3], [1.0, -2.0])
    h = sx.EncoderGradient(enc)
    h.set_level(0, *rows([(3, 1.0), (9, 2.0)]))
    g.merge(h)
    v0, t0 = g.level(0)
    assert t0.sum() == 2 and v0[3, 0] == 2.0 and v0[9, 1] == -4.0
    g.clear()
    assert g.touched_total() == 0 and g.level(0)[0][3, 0] == 0.0 and g.level(0)[0][9, 0] == 0.0
    wrong = sx.EncoderGradient(sx.HashEncoder(small_config(sx, sx.Backend.simplex, 2, 3, table_size=1 << 4)))
    with pytest.raises(ValueError):
        g.merge(wrong)


def test_backward_zero_upstream_leaves_only_zero_slices(sx):                # :389-401
    enc = sx.HashEncoder(small_config(sx, sx.Backend.simplex, 3))
    enc.init_tables(4)
    grad = sx.EncoderGradient(enc)
    enc.encode_backward(np.array([[0.2, 0.6, 0.9]]), np.zeros((1, enc.config.encoded_width())), grad)
    assert grad.touched_total() == enc.config.levels * 4          # the rows are marked ...
    for l in range(grad.levels()):
        assert not grad.level(l)[0].any()                          # ... and hold zeros


def test_backward_one_hot_upstream_recovers_the_weights(sx):                # :403-435
    stream = draws(sx, 28, 2 * 20 * 2).reshape(2, 20, 2)
    for b, backend in enumerate(backends(sx)):
        enc = sx.HashEncoder(small_config(sx, backend, 2))
        enc.init_tables(6)
        cfg = enc.config
        for it in range(20):
            hot_l, hot_f = it % cfg.levels, it % cfg.features
            up = np.zeros((1, cfg.encoded_width()))
            up[0, hot_l * cfg.features + hot_f] = 1.0
            grad = sx.EncoderGradient(enc)
            enc.encode_backward(stream[b, it][None, :], up, grad)
            total = 0.0
            for l in range(cfg.levels):
                v, t = grad.level(l)
                v = v.astype(np.float64)
                for f in range(cfg.features):
                    if l != hot_l or f != hot_f:
                        assert not v[:, f].any()
                assert not v[t == 0].any()
                total += v[:, hot_f].sum()
                if l == hot_l:
                    assert (v[:, hot_f] >= 0.0).all()
            assert abs(total - 1.0) <= 2e-7               # the accumulator is f32 here (fp64 in the reference: 1e-12)


def test_backward_matches_finite_differences_on_table_entries(sx):          # :437-480
    for backend in backends(sx):
        enc = sx.HashEncoder(small_config(sx, backend, 2))
        enc.init_tables(8)
        cfg = enc.config
        x = np.array([[0.37, 0.58]])
        up = draws(sx, 29, cfg.encoded_width(), -1.0, 1.0)[None, :]
        grad = sx.EncoderGradient(enc)
        enc.encode_backward(x, up, grad)

        def loss():
            return float((up[0] * enc.encode(x)[0].astype(np.float64)).sum())

        h, checked = np.float32(1e-3), 0
        for l in range(cfg.levels):
            v, t = grad.level(l)
            for idx in np.flatnonzero(t):
                if checked >= 8:
                    break
                f = int(idx % cfg.features)
                tab = enc.table(l)
                saved = tab[idx * cfg.features + f]
                tab[idx * cfg.features + f] = saved + h
                enc.set_table(l, tab)
                hi = loss()
                tab[idx * cfg.features + f] = saved - h
                enc.set_table(l, tab)
                lo = loss()
                tab[idx * cfg.features + f] = saved
                enc.set_table(l, tab)
                fd = (hi - lo) / (2.0 * float(h))
                analytic = float(v[idx, f])
                assert abs(fd - analytic) < 1e-3 * max(1.0, abs(analytic))
                checked += 1
        assert checked > 0


def test_backward_shape_validation(sx):                                     # :482-491
    enc = sx.HashEncoder(small_config(sx, sx.Backend.simplex, 2))
    good = sx.EncoderGradient(enc)
    bad = sx.EncoderGradient(sx.HashEncoder(small_config(sx, sx.Backend.simplex, 2, 3)))
    W = enc.config.encoded_width()
    with pytest.raises(ValueError):
        enc.encode_backward(np.array([[0.5, 0.5]]), np.zeros((1, W - 1)), good)
    with pytest.raises(ValueError):
        enc.encode_backward(np.array([[0.5, 0.5]]), np.zeros((1, W)), bad)


def test_parameter_count_covers_every_level(sx):                            # :493-497
    cfg = small_config(sx, sx.Backend.simplex, 3, 5)
    assert sx.HashEncoder(cfg).parameter_count() == 5 * cfg.table_size * 2
