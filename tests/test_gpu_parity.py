"""GPU (-m gpu): the CUDA path through the C ABI against the CPU oracle and the committed golden fixtures.

Bars (stated once, used below):
  * vertex selection, hash indices, barycentric weights (fp64): BIT-EXACT
  * encoded features, exact blend (default): BIT-EXACT; fp32-FMA blend: |d| <= FAST_RTOL * sum_k w_k*|entry_k|
  * table gradients (fp32 atomics vs the reference's fp64 accumulator): |d| <= GRAD_RTOL * sum of |contributions|
  * touched rows: exact set equality;  optimizer given identical gradients: BIT-EXACT params and moments
"""
import os

import numpy as np
import pytest

import oracle
from conftest import case_config

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

FAST_RTOL = 4e-7   # three fp32 FMAs + one fp32 weight rounding each
GRAD_RTOL = 2e-6   # fp32 product rounding + fp32 accumulation of <= a few thousand terms per row in these tests
GRAD_ATOL = 1e-28  # contributions below 2^-100 (7.9e-31) are added as +0.0f by design (sxen_device.cuh: canon)


@pytest.fixture(scope="module")
def sx():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2311_15439_b200 as pkg
    assert pkg.device_count() >= 1
    return pkg


def to_sx(sx, cfg: oracle.Config):
    return sx.EncoderConfig(dim=cfg.dim, levels=cfg.levels, table_size=cfg.table_size, features=cfg.features,
                            base_resolution=cfg.base_resolution, growth=cfg.growth, backend=cfg.backend,
                            level_scale=cfg.level_scale)


def dev(a, dtype=None):
    t = torch.as_tensor(np.ascontiguousarray(a), device="cuda:0")
    return t if dtype is None else t.to(dtype)


def make_encoder(sx, cfg, tables=None, seed=None):
    enc = sx.HashEncoder(to_sx(sx, cfg))
    if seed is not None:
        enc.init_tables(seed)
    if tables is not None:
        for l in range(cfg.levels):
            enc.set_table(l, tables[l])
    return enc


def grad_dense(grad, cfg):
    vals = np.zeros((cfg.levels, cfg.table_size, cfg.features), dtype=np.float32)
    tch = np.zeros((cfg.levels, cfg.table_size), dtype=np.uint8)
    for l in range(cfg.levels):
        vals[l], tch[l] = grad.level(l)
    return vals, tch


def abs_contrib(o, cfg, x, up):
    """sum of |w * upstream| per gradient element: the scale fp32 accumulation error is measured against."""
    g, _, _ = o.encode_backward(cfg, x, np.abs(up))
    return g


# ------------------------------------------------------------------------------------------------ golden fixtures
def test_golden_cases_through_the_abi(sx, oracle_lib, golden_encode):
    g = golden_encode
    for name in g["names"].tolist():
        cfg = case_config(g, name)
        enc = make_encoder(sx, cfg, seed=int(g[f"{name}/seed"]))
        assert [enc.resolution(l) for l in range(cfg.levels)] == g[f"{name}/res"].tolist(), name
        assert np.array_equal(np.stack([enc.table(l)[:8] for l in range(cfg.levels)]), g[f"{name}/table_head"]), name
        x = g[f"{name}/x"]
        xd = dev(x)
        feats = enc.encode(xd).cpu().numpy()
        assert np.array_equal(feats.view(np.uint32), g[f"{name}/features"].view(np.uint32)), name
        # vertex chains against the oracle (which test_oracle_golden pins to the reference's merged chains)
        idx, w = enc.encode_debug(xd)
        oi, ow, _, _, _ = oracle_lib.encode_debug(cfg, x)
        assert np.array_equal(idx, oi), name
        assert np.array_equal(w, ow), name
        # backward against the reference's own accumulator contents
        up = g[f"{name}/upstream"]
        grad = sx.EncoderGradient(enc)
        enc.encode_backward(xd, dev(up, torch.float32), grad)
        enc.check()
        vals, tch = grad_dense(grad, cfg)
        lv, rows = g[f"{name}/g_level"], g[f"{name}/g_row"]
        assert int(tch.sum()) == lv.size and tch[lv, rows].all(), name
        # the kernels take f32 upstream: compare with the reference's accumulator for the same rounded upstream
        # (oracle == reference bit-for-bit, test_oracle_golden.py), and with the fixture itself at f32 resolution
        up32 = up.astype(np.float32).astype(np.float64)
        scale = abs_contrib(oracle_lib, cfg, x, up32)[lv, rows]
        want, _, _ = oracle_lib.encode_backward(cfg, x, up32)
        assert (np.abs(vals[lv, rows] - want[lv, rows]) <= GRAD_RTOL * scale + GRAD_ATOL).all(), name
        assert (np.abs(vals[lv, rows] - g[f"{name}/g_val"]) <= (GRAD_RTOL + 1.2e-7) * scale + GRAD_ATOL).all(), name
        # LookupCounters::out_of_bounds: the reference itself clamps a few cube-corner cells when rounding lands y on
        # the upper lattice face (e.g. n=5, x=1); the device must report the same count for encode and for backward
        assert enc.counters().out_of_bounds == 2 * int(g[f"{name}/counters"][1]), name


def test_counters_exact(sx, golden_encode):
    # reference tests/test_encoding.cpp:308-334: touched = k * levels * (n+1); out_of_bounds equals the reference's
    g = golden_encode
    for name in ("small_b0_n2", "small_b0_n5", "small_b1_n3", "c2_n3", "c1_n2", "f1_n4"):
        cfg = case_config(g, name)
        enc = make_encoder(sx, cfg, seed=1)
        x = dev(g[f"{name}/x"])
        enc.reset_counters()
        enc.encode(x)
        c = enc.counters()
        assert c.touched_vertices == int(g[f"{name}/counters"][0])
        assert c.out_of_bounds == int(g[f"{name}/counters"][1])
        cfg_v = cfg.vertices
        assert c.touched_vertices == g[f"{name}/x"].shape[0] * cfg.levels * cfg_v
        enc.reset_counters()
        assert enc.counters().touched_vertices == 0


# ------------------------------------------------------------------------------------------------ kernel variants
@pytest.mark.parametrize("n,growth", [(3, 1.5), (2, 2.0)])
def test_every_tuning_variant_matches_the_oracle(sx, oracle_lib, n, growth):
    # BASELINE level ladder at a table size that keeps 100+ dense gradient comparisons quick (T=2^19 is covered by
    # the golden cases and test_full_size_properties)
    cfg = oracle.Config(dim=n, levels=16, table_size=1 << 16, features=2, base_resolution=16, growth=growth)
    tables = oracle_lib.init_tables(cfg, 42)
    enc = make_encoder(sx, cfg, seed=42)
    N = 5000  # not a multiple of any block size
    x32 = oracle_lib.rng_doubles(99, 1, N * n).reshape(N, n).astype(np.float32)
    x = x32.astype(np.float64)
    up32 = (oracle_lib.rng_doubles(7, 2, N * 32, -1.0, 1.0) * 1e-3).astype(np.float32).reshape(N, 32)
    want, _ = oracle_lib.encode(cfg, tables, x)
    wg, wt, _ = oracle_lib.encode_backward(cfg, x, up32.astype(np.float64))
    scale = abs_contrib(oracle_lib, cfg, x, up32.astype(np.float64))
    # sum_k w_k |e_k| bound for the fast blend
    blend_scale, _ = oracle_lib.encode(cfg, np.abs(tables), x)
    xd, upd = dev(x32), dev(up32)
    for lpt in (1, 2, 4, 16):
        for level_major in (0, 1):
            for exact in (1, 0):
                for agg, merge in (((0, 1), (1 << 20, 1), (0, -1)) if exact else ((0, 1),)):
                    enc.set_tuning(sx.Tuning(levels_per_thread=lpt, block_threads=128 if lpt == 4 else 256,
                                             level_major=level_major, exact_blend=exact, warp_aggregate=agg,
                                             merge_pairs=merge))
                    tag = (lpt, level_major, exact, agg, merge)
                    feats = enc.encode(xd).cpu().numpy()
                    if exact:
                        assert np.array_equal(feats.view(np.uint32), want.view(np.uint32)), tag
                    else:
                        assert (np.abs(feats.astype(np.float64) - want) <= FAST_RTOL * blend_scale).all(), tag
                    grad = sx.EncoderGradient(enc)
                    enc.encode_backward(xd, upd, grad)
                    vals, tch = grad_dense(grad, cfg)
                    assert np.array_equal(tch, wt), tag
                    assert (np.abs(vals - wg) <= GRAD_RTOL * scale + GRAD_ATOL).all(), tag
                    # fused forward+backward == the separate pair
                    grad2 = sx.EncoderGradient(enc)
                    feats2 = enc.encode_forward_backward(xd, upd, grad2).cpu().numpy()
                    assert np.array_equal(feats2.view(np.uint32), feats.view(np.uint32)), tag
                    vals2, tch2 = grad_dense(grad2, cfg)
                    assert np.array_equal(tch2, wt), tag
                    assert (np.abs(vals2 - wg) <= GRAD_RTOL * scale + GRAD_ATOL).all(), tag
                    enc.check()


def test_warp_aggregation_on_coherent_samples(sx, oracle_lib):
    """Many lanes of a warp in the same simplex (ray-marching-like input): merged atomics must sum the same."""
    cfg = oracle.Config(dim=3, levels=8, table_size=1 << 14, features=2, base_resolution=4, growth=1.6)
    rng = np.random.default_rng(3)
    centers = rng.random((64, 3))
    x = (np.repeat(centers, 64, axis=0) + rng.normal(0, 1e-3, (4096, 3))).clip(0, 1)
    x[:64] = centers[0]  # two full warps of identical points
    up = rng.standard_normal((4096, 16)).astype(np.float32)
    enc = make_encoder(sx, cfg, seed=3)
    wg, wt, _ = oracle_lib.encode_backward(cfg, x, up.astype(np.float64))
    scale = abs_contrib(oracle_lib, cfg, x, up.astype(np.float64))
    for lpt in (1, 2, 4):
        enc.set_tuning(sx.Tuning(levels_per_thread=lpt, warp_aggregate=1 << 30))
        grad = sx.EncoderGradient(enc)
        enc.encode_backward(dev(x), dev(up), grad)
        vals, tch = grad_dense(grad, cfg)
        assert np.array_equal(tch, wt)
        assert (np.abs(vals - wg) <= 8 * GRAD_RTOL * scale + GRAD_ATOL).all()


def test_dimension_sweep_and_feature_widths(sx, oracle_lib):
    # BASELINE config 5 shape (n = 2..6, F = 2) at a table size the oracle handles in seconds, plus n = 1, 7, 8 and
    # F in {1, 3, 4, 8, 64} (vector, dynamic and maximum widths)
    shapes = [(n, 2) for n in range(1, 9)] + [(3, 1), (2, 3), (3, 4), (2, 8), (4, 5), (2, 64)]
    for n, F in shapes:
        cfg = oracle.Config(dim=n, levels=6, table_size=1 << 15, features=F, base_resolution=8, growth=1.5)
        tables = oracle_lib.init_tables(cfg, 11)
        enc = make_encoder(sx, cfg, seed=11)
        N = 777
        x = oracle_lib.rng_doubles(5, n, N * n).reshape(N, n)
        up = oracle_lib.rng_doubles(6, n, N * cfg.encoded_width, -1.0, 1.0).astype(np.float32).reshape(N, -1)
        want, _ = oracle_lib.encode(cfg, tables, x)
        oi, ow, _, _, _ = oracle_lib.encode_debug(cfg, x)
        for lpt in (1, 2, 4):
            enc.set_tuning(sx.Tuning(levels_per_thread=lpt))
            feats = enc.encode(dev(x)).cpu().numpy()
            assert np.array_equal(feats.view(np.uint32), want.view(np.uint32)), (n, F, lpt)
        idx, w = enc.encode_debug(dev(x))
        assert np.array_equal(idx, oi) and np.array_equal(w, ow), (n, F)
        grad = sx.EncoderGradient(enc)
        enc.encode_backward(dev(x), dev(up), grad)
        vals, tch = grad_dense(grad, cfg)
        wg, wt, _ = oracle_lib.encode_backward(cfg, x, up.astype(np.float64))
        assert np.array_equal(tch, wt), (n, F)
        scale = abs_contrib(oracle_lib, cfg, x, up.astype(np.float64))
        assert (np.abs(vals - wg) <= GRAD_RTOL * scale + GRAD_ATOL).all(), (n, F)


def test_more_than_32_levels_and_grid_backend(sx, oracle_lib):
    cfg = oracle.Config(dim=2, levels=40, table_size=1 << 12, features=2, base_resolution=4, growth=1.2)
    tables = oracle_lib.init_tables(cfg, 2)
    enc = make_encoder(sx, cfg, seed=2)
    x = oracle_lib.rng_doubles(8, 0, 600).reshape(300, 2)
    want, _ = oracle_lib.encode(cfg, tables, x)
    for lpt in (1, 4, 16):
        enc.set_tuning(sx.Tuning(levels_per_thread=lpt))
        assert np.array_equal(enc.encode(dev(x)).cpu().numpy().view(np.uint32), want.view(np.uint32))
    for n in (1, 2, 3, 5):
        cfg = oracle.Config(dim=n, levels=4, table_size=1 << 12, features=2, base_resolution=4, growth=2.0,
                            backend=oracle.BACKEND_GRID)
        tables = oracle_lib.init_tables(cfg, 9)
        enc = make_encoder(sx, cfg, seed=9)
        x = oracle_lib.rng_doubles(8, n, 200 * n).reshape(200, n)
        want, _ = oracle_lib.encode(cfg, tables, x)
        assert np.array_equal(enc.encode(dev(x)).cpu().numpy().view(np.uint32), want.view(np.uint32)), n
        idx, w = enc.encode_debug(dev(x))
        oi, ow, _, _, _ = oracle_lib.encode_debug(cfg, x)
        assert np.array_equal(idx, oi) and np.array_equal(w, ow), n


# ------------------------------------------------------------------------------------------------ edge cases
def test_empty_boundary_and_invalid_inputs(sx, oracle_lib):
    cfg = oracle.Config(dim=2, levels=2, table_size=1 << 10, features=2, base_resolution=4, growth=2.0)
    tables = oracle_lib.init_tables(cfg, 1)
    enc = make_encoder(sx, cfg, seed=1)
    # empty batch
    out = enc.encode(torch.empty((0, 2), dtype=torch.float64, device="cuda:0"))
    assert tuple(out.shape) == (0, 4)
    assert enc.encode(np.empty((0, 2))).shape == (0, 4)
    # reference tests/test_encoding.cpp:336-346: cube boundary accepted, in bounds
    pts = np.array([[0.0, 0.0], [1.0, 1.0], [1.0, 0.0], [0.999999999, 1.0]])
    want, _ = oracle_lib.encode(cfg, tables, pts)
    enc.reset_counters()
    assert np.array_equal(enc.encode(pts).view(np.uint32), want.view(np.uint32))  # host-buffer entry point
    assert enc.counters().out_of_bounds == 0
    # :348-358: wrong arity, outside the cube, NaN -> std::invalid_argument
    with pytest.raises(ValueError):
        enc.encode(np.array([[0.5, 0.5, 0.5]]))
    for bad in ([1.5, 0.5], [-0.1, 0.5], [float("nan"), 0.5]):
        with pytest.raises(ValueError, match="outside the unit cube"):
            enc.encode(np.array([[0.25, 0.5], bad, [0.5, 0.25]]))
        # device path: asynchronous, surfaced by check(); offending sample writes zeros, the others are correct
        xd = dev(np.array([[0.25, 0.5], bad, [0.5, 0.25]]))
        feats = enc.encode(xd)
        with pytest.raises(ValueError, match="sample 1"):
            enc.check()
        enc.check()  # reported once
        ok, _ = oracle_lib.encode(cfg, tables, np.array([[0.25, 0.5], [0.5, 0.25]]))
        f = feats.cpu().numpy()
        assert np.array_equal(f[[0, 2]].view(np.uint32), ok.view(np.uint32)) and not f[1].any()
    with pytest.raises(ValueError):
        enc.encode(dev(np.zeros((3, 2))), out=torch.empty((3, 5), dtype=torch.float32, device="cuda:0"))
    grad = sx.EncoderGradient(enc)
    with pytest.raises(ValueError):
        enc.encode_backward(dev(np.zeros((3, 2))), dev(np.zeros((3, 5), dtype=np.float32)), grad)
    other = make_encoder(sx, oracle.Config(dim=2, levels=3, table_size=1 << 10, features=2, base_resolution=4))
    with pytest.raises(ValueError, match="shape mismatch"):
        other.encode_backward(dev(np.zeros((3, 2))), dev(np.zeros((3, 6), dtype=np.float32)), grad)


def test_f32_and_f64_coordinates(sx, oracle_lib):
    cfg = oracle.Config(dim=3, levels=16, table_size=1 << 19, features=2, base_resolution=16, growth=1.5)
    tables = oracle_lib.init_tables(cfg, 42)
    enc = make_encoder(sx, cfg, seed=42)
    x = oracle_lib.rng_doubles(99, 1, 3 * 2048).reshape(2048, 3)
    want64, _ = oracle_lib.encode(cfg, tables, x)
    assert np.array_equal(enc.encode(dev(x)).cpu().numpy().view(np.uint32), want64.view(np.uint32))
    x32 = x.astype(np.float32)
    want32, _ = oracle_lib.encode(cfg, tables, x32.astype(np.float64))  # the oracle is fed (double)(float)x, exact
    assert np.array_equal(enc.encode(dev(x32)).cpu().numpy().view(np.uint32), want32.view(np.uint32))
    # device-side counter RNG == CounterRng::next_double
    t = torch.empty(3 * 2048, dtype=torch.float64, device="cuda:0")
    sx.CounterRng(99, 1).fill_device(t)
    assert np.array_equal(t.cpu().numpy(), x.reshape(-1))
    t32 = torch.empty(1000, dtype=torch.float32, device="cuda:0")
    r = sx.CounterRng(7, 2)
    r.fill_device(t32[:400], -1e-3, 1e-3)
    r.fill_device(t32[400:], -1e-3, 1e-3)
    assert np.array_equal(t32.cpu().numpy(), oracle_lib.rng_doubles(7, 2, 1000, -1e-3, 1e-3).astype(np.float32))


def test_host_and_device_entry_points_agree(sx, oracle_lib):
    cfg = oracle.Config(dim=3, levels=16, table_size=1 << 16, features=2, base_resolution=16, growth=1.4)
    enc = make_encoder(sx, cfg, seed=5)
    N = (1 << 18) + 12345  # more than one staging chunk, ragged tail
    x = oracle_lib.rng_doubles(1, 0, 3 * N).reshape(N, 3)
    a = enc.encode(x)
    b = enc.encode(dev(x)).cpu().numpy()
    assert np.array_equal(a.view(np.uint32), b.view(np.uint32))
    up = oracle_lib.rng_doubles(2, 0, 32 * N, -1.0, 1.0).reshape(N, 32)
    g1, g2 = sx.EncoderGradient(enc), sx.EncoderGradient(enc)
    enc.encode_backward(x, up, g1)
    enc.encode_backward(dev(x), dev(up.astype(np.float32)), g2)
    v1, t1 = grad_dense(g1, cfg)
    v2, t2 = grad_dense(g2, cfg)
    assert np.array_equal(t1, t2)
    # same f32 contributions, different atomic order: bounded relative to sum |contribution| per element
    g3 = sx.EncoderGradient(enc)
    enc.encode_backward(dev(x), dev(np.abs(up).astype(np.float32)), g3)
    scale, _ = grad_dense(g3, cfg)
    assert (np.abs(v1 - v2) <= GRAD_RTOL * scale + GRAD_ATOL).all()
    # fused host entry point (f64 and f32 upstream) == encode_host + encode_backward_host
    for upx in (up, up.astype(np.float32)):
        g4 = sx.EncoderGradient(enc)
        f4 = enc.encode_forward_backward(x, upx, g4)
        assert np.array_equal(f4.view(np.uint32), a.view(np.uint32))
        v4, t4 = grad_dense(g4, cfg)
        assert np.array_equal(t4, t1) and (np.abs(v4 - v1) <= GRAD_RTOL * scale + GRAD_ATOL).all()


# ------------------------------------------------------------------------------------------------ accumulator semantics
def test_gradient_accumulator_semantics(sx, oracle_lib):
    # reference tests/test_encoding.cpp:360-401: add/merge/clear; zero upstream leaves only zero slices (but touched)
    cfg = oracle.Config(dim=3, levels=2, table_size=1 << 10, features=2, base_resolution=4, growth=2.0)
    enc = make_encoder(sx, cfg, seed=4)
    x = np.array([[0.2, 0.6, 0.9]])
    g = sx.EncoderGradient(enc)
    assert g.touched_total() == 0
    enc.encode_backward(dev(x), dev(np.zeros((1, 4), dtype=np.float32)), g)
    vals, tch = grad_dense(g, cfg)
    _, wt, _ = oracle_lib.encode_backward(cfg, x, np.zeros((1, 4)))
    assert np.array_equal(tch, wt) and g.touched_total() == int(wt.sum()) and not vals.any()
    # negative-zero contributions (w == 0 at a cell corner, negative upstream) still mark the row touched
    enc.encode_backward(dev(np.array([[0.0, 0.0, 0.0]])), dev(-np.ones((1, 4), dtype=np.float32)), g)
    _, wt2, _ = oracle_lib.encode_backward(cfg, np.array([[0.0, 0.0, 0.0]]), -np.ones((1, 4)))
    assert np.array_equal(grad_dense(g, cfg)[1], wt | wt2)
    # merge = union of touched, sum of values
    h = sx.EncoderGradient(enc)
    up = np.array([[1.0, -2.0, 0.5, 4.0]], dtype=np.float32)
    enc.encode_backward(dev(np.array([[0.7, 0.1, 0.3]])), dev(up), h)
    hv, ht = grad_dense(h, cfg)
    gv, gt = grad_dense(g, cfg)
    g.merge(h)
    mv, mt = grad_dense(g, cfg)
    assert np.array_equal(mt, gt | ht) and np.array_equal(mv, gv + hv)
    with pytest.raises(ValueError, match="shape mismatch"):
        g.merge(sx.EncoderGradient(make_encoder(sx, oracle.Config(dim=3, levels=3, table_size=1 << 10, features=2,
                                                                  base_resolution=4))))
    # upload / download round trip, clear
    g.set_level(1, hv[1] * 3, ht[1])
    v1, t1 = g.level(1)
    assert np.array_equal(v1, hv[1] * 3) and np.array_equal(t1, ht[1])
    g.clear()
    assert g.touched_total() == 0 and not grad_dense(g, cfg)[0].any()


def test_backward_one_hot_recovers_weights(sx, oracle_lib):
    # reference tests/test_encoding.cpp:403-435
    cfg = oracle.Config(dim=2, levels=2, table_size=1 << 10, features=2, base_resolution=4, growth=2.0)
    enc = make_encoder(sx, cfg, seed=6)
    pts = oracle_lib.rng_doubles(28, None, 40).reshape(20, 2)
    for it in range(20):
        hot_l, hot_f = it % 2, it % 2
        up = np.zeros((1, 4), dtype=np.float32)
        up[0, hot_l * 2 + hot_f] = 1.0
        g = sx.EncoderGradient(enc)
        enc.encode_backward(dev(pts[it:it + 1]), dev(up), g)
        vals, tch = grad_dense(g, cfg)
        assert vals[hot_l, :, hot_f].sum() == pytest.approx(1.0, abs=2e-7)
        other = vals.copy()
        other[hot_l, :, hot_f] = 0
        assert not other.any() and (vals >= 0).all()


# ------------------------------------------------------------------------------------------------ optimizers
def test_sparse_adam_bit_exact_given_identical_gradients(sx, oracle_lib):
    cfg = oracle.Config(dim=2, levels=3, table_size=1 << 10, features=2, base_resolution=4, growth=2.0)
    rng = np.random.default_rng(0)
    for F in (2, 3):
        cfg.features = F
        tables = oracle_lib.init_tables(cfg, 8)
        enc = make_encoder(sx, cfg, seed=8)
        opt = sx.SparseAdamState(enc)
        grad = sx.EncoderGradient(enc)
        m, v = np.zeros(tables.size), np.zeros(tables.size)
        ac = oracle.AdamConfig(lr=1e-2)
        for step in range(1, 5):
            touched = (rng.random((cfg.levels, cfg.table_size)) < 0.3).astype(np.uint8)
            g32 = (rng.standard_normal((cfg.levels, cfg.table_size, F)) * 1e-3).astype(np.float32)
            g32[0, :5] = 0.0
            touched[0, :5] = 1  # touched rows with an exactly-zero gradient are still updated (lazy Adam)
            g32 *= touched[..., None]
            for l in range(cfg.levels):
                grad.set_level(l, g32[l], touched[l])
            opt.step(enc, grad, sx.AdamConfig(lr=1e-2), clear_grad=(step % 2 == 0))
            flat = tables.reshape(-1)
            assert oracle_lib.sparse_adam_step(cfg, flat, g32.astype(np.float64), touched, m, v, step, ac) == -1
            got = np.stack([enc.table(l) for l in range(cfg.levels)])
            assert np.array_equal(got.view(np.uint32), tables.view(np.uint32)), (F, step)
            for l in range(cfg.levels):
                gm, gv = opt.moments(l)
                per = cfg.table_size * F
                assert np.array_equal(gm, m[l * per:(l + 1) * per]) and np.array_equal(gv, v[l * per:(l + 1) * per])
            assert grad.touched_total() == (0 if step % 2 == 0 else int(touched.sum()))
            assert opt.step_count() == step
        g32[1, 7, 0] = np.inf
        touched[1, 7] = 1
        for l in range(cfg.levels):
            grad.set_level(l, g32[l], touched[l])
        with pytest.raises(sx.TrainingError, match="non-finite"):
            opt.step(enc, grad, sx.AdamConfig(lr=1e-2))


def test_dense_adam_matches_reference_fixture(sx, golden_neural):
    g = golden_neural
    p = dev(g["adam_p0"].copy())
    opt = sx.AdamState(16)
    for t in range(5):
        opt.step(p, dev(g["adam_g"][t]), sx.AdamConfig(lr=1e-2))
        assert np.array_equal(p.cpu().numpy().view(np.uint32), g["adam_p"][t].view(np.uint32)), t
    bad = g["adam_g"][0].copy()
    bad[5] = np.nan
    with pytest.raises(sx.TrainingError, match="parameter 5"):
        opt.step(p, dev(bad), sx.AdamConfig(lr=1e-2))
    with pytest.raises(ValueError):
        opt.step(p[:8], dev(bad[:8]), sx.AdamConfig())


# ------------------------------------------------------------------------------------------------ BASELINE sizes
@pytest.mark.parametrize("n,growth,T", [(3, 1.5, 1 << 19), (2, 2.0, 1 << 19)])
def test_full_size_properties(sx, oracle_lib, n, growth, T):
    """2^20 samples at the BASELINE shape: size-independent properties + an oracle spot check on a 2^14 subset."""
    cfg = oracle.Config(dim=n, levels=16, table_size=T, features=2, base_resolution=16, growth=growth)
    enc = make_encoder(sx, cfg, seed=42)
    N = 1 << 20
    x = torch.empty((N, n), dtype=torch.float32, device="cuda:0")
    sx.CounterRng(99, 1).fill_device(x)
    up = torch.empty((N, 32), dtype=torch.float32, device="cuda:0")
    sx.CounterRng(7, 2).fill_device(up, -1e-3, 1e-3)
    feats = enc.encode(x)
    # determinism (reference tests/test_encoding.cpp:290-306)
    assert torch.equal(feats, enc.encode(x))
    # oracle spot check, bit-exact
    sub = slice(123456, 123456 + (1 << 14))
    want, _ = oracle_lib.encode(cfg, oracle_lib.init_tables(cfg, 42), x[sub].cpu().numpy().astype(np.float64))
    assert np.array_equal(feats[sub].cpu().numpy().view(np.uint32), want.view(np.uint32))
    # linearity in the table entries (:253-268): doubling every entry doubles every feature, exactly
    tabs = enc.tables_device()
    tabs.mul_(2.0)
    assert torch.equal(enc.encode(x), feats * 2.0)
    # partition of unity (:270-288): constant tables encode to the constant
    tabs.fill_(0.5)
    assert (enc.encode(x) - 0.5).abs().max().item() <= 1e-7
    # backward: per (level, feature), gradients sum to the upstream column sums (weights sum to one)
    grad = sx.EncoderGradient(enc)
    enc.encode_backward(x, up, grad)
    gsum = grad.device_view().view(16, T, 2).double().sum(dim=1).reshape(-1)
    usum = up.double().sum(dim=0)
    denom = up.double().abs().sum(dim=0)
    assert ((gsum - usum).abs() <= 1e-5 * denom).all()
    # every sample touches L*(n+1) rows; the union cannot exceed that, nor the table
    assert 0 < grad.touched_total() <= min(16 * T, N * 16 * (n + 1))
    # fused kernel: same features, same gradients up to atomic ordering
    grad2 = sx.EncoderGradient(enc)
    f2 = enc.encode_forward_backward(x, up, grad2)
    assert (f2 - 0.5).abs().max().item() <= 1e-7
    assert grad2.touched_total() == grad.touched_total()
    d = (grad2.device_view() - grad.device_view()).abs().max().item()
    assert d <= 1e-5 * up.abs().max().item() * 64
    enc.check()
    c = enc.counters()
    assert c.out_of_bounds == 0


# ------------------------------------------------------------------------------------------------ round-1 additions
@pytest.mark.parametrize("n,growth", [(3, 1.5), (2, 2.0)])
def test_coarse_replicas_and_cache_policies_do_not_change_results(sx, oracle_lib, n, growth):
    """Replicated dense accumulators for the coarse levels (folded in-call) and the L2 eviction policies are pure
    scheduling: touched sets exact, gradients within the fp32 bar, features bit-identical, under every combination."""
    cfg = oracle.Config(dim=n, levels=16, table_size=1 << 16, features=2, base_resolution=16, growth=growth)
    tables = oracle_lib.init_tables(cfg, 42)
    enc = make_encoder(sx, cfg, seed=42)
    N = 20000
    x32 = oracle_lib.rng_doubles(5, 1, N * n).reshape(N, n).astype(np.float32)
    x32[:64] = x32[0]          # a warp and a half of identical samples: maximum same-address pressure
    x32[64:128, 0] = 0.0       # and a face of the cube
    x = x32.astype(np.float64)
    up32 = (oracle_lib.rng_doubles(6, 2, N * 32, -1.0, 1.0)).astype(np.float32).reshape(N, 32)
    up32[::7] = 0.0            # exact-zero contributions still mark their rows touched
    want, _ = oracle_lib.encode(cfg, tables, x)
    wg, wt, _ = oracle_lib.encode_backward(cfg, x, up32.astype(np.float64))
    scale = abs_contrib(oracle_lib, cfg, x, up32.astype(np.float64))
    xd, upd = dev(x32), dev(up32)
    for rep in (1, 0, -1):   # forced on (N is below the automatic threshold), library default, off
        for hints in (-1, 0, 5, 8, 10, 15):
            for lm, lpt in ((0, 2), (1, 4), (0, 1)):
                enc.set_tuning(sx.Tuning(levels_per_thread=lpt, level_major=lm, coarse_replicas=rep, cache_hints=hints))
                tag = (rep, hints, lm, lpt)
                grad = sx.EncoderGradient(enc)
                feats = enc.encode_forward_backward(xd, upd, grad).cpu().numpy()
                assert np.array_equal(feats.view(np.uint32), want.view(np.uint32)), tag
                vals, tch = grad_dense(grad, cfg)
                assert np.array_equal(tch, wt), tag
                assert (np.abs(vals - wg) <= GRAD_RTOL * scale + GRAD_ATOL).all(), tag
                # a second batch into the same accumulator doubles it (the replicas were re-armed by the fold)
                enc.encode_backward(xd, upd, grad)
                vals2, tch2 = grad_dense(grad, cfg)
                assert np.array_equal(tch2, wt), tag
                assert (np.abs(vals2 - 2 * wg) <= 2 * GRAD_RTOL * scale + GRAD_ATOL).all(), tag
    enc.check()


def test_accumulator_of_another_lattice_falls_back_to_hashed_rows(sx, oracle_lib):
    """An accumulator is shape-compatible with any encoder of the same (L, T, F) -- src/encoding.cpp:323-325 -- but its
    replicas are laid out for the lattice it was created from; with another ladder the launch must not use them."""
    cfg_a = oracle.Config(dim=2, levels=4, table_size=1 << 12, features=2, base_resolution=4, growth=2.0)
    cfg_b = oracle.Config(dim=2, levels=4, table_size=1 << 12, features=2, base_resolution=7, growth=1.7)
    enc_a, enc_b = make_encoder(sx, cfg_a, seed=1), make_encoder(sx, cfg_b, seed=1)
    N = 3000
    x = oracle_lib.rng_doubles(9, 1, N * 2).reshape(N, 2)
    up = oracle_lib.rng_doubles(9, 2, N * 8, -1.0, 1.0).reshape(N, 8)
    grad = sx.EncoderGradient(enc_a)        # replicas sized for cfg_a's lattice
    enc_b.encode_backward(dev(x), dev(up, torch.float32), grad)
    wg, wt, _ = oracle_lib.encode_backward(cfg_b, x, up.astype(np.float32).astype(np.float64))
    scale = abs_contrib(oracle_lib, cfg_b, x, up)
    vals, tch = grad_dense(grad, cfg_b)
    assert np.array_equal(tch, wt)
    assert (np.abs(vals - wg) <= GRAD_RTOL * scale + GRAD_ATOL).all()


def test_level_ranges_compose_to_the_full_launch(sx, oracle_lib):
    """encode_backward / encode_forward_backward restricted to level ranges: the chunks together equal the whole launch
    (features bit-identical, touched sets equal, gradients within the fp32 bar), and a chunk leaves the other levels'
    slices of the feature rows and of the accumulator alone."""
    cfg = oracle.Config(dim=3, levels=16, table_size=1 << 15, features=2, base_resolution=16, growth=1.5)
    tables = oracle_lib.init_tables(cfg, 42)
    enc = make_encoder(sx, cfg, seed=42)
    N = 7001
    x32 = oracle_lib.rng_doubles(99, 1, N * 3).reshape(N, 3).astype(np.float32)
    up32 = oracle_lib.rng_doubles(7, 2, N * 32, -1.0, 1.0).astype(np.float32).reshape(N, 32)
    want, _ = oracle_lib.encode(cfg, tables, x32.astype(np.float64))
    wg, wt, _ = oracle_lib.encode_backward(cfg, x32.astype(np.float64), up32.astype(np.float64))
    scale = abs_contrib(oracle_lib, cfg, x32.astype(np.float64), up32.astype(np.float64))
    xd, upd = dev(x32), dev(up32)
    for chunks in (2, 4, 5, 16):
        grad = sx.EncoderGradient(enc)
        out = torch.full((N, 32), float("nan"), dtype=torch.float32, device="cuda:0")
        ranges = sx.level_ranges(16, chunks)
        for i, (first, count) in enumerate(ranges):
            enc.encode_forward_backward(xd, upd, grad, out=out, levels=(first, count))
            if i == 0:
                o = out.cpu().numpy()
                assert np.isnan(o[:, count * 2:]).all() and not np.isnan(o[:, :count * 2]).any()
                _, tch = grad_dense(grad, cfg)
                assert not tch[count:].any() and np.array_equal(tch[:count], wt[:count])
        assert np.array_equal(out.cpu().numpy().view(np.uint32), want.view(np.uint32)), chunks
        vals, tch = grad_dense(grad, cfg)
        assert np.array_equal(tch, wt), chunks
        assert (np.abs(vals - wg) <= GRAD_RTOL * scale + GRAD_ATOL).all(), chunks
        grad_b = sx.EncoderGradient(enc)
        for first, count in ranges:
            enc.encode_backward(xd, upd, grad_b, levels=(first, count))
        vb, tb = grad_dense(grad_b, cfg)
        assert np.array_equal(tb, wt) and (np.abs(vb - wg) <= GRAD_RTOL * scale + GRAD_ATOL).all(), chunks
    with pytest.raises(ValueError):
        enc.encode_backward(xd, upd, sx.EncoderGradient(enc), levels=(10, 7))
    assert enc.counters().out_of_bounds == 0


@pytest.mark.parametrize("n,growth", [(3, 1.5), (2, 2.0)])
def test_tuned_grid_backend_matches_the_oracle(sx, oracle_lib, n, growth):
    """gather_grid (src/encoding.cpp:244-285) through the tuned F == 2 kernel (2^n corners in registers, pair-merged
    reds, coarse-level replicas): corner indices and weights bit-exact, features bit-exact, gradients within the fp32 bar."""
    cfg = oracle.Config(dim=n, levels=16, table_size=1 << 16, features=2, base_resolution=16, growth=growth, backend=1)
    tables = oracle_lib.init_tables(cfg, 42)
    enc = make_encoder(sx, cfg, seed=42)
    N = 6001
    x32 = oracle_lib.rng_doubles(99, 1, N * n).reshape(N, n).astype(np.float32)
    x32[:40] = 1.0             # the far corner of the cube (legal: clamped to nextafter(1, 0) first)
    x32[40:80, 0] = 0.0
    x = x32.astype(np.float64)
    up32 = oracle_lib.rng_doubles(7, 2, N * 32, -1.0, 1.0).astype(np.float32).reshape(N, 32)
    want, _ = oracle_lib.encode(cfg, tables, x)
    wg, wt, _ = oracle_lib.encode_backward(cfg, x, up32.astype(np.float64))
    scale = abs_contrib(oracle_lib, cfg, x, up32.astype(np.float64))
    xd, upd = dev(x32), dev(up32)
    idx, w = enc.encode_debug(xd)
    oi, ow, _, _, _ = oracle_lib.encode_debug(cfg, x)
    assert np.array_equal(idx, oi) and np.array_equal(w, ow)
    for lpt in (1, 2):
        for lm in (0, 1):
            for rep, merge in ((1, 1), (-1, 1), (1, -1)):
                enc.set_tuning(sx.Tuning(levels_per_thread=lpt, level_major=lm, coarse_replicas=rep, merge_pairs=merge))
                tag = (lpt, lm, rep, merge)
                feats = enc.encode(xd).cpu().numpy()
                assert np.array_equal(feats.view(np.uint32), want.view(np.uint32)), tag
                grad = sx.EncoderGradient(enc)
                enc.encode_backward(xd, upd, grad)
                vals, tch = grad_dense(grad, cfg)
                assert np.array_equal(tch, wt), tag
                assert (np.abs(vals - wg) <= GRAD_RTOL * scale + GRAD_ATOL).all(), tag
                grad2 = sx.EncoderGradient(enc)
                feats2 = enc.encode_forward_backward(xd, upd, grad2).cpu().numpy()
                assert np.array_equal(feats2.view(np.uint32), want.view(np.uint32)), tag
                vals2, tch2 = grad_dense(grad2, cfg)
                assert np.array_equal(tch2, wt), tag
                assert (np.abs(vals2 - wg) <= GRAD_RTOL * scale + GRAD_ATOL).all(), tag
    enc.check()


def test_maximum_sizes(sx, oracle_lib):
    """The reference's limits (src/encoding.cpp:14-15,28-58): 8 dimensions, 64 features, finest resolution 2^26, and the
    largest table its CLI accepts (2^24 rows, tools/sxen_main.cpp:52-54).  Indices, weights and features bit-exact;
    the same limits rejected one step further."""
    # (a) largest table, finest legal resolution: one level at res 2^26 in a 2^24-row table (128 MiB)
    cfg = oracle.Config(dim=3, levels=1, table_size=1 << 24, features=2, base_resolution=1 << 26, growth=2.0)
    enc = make_encoder(sx, cfg, seed=5)
    x = oracle_lib.rng_doubles(3, 1, 3 * 4096).reshape(4096, 3)
    x[0], x[1] = 0.0, 1.0
    idx, w = enc.encode_debug(dev(x))
    oi, ow, _, _, _ = oracle_lib.encode_debug(cfg, x)
    assert np.array_equal(idx, oi) and np.array_equal(w, ow)
    assert int(idx.max()) < (1 << 24) and int(idx.max()) > (1 << 23)  # the whole index range is in use
    want, _ = oracle_lib.encode(cfg, oracle_lib.init_tables(cfg, 5), x)
    assert np.array_equal(enc.encode(dev(x)).cpu().numpy().view(np.uint32), want.view(np.uint32))
    grad = sx.EncoderGradient(enc)
    up = oracle_lib.rng_doubles(4, 2, 2 * 4096, -1.0, 1.0).reshape(4096, 2).astype(np.float32)
    enc.encode_backward(dev(x), dev(up), grad)
    wg, wt, _ = oracle_lib.encode_backward(cfg, x, up.astype(np.float64))
    vals, tch = grad.level(0)
    assert np.array_equal(tch, wt[0])
    scale = abs_contrib(oracle_lib, cfg, x, up.astype(np.float64))[0]
    assert (np.abs(vals - wg[0]) <= GRAD_RTOL * scale + GRAD_ATOL).all()
    del grad, enc
    # (b) 8 dimensions x 64 features (generic kernel), both backends
    for backend in (0, 1):
        cfg = oracle.Config(dim=8, levels=2, table_size=1 << 12, features=64, base_resolution=3, growth=2.0, backend=backend)
        enc = make_encoder(sx, cfg, seed=6)
        x = oracle_lib.rng_doubles(8, 1, 8 * 257).reshape(257, 8)
        want, _ = oracle_lib.encode(cfg, oracle_lib.init_tables(cfg, 6), x)
        assert np.array_equal(enc.encode(dev(x)).cpu().numpy().view(np.uint32), want.view(np.uint32)), backend
        idx, w = enc.encode_debug(dev(x))
        oi, ow, _, _, _ = oracle_lib.encode_debug(cfg, x)
        assert np.array_equal(idx, oi) and np.array_equal(w, ow), backend
    # (c) one step past each limit is rejected exactly as EncoderConfig::validate does
    for bad in (dict(dim=9), dict(features=65), dict(base_resolution=(1 << 26) + 1), dict(levels=2, base_resolution=1 << 26),
                dict(table_size=(1 << 12) + 1), dict(dim=0), dict(levels=0), dict(growth=1.0)):
        kw = dict(dim=3, levels=1, table_size=1 << 12, features=2, base_resolution=16, growth=2.0)
        kw.update(bad)
        with pytest.raises(ValueError):
            sx.HashEncoder(sx.EncoderConfig(**kw))


def test_fused_call_counts_and_big_table_split(sx, oracle_lib):
    """(a) The fused walk stands for the reference's encode + encode_backward pair, counters included: touched and
    out-of-bounds both count twice.  (b) With tables beyond L2 and the launch shape left to the library, the fused entry
    point runs as a forward plus a backward launch: same features (bit-exact), same gradients."""
    cfg = oracle.Config(dim=5, levels=3, table_size=1 << 12, features=2, base_resolution=3, growth=2.0)
    enc = make_encoder(sx, cfg, seed=1)
    x = np.ones((64, 5))  # the far corner: the reference clamps some cells there at n = 5 (golden small_b0_n5)
    up = np.ones((64, 6), dtype=np.float32)
    enc.reset_counters()
    enc.encode(dev(x))
    once = enc.counters()
    enc.reset_counters()
    enc.encode_forward_backward(dev(x), dev(up), sx.EncoderGradient(enc))
    both = enc.counters()
    assert both.touched_vertices == 2 * once.touched_vertices
    assert both.out_of_bounds == 2 * once.out_of_bounds
    # (b) 2^22-row tables, 12 levels = 384 MiB: the library's auto path splits the fused call
    cfg = oracle.Config(dim=3, levels=12, table_size=1 << 22, features=2, base_resolution=16, growth=1.5)
    enc = make_encoder(sx, cfg, seed=42)
    N = 50000
    x32 = oracle_lib.rng_doubles(99, 1, N * 3).reshape(N, 3).astype(np.float32)
    up32 = oracle_lib.rng_doubles(7, 2, N * 24, -1.0, 1.0).astype(np.float32).reshape(N, 24)
    launches = sx.launch_count()
    g_auto = sx.EncoderGradient(enc)
    f_auto = enc.encode_forward_backward(dev(x32), dev(up32), g_auto)
    auto_launches = sx.launch_count() - launches
    enc.set_tuning(sx.Tuning(level_major=0))
    launches = sx.launch_count()
    g_fused = sx.EncoderGradient(enc)
    f_fused = enc.encode_forward_backward(dev(x32), dev(up32), g_fused)
    fused_launches = sx.launch_count() - launches
    assert auto_launches == fused_launches + 1  # (grad creation launches are equal on both sides)
    assert torch.equal(f_auto, f_fused)
    sub = slice(0, 4096)
    want, _ = oracle_lib.encode(cfg, oracle_lib.init_tables(cfg, 42), x32[sub].astype(np.float64))
    assert np.array_equal(f_auto[sub].cpu().numpy().view(np.uint32), want.view(np.uint32))
    assert g_auto.touched_total() == g_fused.touched_total()
    d = (g_auto.device_view() - g_fused.device_view()).abs().max().item()
    assert d <= 1e-5


def test_random_configurations_match_the_oracle(sx, oracle_lib):
    """Seeded fuzz over the whole EncoderConfig surface (dim 1..8, both backends, raw / equal-memory ladders, F in
    1..8, odd level counts, tiny and mid tables, growths from barely above 1 to 2.5) with samples that include exact 0 / 1
    coordinates and repeated points: indices, weights, features bit-exact, touched sets exact, gradients within the fp32
    bar, fused == separate, counters equal to the oracle's."""
    rng = np.random.default_rng(20240229)
    done = 0
    cases = int(os.environ.get("SXEN_FUZZ_CASES", "120"))   # a longer soak: SXEN_FUZZ_CASES=2000
    while done < cases:
        n = int(rng.integers(1, 9))
        backend = int(rng.integers(0, 2))
        if backend == oracle.BACKEND_GRID and n > 5:
            continue  # 2^n corners x the oracle's Python-side loops: keep the CPU side in seconds
        cfg = oracle.Config(dim=n, levels=int(rng.integers(1, 12)), table_size=1 << int(rng.integers(4, 15)),
                            features=int(rng.choice([1, 2, 2, 2, 3, 4, 8])), base_resolution=int(rng.integers(1, 20)),
                            growth=float(rng.choice([1.05, 1.26, 1.5, 2.0, 2.5])), backend=backend,
                            level_scale=int(rng.integers(0, 2)))
        if oracle_lib.validate(cfg) != 0:   # e.g. the finest resolution above 2^26 (src/encoding.cpp:52-57)
            with pytest.raises(ValueError):
                sx.HashEncoder(to_sx(sx, cfg))      # the same rejection on the device side
            continue
        done += 1
        seed = int(rng.integers(1, 1 << 30))
        tables = oracle_lib.init_tables(cfg, seed)
        enc = make_encoder(sx, cfg, seed=seed)
        N = int(rng.integers(1, 600))
        x = rng.random((N, n))
        x[rng.random((N, n)) < 0.03] = 0.0
        x[rng.random((N, n)) < 0.03] = 1.0
        if N > 4:
            x[N // 2] = x[0]
        x32 = x.astype(np.float32)
        x = x32.astype(np.float64)
        up = (rng.standard_normal((N, cfg.encoded_width)) * 1e-2).astype(np.float32)
        tag = (cfg, N)
        want, bad = oracle_lib.encode(cfg, tables, x)
        assert bad == -1
        oi, ow, _, _, _ = oracle_lib.encode_debug(cfg, x)
        wg, wt, _ = oracle_lib.encode_backward(cfg, x, up.astype(np.float64))
        scale = abs_contrib(oracle_lib, cfg, x, up.astype(np.float64))
        enc.set_tuning(sx.Tuning(levels_per_thread=int(rng.choice([0, 1, 2, 4])), level_major=int(rng.integers(-1, 2)),
                                 coarse_replicas=int(rng.choice([0, 1, -1]))))
        xd, upd = dev(x32), dev(up)
        idx, w = enc.encode_debug(xd)
        assert np.array_equal(idx, oi) and np.array_equal(w, ow), tag
        feats = enc.encode(xd).cpu().numpy()
        assert np.array_equal(feats.view(np.uint32), want.view(np.uint32)), tag
        grad = sx.EncoderGradient(enc)
        enc.encode_backward(xd, upd, grad)
        vals, tch = grad_dense(grad, cfg)
        assert np.array_equal(tch, wt), tag
        assert (np.abs(vals - wg) <= GRAD_RTOL * scale + GRAD_ATOL).all(), tag
        grad2 = sx.EncoderGradient(enc)
        feats2 = enc.encode_forward_backward(xd, upd, grad2).cpu().numpy()
        assert np.array_equal(feats2.view(np.uint32), want.view(np.uint32)), tag
        vals2, tch2 = grad_dense(grad2, cfg)
        assert np.array_equal(tch2, wt) and (np.abs(vals2 - wg) <= GRAD_RTOL * scale + GRAD_ATOL).all(), tag
        enc.check()


@pytest.mark.parametrize("dim,levels,chunk,lpt", [(3, 16, 8, 2), (3, 16, 4, 2), (3, 12, 8, 4), (2, 16, 8, 1), (3, 10, 4, 2), (3, 16, 0, 0)])
def test_chunked_fused_launch_matches_the_oracle(sx, oracle_lib, dim, levels, chunk, lpt):
    """sxen_tuning.level_chunk: one fused launch whose grid walks the levels in contiguous ranges (blockIdx.y = range,
    sample-major inside a range -- the library default at dim 3, T = 2^19, 16 levels).  Same features bit for bit as the
    oracle (HashEncoder::encode, src/encoding.cpp:295-315), same touched rows, gradients to the fp32-atomic bar
    (encode_backward, :317-335); ragged sample counts and level counts that the range size does not divide included."""
    cfg = oracle.Config(dim=dim, levels=levels, table_size=1 << 19, features=2, base_resolution=16,
                        growth=1.5 if dim == 3 else 2.0)
    enc = make_encoder(sx, cfg, seed=42)
    enc.set_tuning(sx.Tuning(levels_per_thread=lpt, level_major=0 if chunk else -1, level_chunk=chunk))
    N = 3001
    x32 = oracle_lib.rng_doubles(99, 1, N * dim).reshape(N, dim).astype(np.float32)
    up32 = oracle_lib.rng_doubles(7, 2, N * levels * 2, -1.0, 1.0).astype(np.float32).reshape(N, levels * 2)
    grad = sx.EncoderGradient(enc)
    feats = enc.encode_forward_backward(dev(x32), dev(up32), grad)
    enc.check()
    xd, upd = x32.astype(np.float64), up32.astype(np.float64)
    want, bad = oracle_lib.encode(cfg, oracle_lib.init_tables(cfg, 42), xd)
    assert bad == -1
    assert np.array_equal(feats.cpu().numpy().view(np.uint32), want.view(np.uint32))
    og, ot, _ = oracle_lib.encode_backward(cfg, xd, upd)
    scale = abs_contrib(oracle_lib, cfg, xd, upd)
    gv, gt = grad_dense(grad, cfg)
    assert np.array_equal(gt, ot)
    assert (np.abs(gv - og) <= GRAD_RTOL * scale + GRAD_ATOL).all()


@pytest.mark.parametrize("dim", [2, 4, 5, 6])
def test_config5_table_size_under_the_library_launch_shape(sx, oracle_lib, dim):
    """BASELINE configs[4] as stated -- n = 2..6 at L=16, F=2, T=2^22 (512 MiB of tables) -- under the launch shape the
    library picks on its own there (level-major, two levels per thread, the fused call split into a forward and a backward
    launch, evict_last hints): a 2^14-sample batch against the oracle.  Indices / weights / features bit for bit, touched
    rows exact, gradients to the fp32-atomic bar.  (n = 3 at this size: test_level_major... above.)"""
    cfg = oracle.Config(dim=dim, levels=16, table_size=1 << 22, features=2, base_resolution=16, growth=1.5 if dim > 2 else 2.0)
    enc = make_encoder(sx, cfg, seed=42)
    N = 1 << 14
    x32 = oracle_lib.rng_doubles(99, 1, N * dim).reshape(N, dim).astype(np.float32)
    up32 = oracle_lib.rng_doubles(7, 2, N * 32, -1.0, 1.0).astype(np.float32).reshape(N, 32)
    xd, upd = x32.astype(np.float64), up32.astype(np.float64)
    t = enc.tuning()
    assert t.level_major == -1 and t.levels_per_thread == 0 and t.cache_hints == -1   # everything left to the library
    grad = sx.EncoderGradient(enc)
    launches = sx.launch_count()
    feats = enc.encode_forward_backward(dev(x32), dev(up32), grad)
    assert sx.launch_count() - launches >= 2   # forward launch + backward launch (+ fold)
    enc.check()
    idx, w = enc.encode_debug(dev(x32))
    oi, ow, _, _, _ = oracle_lib.encode_debug(cfg, xd)
    assert np.array_equal(idx, oi) and np.array_equal(w, ow)
    want, bad = oracle_lib.encode(cfg, oracle_lib.init_tables(cfg, 42), xd)
    assert bad == -1 and np.array_equal(feats.cpu().numpy().view(np.uint32), want.view(np.uint32))
    og, ot, _ = oracle_lib.encode_backward(cfg, xd, upd)
    scale = abs_contrib(oracle_lib, cfg, xd, upd)
    for l in range(16):   # level by level: the dense [16, 2^22, 2] arrays are 512 MiB each on the host
        gv, gt = grad.level(l)
        assert np.array_equal(gt, ot[l]), (dim, l)
        assert (np.abs(gv - og[l]) <= GRAD_RTOL * scale[l] + GRAD_ATOL).all(), (dim, l)
