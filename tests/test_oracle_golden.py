"""CPU: pin oracle/sxen_oracle.c against the reference's golden vectors.

Sources of truth: (1) values frozen in the reference's own tests and in SURVEY.md 8c (typed in below),
(2) fixtures under tests/golden/ generated from the compiled, unmodified reference.
"""
import numpy as np
import pytest

import oracle
from oracle import AdamConfig, Config, MlpConfig
from conftest import case_config, merge_chain


# ---------------------------------------------------------------- SURVEY 8c frozen values
def test_rng_frozen(oracle_lib):
    o = oracle_lib
    assert o.mix64(0) == 16294208416658607535
    assert o.hash_combine(42, 1) == 9692408228951597300
    assert set(o.rng_u64(1234, 0, 2).tolist()) == {15934349690077123996, 541818966539761233}
    assert o.rng_doubles(99, None, 1)[0] == 0.88088003301114937


def test_skew_constants_frozen(oracle_lib):
    s2, s3 = oracle_lib.skew_constants(2), oracle_lib.skew_constants(3)
    assert s2.tolist() == [0.3660254037844386, 0.21132486540518708, 1.7320508075688772]
    assert s3.tolist() == [0.33333333333333331, 0.16666666666666666, 2.0]
    for n in range(1, 9):  # reference tests/test_lattice.cpp:39-45
        f, g, s = oracle_lib.skew_constants(n)
        assert abs(f - g - n * f * g) < 1e-15
        assert s == pytest.approx(np.sqrt(n + 1.0), rel=1e-15)


def test_resolution_ladders_frozen(oracle_lib):
    cfg = Config(dim=3, levels=16, table_size=1 << 19, base_resolution=16, growth=1.5)
    assert oracle_lib.resolutions(cfg) == [16, 24, 36, 54, 81, 121, 182, 273, 410, 615, 922, 1383, 2075, 3113, 4670, 7006]
    cfg = Config(dim=2, levels=16, table_size=1 << 19, base_resolution=16, growth=2.0)
    assert oracle_lib.resolutions(cfg) == [16 << l for l in range(16)]
    # reference tests/test_encoding.cpp:88-106
    cfg = Config(dim=2, levels=4, table_size=1 << 10, base_resolution=16, growth=2.0)
    assert [oracle_lib.level_resolution(cfg, l) for l in (0, 1, 3)] == [16, 32, 128]
    assert oracle_lib.equal_memory_multiplier(2) == pytest.approx(3.0 ** 0.25, rel=1e-12)
    assert oracle_lib.equal_memory_multiplier(3) == pytest.approx(np.cbrt(4.0), rel=1e-12)
    cfg.level_scale = oracle.SCALE_EQUAL_MEMORY
    assert oracle_lib.level_resolution(cfg, 0) == int(np.floor(16.0 * 3.0 ** 0.25))
    cfg.backend = oracle.BACKEND_GRID
    assert oracle_lib.level_resolution(cfg, 0) == 16


def test_hash_frozen(oracle_lib):
    assert oracle_lib.hash_coords([1, 2]) == 1013904227
    assert oracle_lib.hash_coords([1, 2]) & ((1 << 19) - 1) == 455523
    assert oracle_lib.hash_coords([1, 2, 3]) == 2892625372
    assert oracle_lib.hash_coords([1, 2, 3]) & ((1 << 19) - 1) == 128476
    for n in range(1, 9):  # reference tests/test_encoding.cpp:39-45
        assert oracle_lib.hash_coords([0] * n) == 0


def test_lattice_frozen(oracle_lib):
    # reference tests/test_lattice.cpp:127-150, 169-184
    perm, _ = oracle_lib.subdivide([0.3, 0.6])
    assert perm.tolist() == [1, 0]
    perm, srt = oracle_lib.subdivide([0.7, 0.5, 0.2])
    assert perm.tolist() == [0, 1, 2]
    w = oracle_lib.barycentric(srt)
    assert np.allclose(w, [0.3, 0.2, 0.3, 0.2], atol=1e-12)
    assert oracle_lib.barycentric([0.0, 0.0]).tolist() == [1.0, 0.0, 0.0]
    perm, _ = oracle_lib.subdivide([0.5, 0.5])  # ties keep ascending axis order
    assert perm.tolist() == [0, 1]


FROZEN_POINTS = [
    # (cfg, level, x, base, perm, idx, w, feature0 or None, table seed)
    (Config(dim=2, levels=1, table_size=1 << 10, features=2, base_resolution=4, growth=2.0), 0, [0.25, 0.5],
     [1, 1], [1, 0], [432, 867, 864], [0.21132486540518691, 0.57735026918962573, 0.21132486540518736],
     2.80681197e-05, 123),
    (Config(dim=3, levels=16, table_size=1 << 19, features=2, base_resolution=16, growth=1.5), 0, [0.31, 0.77, 0.12],
     [5, 9, 4], [0, 1, 2], [137576, 137579, 237240, 95493],
     [.32000000000000028, .32000000000000028, .19999999999999929, .16000000000000014], -2.46729196e-05, 42),
    (Config(dim=3, levels=16, table_size=1 << 19, features=2, base_resolution=16, growth=1.5), 15, [0.31, 0.77, 0.12],
     [2487, 4098, 1821], [2, 1, 0], [193588, 89251, 139986, 139997],
     [.44000000000028194, .049999999999499778, .38000000000010914, .13000000000010914], -2.21245955e-05, 42),
    (Config(dim=3, levels=16, table_size=1 << 19, features=2, base_resolution=16, growth=1.5), 15, [1.0, 0.0, 1.0],
     [5838, 2335, 5838], [1, 0, 2], [500807, 474632, 474633, 386708],
     [.66666666666696983, 9.0949470177292824e-13, 0.0, .33333333333212067], None, 42),
    (Config(dim=2, levels=16, table_size=1 << 19, features=2, base_resolution=16, growth=2.0), 15,
     [1000.5 / 2048, 77.5 / 2048], [206194, 69773], [1, 0], [78607, 177500, 177501],
     [.47020313914981671, .059593721671262756, .47020313917892054], None, 42),
]


@pytest.mark.parametrize("case", FROZEN_POINTS, ids=lambda c: f"n{c[0].dim}_l{c[1]}")
def test_gather_frozen_points(oracle_lib, case):
    cfg, level, x, base, perm, idx, w, f0, seed = case
    gi, gw, gb, gp, bad = oracle_lib.encode_debug(cfg, np.array([x]))
    assert bad == -1
    assert gb[0, level].tolist() == base
    assert gp[0, level].tolist() == perm
    assert gi[0, level].tolist() == idx
    assert np.allclose(gw[0, level], w, rtol=0, atol=5e-16)
    if f0 is not None:
        tables = oracle_lib.init_tables(cfg, seed)
        out, _ = oracle_lib.encode(cfg, tables, np.array([x]))
        assert out[0, level * cfg.features] == pytest.approx(f0, rel=2e-8)


def test_table_init_frozen(oracle_lib):
    cfg = Config(dim=2, levels=1, table_size=1 << 10, features=2, base_resolution=4, growth=2.0)
    t = oracle_lib.init_tables(cfg, 123)
    assert np.allclose(t[0, :4], [1.44627611e-05, 7.30800602e-05, 2.1084421e-05, -8.23445953e-05], rtol=2e-8)


# ---------------------------------------------------------------- fixtures from the compiled reference
def test_scalar_fixtures(oracle_lib, golden_scalar):
    g, o = golden_scalar, oracle_lib
    assert [o.mix64(int(z)) for z in g["mix64_in"]] == g["mix64_out"].tolist()
    zs = g["mix64_in"]
    assert [o.hash_combine(int(a), int(b)) for a in zs for b in zs[:4]] == g["hash_combine_out"].tolist()
    assert np.array_equal(o.rng_u64(1234, 0, 16), g["rng_1234_0_u64"])
    assert np.array_equal(o.rng_u64(99, None, 16), g["rng_99_u64"])
    assert np.array_equal(o.rng_doubles(99, None, 16), g["rng_99_double"])
    assert np.array_equal(o.rng_doubles(7, 2, 16, -1.0, 1.0), g["rng_7_2_ranged"])
    assert np.array_equal(np.stack([o.skew_constants(n) for n in range(1, 9)]), g["skew"])
    assert np.array_equal([o.equal_memory_multiplier(n) for n in range(1, 9)], g["eqmem"])
    for c, n, h in zip(g["hash_coords_in"], g["hash_coords_n"], g["hash_coords_out"]):
        assert o.hash_coords(c[:n]) == h
    for fr, perm, srt, w, n in zip(g["sub_fracs"], g["sub_perm"], g["sub_sorted"], g["sub_w"], g["sub_n"]):
        p, s = o.subdivide(fr[:n])
        assert np.array_equal(p, perm[:n]) and np.array_equal(s, srt[:n])
        assert np.array_equal(o.barycentric(s), w[: n + 1])
    ladders = {
        "res_b16_g1.5": Config(dim=3, levels=16, base_resolution=16, growth=1.5, table_size=1 << 19),
        "res_b16_g2": Config(dim=2, levels=16, base_resolution=16, growth=2.0, table_size=1 << 19),
        "res_eqmem_n2": Config(dim=2, levels=10, base_resolution=16, growth=1.6, level_scale=oracle.SCALE_EQUAL_MEMORY),
        "res_eqmem_n5": Config(dim=5, levels=10, base_resolution=7, growth=1.37, level_scale=oracle.SCALE_EQUAL_MEMORY),
        "res_grid_eqmem": Config(dim=3, levels=6, base_resolution=16, growth=1.5, backend=oracle.BACKEND_GRID,
                                 level_scale=oracle.SCALE_EQUAL_MEMORY),
    }
    for k, cfg in ladders.items():
        assert o.resolutions(cfg) == g[k].tolist()


def test_encode_fixtures_bit_exact(oracle_lib, golden_encode):
    g, o = golden_encode, oracle_lib
    for name in g["names"].tolist():
        cfg = case_config(g, name)
        assert o.validate(cfg) == 0
        assert o.resolutions(cfg) == g[f"{name}/res"].tolist()
        tables = o.init_tables(cfg, int(g[f"{name}/seed"]))
        assert np.array_equal(tables[:, :8], g[f"{name}/table_head"]), name
        x = g[f"{name}/x"]
        counters = np.zeros(2, dtype=np.uint64)
        out, bad = o.encode(cfg, tables, x, counters)
        assert bad == -1
        assert np.array_equal(out.view(np.uint32), g[f"{name}/features"].view(np.uint32)), name
        assert counters.tolist() == g[f"{name}/counters"].tolist(), name
        # vertex chains: indices bit-exact, weights bit-exact (duplicates merged as the accumulator does)
        idx, w, _, _, _ = o.encode_debug(cfg, x)
        gi, gw, gc = g[f"{name}/idx"], g[f"{name}/w"], g[f"{name}/cnt"]
        for s in range(x.shape[0]):
            for l in range(cfg.levels):
                mi, mw = merge_chain(idx[s, l], w[s, l])
                k = int(gc[s, l])
                assert mi == gi[s, l, :k].tolist(), (name, s, l)
                assert mw == gw[s, l, :k].tolist(), (name, s, l)
        # backward: same dense accumulator contents
        grad, touched, bad = o.encode_backward(cfg, x, g[f"{name}/upstream"])
        assert bad == -1
        lv, rows, vals = g[f"{name}/g_level"], g[f"{name}/g_row"], g[f"{name}/g_val"]
        assert int(touched.sum()) == lv.size, name
        assert np.array_equal(grad[lv, rows], vals), name
        assert touched[lv, rows].all()


def test_mlp_fixtures(oracle_lib, golden_neural):
    g, o = golden_neural, oracle_lib
    mc = MlpConfig(32, 64, 2, 3)
    p = o.mlp_init(mc, int(g["mlp_seed"]))
    assert np.array_equal(p, g["mlp_params"])
    out, acts = o.mlp_forward(mc, p, g["mlp_in"])
    assert np.array_equal(out, g["mlp_out"])
    grad, ig = o.mlp_backward(mc, p, acts, g["mlp_up"])
    assert np.array_equal(ig, g["mlp_input_grad"])
    # the reference sums per-sample grads in the same order, so the batch gradient is bit-identical too
    assert np.array_equal(grad, g["mlp_grad"])
    for tag, mc2 in (("h0", MlpConfig(5, 7, 0, 2)), ("h1", MlpConfig(6, 9, 1, 1))):
        p2 = o.mlp_init(mc2, 11)
        assert np.array_equal(p2, g[f"mlp_{tag}_params"])
        o2, a2 = o.mlp_forward(mc2, p2, g[f"mlp_{tag}_in"])
        assert np.array_equal(o2, g[f"mlp_{tag}_out"])
        g2, ig2 = o.mlp_backward(mc2, p2, a2, g[f"mlp_{tag}_up"])
        assert np.array_equal(g2, g[f"mlp_{tag}_grad"]) and np.array_equal(ig2, g[f"mlp_{tag}_input_grad"])


def test_adam_fixtures(oracle_lib, golden_neural):
    g, o = golden_neural, oracle_lib
    ac = AdamConfig(lr=1e-2)
    p = g["adam_p0"].copy()
    m, v = np.zeros(16), np.zeros(16)
    for t in range(5):
        assert o.adam_step(p, g["adam_g"][t], m, v, t + 1, ac) == -1
        assert np.array_equal(p, g["adam_p"][t]), t
    bad = g["adam_g"][0].copy()
    bad[5] = np.nan
    assert o.adam_step(p, bad, m, v, 6, ac) == 5  # TrainingError index, reference src/optimizer.cpp:35-37


@pytest.mark.parametrize("threads", [1])
def test_train_fixture_single_thread_bit_exact(oracle_lib, golden_neural, threads):
    """Replays reference train_field (1 worker) with the oracle's pieces: loss curve, tables and MLP bit-identical."""
    g, o = golden_neural, oracle_lib
    c = g["train_cfg"]
    cfg = Config(dim=int(c[0]), levels=int(c[1]), table_size=int(c[2]), features=int(c[3]), base_resolution=int(c[4]),
                 growth=2.0)
    mc = MlpConfig(*[int(v) for v in g["train_mlp"]])
    tables = o.init_tables(cfg, 42)
    params = o.mlp_init(mc, o.hash_combine(42, 1))
    tm, tv = np.zeros(tables.size), np.zeros(tables.size)
    mm, mv = np.zeros(params.size), np.zeros(params.size)
    coords, targets = g["train_coords"], g["train_targets"]
    for step in range(coords.shape[0]):
        loss, tg, touched, mg, _ = o.train_grads(cfg, mc, tables, params, coords[step], targets[step])
        assert loss == g["train_loss_t1"][step], step
        flat = tables.reshape(-1)
        assert o.sparse_adam_step(cfg, flat, tg, touched, tm, tv, step + 1, AdamConfig(lr=1e-2)) == -1
        assert o.adam_step(params, mg, mm, mv, step + 1, AdamConfig(lr=1e-3)) == -1
    assert np.array_equal(tables, g["train_tables_t1"])
    assert np.array_equal(params, g["train_mlp_params_t1"])


def test_validation_codes(oracle_lib):
    # reference tests/test_encoding.cpp:108-138
    ok = Config(dim=2, levels=2, table_size=1 << 10, features=2, base_resolution=4, growth=2.0)
    assert oracle_lib.validate(ok) == 0
    for field, value in [("dim", 0), ("dim", 9), ("levels", 0), ("table_size", 1000), ("features", 0),
                         ("features", 65), ("base_resolution", 0), ("growth", 1.0), ("growth", float("nan")),
                         ("growth", float("inf")), ("levels", 40)]:
        bad = Config(**{**ok.__dict__, field: value})
        assert oracle_lib.validate(bad) != 0, (field, value)


def test_input_rejection(oracle_lib):
    # reference tests/test_encoding.cpp:348-358 : out-of-cube and NaN coordinates are rejected, 0 and 1 are legal
    cfg = Config(dim=2, levels=2, table_size=1 << 10, features=2, base_resolution=4, growth=2.0)
    t = oracle_lib.init_tables(cfg, 1)
    for x in ([1.5, 0.5], [-0.1, 0.5], [float("nan"), 0.5]):
        _, bad = oracle_lib.encode(cfg, t, np.array([[0.5, 0.5], x]))
        assert bad == 1
    counters = np.zeros(2, dtype=np.uint64)
    _, bad = oracle_lib.encode(cfg, t, np.array([[0.0, 0.0], [1.0, 1.0], [1.0, 0.0], [0.999999999, 1.0]]), counters)
    assert bad == -1 and counters[1] == 0  # :336-346 boundary points stay in bounds
