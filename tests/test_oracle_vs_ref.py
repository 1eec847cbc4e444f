"""CPU: the oracle restatement against the live, unmodified reference library (oracle/_ref) on seeded random
inputs larger than the committed fixtures.  Skipped when neither the prebuilt .so nor /root/reference exists."""
import numpy as np
import pytest

import oracle
from oracle import Config, MlpConfig

CONFIGS = [
    Config(dim=3, levels=16, table_size=1 << 19, features=2, base_resolution=16, growth=1.5),
    Config(dim=2, levels=16, table_size=1 << 19, features=2, base_resolution=16, growth=2.0),
    Config(dim=4, levels=6, table_size=1 << 15, features=4, base_resolution=8, growth=1.5,
           level_scale=oracle.SCALE_EQUAL_MEMORY),
    Config(dim=6, levels=4, table_size=1 << 14, features=1, base_resolution=4, growth=2.0),
    Config(dim=3, levels=5, table_size=1 << 14, features=2, base_resolution=4, growth=2.0, backend=oracle.BACKEND_GRID),
]


@pytest.mark.parametrize("cfg", CONFIGS, ids=lambda c: f"n{c.dim}_L{c.levels}_F{c.features}_b{c.backend}")
def test_encode_and_backward_match_reference(oracle_lib, ref_lib, cfg):
    rng = np.random.default_rng(cfg.dim * 100 + cfg.levels)
    N = 3000
    x = rng.random((N, cfg.dim))
    x[:8] = rng.integers(0, 2, size=(8, cfg.dim)).astype(np.float64)  # cube corners incl. x == 1.0
    x[8:16] = (x[8:16] * 8).round() / 8  # exact ties / lattice-aligned points
    enc = ref_lib.encoder(cfg)
    enc.init_tables(17)
    tables = oracle_lib.init_tables(cfg, 17)
    assert np.array_equal(tables, enc.tables())
    a, bad = oracle_lib.encode(cfg, tables, x)
    b, rbad, st = enc.encode(x)
    assert bad == -1 and rbad == -1 and st == 0
    assert np.array_equal(a.view(np.uint32), b.view(np.uint32))
    up = rng.standard_normal((N, cfg.encoded_width))
    g1, t1, _ = oracle_lib.encode_backward(cfg, x, up)
    g2, t2, _, _, st = enc.encode_backward(x, up)
    assert st == 0
    assert np.array_equal(t1, t2) and np.array_equal(g1, g2)


def test_reference_rejects_what_oracle_rejects(oracle_lib, ref_lib):
    cfg = Config(dim=2, levels=2, table_size=1 << 10, features=2, base_resolution=4, growth=2.0)
    enc = ref_lib.encoder(cfg)
    t = oracle_lib.init_tables(cfg, 0)
    for x in ([1.5, 0.5], [-1e-300, 0.5], [float("nan"), 0.5], [0.5, float("inf")]):
        pts = np.array([[0.25, 0.5], x])
        _, bad = oracle_lib.encode(cfg, t, pts)
        _, rbad, st = enc.encode(pts)
        assert bad == rbad == 1 and st == 1  # std::invalid_argument


def test_mlp_matches_reference(oracle_lib, ref_lib):
    mc = MlpConfig(32, 64, 2, 3)
    rng = np.random.default_rng(5)
    mlp = ref_lib.mlp(mc)
    mlp.init(99)
    p = oracle_lib.mlp_init(mc, 99)
    assert np.array_equal(p, mlp.params())
    inp = rng.standard_normal((200, 32)).astype(np.float32)
    up = rng.standard_normal((200, 3))
    out_r, grad_r, ig_r = mlp.forward_backward(inp, up)
    out_o, acts = oracle_lib.mlp_forward(mc, p, inp)
    grad_o, ig_o = oracle_lib.mlp_backward(mc, p, acts, up)
    assert np.array_equal(out_o, out_r) and np.array_equal(ig_o, ig_r) and np.array_equal(grad_o, grad_r)
