"""GPU (-m gpu): the "SXEN"/"SXML" checkpoint format (src/checkpoint.cpp:81-175).  Files written by the unmodified
reference (tests/golden/ref_checkpoint*.sxen) load into the device encoder/MLP with identical parameters, and saving
them again reproduces the reference's bytes exactly -- so B200-trained models load into the reference and back."""
import os

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu
GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


@pytest.fixture(scope="module")
def sx():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2311_15439_b200 as pkg
    return pkg


def test_reference_checkpoint_round_trip_is_byte_exact(sx, tmp_path):
    g = np.load(os.path.join(GOLDEN, "checkpoint_cases.npz"))
    for name, with_mlp in (("ref_checkpoint.sxen", True), ("ref_checkpoint_nomlp.sxen", False)):
        src = os.path.join(GOLDEN, name)
        enc, mlp = sx.load_checkpoint(src)
        cfg = enc.config
        assert [cfg.dim, cfg.levels, cfg.table_size, cfg.features, cfg.base_resolution] == g["cfg"].tolist()
        assert cfg.growth == float(g["growth"]) and cfg.backend == 0
        assert np.array_equal(np.stack([enc.table(l) for l in range(cfg.levels)]), g["tables"])
        assert (mlp is not None) == with_mlp
        if with_mlp:
            mc = mlp.config
            assert [mc.input_width, mc.hidden_width, mc.hidden_layers, mc.output_width] == g["mlp"].tolist()
            assert np.array_equal(mlp.parameters(), g["mlp_params"])
        out = str(tmp_path / name)
        sx.save_checkpoint(out, enc, mlp)
        assert open(out, "rb").read() == open(src, "rb").read()


def test_reference_reads_what_the_device_writes(sx, ref_lib, tmp_path):
    """Live cross-check when the reference library is available: train a few steps on the GPU, save, load with the
    reference, compare parameters."""
    cfg = sx.EncoderConfig(dim=2, levels=4, table_size=1 << 8, features=2, base_resolution=4, growth=2.0)
    enc = sx.HashEncoder(cfg)
    enc.init_tables(3)
    mlp = sx.Mlp(sx.MlpConfig(8, 16, 2, 3))
    mlp.init_params(4)
    tr = sx.Trainer(enc, mlp)
    x = torch.rand((512, 2), dtype=torch.float64, device="cuda:0")
    tr.step(x, torch.rand((512, 3), dtype=torch.float64, device="cuda:0"), sx.AdamConfig(1e-2), sx.AdamConfig(1e-3))
    path = str(tmp_path / "gpu.sxen")
    sx.save_checkpoint(path, enc, mlp)
    c, tables, m, params = ref_lib.load_checkpoint(path)
    assert (c.dim, c.levels, c.table_size, c.features, c.base_resolution, c.growth) == (2, 4, 256, 2, 4, 2.0)
    assert np.array_equal(tables, np.stack([enc.table(l) for l in range(4)]))
    assert (m.input_width, m.hidden_width, m.hidden_layers, m.output_width) == (8, 16, 2, 3)
    assert np.array_equal(params, mlp.parameters())


def test_malformed_checkpoints_raise_io_error(sx, tmp_path):
    good = open(os.path.join(GOLDEN, "ref_checkpoint.sxen"), "rb").read()
    cases = {"magic": b"XXXX" + good[4:], "version": good[:4] + (7).to_bytes(4, "little") + good[8:],
             "truncated": good[:100], "trailing": good + b"\x00", "backend": good[:36] + (5).to_bytes(4, "little") + good[40:],
             "table_size": good[:16] + (1000).to_bytes(4, "little") + good[20:]}
    for name, blob in cases.items():
        p = str(tmp_path / f"{name}.sxen")
        open(p, "wb").write(blob)
        with pytest.raises(sx.IoError):
            sx.load_checkpoint(p)
    with pytest.raises(sx.IoError):
        sx.load_checkpoint(str(tmp_path / "missing.sxen"))


# ---- the reference's own `checkpoint` suite (/root/reference/proj/tests/test_checkpoint.cpp), case by case
def sample_config(sx, **kw):                             # :20-31
    base = dict(dim=3, levels=3, table_size=1 << 8, features=2, base_resolution=5, growth=1.7, backend=sx.Backend.simplex,
                level_scale=sx.LevelScale.raw)
    base.update(kw)
    return sx.EncoderConfig(**base)


def test_suite_encoder_only_round_trip_is_bit_exact(sx, tmp_path):          # :47-71
    cfg = sample_config(sx)
    enc = sx.HashEncoder(cfg)
    enc.init_tables(71)
    path = str(tmp_path / "enc_only.ckpt")
    sx.save_checkpoint(path, enc)
    got, mlp = sx.load_checkpoint(path)
    assert mlp is None
    g = got.config
    assert (g.dim, g.levels, g.table_size, g.features, g.base_resolution, g.growth, g.backend) == \
           (cfg.dim, cfg.levels, cfg.table_size, cfg.features, cfg.base_resolution, cfg.growth, cfg.backend)
    for l in range(cfg.levels):
        assert got.resolution(l) == enc.resolution(l)
        assert np.array_equal(got.table(l).view(np.uint32), enc.table(l).view(np.uint32))


def test_suite_encoder_plus_head_round_trip_is_bit_exact(sx, tmp_path):     # :73-99
    cfg = sample_config(sx)
    enc = sx.HashEncoder(cfg)
    enc.init_tables(72)
    mc = sx.MlpConfig(cfg.encoded_width(), 12, 2, 3)
    mlp = sx.Mlp(mc)
    mlp.init_params(73)
    path = str(tmp_path / "enc_mlp.ckpt")
    sx.save_checkpoint(path, enc, mlp)
    _, got = sx.load_checkpoint(path)
    assert got is not None
    gm = got.config
    assert (gm.input_width, gm.hidden_width, gm.hidden_layers, gm.output_width) == (mc.input_width, 12, 2, 3)
    assert np.array_equal(got.parameters().view(np.uint32), mlp.parameters().view(np.uint32))


def test_suite_level_scale_is_a_loader_parameter_not_file_state(sx, tmp_path):   # :101-116
    cfg = sample_config(sx, level_scale=sx.LevelScale.equal_memory)
    enc = sx.HashEncoder(cfg)
    enc.init_tables(74)
    path = str(tmp_path / "scale_mode.ckpt")
    sx.save_checkpoint(path, enc)
    raw, _ = sx.load_checkpoint(path)                    # default: raw
    assert raw.config.level_scale == sx.LevelScale.raw and raw.resolution(0) != enc.resolution(0)
    matched, _ = sx.load_checkpoint(path, sx.LevelScale.equal_memory)
    assert matched.config.level_scale == sx.LevelScale.equal_memory
    assert [matched.resolution(l) for l in range(cfg.levels)] == [enc.resolution(l) for l in range(cfg.levels)]


def test_suite_corrupt_missing_and_unwritable_are_io_errors(sx, tmp_path):  # :118-165
    enc = sx.HashEncoder(sample_config(sx))
    enc.init_tables(75)
    good = str(tmp_path / "good.ckpt")
    sx.save_checkpoint(good, enc)
    data = open(good, "rb").read()
    assert len(data) > 64
    cases = {"bad_magic": b"Z" + data[1:], "bad_version": data[:4] + bytes([99]) + data[5:],
             "truncated": data[:-7], "trailing": data + b"x"}
    for name, blob in cases.items():
        p = str(tmp_path / f"{name}.ckpt")
        open(p, "wb").write(blob)
        with pytest.raises(sx.IoError):
            sx.load_checkpoint(p)
    with pytest.raises(sx.IoError):
        sx.load_checkpoint(str(tmp_path / "does_not_exist.ckpt"))
    with pytest.raises(sx.IoError):
        sx.save_checkpoint("/nonexistent-dir/x.ckpt", enc)
