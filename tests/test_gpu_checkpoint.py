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
