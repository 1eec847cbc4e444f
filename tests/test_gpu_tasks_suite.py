"""GPU (-m gpu): the reference's own `tasks` test suite (/root/reference/proj/tests/test_tasks.cpp), case by case, against
the device path -- same configurations (task_encoder: 4 levels, T = 2^12, F = 2, base 4, growth 2; quick_train: batch 256,
record_every 50), same assertions.  Determinism cases run in the reproducible mode, where the device path makes the same
promise as the reference (bit-identical runs for a fixed seed)."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def sx():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2311_15439_b200 as pkg
    return pkg


def task_encoder(sx, backend, dim):       # tests/test_tasks.cpp:12-24
    return sx.EncoderConfig(dim=dim, levels=4, table_size=1 << 12, features=2, base_resolution=4, growth=2.0, backend=backend,
                            level_scale=sx.LevelScale.raw)


def quick_train(sx, steps, batch=256, **kw):     # :26-33
    return sx.TrainConfig(steps=steps, batch_size=batch, threads=1, record_every=50, **kw)


def constant_image(w, h, value):          # :35-41
    return np.full((h, w, 3), value, dtype=np.float64)


def test_psnr_cap_identity_and_scale(sx):                                   # :47-53
    assert sx.psnr_from_mse(0.0) == 99.0 and sx.psnr_from_mse(-1.0) == 99.0 and sx.psnr_from_mse(1e-12) == 99.0
    assert abs(sx.psnr_from_mse(1.0)) <= 1e-12 and abs(sx.psnr_from_mse(0.01) - 20.0) <= 1e-12 * 20


def test_image_metrics(sx):                                                 # :55-61
    img = sx.make_test_image(24, 16, 3)
    assert sx.image_mse(img, img) == 0.0 and sx.image_psnr(img, img) == 99.0
    with pytest.raises(ValueError):
        sx.image_mse(img, sx.make_test_image(16, 24, 3))


def test_procedural_image_is_deterministic_seed_sensitive_and_in_range(sx):  # :74-93
    a, b, c = sx.make_test_image(32, 32, 7), sx.make_test_image(32, 32, 7), sx.make_test_image(32, 32, 8)
    assert np.array_equal(a, b) and not np.array_equal(a, c)
    assert a.min() >= 0.0 and a.max() <= 1.0 and a.max() - a.min() > 0.2


def test_zero_model_renders_black(sx):                                      # :95-114
    cfg = task_encoder(sx, sx.Backend.simplex, 2)
    enc = sx.HashEncoder(cfg)
    mlp = sx.Mlp(sx.MlpConfig(cfg.encoded_width(), 8, 1, 3))                # zero weights
    img = sx.render_image(enc, mlp, 20, 12, 1)
    assert img.shape == (12, 20, 3) and not img.any()
    with pytest.raises(ValueError):
        sx.render_image(enc, sx.Mlp(sx.MlpConfig(cfg.encoded_width(), 8, 1, 2)), 4, 4, 1)


def test_constant_gray_image_passes_50_db_within_500_steps(sx):             # :116-121
    res = sx.fit_image(constant_image(64, 64, 0.5), task_encoder(sx, sx.Backend.simplex, 2), quick_train(sx, 500))
    assert res.final_psnr > 50.0
    # (the encoded width here is 8: the tensor-core head covers 16 and 32 and says so instead of falling back)
    with pytest.raises(ValueError, match="tensor-core path covers"):
        sx.fit_image(constant_image(8, 8, 0.5), task_encoder(sx, sx.Backend.simplex, 2), quick_train(sx, 1),
                     sx.FitImageOptions(mlp_precision=1))


def test_fit_image_validates_the_encoder_dimension(sx):                     # :123-127
    with pytest.raises(ValueError):
        sx.fit_image(constant_image(8, 8, 0.5), task_encoder(sx, sx.Backend.simplex, 3), quick_train(sx, 1))


def test_zero_step_fit_reports_a_finite_reproducible_baseline(sx):          # :129-136
    img = sx.make_test_image(32, 32, 9)
    a = sx.fit_image(img, task_encoder(sx, sx.Backend.simplex, 2), quick_train(sx, 0))
    b = sx.fit_image(img, task_encoder(sx, sx.Backend.simplex, 2), quick_train(sx, 0))
    assert np.isfinite(a.final_psnr) and abs(a.final_psnr - b.final_psnr) <= 1e-9 and a.train.steps_run == 0


def test_image_fit_learns(sx):                                              # :138-150
    res = sx.fit_image(sx.make_test_image(48, 48, 10), task_encoder(sx, sx.Backend.simplex, 2), quick_train(sx, 300))
    curve = res.train.loss_curve
    assert len(curve) >= 2 and curve[-1][1] < curve[0][1]
    assert len(res.psnr_curve) == len(curve)
    for (s0, p), (s1, l) in zip(res.psnr_curve, curve):
        assert s0 == s1 and abs(p - sx.psnr_from_mse(l)) <= 1e-12 * max(1.0, abs(p))


def _field_spec(sx):
    return sx.NoiseFieldSpec(dim=2, seed=7, kind=sx.NoiseKind.perlin, octaves=1, frequency=4.0)


def test_field_regression_beats_a_tenth_of_the_variance(sx):                # :152-166
    res = sx.fit_field(_field_spec(sx), task_encoder(sx, sx.Backend.simplex, 2), quick_train(sx, 300),
                       sx.FitFieldOptions(holdout_samples=1 << 12))
    assert res.field_variance > 1e-4 and res.holdout_mse < 0.1 * res.field_variance


def test_simplex_and_grid_land_within_2x_on_the_same_field(sx):             # :168-187
    opt = sx.FitFieldOptions(holdout_samples=1 << 12)
    s = sx.fit_field(_field_spec(sx), task_encoder(sx, sx.Backend.simplex, 2), quick_train(sx, 300), opt).holdout_mse
    g = sx.fit_field(_field_spec(sx), task_encoder(sx, sx.Backend.grid, 2), quick_train(sx, 300), opt).holdout_mse
    assert s > 0.0 and g > 0.0 and 0.5 < s / g < 2.0


def test_field_fit_is_deterministic_for_a_fixed_seed(sx):                   # :189-204, in the reproducible mode
    spec = sx.NoiseFieldSpec(dim=3, seed=5, kind=sx.NoiseKind.simplex, octaves=1, frequency=3.0)
    opt = sx.FitFieldOptions(holdout_samples=1 << 10)
    runs = [sx.fit_field(spec, task_encoder(sx, sx.Backend.simplex, 3), quick_train(sx, 50, reproducible=True), opt).holdout_mse
            for _ in range(2)]
    assert runs[0] == runs[1]


def test_fit_field_validates_dimensions_and_holdout_size(sx):               # :206-216
    spec = sx.NoiseFieldSpec(dim=3)
    with pytest.raises(ValueError):
        sx.fit_field(spec, task_encoder(sx, sx.Backend.simplex, 2), quick_train(sx, 1))
    with pytest.raises(ValueError):
        sx.fit_field(spec, task_encoder(sx, sx.Backend.simplex, 3), quick_train(sx, 1), sx.FitFieldOptions(holdout_samples=1))
