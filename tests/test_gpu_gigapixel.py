"""GPU (-m gpu): BASELINE configs[2] as written -- fit_image on a 32768 x 32768 procedural image that is never stored.

The reference's sampler (src/tasks.cpp:112-126) draws idx = CounterRng(seed, step).next_below(w*h) and reads the pixel
from the ImageDataset; make_test_image (src/image.cpp:68-96) defines every pixel as a function of its centre, so the
target can be evaluated where it is drawn (sxen_sample_test_image_batch).  Parity:
  * on a stored image (64 x 64): coordinates bit-identical to sxen_sample_image_batch, targets equal to the stored pixels
  * at 32768 x 32768: indices / coordinates bit-exact and targets within NOISE_ATOL of the REFERENCE's own
    noise_field_value at those pixels (tests/golden/gigapixel_sampler.npz, make_golden.py gigapixel)
  * a short sharded-shaped fit runs and learns
"""
import os

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

NOISE_ATOL = 1e-12   # log / cos / sin of the gradient table are CUDA's, not glibc's (same bar as test_gpu_tasks.py)
GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "gigapixel_sampler.npz")


@pytest.fixture(scope="module")
def sx():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2311_15439_b200 as pkg
    return pkg


def test_procedural_sampler_equals_the_stored_image_sampler(sx):
    img = sx.make_test_image(64, 48, 7)
    image_dev = torch.as_tensor(img, device="cuda:0").contiguous()
    stored = sx.image_sampler(image_dev.reshape(-1), 64, 48, 1234)
    onfly = sx.test_image_sampler(64, 48, 7, 1234)
    for step in (0, 3, 1000):
        c0, t0 = stored(step, 5000)
        c1, t1 = onfly(step, 5000)
        assert torch.equal(c0, c1)
        assert (t0 - t1).abs().max().item() <= 1e-15   # the same device noise kernels evaluate both
    # a rank's chunk of the batch: samples [first, first + count) of the same stream
    part = sx.test_image_sampler(64, 48, 7, 1234, first=1200, count=700)
    c2, t2 = part(3, 5000)
    c1, t1 = onfly(3, 5000)
    assert torch.equal(c2, c1[1200:1900]) and torch.equal(t2, t1[1200:1900])
    with pytest.raises(ValueError):
        sx.test_image_sampler(0, 4, 7, 1)(0, 4)


def test_gigapixel_sampler_matches_the_reference(sx):
    g = np.load(GOLD)
    W, H = int(g["width"]), int(g["height"])
    assert W == H == 32768
    sampler = sx.test_image_sampler(W, H, int(g["image_seed"]), int(g["train_seed"]))
    for step in (0, 7):
        coords, targets = sampler(step, 1 << 16)     # a 2^16-sample batch; the fixture holds its first 1024 draws
        c, t = coords[:1024].cpu().numpy(), targets[:1024].cpu().numpy()
        assert np.array_equal(c, g[f"step{step}/coords"])
        idx = np.rint(c[:, 1] * H - 0.5).astype(np.int64) * W + np.rint(c[:, 0] * W - 0.5).astype(np.int64)
        assert np.array_equal(idx, g[f"step{step}/idx"])
        assert np.abs(t - g[f"step{step}/targets"]).max() <= NOISE_ATOL
        full = targets.cpu().numpy()
        assert full.min() >= 0.0 and full.max() <= 1.0 and full.std() > 0.05


def test_gigapixel_fit_learns(sx):
    """configs[2] shape at a reduced step count: L=16 F=2 T=2^19, base 16, growth 2.0 (finest 524288 >= 32768), 2^18
    samples per step for 40 steps with the tcgen05 head; PSNR over the first 2^20 pixels."""
    cfg = sx.EncoderConfig(dim=2, levels=16, table_size=1 << 19, features=2, base_resolution=16, growth=2.0)
    tc = sx.TrainConfig(batch_size=1 << 18, steps=40, record_every=1)
    res = sx.fit_test_image(32768, 32768, 7, cfg, tc, sx.FitImageOptions(mlp_precision=1), psnr_pixels=1 << 20)
    loss = [v for _, v in res.train.loss_curve]
    assert loss[-1] < 0.2 * loss[0]
    assert res.final_psnr > 18.0
    # the error kernel agrees with the sampler's targets: MSE over a pixel range == mean squared error against the targets
    # the sampler would hand out for those pixels (checked on a row of the image through both paths)
    mse_a = sx.test_image_mse(res.encoder, res.mlp, 32768, 32768, 7, first_pixel=5 * 32768, count=4096)
    coords = torch.empty((4096, 2), dtype=torch.float64, device="cuda:0")
    import ctypes as C
    assert sx.lib.sxen_pixel_centers(32768, 32768, 5 * 32768, 4096, C.c_void_p(coords.data_ptr()), None) == 0
    pred = res.mlp.forward(res.encoder.encode(coords)).double().clamp(0, 1)
    # targets of exactly those pixels: evaluate the image through make_test_image's definition on a strip is not stored, so
    # compare with the noise kernels directly
    shared = sx.NoiseFieldSpec(dim=2, seed=sx.hash_combine(7, 0xAB), kind=sx.NoiseKind.perlin, octaves=4, frequency=4.0)
    base = sx.noise_field_value(shared, coords)
    tgt = torch.stack([torch.clamp(0.5 + 0.62 * (0.45 * base + 0.55 * sx.noise_field_value(
        sx.NoiseFieldSpec(dim=2, seed=sx.hash_combine(7, c + 1), kind=sx.NoiseKind.perlin, octaves=5, frequency=8.0), coords)),
        0.0, 1.0) for c in range(3)], dim=1)
    mse_b = ((pred - tgt) ** 2).mean().item()
    assert abs(mse_a - mse_b) <= 1e-12 + 1e-9 * mse_b
