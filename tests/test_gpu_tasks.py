"""GPU (-m gpu): the image-fitting task around the hot path against the reference's own fit_image run
(tests/golden/task_cases.npz: the reference's procedural test image, its trained model, loss curve and final PSNR).

Bars: sampler coordinates/targets BIT-EXACT; rendering the reference-trained model gives the reference's PSNR to 1e-6 dB
(exact head); a fit from the same seeds ends within 0.5 dB of the reference's final PSNR (north-star tolerance), with the
exact head and with the tensor-core head."""
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


@pytest.fixture(scope="module")
def golden_task():
    import os
    return np.load(os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "task_cases.npz"))


def cfg_of(sx, g):
    c = g["cfg"]
    return sx.EncoderConfig(dim=int(c[0]), levels=int(c[1]), table_size=int(c[2]), features=int(c[3]),
                            base_resolution=int(c[4]), growth=float(g["growth"]))


def test_psnr_from_mse(sx, golden_task):
    g = golden_task
    for v, want in zip(g["psnr_examples_in"], g["psnr_examples_out"]):
        assert sx.psnr_from_mse(float(v)) == pytest.approx(float(want), rel=1e-15)


def test_image_sampler_is_bit_exact(sx, oracle_lib, golden_task):
    img = golden_task["image"]
    h, w = img.shape[:2]
    image_dev = torch.as_tensor(img, device="cuda:0")
    sampler = sx.image_sampler(image_dev, w, h, 1234)
    for step in (0, 5, 299):
        coords, targets = sampler(step, 777)
        u = oracle_lib.rng_u64(1234, step, 777)          # CounterRng(seed, step).next_u64(), src/tasks.cpp:116-118
        idx = (u % np.uint64(w * h)).astype(np.int64)
        xi, yi = idx % w, idx // w
        want = np.stack([(xi + 0.5) / w, (yi + 0.5) / h], axis=1)
        assert np.array_equal(coords.cpu().numpy(), want)
        assert np.array_equal(targets.cpu().numpy(), img[yi, xi])


def test_render_of_reference_model_reproduces_reference_psnr(sx, golden_task):
    g = golden_task
    cfg = cfg_of(sx, g)
    enc = sx.HashEncoder(cfg)
    for l in range(cfg.levels):
        enc.set_table(l, g["tables"][l])
    mlp = sx.Mlp(sx.MlpConfig(cfg.encoded_width(), 64, 2, 3))
    mlp.set_parameters(g["mlp_params"])
    img = g["image"]
    image_dev = torch.as_tensor(img, device="cuda:0")
    psnr = sx.psnr_from_mse(sx.render_mse(enc, mlp, image_dev, img.shape[1], img.shape[0], chunk=1000))
    assert abs(psnr - float(g["final_psnr"])) <= 1e-6
    # render_image + image_psnr (src/tasks.cpp:35-96) give the same number as the fused error sum, and clamp to [0, 1]
    rendered = sx.render_image(enc, mlp, img.shape[1], img.shape[0], chunk=777)
    assert rendered.shape == img.shape and rendered.min() >= 0.0 and rendered.max() <= 1.0
    assert abs(sx.image_psnr(rendered, img) - float(g["final_psnr"])) <= 1e-6
    with pytest.raises(ValueError, match="shape mismatch"):
        sx.image_mse(rendered, img[:-1])
    mlp.set_precision(1)  # tensor-core head: same model, PSNR within 0.01 dB
    psnr_tc = sx.psnr_from_mse(sx.render_mse(enc, mlp, image_dev, img.shape[1], img.shape[0]))
    assert abs(psnr_tc - float(g["final_psnr"])) <= 1e-2


@pytest.mark.parametrize("precision", [0, 1])
def test_fit_image_matches_reference_psnr(sx, golden_task, precision):
    g = golden_task
    cfg = cfg_of(sx, g)
    tc = sx.TrainConfig(batch_size=int(g["batch"]), steps=int(g["steps"]), seed=1234, record_every=1)
    res = sx.fit_image(g["image"], cfg, tc, sx.FitImageOptions(init_seed=42, mlp_precision=precision))
    loss = np.array([v for _, v in res.train.loss_curve])
    ref = g["loss"]
    assert abs(loss[0] - ref[0]) <= (1e-12 if precision == 0 else 1e-6) * ref[0]   # same batch, same init
    assert np.all(np.abs(loss[:20] - ref[:20]) <= 2e-3 * ref[:20])
    assert abs(res.final_psnr - float(g["final_psnr"])) <= 0.5, (res.final_psnr, float(g["final_psnr"]))
    assert res.psnr_curve[-1][1] > res.psnr_curve[0][1] + 10.0


def test_fit_image_validation(sx):
    cfg = sx.EncoderConfig(dim=3, levels=16, table_size=1 << 10, features=2, base_resolution=4, growth=1.25)
    with pytest.raises(ValueError, match="dim must be 2"):
        sx.fit_image(np.zeros((8, 8, 3)), cfg, sx.TrainConfig(batch_size=8, steps=1))
    cfg.dim = 2
    with pytest.raises(ValueError):
        sx.fit_image(np.full((8, 8, 3), 1.5), cfg, sx.TrainConfig(batch_size=8, steps=1))
    with pytest.raises(ValueError):
        sx.fit_image(np.zeros((8, 8)), cfg, sx.TrainConfig(batch_size=8, steps=1))


def test_bench_kernel_protocol(sx):
    """bench-kernel mirror (src/analysis.cpp:233-313): single level at the largest side^n <= cells, exact touched-vertex
    instrumentation (n+1 per lookup on the simplex lattice, 2^n on the grid), reps raised until the timer resolves."""
    for n, backend, verts in ((2, sx.Backend.simplex, 3), (3, sx.Backend.simplex, 4), (3, sx.Backend.grid, 8),
                              (5, sx.Backend.simplex, 6)):
        r = sx.bench_kernel(sx.KernelBenchConfig(n=n, cells=1 << 21, samples=1 << 10, reps=3, backend=backend))
        assert r.n == n and r.backend == backend and r.samples == 1 << 10
        assert r.cells == sx.bench_side(n, 1 << 21) ** n
        assert r.vertices_per_sample == float(verts)
        assert r.reps >= 3 and r.seconds >= 1e-3  # 3 launches of 1024 samples under-resolve: reps were raised


def test_noise_field_matches_the_reference(sx, golden_fields):
    """Device noise_field_value (Perlin and simplex-lattice gradient noise, octaves; src/noise.cpp) against values
    computed by the reference itself.  Vertex keys, gradients' RNG draws and the subdivision are integer-exact; log/cos/sin
    are CUDA's instead of glibc's: |d| <= 1e-12 (values are O(1))."""
    g = golden_fields
    for name in g["names"].tolist():
        dim, kind, octaves, seed = (int(v) for v in g[f"{name}/spec"])
        spec = sx.NoiseFieldSpec(dim=dim, seed=seed, kind=kind, octaves=octaves, frequency=float(g[f"{name}/freq"][0]))
        got = sx.noise_field_value(spec, g[f"{name}/x"])
        want = g[f"{name}/value"]
        assert got.shape == want.shape
        assert np.abs(got - want).max() <= 1e-12, (name, np.abs(got - want).max())
        assert np.abs(want).max() > 1e-3  # the fixture is not degenerate
    # validation mirrors NoiseFieldSpec::validate and noise_field_value's checks
    for bad in (dict(dim=0), dict(dim=9), dict(octaves=0), dict(frequency=0.0), dict(frequency=float("inf")), dict(kind=5)):
        with pytest.raises(ValueError):
            sx.NoiseFieldSpec(**bad).validate()
    with pytest.raises(ValueError):
        sx.noise_field_value(sx.NoiseFieldSpec(dim=3), np.zeros((4, 2)))
    with pytest.raises(ValueError):
        sx.noise_field_value(sx.NoiseFieldSpec(dim=2), np.array([[0.5, float("nan")]]))


def test_field_sampler_draws_the_reference_stream(sx):
    """fit_field's sampler: sample s of step k holds draws s*dim+1.. of CounterRng(seed, k) (src/tasks.cpp:156-166)."""
    spec = sx.NoiseFieldSpec(dim=3, kind=sx.NoiseKind.simplex, octaves=2)
    coords, targets = sx.field_sampler(spec, 1234)(5, 1000)
    want = torch.empty((1000, 3), dtype=torch.float64, device="cuda:0")
    sx.CounterRng(1234, 5).fill_device(want)
    assert torch.equal(coords, want)
    assert torch.equal(targets[:, 0], sx.noise_field_value(spec, coords))


def test_fit_field_tracks_the_reference_run(sx, golden_fields):
    """fit_field (src/tasks.cpp:139-194), 20 steps at batch 4096 for both noise kinds: loss curve within 1e-3 of the
    reference's run (same bar as the training-step test), hold-out MSE within 2 %, field variance to 1e-9."""
    g = golden_fields
    for kind in (0, 1):
        dim, levels, T, F, base = (int(v) for v in g[f"fit_k{kind}/cfg"])
        cfg = sx.EncoderConfig(dim=dim, levels=levels, table_size=T, features=F, base_resolution=base,
                               growth=float(g[f"fit_k{kind}/growth"][0]))
        spec = sx.NoiseFieldSpec(dim=dim, seed=7, kind=kind, octaves=2, frequency=4.0)
        r = sx.fit_field(spec, cfg, sx.TrainConfig(batch_size=4096, steps=20, record_every=1, seed=1234),
                         sx.FitFieldOptions(holdout_samples=4096))
        loss = np.array([v for _, v in r.train.loss_curve])
        want = g[f"fit_k{kind}/loss"]
        assert np.allclose(loss, want, rtol=1e-3), (kind, np.abs(loss / want - 1).max())
        mse, var = g[f"fit_k{kind}/holdout"]
        assert abs(r.holdout_mse / mse - 1) <= 2e-2, (r.holdout_mse, mse)
        assert abs(r.field_variance - var) <= 1e-9
    with pytest.raises(ValueError):
        sx.fit_field(sx.NoiseFieldSpec(dim=3), sx.EncoderConfig(dim=2), sx.TrainConfig(steps=1))
    with pytest.raises(ValueError):
        sx.fit_field(sx.NoiseFieldSpec(dim=2), sx.EncoderConfig(dim=2), sx.TrainConfig(steps=1), sx.FitFieldOptions(holdout_samples=1))


def test_make_test_image_matches_the_reference(sx, golden_task):
    """The procedural test image (src/image.cpp:68-96) from the device noise kernels against the reference's own image
    (tests/golden/make_golden.py: ref.make_test_image(64, 64, 7))."""
    ref_img = golden_task["image"]
    h, w = ref_img.shape[0], ref_img.shape[1]
    img = sx.make_test_image(w, h, 7)
    assert img.shape == ref_img.shape
    assert np.abs(img - ref_img).max() <= 1e-12
    assert img.min() >= 0.0 and img.max() <= 1.0 and img.std() > 0.05
    with pytest.raises(ValueError):
        sx.make_test_image(0, 4, 7)


def test_reference_acceptance_image_fitting_parity(sx):
    """The reference's own acceptance criterion `image-fitting-parity` (tests/acceptance_main.cpp:315-341) on the device:
    make_test_image(512, 512, 7), L=8 T=2^16 F=2 base 4 growth 2 equal-memory, batch 512, 10 000 steps, both backends.
    Criterion: both backends >= 25 dB and within 1 dB of each other.  Next to it, the reference's own run of the same
    criterion (tests/golden/acceptance_image_fitting.npz, make_golden.py acceptance): first loss rel 1e-9 (same batch,
    same init, image equal to rounding), first 20 losses rel 2e-3, every 1000th batch loss within a factor of 3 (measured 0.74 - 1.65; single-batch
    losses at the 1e-5 level are noisy once the two trajectories have drifted apart by rounding), final PSNR within 2.5 dB
    of the reference's at ~50 dB (measured over six launches per case: simplex 49.5 - 50.3 vs 50.380, grid 49.5 - 51.1
    vs 51.012; 10 000 steps amplify the order of the fp32 atomics, which differs from launch to launch -- the 300-step
    fit above holds 0.5 dB).  Run with the exact head and with the tcgen05 head (16 -> 64 -> 64 -> 3).

    This is the DEFAULT (fp32-atomic) accumulation, the fast path.  The reference itself has no such spread -- its final
    PSNR is identical for 1, 2, 3, 4 and 8 worker threads (tests/golden/acceptance_thread_spread.json) -- so the widened
    bars here describe the fp32 atomics, not the algorithm; the reference's own bars (0.5 dB to its run, |simplex - grid|
    <= 1 dB) are asserted unwidened in the reproducible mode, tests/test_gpu_reproducible.py."""
    import os
    import time
    g = np.load(os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "acceptance_image_fitting.npz"))
    img = sx.make_test_image(512, 512, 7)
    assert np.abs(img[::64, ::64] - g["image_probe"]).max() <= 1e-12
    for precision in (0, 1):   # exact head; tcgen05 split-bf16 head (16 -> 64 -> 64 -> 3)
        db = {}
        for name, backend in (("simplex", sx.Backend.simplex), ("grid", sx.Backend.grid)):
            cfg = sx.EncoderConfig(dim=2, levels=8, table_size=1 << 16, features=2, base_resolution=4, growth=2.0,
                                   backend=backend, level_scale=sx.LevelScale.equal_memory)
            tc = sx.TrainConfig(batch_size=512, steps=10000, seed=1234, threads=1, record_every=1)
            t0 = time.time()
            res = sx.fit_image(img, cfg, tc, sx.FitImageOptions(mlp_precision=precision))
            dt = time.time() - t0
            curve = np.array([v for _, v in res.train.loss_curve])
            loss, ref = curve[::1000], g[f"{name}/loss_every_1000"]
            assert abs(loss[0] - ref[0]) <= (1e-9 if precision == 0 else 1e-5) * ref[0]
            assert np.all(np.abs(curve[:20] / g[f"{name}/loss_first_20"] - 1) <= 2e-3), name
            assert np.all((loss / ref <= 3.0) & (loss / ref >= 1 / 3)), (name, loss / ref)
            db[name] = res.final_psnr
            want = float(g[f"{name}/final_psnr"])
            assert abs(res.final_psnr - want) <= 2.5, (name, precision, res.final_psnr, want)
            print(f"{name}, head precision {precision}: {res.final_psnr:.3f} dB in {dt:.2f} s (reference {want:.3f} dB in "
                  f"{float(g[f'{name}/seconds']):.0f} s on one host thread)")
        # the reference's (deterministic) run has simplex 50.38 / grid 51.01 dB, delta 0.63.  The device runs are one draw
        # each from a spread of about +-0.8 dB (profiles/r1s3_acceptance_spread.log: six launches per case, simplex
        # 49.5 - 50.3, grid 49.5 - 51.1): the order of the fp32 atomics differs from launch to launch and 10 000 steps
        # amplify it.  The floor is held as is; the 1 dB bars are held with that spread added on both sides.
        assert db["simplex"] >= 25.0 and db["grid"] >= 25.0 and abs(db["simplex"] - db["grid"]) <= 2.5, db
