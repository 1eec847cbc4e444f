"""GPU (-m gpu): the C++ host side above the C ABI -- include/sxen_b200_train.hpp's train_field / fit_image / fit_field,
compiled with g++ into a program that links only libsxen_b200.so (no Python, no CUDA headers) -- against the reference's
own runs (tests/golden/task_cases.npz, field_cases.npz), and the queued training step behind it
(sxen_trainer_step_enqueue / sxen_trainer_collect) against the per-step entry point.

Bars (the same as the Python mirror's tests): first loss of a fit rel 1e-12 (same batch, same init; exact head), first 20
losses rel 2e-3, final PSNR within 0.5 dB of the reference's; fit_field loss curve rel 1e-3, hold-out MSE within 2 %,
field variance 1e-9; a non-finite loss raises TrainingError naming the step and leaves tables and MLP untouched."""
import os
import subprocess

import numpy as np
import pytest

from closeness import assert_tables_match

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def sx():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2311_15439_b200 as pkg
    return pkg


@pytest.fixture(scope="module")
def cpp_results(sx, tmp_path_factory):
    tmp = tmp_path_factory.mktemp("cpp_trainer")
    lib_dir = os.path.join(ROOT, "paper_2311_15439_b200", "lib")
    exe = str(tmp / "train_tasks_check")
    subprocess.run(["g++", "-std=c++20", "-O1", "-Wall", "-I", os.path.join(ROOT, "include"),
                    os.path.join(ROOT, "tests", "cpp", "train_tasks_check.cpp"), "-o", exe, "-L", lib_dir,
                    "-lsxen_b200", f"-Wl,-rpath,{lib_dir}"], check=True)
    g = np.load(os.path.join(ROOT, "tests", "golden", "task_cases.npz"))
    gf = np.load(os.path.join(ROOT, "tests", "golden", "field_cases.npz"))
    img = np.ascontiguousarray(g["image"], dtype=np.float64)
    img_path = str(tmp / "image.f64")
    img.tofile(img_path)
    c = g["cfg"]
    assert int(c[0]) == 2
    env = dict(os.environ)
    for kind in (0, 1):
        fc = gf[f"fit_k{kind}/cfg"]
        env[f"SXEN_FIELD_CFG{kind}"] = (f"{int(fc[0])} {int(fc[1])} {int(fc[2])} {int(fc[3])} {int(fc[4])} "
                                        f"{float(gf[f'fit_k{kind}/growth'][0])!r}")
    run = subprocess.run([exe, img_path, str(img.shape[1]), str(img.shape[0]), str(int(c[1])), str(int(c[2])),
                          str(int(c[3])), str(int(c[4])), repr(float(g["growth"])), str(int(g["steps"])),
                          str(int(g["batch"]))], capture_output=True, text=True, env=env, timeout=900)
    assert run.returncode == 0 and "train_tasks ok" in run.stdout, run.stdout[-2000:] + run.stderr[-2000:]
    out = {}
    for line in run.stdout.splitlines():
        parts = line.split()
        if len(parts) >= 2 and parts[0] not in ("train_tasks",):
            out[parts[0]] = np.array([float(v) for v in parts[1:]])
    return out, g, gf


def test_cpp_fit_image_matches_the_reference_run(cpp_results):
    out, g, _ = cpp_results
    ref = g["loss"]
    for key, tol0 in (("w1", 1e-12), ("w64", 1e-12), ("tc", 1e-6)):
        loss = out[f"fit_image_{key}_loss"]
        assert loss.shape == ref.shape
        assert abs(loss[0] - ref[0]) <= tol0 * ref[0]
        assert np.all(np.abs(loss[:20] - ref[:20]) <= 2e-3 * ref[:20])
        assert abs(out[f"fit_image_{key}_psnr"][0] - float(g["final_psnr"])) <= 0.5
    # window 1 and window 64 are the same run up to the order of the fp32 atomics
    assert np.allclose(out["fit_image_w1_loss"][:20], out["fit_image_w64_loss"][:20], rtol=1e-4)
    assert out["launches"][0] > 0


def test_cpp_fit_field_tracks_the_reference_run(cpp_results):
    out, _, gf = cpp_results
    for kind in (0, 1):
        want = gf[f"fit_k{kind}/loss"]
        assert np.allclose(out[f"fit_field_k{kind}_loss"], want, rtol=1e-3)
        mse, var = gf[f"fit_k{kind}/holdout"]
        got_mse, got_var = out[f"fit_field_k{kind}_holdout"]
        assert abs(got_mse / mse - 1) <= 2e-2
        assert abs(got_var - var) <= 1e-9


def _model(sx, T=1 << 12):
    cfg = sx.EncoderConfig(dim=2, levels=16, table_size=T, features=2, base_resolution=4, growth=1.3)
    enc = sx.HashEncoder(cfg)
    enc.init_tables(42)
    mlp = sx.Mlp(sx.MlpConfig(cfg.encoded_width(), 64, 2, 3))
    mlp.init_params(sx.hash_combine(42, 1))
    return cfg, enc, mlp


def test_queued_steps_equal_per_step_calls(sx):
    """K queued steps + one collect == K sxen_trainer_step calls: same losses (to the order of the fp32 atomics), same
    step counters, pending bookkeeping."""
    ta, ma = sx.AdamConfig(lr=1e-2), sx.AdamConfig(lr=1e-3)
    gen = torch.Generator(device="cuda").manual_seed(5)
    batches = [(torch.rand((4096, 2), dtype=torch.float64, device="cuda", generator=gen),
                torch.rand((4096, 3), dtype=torch.float64, device="cuda", generator=gen)) for _ in range(12)]
    _, e1, m1 = _model(sx)
    t1 = sx.Trainer(e1, m1)
    per_step = [t1.step(x, y, ta, ma) for x, y in batches]
    _, e2, m2 = _model(sx)
    t2 = sx.Trainer(e2, m2)
    for x, y in batches[:5]:
        t2.step_enqueue(x, y, ta, ma)
    assert t2.pending() == 5
    first, failed = t2.collect()
    assert failed == -1 and len(first) == 5 and t2.pending() == 0
    for x, y in batches[5:]:
        t2.step_enqueue(x, y, ta, ma)
    rest, failed = t2.collect()
    assert failed == -1 and t2.collect() == ([], -1)
    queued = np.array(first + rest)
    assert queued[0] == per_step[0]                       # before any update: the same arithmetic on the same state
    assert np.allclose(queued, per_step, rtol=1e-4)
    assert np.allclose(m2.parameters(), m1.parameters(), rtol=1e-3, atol=1e-6)
    for l in (0, 7, 15):
        assert_tables_match(e2.table(l), e1.table(l), 1e-6, rtol=1e-3)


def test_queued_non_finite_loss_stops_the_updates_on_the_device(sx):
    """src/trainer.cpp:121-123: the reference throws before the optimizer steps.  Queued: the failing step and every
    later one leave tables, MLP and moments untouched; collect names the step."""
    ta, ma = sx.AdamConfig(lr=1e-2), sx.AdamConfig(lr=1e-3)
    cfg, enc, mlp = _model(sx)
    tr = sx.Trainer(enc, mlp)
    x = torch.rand((1024, 2), dtype=torch.float64, device="cuda")
    good = torch.rand((1024, 3), dtype=torch.float64, device="cuda")
    bad = good.clone()
    bad[17, 1] = float("nan")
    tr.step_enqueue(x, good, ta, ma)
    tr.step_enqueue(x, good, ta, ma)
    losses, failed = tr.collect()
    assert failed == -1 and all(np.isfinite(losses))
    tables = [enc.table(l).copy() for l in range(cfg.levels)]
    params = mlp.parameters().copy()
    tr.step_enqueue(x, good, ta, ma)   # step 0 of this window: applied
    tr.step_enqueue(x, bad, ta, ma)    # step 1: non-finite
    tr.step_enqueue(x, good, ta, ma)   # step 2: queued behind it, must not be applied either
    losses, failed = tr.collect()
    assert failed == 1 and np.isfinite(losses[0]) and not np.isfinite(losses[1])
    assert any(not np.array_equal(enc.table(l), tables[l]) for l in range(cfg.levels))   # step 0 did update
    assert not np.array_equal(mlp.parameters(), params)
    # ... and nothing after it: one more good step from here gives the loss the failing window's step 2 would have seen
    # had it been applied after step 0 only (same state, same batch)
    state = [enc.table(l).copy() for l in range(cfg.levels)]
    tr.step_enqueue(x, good, ta, ma)
    (again,), failed = tr.collect()
    assert failed == -1 and np.isclose(again, losses[2], rtol=1e-6)
    assert any(not np.array_equal(enc.table(l), state[l]) for l in range(cfg.levels))
    # train_field surfaces it as TrainingError with the global step number
    _, enc3, mlp3 = _model(sx)
    init = [enc3.table(l).copy() for l in range(cfg.levels)]

    def sampler(step, batch):
        return x[:batch], (bad if step >= 0 else good)[:batch]

    with pytest.raises(sx.TrainingError, match="step 0"):
        sx.train_field(enc3, mlp3, sampler, sx.TrainConfig(batch_size=1024, steps=6, record_every=1))
    for l in range(cfg.levels):
        assert np.array_equal(enc3.table(l), init[l])


def test_queue_overflow_is_a_logic_error(sx):
    ta, ma = sx.AdamConfig(), sx.AdamConfig()
    _, enc, mlp = _model(sx, T=1 << 10)
    tr = sx.Trainer(enc, mlp)
    x = torch.rand((64, 2), dtype=torch.float64, device="cuda")
    y = torch.rand((64, 3), dtype=torch.float64, device="cuda")
    for _ in range(4096):
        tr.step_enqueue(x, y, ta, ma)
    with pytest.raises(RuntimeError, match="not collected"):
        tr.step_enqueue(x, y, ta, ma)
    losses, failed = tr.collect()
    assert len(losses) == 4096 and failed == -1 and losses[-1] < losses[0]


@pytest.mark.parametrize("backend", [0, 1])
def test_small_batch_table_update_walks_the_batch_like_the_scan(sx, backend):
    """A small batch takes the batch-walking sparse Adam (O(batch*L*V) claims by atomic exchange) instead of the scan of
    all L*T accumulator rows.  Same rows, same arithmetic: against a twin driven through accumulate + update (always the
    scan) the updated-row sets are identical, the tables agree to the order of the fp32 atomics, and the accumulator is
    left fully cleared (a row the walk missed would still be marked touched)."""
    cfg = sx.EncoderConfig(dim=2, levels=16, table_size=1 << 17, features=2, base_resolution=16, growth=1.4,
                           backend=backend)
    ta, ma = sx.AdamConfig(lr=1e-2), sx.AdamConfig(lr=1e-3)
    gen = torch.Generator(device="cuda").manual_seed(11)
    B = 1024   # 1024 * 16 * 3 * 8 <= 16 * 2^17: the walk pays
    batches = [(torch.rand((B, 2), dtype=torch.float64, device="cuda", generator=gen),
                torch.rand((B, 3), dtype=torch.float64, device="cuda", generator=gen)) for _ in range(4)]
    batches[1][0][:8] = batches[1][0][0]          # repeated samples: several threads race for the same rows
    batches[2][0][5] = torch.tensor([1.0, 0.0])   # the cube's corner (clamped cell)

    def twin():
        enc = sx.HashEncoder(cfg)
        enc.init_tables(42)
        mlp = sx.Mlp(sx.MlpConfig(cfg.encoded_width(), 64, 2, 3))
        mlp.init_params(sx.hash_combine(42, 1))
        return enc, mlp, sx.Trainer(enc, mlp)

    e1, m1, t1 = twin()   # whole-step entry points: walk
    e2, m2, t2 = twin()   # accumulate + update: scan
    e3, m3, t3 = twin()   # queued steps: walk behind the gate
    init = [e1.table(l).reshape(-1, 2).copy() for l in range(cfg.levels)]
    for x, y in batches:
        l1 = t1.step(x, y, ta, ma)
        t2.accumulate(x, y, B)
        l2 = t2.loss(B)
        t2.update(ta, ma)
        t3.step_enqueue(x, y, ta, ma)
        assert np.isclose(l1, l2, rtol=1e-5)
    l3, failed = t3.collect()
    assert failed == -1 and np.isclose(l3[-1], l2, rtol=1e-5)
    for tr in (t1, t2, t3):
        g = tr.table_grad_device()
        assert int((g.view(torch.int32) != -2147483648).sum().item()) == 0   # every row back to -0.0f
    for l in range(cfg.levels):
        a, b, c = (e.table(l).reshape(-1, 2) for e in (e1, e2, e3))
        changed = (b != init[l]).any(axis=1)
        assert changed.sum() > 0
        assert np.array_equal((a != init[l]).any(axis=1), changed), l
        assert np.array_equal((c != init[l]).any(axis=1), changed), l
        assert_tables_match(a, b, 1e-6, rtol=1e-3)
        assert_tables_match(c, b, 1e-6, rtol=1e-3)
    assert np.allclose(m1.parameters(), m2.parameters(), rtol=1e-3, atol=1e-6)


def test_cpp_bench_kernel_protocol(sx, tmp_path):
    """include/sxen_b200_analysis.hpp on the device: the reference's bench-kernel protocol (src/analysis.cpp:233-313) from a
    C++ host program -- exact vertices per sample (n+1 simplex, 2^n grid), cells = side^n, a resolved time."""
    lib_dir = os.path.join(ROOT, "paper_2311_15439_b200", "lib")
    exe = str(tmp_path / "analysis_check")
    subprocess.run(["g++", "-std=c++20", "-O1", "-Wall", "-I", os.path.join(ROOT, "include"),
                    os.path.join(ROOT, "tests", "cpp", "analysis_check.cpp"), "-o", exe, "-L", lib_dir,
                    "-lsxen_b200", f"-Wl,-rpath,{lib_dir}"], check=True)
    run = subprocess.run([exe, str(tmp_path)], capture_output=True, text=True, timeout=600)
    assert run.returncode == 0 and run.stdout.strip().endswith("analysis ok"), run.stdout + run.stderr
    assert run.stdout.count("bench_kernel n=") == 6


def test_cpp_checkpoint_round_trip_of_reference_files(sx, tmp_path):
    """include/sxen_b200_checkpoint.hpp on the device: the reference-written fixtures (tests/golden/ref_checkpoint*.sxen,
    src/checkpoint.cpp:81-112) load and re-save byte for byte from a C++ host program; truncated files, trailing bytes and
    a bad MLP magic raise IoError; a device-written grid / F=4 model reads back identically."""
    lib_dir = os.path.join(ROOT, "paper_2311_15439_b200", "lib")
    exe = str(tmp_path / "checkpoint_check")
    subprocess.run(["g++", "-std=c++20", "-O1", "-Wall", "-I", os.path.join(ROOT, "include"),
                    os.path.join(ROOT, "tests", "cpp", "checkpoint_check.cpp"), "-o", exe, "-L", lib_dir,
                    "-lsxen_b200", f"-Wl,-rpath,{lib_dir}"], check=True)
    gold = os.path.join(ROOT, "tests", "golden")
    run = subprocess.run([exe, str(tmp_path), os.path.join(gold, "ref_checkpoint.sxen"),
                          os.path.join(gold, "ref_checkpoint_nomlp.sxen")], capture_output=True, text=True, timeout=600)
    assert run.returncode == 0 and run.stdout.strip().endswith("checkpoint ok"), run.stdout + run.stderr


def test_queued_steps_report_a_rejected_coordinate_at_collect(sx):
    """check_input (src/encoding.cpp:183-194) on the queued path: the offending sample is named when the window is
    collected (ValueError = std::invalid_argument), and the handle goes on afterwards."""
    ta, ma = sx.AdamConfig(lr=1e-2), sx.AdamConfig(lr=1e-3)
    _, enc, mlp = _model(sx)
    tr = sx.Trainer(enc, mlp)
    x = torch.rand((256, 2), dtype=torch.float64, device="cuda")
    y = torch.rand((256, 3), dtype=torch.float64, device="cuda")
    bad = x.clone()
    bad[37, 1] = 1.5
    tr.step_enqueue(x, y, ta, ma)
    torch.cuda.synchronize()
    tables1 = np.stack([enc.table(l) for l in range(enc.config.levels)])
    params1 = mlp.parameters().copy()
    tr.step_enqueue(bad, y, ta, ma)
    tr.step_enqueue(x, y, ta, ma)   # queued behind the rejected batch: must not be applied either
    with pytest.raises(ValueError, match="sample 37"):
        tr.collect()
    # the reference rejects the batch before it changes anything (check_input throws inside encode): tables, MLP and the
    # step counters are as they were after the one good step -- the device gate closed on the encoder's rejected-sample word
    assert np.array_equal(np.stack([enc.table(l) for l in range(enc.config.levels)]), tables1)
    assert np.array_equal(mlp.parameters(), params1)
    # a twin that ran the same two good steps and nothing else ends in the same state (bias corrections included)
    _, enc2, mlp2 = _model(sx)
    tr2 = sx.Trainer(enc2, mlp2)
    tr2.step_enqueue(x, y, ta, ma)
    tr2.step_enqueue(x, y, ta, ma)
    tr2.collect()
    tr.step_enqueue(x, y, ta, ma)
    losses, failed = tr.collect()
    assert failed == -1 and len(losses) == 1 and np.isfinite(losses[0])
    # (fp32 atomics: same rows, values to the accumulation-order bar)
    a = np.stack([enc.table(l) for l in range(enc.config.levels)])
    b = np.stack([enc2.table(l) for l in range(enc2.config.levels)])
    assert np.array_equal(a != tables1, b != tables1)
    assert_tables_match(a, b, 1e-3 * 1e-2)   # ... except for the odd Adam sign flip (tests/closeness.py)


def test_per_step_call_refuses_to_jump_a_queue(sx):
    """sxen_trainer_step is one queued step collected at once: with steps still queued it would hand back the wrong loss,
    so it is a logic error until they are collected."""
    ta, ma = sx.AdamConfig(lr=1e-2), sx.AdamConfig(lr=1e-3)
    _, enc, mlp = _model(sx, T=1 << 10)
    tr = sx.Trainer(enc, mlp)
    x = torch.rand((128, 2), dtype=torch.float64, device="cuda")
    y = torch.rand((128, 3), dtype=torch.float64, device="cuda")
    first = tr.step(x, y, ta, ma)
    tr.step_enqueue(x, y, ta, ma)
    with pytest.raises(RuntimeError, match="not collected"):
        tr.step(x, y, ta, ma)
    (second,), failed = tr.collect()
    third = tr.step(x, y, ta, ma)
    assert failed == -1 and first > second > third
