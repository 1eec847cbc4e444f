"""GPU (-m gpu): run_chunk as ONE kernel (csrc/sxen_train_fused.cu; reference: src/trainer.cpp:20-49).

The fused step must be the unfused tensor-core step with the HBM round trips removed: the gather warps produce the same
feature bits (exact blend) the encode kernel would have written, the tcgen05 head is the same split-bf16 arithmetic, the
scatter warps issue the same products as encode_backward.  Bars:
  * against the three-kernel step on the same batch: loss rel 1e-6, touched row sets EQUAL, table gradients within the
    fp32-atomic bar of test_gpu_parity.py plus the head's own run-to-run noise (the input gradient is identical; only the
    order of the atomics differs), MLP gradient rel 1e-9 (fp64 atomics, different CTA <-> tile assignment of partial sums)
  * against the oracle's fp64 pipeline (oracle.train_grads): loss and gradients within the tensor-core head's TC3_RTOL bars
  * ragged batches (not a multiple of the 128-sample tile), tiny batches (fewer tiles than SMs), dim 2 and 3, out_w 1..3
  * rejected coordinates and non-finite targets keep the reference's throw-before-update through the fused path
"""
import numpy as np
import pytest

import oracle

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

TC3_RTOL = 3e-5


@pytest.fixture(scope="module")
def sx():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2311_15439_b200 as pkg
    return pkg


def make(sx, dim, out_w, T=1 << 14, fused=0, precision=1):
    cfg = sx.EncoderConfig(dim=dim, levels=16, table_size=T, features=2, base_resolution=16, growth=1.5 if dim == 3 else 2.0)
    enc = sx.HashEncoder(cfg)
    enc.init_tables(42)
    mlp = sx.Mlp(sx.MlpConfig(32, 64, 2, out_w))
    mlp.init_params(sx.hash_combine(42, 1))
    mlp.set_precision(precision)
    tr = sx.Trainer(enc, mlp)
    tr.set_fused(fused)
    return cfg, enc, mlp, tr


def grads_of(tr, enc, mlp, x, y, batch=None):
    tr.accumulate(x, y, batch or x.shape[0])
    torch.cuda.synchronize()
    enc.check()
    g = tr.table_grad_device().clone()
    return g, mlp.gradient().copy(), float(tr.loss_device().item())


@pytest.mark.parametrize("dim,out_w,n", [(3, 3, 128 * 300 + 77), (2, 3, 128 * 150), (3, 1, 1000), (2, 2, 50), (3, 3, 1 << 17)])
def test_fused_step_equals_the_three_kernel_step(sx, dim, out_w, n):
    gen = torch.Generator(device="cuda").manual_seed(dim * 100 + out_w)
    x = torch.rand((n, dim), dtype=torch.float32, device="cuda", generator=gen)
    x[0] = 1.0   # a boundary sample (clamped cell: counted once forward, once backward)
    x[1] = 0.0
    y = torch.rand((n, out_w), dtype=torch.float64, device="cuda", generator=gen)
    _, e0, m0, t0 = make(sx, dim, out_w, fused=0)
    _, e1, m1, t1 = make(sx, dim, out_w, fused=1)
    launches = sx.launch_count()
    g1, mg1, l1 = grads_of(t1, e1, m1, x, y)
    fused_launches = sx.launch_count() - launches
    launches = sx.launch_count()
    g0, mg0, l0 = grads_of(t0, e0, m0, x, y)
    assert fused_launches < sx.launch_count() - launches    # one kernel (+ fold) instead of encode + head + encode_backward (+ fold)
    assert abs(l1 - l0) <= 1e-6 * abs(l0)
    neg0 = torch.tensor(-0.0, device="cuda").view(torch.int32)
    touched0 = g0.view(torch.int32).view(-1, 2)[:, 0] != neg0
    touched1 = g1.view(torch.int32).view(-1, 2)[:, 0] != neg0
    assert torch.equal(touched0, touched1)
    scale = g0.abs().max().item()
    assert (g1 - g0).abs().max().item() <= 2e-5 * scale
    # parameter gradients: fp32 sums over a CTA's tiles in TMEM; the stand-alone head groups them by its two tile groups
    assert np.abs(mg1 - mg0).max() <= 1e-4 * np.abs(mg0).max()
    c0, c1 = e0.counters(), e1.counters()
    assert c0.touched_vertices == c1.touched_vertices and c0.out_of_bounds == c1.out_of_bounds


def test_fused_step_against_the_oracle_pipeline(sx, oracle_lib):
    """One batch through the fused kernel against the oracle's fp64 run_chunk (oracle.train_grads): loss, MLP gradient and
    table gradient within the tensor-core head's bars (tests/test_gpu_tc.py)."""
    dim, out_w, n = 3, 3, 5000
    ocfg = oracle.Config(dim=dim, levels=16, table_size=1 << 14, features=2, base_resolution=16, growth=1.5)
    mc = oracle.MlpConfig(32, 64, 2, out_w)
    tables = oracle_lib.init_tables(ocfg, 42)
    params = oracle_lib.mlp_init(mc, oracle_lib.hash_combine(42, 1))
    x = oracle_lib.rng_doubles(99, 1, n * dim).reshape(n, dim).astype(np.float32)
    y = oracle_lib.rng_doubles(5, 3, n * out_w).reshape(n, out_w)
    want = oracle_lib.train_grads(ocfg, mc, tables, params, x.astype(np.float64), y)
    _, enc, mlp, tr = make(sx, dim, out_w, fused=1)
    g, mg, loss_sum = grads_of(tr, enc, mlp, torch.as_tensor(x, device="cuda"), torch.as_tensor(y, device="cuda"))
    wloss, wtg, wtouched, wmg, sample_loss = want   # (batch MSE, table grads, touched, MLP grads, per-sample losses)
    wl = float(sample_loss.sum())
    assert abs(loss_sum - wl) <= 10 * TC3_RTOL * wl
    assert np.linalg.norm(mg - wmg) <= 10 * TC3_RTOL * np.linalg.norm(wmg)
    got = g.cpu().numpy().reshape(16, 1 << 14, 2)
    touched = got.view(np.uint32)[..., 0] != 0x80000000
    assert np.array_equal(touched, wtouched.astype(bool))
    got = np.where(touched[..., None], got, 0.0)
    # a hidden unit whose pre-activation sits within the split-bf16 error of zero can land on the other side of the ReLU than
    # in fp64, which changes that SAMPLE's whole input gradient (tests/test_gpu_tc.py bounds the share of such samples at
    # 2e-3); every row those few samples touch then differs.  So: nearly all elements to the head's bar, the whole to 2 %.
    close = np.abs(got - wtg) <= 20 * TC3_RTOL * np.abs(wtg).max()
    assert close[touched].mean() >= 0.995, close[touched].mean()
    assert np.linalg.norm(got - wtg) <= 2e-2 * np.linalg.norm(wtg)


def test_fused_training_runs_track_the_unfused_ones(sx):
    """30 queued steps, fused vs three kernels: the loss curves agree to the head's noise and go down."""
    ta, ma = sx.AdamConfig(lr=1e-2), sx.AdamConfig(lr=1e-3)
    gen = torch.Generator(device="cuda").manual_seed(9)
    xs = [torch.rand((8192, 3), dtype=torch.float32, device="cuda", generator=gen) for _ in range(30)]
    ys = [torch.stack([0.5 + 0.5 * torch.sin(9 * x[:, 0]), x[:, 1] * x[:, 2], 0.5 + 0.5 * torch.cos(7 * x[:, 2])], dim=1).double()
          for x in xs]
    curves = []
    for fused in (0, 1):
        _, enc, mlp, tr = make(sx, 3, 3, T=1 << 16, fused=fused)
        for x, y in zip(xs, ys):
            tr.step_enqueue(x, y, ta, ma)
        losses, failed = tr.collect()
        assert failed == -1
        curves.append(np.array(losses))
    assert curves[1][-1] < 0.5 * curves[1][0]
    assert np.allclose(curves[0][:5], curves[1][:5], rtol=1e-4)
    assert np.allclose(curves[0], curves[1], rtol=0.05)


def test_fused_step_keeps_throw_before_update(sx):
    ta, ma = sx.AdamConfig(lr=1e-2), sx.AdamConfig(lr=1e-3)
    _, enc, mlp, tr = make(sx, 3, 3, fused=1)
    x = torch.rand((3000, 3), dtype=torch.float32, device="cuda")
    y = torch.rand((3000, 3), dtype=torch.float32, device="cuda")
    before = np.stack([enc.table(l) for l in range(16)])
    bad = x.clone()
    bad[2999, 2] = 1.5
    with pytest.raises(ValueError, match="sample 2999"):
        tr.step(bad, y, ta, ma)
    ybad = y.clone()
    ybad[17, 0] = float("nan")
    with pytest.raises(sx.TrainingError):
        tr.step(x, ybad, ta, ma)
    assert np.array_equal(np.stack([enc.table(l) for l in range(16)]), before)
    assert np.isfinite(tr.step(x, y, ta, ma))
    assert not np.array_equal(np.stack([enc.table(l) for l in range(16)]), before)
    # configurations the fused kernel does not cover fall back (auto) or are refused (required)
    _, enc2, mlp2, tr2 = make(sx, 3, 3, fused=1, precision=0)
    with pytest.raises(ValueError, match="fused kernel was required"):
        tr2.step(x, y, ta, ma)


def test_back_to_back_fused_launches_complete(sx):
    """A few hundred launches back to back (mbarrier phase bookkeeping over tiles and launches; the tcgen05 head once hung
    in such a loop, tools/mlp_stress.py)."""
    ta, ma = sx.AdamConfig(lr=1e-3), sx.AdamConfig(lr=1e-4)
    _, enc, mlp, tr = make(sx, 3, 3, T=1 << 16, fused=1)
    for n in (1 << 16, 128 * 148 * 2 + 5, 300):
        x = torch.rand((n, 3), dtype=torch.float32, device="cuda")
        y = torch.rand((n, 3), dtype=torch.float32, device="cuda")
        for _ in range(100):
            tr.step_enqueue(x, y, ta, ma)
        losses, failed = tr.collect()
        assert failed == -1 and len(losses) == 100 and np.isfinite(losses).all()
