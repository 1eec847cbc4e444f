"""GPU (-m gpu): the reference's own `neural` test suite (/root/reference/proj/tests/test_neural.cpp), case by case,
against the device path -- same shapes, seeds, samplers and tolerances.  The dense matrix-product oracle of
tests/oracles.hpp is tests/independent.py's `mlp_forward` (numpy, fp64).  The reference's per-sample calls become batches
of one; its MlpWorkspace / MlpGradient live inside the Mlp handle.  Bit-identical loss curves are promised in the
reproducible mode (the device's counterpart of "fixed seed and thread count")."""
import math

import numpy as np
import pytest

from independent import mlp_forward

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def sx():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2311_15439_b200 as pkg
    return pkg


def dev(a):
    return torch.as_tensor(np.ascontiguousarray(a), device="cuda:0")


def tiny_mlp(sx, i, h, l, o):                            # tests/test_neural.cpp:19-26
    return sx.MlpConfig(input_width=i, hidden_width=h, hidden_layers=l, output_width=o)


def random_input(sx, width, seed):                       # :28-33  (float)(next_double(-1, 1))
    t = torch.empty(width, dtype=torch.float64, device="cuda:0")
    sx.CounterRng(seed).fill_device(t, -1.0, 1.0)
    return t.to(torch.float32).reshape(1, width)


def layers(mlp):
    L = mlp.layer_count()
    cfg = mlp.config
    return ([mlp.weights(l).reshape(cfg.layer_output_width(l), cfg.layer_input_width(l)) for l in range(L)],
            [mlp.biases(l) for l in range(L)])


def small_encoder(sx, levels=2, log2t=8):
    return sx.EncoderConfig(dim=2, levels=levels, table_size=1 << log2t, features=2, base_resolution=4)


def test_config_validation(sx):                                             # :39-48
    tiny_mlp(sx, 4, 8, 2, 3).validate()
    tiny_mlp(sx, 4, 8, 0, 3).validate()                  # single affine map
    for bad in ((0, 8, 2, 3), (4, 0, 2, 3), (4, 8, -1, 3), (4, 8, 2, 0)):
        with pytest.raises(ValueError):
            tiny_mlp(sx, *bad).validate()
    assert tiny_mlp(sx, 4, 8, 2, 3).layer_count() == 3 and tiny_mlp(sx, 4, 8, 0, 3).layer_count() == 1


def test_zero_parameters_produce_zero_output(sx):                           # :50-56
    mlp = sx.Mlp(tiny_mlp(sx, 6, 12, 2, 4))              # parameters start zeroed
    assert not mlp.forward(random_input(sx, 6, 31)).cpu().numpy().any()


def test_identity_single_layer_passes_input_through(sx):                    # :58-66
    mlp = sx.Mlp(tiny_mlp(sx, 5, 1, 0, 5))
    p = mlp.parameters()
    for o in range(5):
        p[o * 5 + o] = 1.0
    mlp.set_parameters(p)
    x = random_input(sx, 5, 32)                          # includes negatives; the output has no activation
    assert np.array_equal(mlp.forward(x).cpu().numpy(), x.cpu().numpy())


def test_forward_matches_the_dense_matrix_product_oracle(sx):               # :68-81
    mlp = sx.Mlp(tiny_mlp(sx, 8, 16, 2, 3))
    mlp.init_params(41)
    ws, bs = layers(mlp)
    x = torch.cat([random_input(sx, 8, 1000 + it) for it in range(200)])
    got = mlp.forward(x).cpu().numpy().astype(np.float64)
    want = mlp_forward(mlp.config, ws, bs, x.cpu().numpy())
    assert (np.abs(got - want) <= 1e-5 * np.maximum(1.0, np.abs(want))).all()
    one = mlp.forward(x[17:18]).cpu().numpy()            # a batch of one says the same, bit for bit
    assert np.array_equal(one[0].view(np.uint32), mlp.forward(x).cpu().numpy()[17].view(np.uint32))


def test_initialization_is_seed_deterministic_and_bias_free(sx):            # :83-100
    a, b, c = (sx.Mlp(tiny_mlp(sx, 8, 16, 2, 3)) for _ in range(3))
    a.init_params(7)
    b.init_params(7)
    c.init_params(8)
    assert np.array_equal(a.parameters().view(np.uint32), b.parameters().view(np.uint32))
    for l in range(a.layer_count()):
        assert not a.biases(l).any()
    assert (a.parameters() != c.parameters()).any()


def test_backward_requires_a_cached_forward_pass(sx):                       # :102-109
    mlp = sx.Mlp(tiny_mlp(sx, 4, 8, 1, 2))
    mlp.init_params(1)
    with pytest.raises(RuntimeError):                    # std::logic_error
        mlp.backward(dev(np.array([[1.0, 1.0]])))


def test_zero_upstream_produces_zero_gradients_everywhere(sx):              # :111-121
    mlp = sx.Mlp(tiny_mlp(sx, 4, 8, 2, 2))
    mlp.init_params(2)
    mlp.forward(random_input(sx, 4, 33))
    ig = mlp.backward(dev(np.zeros((1, 2))))
    assert not mlp.gradient().any() and not ig.cpu().numpy().any()


def test_single_affine_layer_has_the_closed_form_gradient(sx):              # :123-151
    mlp = sx.Mlp(tiny_mlp(sx, 3, 1, 0, 2))
    mlp.init_params(3)
    x = random_input(sx, 3, 34)
    xin = x.cpu().numpy()[0].astype(np.float64)
    up = np.array([0.7, -1.3])
    mlp.forward(x)
    ig = mlp.backward(dev(up[None, :])).cpu().numpy()[0]
    g = mlp.gradient()
    gw, gb = g[:6].reshape(2, 3), g[6:8]
    assert (np.abs(gb - up) <= 1e-12 * np.abs(up)).all()
    want_w = up[:, None] * xin[None, :]
    assert (np.abs(gw - want_w) <= 1e-6 * np.abs(want_w)).all()
    want_ig = up @ mlp.weights(0).reshape(2, 3).astype(np.float64)
    assert (np.abs(ig - want_ig) <= 1e-6 * np.abs(want_ig)).all()


def test_backward_accumulates_across_calls(sx):                             # :153-170
    once, twice = sx.Mlp(tiny_mlp(sx, 4, 8, 1, 2)), sx.Mlp(tiny_mlp(sx, 4, 8, 1, 2))
    x = random_input(sx, 4, 35)
    up = dev(np.array([[0.4, 0.9]]))
    for m, reps in ((once, 1), (twice, 2)):
        m.init_params(4)
        for _ in range(reps):
            m.forward(x)
            m.backward(up)
    a, b = once.gradient(), twice.gradient()
    assert a.any() and (np.abs(b - 2.0 * a) <= 1e-12 * np.abs(2.0 * a)).all()


def test_gradient_merge_and_clear(sx):                                      # :172-190
    # MlpGradient::merge is a sum: two handles with the same parameters, each holding one backward, against one handle
    # that accumulated both
    cfg = tiny_mlp(sx, 3, 4, 1, 2)
    a, b, both = sx.Mlp(cfg), sx.Mlp(cfg), sx.Mlp(cfg)
    for m in (a, b, both):
        m.init_params(5)
    xa, xb = random_input(sx, 3, 36), random_input(sx, 3, 37)
    ua, ub = dev(np.array([[1.0, 2.0]])), dev(np.array([[-0.5, 0.25]]))
    a.forward(xa); a.backward(ua)
    b.forward(xb); b.backward(ub)
    both.forward(xa); both.backward(ua)
    both.forward(xb); both.backward(ub)
    total = a.gradient() + b.gradient()
    assert (np.abs(both.gradient() - total) <= 1e-12 * np.abs(total) + 1e-300).all()
    merged = a.gradient_device() + b.gradient_device()    # the device views add like the host copies
    assert np.array_equal(merged.cpu().numpy(), total)
    a.clear_gradient()
    assert not a.gradient().any()


def test_full_stack_gradients_match_central_finite_differences(sx):         # :192-228
    mlp = sx.Mlp(tiny_mlp(sx, 4, 8, 2, 2))
    mlp.init_params(45)
    x = random_input(sx, 4, 38)
    up = np.array([0.8, -0.6])
    mlp.forward(x)
    mlp.backward(dev(up[None, :]))
    grad = mlp.gradient()
    params = mlp.parameters()

    def loss(p):
        mlp.set_parameters(p)
        return float((up * mlp.forward(x).cpu().numpy()[0].astype(np.float64)).sum())

    h = 1e-3
    picks = np.random.default_rng(39).integers(0, params.size, size=10)
    for pi in picks:
        p = params.copy()
        p[pi] = np.float32(float(params[pi]) + h)
        hi = loss(p)
        p[pi] = np.float32(float(params[pi]) - h)
        lo = loss(p)
        fd = (hi - lo) / (2.0 * h)
        assert abs(fd - grad[pi]) <= 1e-3 * max(1.0, abs(grad[pi]))
    mlp.set_parameters(params)


def test_adam_zero_gradient_leaves_parameters_unchanged(sx):                # :230-239
    params = dev(np.array([0.5, -0.25, 1.0], dtype=np.float32))
    opt = sx.AdamState(3)
    opt.step(params, dev(np.zeros(3)), sx.AdamConfig())
    assert opt.step_count() == 1
    assert np.array_equal(params.cpu().numpy(), np.array([0.5, -0.25, 1.0], dtype=np.float32))


def test_adam_first_step_closed_form(sx):                                   # :241-251
    params = dev(np.array([1.0, 1.0], dtype=np.float32))
    opt = sx.AdamState(2)
    opt.step(params, dev(np.array([0.5, -0.02])), sx.AdamConfig(lr=0.1))
    p = params.cpu().numpy().astype(np.float64)
    assert abs(p[0] - 0.9) <= 1e-6 * 0.9 and abs(p[1] - 1.1) <= 1e-6 * 1.1


def test_adam_constant_gradient_approaches_a_fixed_step_of_lr(sx):          # :253-267
    params = dev(np.array([0.0], dtype=np.float32))
    grads = dev(np.array([0.3]))
    cfg = sx.AdamConfig(lr=0.01)
    opt = sx.AdamState(1)
    prev = last = 0.0
    for _ in range(200):
        opt.step(params, grads, cfg)
        now = float(params.cpu().numpy()[0])
        last, prev = now - prev, now
    assert abs(last + cfg.lr) <= 0.05 * cfg.lr


def test_adam_non_finite_gradient_raises_a_training_error(sx):              # :269-274
    params = dev(np.array([0.0], dtype=np.float32))
    with pytest.raises(sx.TrainingError):
        sx.AdamState(1).step(params, dev(np.array([float("nan")])), sx.AdamConfig())
    assert float(params.cpu().numpy()[0]) == 0.0         # thrown before the update


def test_sparse_table_update_touches_only_accumulated_entries(sx):          # :276-309
    cfg = small_encoder(sx, 2, 6)
    enc = sx.HashEncoder(cfg)
    enc.init_tables(9)
    before0, before1 = enc.table(0), enc.table(1)
    grad = sx.EncoderGradient(enc)
    v, t = np.zeros((cfg.table_size, 2), dtype=np.float32), np.zeros(cfg.table_size, dtype=np.uint8)
    v[5], t[5] = (0.25, -0.5), 1                          # grad.add(0, 5, 1.0, {0.25, -0.5})
    grad.set_level(0, v, t)
    opt_cfg = sx.AdamConfig(lr=0.05)
    opt = sx.SparseAdamState(enc)
    opt.step(enc, grad, opt_cfg)
    assert opt.step_count() == 1
    after0 = enc.table(0)
    for i in range(before0.size):
        if i == 10:
            assert abs(float(after0[i]) - (float(before0[i]) - opt_cfg.lr)) <= 1e-5 * abs(float(before0[i]) - opt_cfg.lr)
        elif i == 11:
            assert abs(float(after0[i]) - (float(before0[i]) + opt_cfg.lr)) <= 1e-5 * abs(float(before0[i]) + opt_cfg.lr)
        else:
            assert after0[i] == before0[i]
    assert np.array_equal(enc.table(1), before1)


def uniform_sampler(sx, seed, dim, target):
    """CounterRng(seed, step) coordinates; target(coords) -> [B, out] (tests/test_neural.cpp:328-333, :386-393)."""
    def sampler(step, b):
        x = torch.empty((b, dim), dtype=torch.float64, device="cuda:0")
        sx.CounterRng(seed, step).fill_device(x)
        return x, target(x)
    return sampler


def constant_sampler(coord, target, dim=2):
    def sampler(step, b):
        return (torch.full((b, dim), coord, dtype=torch.float64, device="cuda:0"),
                torch.full((b, 1), target, dtype=torch.float64, device="cuda:0"))
    return sampler


def test_training_drives_a_constant_target_below_1e6_in_200_steps(sx):      # :311-338
    ecfg = small_encoder(sx, 2, 8)
    enc = sx.HashEncoder(ecfg)
    enc.init_tables(10)
    mlp = sx.Mlp(tiny_mlp(sx, ecfg.encoded_width(), 16, 1, 1))
    mlp.init_params(11)
    tcfg = sx.TrainConfig(batch_size=256, steps=200, seed=12, threads=1)
    tcfg.mlp_adam.lr = 1e-2                               # the output bias alone can represent the target
    sampler = uniform_sampler(sx, 100, 2, lambda x: torch.full((x.shape[0], 1), 0.35, dtype=torch.float64, device=x.device))
    res = sx.train_field(enc, mlp, sampler, tcfg)
    assert res.steps_run == 200 and res.final_loss < 1e-6


def test_zero_training_steps_leave_every_parameter_untouched(sx):           # :340-368
    ecfg = small_encoder(sx, 2, 6)
    enc = sx.HashEncoder(ecfg)
    enc.init_tables(13)
    mlp = sx.Mlp(tiny_mlp(sx, ecfg.encoded_width(), 8, 1, 1))
    mlp.init_params(14)
    tables_before, params_before = enc.table(0), mlp.parameters()
    res = sx.train_field(enc, mlp, constant_sampler(0.5, 0.0), sx.TrainConfig(steps=0, batch_size=8, threads=1))
    assert res.steps_run == 0 and res.loss_curve == []
    assert np.array_equal(enc.table(0), tables_before) and np.array_equal(mlp.parameters(), params_before)


def test_fixed_seed_gives_a_bit_identical_loss_curve(sx):                   # :370-408
    def run():
        ecfg = small_encoder(sx, 2, 8)
        enc = sx.HashEncoder(ecfg)
        enc.init_tables(15)
        mlp = sx.Mlp(tiny_mlp(sx, ecfg.encoded_width(), 16, 1, 1))
        mlp.init_params(16)
        tcfg = sx.TrainConfig(batch_size=64, steps=40, record_every=5, seed=17, threads=1, reproducible=True)
        sampler = uniform_sampler(sx, 200, 2, lambda x: (torch.sin(6.0 * x[:, 0]) * torch.cos(4.0 * x[:, 1]))[:, None])
        return sx.train_field(enc, mlp, sampler, tcfg).loss_curve

    a, b = run(), run()
    assert len(a) == len(b) == 9 and [s for s, _ in a] == [0, 5, 10, 15, 20, 25, 30, 35, 39]
    for (sa, la), (sb, lb) in zip(a, b):
        assert sa == sb and la == lb                      # bit-identical
    assert a[-1][1] < a[0][1]


def test_loss_curve_records_step_zero_the_cadence_and_the_final_step(sx):   # :410-437
    ecfg = small_encoder(sx, 1, 6)
    enc = sx.HashEncoder(ecfg)
    mlp = sx.Mlp(tiny_mlp(sx, ecfg.encoded_width(), 8, 1, 1))
    mlp.init_params(18)
    res = sx.train_field(enc, mlp, constant_sampler(0.25, 0.5),
                         sx.TrainConfig(batch_size=8, steps=10, record_every=4, threads=1))
    assert [s for s, _ in res.loss_curve] == [0, 4, 8, 9]
    assert all(math.isfinite(l) for _, l in res.loss_curve)


def test_width_mismatch_between_encoder_aux_and_head_is_rejected(sx):       # :439-462
    ecfg = small_encoder(sx, 2, 6)
    enc = sx.HashEncoder(ecfg)
    mlp = sx.Mlp(tiny_mlp(sx, ecfg.encoded_width() + 1, 8, 1, 1))
    with pytest.raises(ValueError):
        sx.train_field(enc, mlp, lambda s, b: None, sx.TrainConfig(threads=1))

    def ok(step, b):                                      # now the widths line up
        f = lambda v, w: torch.full((b, w), v, dtype=torch.float64, device="cuda:0")
        return f(0.5, 2), f(0.7, 1), f(0.1, 1)

    res = sx.train_field(enc, mlp, ok, sx.TrainConfig(threads=1, aux_dims=1, steps=1, batch_size=4))
    assert res.steps_run == 1


def test_a_non_finite_target_aborts_with_a_training_error(sx):              # :464-484
    ecfg = small_encoder(sx, 1, 6)
    enc = sx.HashEncoder(ecfg)
    mlp = sx.Mlp(tiny_mlp(sx, ecfg.encoded_width(), 8, 1, 1))
    mlp.init_params(19)
    before = mlp.parameters()
    with pytest.raises(sx.TrainingError):
        sx.train_field(enc, mlp, constant_sampler(0.5, float("inf")), sx.TrainConfig(batch_size=4, steps=5, threads=1))
    assert np.array_equal(mlp.parameters(), before)       # thrown before any update (src/trainer.cpp:121-123)


def test_host_span_calls_equal_the_device_calls(sx):
    """Mlp::forward / backward through the host-buffer entry points (sxen_mlp_forward_host / _backward_host: the
    reference's span signatures, include/sxen/mlp.hpp:94-99) against the device-pointer calls: same bits."""
    mlp_h, mlp_d = sx.Mlp(tiny_mlp(sx, 8, 16, 2, 3)), sx.Mlp(tiny_mlp(sx, 8, 16, 2, 3))
    mlp_h.init_params(41)
    mlp_d.init_params(41)
    x = torch.cat([random_input(sx, 8, 2000 + it) for it in range(37)])
    up = np.linspace(-1.0, 1.0, 37 * 3).reshape(37, 3)
    with pytest.raises(RuntimeError):                    # std::logic_error, before anything is copied
        mlp_h.backward(up)
    out_h = mlp_h.forward(x.cpu().numpy())
    assert isinstance(out_h, np.ndarray) and np.array_equal(out_h.view(np.uint32), mlp_d.forward(x).cpu().numpy().view(np.uint32))
    ig_h = mlp_h.backward(up)
    ig_d = mlp_d.backward(dev(up)).cpu().numpy()
    assert ig_h.dtype == np.float64 and np.array_equal(ig_h, ig_d)
    gh, gd = mlp_h.gradient(), mlp_d.gradient()
    assert (np.abs(gh - gd) <= 1e-12 * np.abs(gd) + 1e-300).all()
    with pytest.raises(ValueError):
        mlp_h.forward(np.zeros((2, 7), dtype=np.float32))
    with pytest.raises(ValueError):
        mlp_h.backward(np.zeros((36, 3)))                 # batch differs from the forward's
    assert mlp_h.forward(np.zeros((0, 8), dtype=np.float32)).shape == (0, 3)
