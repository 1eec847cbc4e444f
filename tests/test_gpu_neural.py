"""GPU (-m gpu): MLP head, loss and training step through the C ABI against the oracle / reference fixtures.

Bars: forward activations and per-sample input gradients BIT-EXACT (fp64 accumulation in the reference's order);
parameter gradients rel 1e-12 (fp64 reassociation only); first-step loss rel 1e-13; loss curve of a 12-step run within
1e-3 of the reference's (table gradients are fp32 atomics, Adam amplifies sign flips of near-zero gradients)."""
import os

import numpy as np
import pytest

import oracle
from closeness import assert_tables_match, sums_close

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


def test_mlp_matches_reference_fixture(sx, golden_neural):
    g = golden_neural
    mlp = sx.Mlp(sx.MlpConfig(32, 64, 2, 3))
    assert mlp.parameter_count() == 6467 == g["mlp_params"].size
    mlp.init_params(int(g["mlp_seed"]))
    assert np.array_equal(mlp.parameters().view(np.uint32), g["mlp_params"].view(np.uint32))  # Mlp::init_params
    assert not mlp.biases(1).any() and mlp.weights(0).size == 32 * 64
    out = mlp.forward(dev(g["mlp_in"]))
    assert np.array_equal(out.cpu().numpy().view(np.uint32), g["mlp_out"].view(np.uint32))
    ig = mlp.backward(dev(g["mlp_up"]))
    assert np.array_equal(ig.cpu().numpy(), g["mlp_input_grad"])
    grad = mlp.gradient()
    assert sums_close(grad, g["mlp_grad"], 1e-12)
    # gradient accumulates across calls (MlpGradient semantics) and clears
    mlp.forward(dev(g["mlp_in"]))
    mlp.backward(dev(g["mlp_up"]))
    assert sums_close(mlp.gradient(), 2 * g["mlp_grad"], 1e-12)
    mlp.clear_gradient()
    assert not mlp.gradient().any()
    ig32 = mlp.backward(dev(g["mlp_up"]), dtype=torch.float32)
    assert np.array_equal(ig32.cpu().numpy(), g["mlp_input_grad"].astype(np.float32))


@pytest.mark.parametrize("tag,shape", [("h0", (5, 7, 0, 2)), ("h1", (6, 9, 1, 1))])
def test_mlp_odd_shapes(sx, golden_neural, tag, shape):
    g = golden_neural
    mlp = sx.Mlp(sx.MlpConfig(*shape))
    mlp.init_params(11)
    assert np.array_equal(mlp.parameters(), g[f"mlp_{tag}_params"])
    out = mlp.forward(dev(g[f"mlp_{tag}_in"]))
    assert np.array_equal(out.cpu().numpy().view(np.uint32), g[f"mlp_{tag}_out"].view(np.uint32))
    ig = mlp.backward(dev(g[f"mlp_{tag}_up"]))
    assert np.array_equal(ig.cpu().numpy(), g[f"mlp_{tag}_input_grad"])
    assert sums_close(mlp.gradient(), g[f"mlp_{tag}_grad"], 1e-12)


def test_mlp_against_oracle_large_batch(sx, oracle_lib):
    mc = oracle.MlpConfig(32, 64, 2, 3)
    rng = np.random.default_rng(1)
    p = oracle_lib.mlp_init(mc, 5)
    p[-3:] = [0.1, -0.2, 0.3]  # non-zero biases
    inp = rng.standard_normal((3001, 32)).astype(np.float32) * 1e-2
    up = rng.standard_normal((3001, 3)) * 1e-4
    want, acts = oracle_lib.mlp_forward(mc, p, inp)
    wg, wig = oracle_lib.mlp_backward(mc, p, acts, up)
    mlp = sx.Mlp(sx.MlpConfig(32, 64, 2, 3))
    mlp.set_parameters(p)
    out = mlp.forward(dev(inp))
    assert np.array_equal(out.cpu().numpy().view(np.uint32), want.view(np.uint32))
    ig = mlp.backward(dev(up))
    assert np.array_equal(ig.cpu().numpy(), wig)
    assert sums_close(mlp.gradient(), wg, 1e-11)


@pytest.mark.parametrize("hidden,layers", [(1024, 2), (700, 1), (4096, 1)])
def test_wide_heads_train(sx, oracle_lib, hidden, layers):
    """MlpConfig::validate admits widths up to 2^14 (src/mlp.cpp:13) and the reference trains them; the exact backward
    shrinks its per-block sample tile until the layer fits shared memory (a 1024-wide head used to be created, run forward
    and then refuse its first training step).  Forward bit-exact, input gradient bit-exact, parameter gradient rel 1e-11."""
    mc = oracle.MlpConfig(8, hidden, layers, 2)
    rng = np.random.default_rng(hidden)
    p = oracle_lib.mlp_init(mc, 9)
    inp = rng.standard_normal((70, 8)).astype(np.float32) * 1e-1
    up = rng.standard_normal((70, 2)) * 1e-3
    want, acts = oracle_lib.mlp_forward(mc, p, inp)
    wg, wig = oracle_lib.mlp_backward(mc, p, acts, up)
    mlp = sx.Mlp(sx.MlpConfig(8, hidden, layers, 2))
    mlp.set_parameters(p)
    out = mlp.forward(dev(inp))
    assert np.array_equal(out.cpu().numpy().view(np.uint32), want.view(np.uint32))
    ig = mlp.backward(dev(up))
    assert np.array_equal(ig.cpu().numpy(), wig)
    assert sums_close(mlp.gradient(), wg, 1e-11)


def test_mlp_validation_and_errors(sx):
    # reference tests/test_neural.cpp: width validation, backward before forward
    for bad in ((0, 64, 2, 3), (32, 64, 2, 0), (32, 64, -1, 3), (32, 0, 1, 3), (1 << 15, 64, 2, 3)):
        with pytest.raises(ValueError):
            sx.MlpConfig(*bad).validate()
    sx.MlpConfig(32, 0, 0, 3).validate()  # hidden_width is irrelevant without hidden layers
    mlp = sx.Mlp(sx.MlpConfig(4, 8, 1, 2))
    with pytest.raises(RuntimeError, match="before forward"):  # std::logic_error
        mlp.backward(dev(np.zeros((3, 2))))
    with pytest.raises(ValueError):
        mlp.forward(dev(np.zeros((3, 5), dtype=np.float32)))
    mlp.forward(dev(np.zeros((3, 4), dtype=np.float32)))
    with pytest.raises(ValueError):
        mlp.backward(dev(np.zeros((3, 3))))
    with pytest.raises(ValueError):
        mlp.backward(dev(np.zeros((4, 2))))  # batch differs from the forward's
    with pytest.raises(ValueError):
        mlp.set_parameters(np.zeros(5))


def test_training_step_matches_reference_run(sx, oracle_lib, golden_neural):
    g = golden_neural
    c = g["train_cfg"]
    cfg = sx.EncoderConfig(dim=int(c[0]), levels=int(c[1]), table_size=int(c[2]), features=int(c[3]),
                           base_resolution=int(c[4]), growth=2.0)
    mc = sx.MlpConfig(*[int(v) for v in g["train_mlp"]])
    enc = sx.HashEncoder(cfg)
    enc.init_tables(42)
    mlp = sx.Mlp(mc)
    mlp.init_params(sx.hash_combine(42, 1))  # src/tasks.cpp:104-107
    coords, targets = g["train_coords"], g["train_targets"]
    steps, batch = coords.shape[0], coords.shape[1]

    def sampler(step, b):
        assert b == batch
        return dev(coords[step]), dev(targets[step])

    res = sx.train_field(enc, mlp, sampler, sx.TrainConfig(batch_size=batch, steps=steps, record_every=1))
    loss = np.array([v for _, v in res.loss_curve])
    ref = g["train_loss_t1"]
    assert res.steps_run == steps and len(loss) == steps
    assert abs(loss[0] - ref[0]) <= 1e-13 * ref[0]
    assert np.all(np.abs(loss - ref) <= 1e-3 * ref), (loss, ref)
    # the reference's own multi-worker run differs from its single-worker run by reassociation only; so must we
    assert np.all(np.abs(loss - g["train_loss_t3"]) <= 1e-3 * ref)
    tabs = np.stack([enc.table(l) for l in range(cfg.levels)])
    close = np.abs(tabs - g["train_tables_t1"]) <= 1e-6
    assert close.mean() >= 0.99, close.mean()
    assert np.abs(mlp.parameters() - g["train_mlp_params_t1"]).max() <= 1e-4
    # untouched rows never move (lazy Adam): every entry the reference left at its init value is at its init value here
    init = oracle_lib.init_tables(oracle.Config(dim=cfg.dim, levels=cfg.levels, table_size=cfg.table_size,
                                                features=cfg.features, base_resolution=cfg.base_resolution, growth=2.0), 42)
    untouched = g["train_tables_t1"] == init
    assert np.array_equal(tabs[untouched], init[untouched])


def test_training_errors(sx):
    cfg = sx.EncoderConfig(dim=2, levels=2, table_size=1 << 8, features=2, base_resolution=4, growth=2.0)
    enc = sx.HashEncoder(cfg)
    with pytest.raises(ValueError, match="MLP input width"):  # src/trainer.cpp:61-65
        sx.Trainer(enc, sx.Mlp(sx.MlpConfig(5, 8, 1, 1)))
    mlp = sx.Mlp(sx.MlpConfig(4, 8, 1, 1))
    mlp.init_params(1)
    enc.init_tables(1)
    tr = sx.Trainer(enc, mlp)
    x = dev(np.random.default_rng(0).random((32, 2)))
    t = dev(np.full((32, 1), np.nan))
    with pytest.raises(sx.TrainingError, match="non-finite"):  # src/trainer.cpp:121-123
        tr.step(x, t, sx.AdamConfig(1e-2), sx.AdamConfig(1e-3))
    with pytest.raises(ValueError):
        sx.train_field(enc, mlp, None, sx.TrainConfig(batch_size=8, steps=1))
    with pytest.raises(ValueError):
        sx.train_field(enc, mlp, lambda s, b: None, sx.TrainConfig(batch_size=0, steps=1))


def test_constant_target_converges(sx):
    # reference tests/test_neural.cpp:311-338: a constant field is learned quickly
    cfg = sx.EncoderConfig(dim=2, levels=4, table_size=1 << 10, features=2, base_resolution=4, growth=2.0)
    enc = sx.HashEncoder(cfg)
    enc.init_tables(42)
    mlp = sx.Mlp(sx.MlpConfig(8, 16, 2, 1))
    mlp.init_params(sx.hash_combine(42, 1))

    def sampler(step, b):
        x = torch.empty((b, 2), dtype=torch.float64, device="cuda:0")
        sx.CounterRng(1234, step).fill_device(x)
        return x, torch.full((b, 1), 0.7, dtype=torch.float64, device="cuda:0")

    res = sx.train_field(enc, mlp, sampler, sx.TrainConfig(batch_size=256, steps=300, record_every=50))
    assert res.loss_curve[0][1] > 0.1 and res.final_loss < 1e-3


def test_overlapped_distributed_step_on_one_rank_equals_the_plain_step(sx):
    """Trainer.distributed_step (level-chunked backward, gradient exchange on a second stream) through a 1-rank NCCL
    group must reproduce Trainer.step: same loss bits, same tables after the update.  (>1 GPU is not available to the
    tests; the chunking and the -0.0 algebra across ranks are covered on gloo in test_distributed_cpu.py.)"""
    import os
    import torch.distributed as dist
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ.setdefault("MASTER_PORT", "29631")
    created = False
    if not dist.is_initialized():
        dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda:0"))
        created = True
    try:
        cfg = sx.EncoderConfig(dim=3, levels=16, table_size=1 << 14, features=2, base_resolution=16, growth=1.5)
        N = 6000
        x = torch.rand((N, 3), dtype=torch.float32, device="cuda:0")
        tgt = torch.rand((N, 3), dtype=torch.float32, device="cuda:0")
        ta, ma = sx.AdamConfig(lr=1e-2), sx.AdamConfig(lr=1e-3)
        results = []
        for mode in ("plain", "overlapped"):
            enc = sx.HashEncoder(cfg)
            enc.init_tables(42)
            mlp = sx.Mlp(sx.MlpConfig(32, 64, 2, 3))
            mlp.init_params(sx.hash_combine(42, 1))
            tr = sx.Trainer(enc, mlp)
            losses = []
            for _ in range(3):
                if mode == "plain":
                    losses.append(tr.step(x, tgt, ta, ma))
                else:
                    losses.append(tr.distributed_step(x, tgt, ta, ma, level_chunks=4))
            torch.cuda.synchronize()
            results.append((losses, np.stack([enc.table(l) for l in range(16)]), mlp.parameters()))
        (l0, t0, p0), (l1, t1, p1) = results
        # same kernels on the same data; only the fp32 atomic order differs between runs
        assert np.allclose(l0, l1, rtol=1e-5), (l0, l1)   # (1e-5: room for the other branch of an Adam sign flip, tests/closeness.py)
        assert_tables_match(t0, t1, 2e-3 * 1e-2 + 1e-7)
        assert np.allclose(p0, p1, rtol=0, atol=1e-5)
        with pytest.raises(RuntimeError):  # std::logic_error
            tr.accumulate_tables(x[:100], 0, 16)  # no matching accumulate_head
    finally:
        if created:
            dist.destroy_process_group()


def test_training_with_aux_inputs_matches_reference_run(sx):
    """TrainConfig::aux_dims (src/trainer.cpp:32-35,59-65): pass-through inputs appended after the encoding.  Against the
    reference's own 12-step run with 2 aux inputs (tests/golden/aux_cases.npz, make_golden.py aux): first loss rel 1e-13,
    loss curve rel 1e-3, final tables / parameters close; the width rule and the missing-aux error as the reference's
    test (tests/test_neural.cpp:439-462)."""
    import os
    g = np.load(os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "aux_cases.npz"))
    c = g["cfg"]
    cfg = sx.EncoderConfig(dim=int(c[0]), levels=int(c[1]), table_size=int(c[2]), features=int(c[3]),
                           base_resolution=int(c[4]), growth=float(g["growth"]))
    aux_dims = int(g["aux_dims"])
    mc = sx.MlpConfig(*[int(v) for v in g["mlp"]])
    coords, aux, targets = g["coords"], g["aux"], g["targets"]
    steps, batch = coords.shape[0], coords.shape[1]

    def run(aux_dtype, per_step):
        enc = sx.HashEncoder(cfg)
        enc.init_tables(42)
        mlp = sx.Mlp(mc)
        mlp.init_params(sx.hash_combine(42, 1))
        if per_step:   # the per-step entry point
            tr = sx.Trainer(enc, mlp, aux_dims)
            loss = []
            for s in range(steps):
                tr.set_aux(dev(aux[s]).to(aux_dtype))
                loss.append(tr.step(dev(coords[s]), dev(targets[s]), sx.AdamConfig(lr=1e-2), sx.AdamConfig(lr=1e-3)))
            return enc, mlp, np.array(loss)

        def sampler(step, b):
            assert b == batch
            return dev(coords[step]), dev(aux[step]).to(aux_dtype), dev(targets[step])

        res = sx.train_field(enc, mlp, sampler, sx.TrainConfig(batch_size=batch, steps=steps, record_every=1,
                                                               aux_dims=aux_dims))
        return enc, mlp, np.array([v for _, v in res.loss_curve])

    ref = g["loss"]
    for aux_dtype, per_step in ((torch.float64, False), (torch.float64, True), (torch.float32, False)):
        enc, mlp, loss = run(aux_dtype, per_step)
        assert abs(loss[0] - ref[0]) <= 1e-13 * ref[0], (aux_dtype, per_step)   # aux is narrowed to float either way (:33)
        assert np.all(np.abs(loss - ref) <= 1e-3 * ref), (loss, ref)
        tabs = np.stack([enc.table(l) for l in range(cfg.levels)])
        assert (np.abs(tabs - g["tables"]) <= 1e-6).mean() >= 0.99
        assert np.abs(mlp.parameters() - g["mlp_params"]).max() <= 1e-4

    enc = sx.HashEncoder(cfg)
    mlp = sx.Mlp(mc)
    with pytest.raises(ValueError, match="encoded width"):
        sx.Trainer(enc, mlp)                       # aux_dims = 0: widths do not line up
    with pytest.raises(ValueError, match="encoded width"):
        sx.Trainer(enc, mlp, aux_dims + 1)
    with pytest.raises(ValueError):
        sx.Trainer(enc, mlp, -1)
    tr = sx.Trainer(enc, mlp, aux_dims)
    with pytest.raises(RuntimeError, match="no aux inputs"):
        tr.step(dev(coords[0]), dev(targets[0]), sx.AdamConfig(), sx.AdamConfig())
    with pytest.raises(ValueError):
        tr.set_aux(dev(aux[0][:, :1]))


def test_random_trainer_shapes_match_the_oracle(sx, oracle_lib):
    """Seeded fuzz of the gradient pass of one training step (run_chunk, src/trainer.cpp:20-49) over encoder and head
    shapes the fixed cases do not visit: dim 1..6, F in {1, 2, 4}, 1..3 hidden layers of odd widths, 1..4 outputs, ragged
    batches, a global batch larger than the local chunk (a rank's share).  Exact head: loss rel 1e-12, MLP gradients rel
    1e-9, table gradients within the fp32-atomics bar, touched sets exact."""
    rng = np.random.default_rng(77)
    for case in range(int(os.environ.get("SXEN_FUZZ_CASES", "24"))):
        n = int(rng.integers(1, 7))
        cfg = oracle.Config(dim=n, levels=int(rng.integers(1, 9)), table_size=1 << int(rng.integers(6, 13)),
                            features=int(rng.choice([1, 2, 2, 4])), base_resolution=int(rng.integers(2, 12)),
                            growth=float(rng.choice([1.3, 1.5, 2.0])), backend=int(rng.integers(0, 2)) if n <= 4 else 0)
        assert oracle_lib.validate(cfg) == 0
        layers = int(rng.integers(1, 4))
        mc = oracle.MlpConfig(cfg.encoded_width, int(rng.choice([8, 16, 33, 64])), layers, int(rng.integers(1, 5)))
        seed = int(rng.integers(1, 1 << 30))
        tables = oracle_lib.init_tables(cfg, seed)
        tables = (tables.astype(np.float64) * 2000.0).astype(np.float32)   # O(0.1) features: every layer's ReLU is exercised
        params = oracle_lib.mlp_init(mc, seed + 1)
        B = int(rng.integers(1, 300))
        global_batch = B + int(rng.integers(0, 3)) * 17
        x = rng.random((B, n))
        x[rng.random((B, n)) < 0.02] = 1.0
        tgt = rng.random((B, mc.output_width))
        loss, wtg, wtouched, wmg, _ = oracle_lib.train_grads(cfg, mc, tables, params, x, tgt, global_batch)
        enc = sx.HashEncoder(sx.EncoderConfig(dim=cfg.dim, levels=cfg.levels, table_size=cfg.table_size,
                                              features=cfg.features, base_resolution=cfg.base_resolution,
                                              growth=cfg.growth, backend=cfg.backend))
        for l in range(cfg.levels):
            enc.set_table(l, tables[l])
        mlp = sx.Mlp(sx.MlpConfig(mc.input_width, mc.hidden_width, mc.hidden_layers, mc.output_width))
        mlp.set_parameters(params)
        tr = sx.Trainer(enc, mlp)
        tr.accumulate(dev(x), dev(tgt), global_batch)
        tag = (case, cfg, mc, B, global_batch)
        # both divide this chunk's sum by (global_batch * out_w), as the reference does once all chunks are in (:120)
        got_loss = tr.loss(global_batch)
        assert abs(got_loss - loss) <= 1e-12 * abs(loss), tag
        assert sums_close(mlp.gradient(), wmg, 1e-9), tag
        g = tr.table_grad_device().cpu().numpy().reshape(cfg.levels, cfg.table_size, cfg.features)
        touched = (g[..., 0].view(np.uint32) != 0x80000000).astype(np.uint8)
        assert np.array_equal(touched, wtouched), tag
        vals = np.where(touched[..., None].astype(bool), g, 0.0)
        scale = np.abs(wtg).max() + 1e-30
        assert np.abs(vals - wtg).max() <= 2e-5 * scale, (tag, np.abs(vals - wtg).max() / scale)
