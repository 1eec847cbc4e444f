"""GPU (-m gpu): BASELINE configs[3] AT ITS STATED SIZE -- NeRF-style dense sampling: 3D simplex encode (L=16 F=2 T=2^19,
base 16, growth 1.5) + the 64-wide tcgen05 head (32 -> 64 -> 64 -> 3, split bf16), 2^24 samples in ONE training-step
accumulation (run_chunk over the whole batch, /root/reference/proj/src/trainer.cpp:20-49, merged as :101-128).

The CPU oracle cannot run 2^24 samples in seconds, so the size itself is held by size-independent properties and the
arithmetic by an oracle spot check inside the same normalisation:
  * additivity over the reference's worker chunks: one 2^24-sample accumulation == sixteen 2^20-sample accumulations with
    the same global batch (what `train_field`'s workers / the sharded step's ranks each contribute): same touched rows,
    table gradients within the fp32 order-of-atomics bar, MLP gradients and loss sum alike;
  * a 4096-sample slice of the same batch, accumulated alone with global_batch = 2^24, against the oracle's
    encode -> mlp_forward -> MSE upstream -> mlp_backward -> encode_backward chain: features bit-exact, loss within the
    tensor-core head's bar, touched rows exact, table gradients within the head's bar (ReLU-flip stragglers bounded as in
    tests/test_gpu_tc.py);
  * the step that follows is applied and lowers the loss on the same batch."""
import numpy as np
import pytest

import oracle

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

TC3_RTOL = 1.5e-5        # the head's bar, tests/test_gpu_tc.py
ORDER_RTOL = 1e-5        # two runs of the same fp32 atomics in another order, relative to the level's largest entry
                         # (measured 7e-8 .. 1.3e-6 per level, profiles/r2s4_config4_margins.log)
UNTOUCHED = np.int32(-2147483648)  # bit pattern of -0.0f, the accumulator's "row not touched" marker
N = 1 << 24
CHUNK = 1 << 20


@pytest.fixture(scope="module")
def sx():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2311_15439_b200 as pkg
    return pkg


def make(sx):
    cfg = sx.EncoderConfig(dim=3, levels=16, table_size=1 << 19, features=2, base_resolution=16, growth=1.5)
    enc = sx.HashEncoder(cfg)
    enc.init_tables(42)
    mlp = sx.Mlp(sx.MlpConfig(32, 64, 2, 3))
    mlp.init_params(sx.hash_combine(42, 1))
    mlp.set_precision(1)
    return enc, mlp


def batch(sx):
    x = torch.empty((N, 3), dtype=torch.float32, device="cuda:0")
    sx.CounterRng(99, 1).fill_device(x)
    # the procedural radiance-like target of tools/config_runs.py (C4), evaluated on the device
    tgt = torch.stack([0.5 + 0.5 * torch.sin(40 * x[:, 0]) * torch.cos(31 * x[:, 1]), x[:, 0] * x[:, 2],
                       0.5 + 0.5 * torch.cos(57 * x[:, 2])], dim=1).contiguous()
    return x, tgt


def accumulated(sx, enc, mlp, x, tgt, pieces):
    """Table-gradient accumulator [L, T*F] (host), MLP gradient, loss -- of the given sample ranges under global batch N."""
    mlp.clear_gradient()
    tr = sx.Trainer(enc, mlp)
    for b, e in pieces:
        tr.accumulate(x[b:e], tgt[b:e], N)
    loss = tr.loss(N)
    g = tr.table_grad_device().clone().cpu().numpy().reshape(16, -1)
    m = mlp.gradient().copy()
    del tr
    return g, m, loss


def test_config4_accumulation_is_additive_over_worker_chunks_and_matches_the_oracle(sx, oracle_lib):
    enc, mlp = make(sx)
    x, tgt = batch(sx)
    g1, m1, loss1 = accumulated(sx, enc, mlp, x, tgt, [(0, N)])
    g16, m16, loss16 = accumulated(sx, enc, mlp, x, tgt, [(c * CHUNK, (c + 1) * CHUNK) for c in range(N // CHUNK)])
    assert np.isfinite(loss1) and 0.0 < loss1 < 1.0
    assert abs(loss1 - loss16) <= 1e-12 * loss1, (loss1, loss16)      # the same per-sample errors, fp64 sums (measured 8e-16)
    t1, t16 = g1.view(np.int32) != UNTOUCHED, g16.view(np.int32) != UNTOUCHED
    assert np.array_equal(t1, t16)
    assert t1[15].mean() > 0.99 and t1[0].sum() <= 2 * 17 ** 3        # fine levels: every row hit; level 0: its 17^3 vertices
    for l in range(16):
        d = np.abs(g1[l] - g16[l]).max()
        assert d <= ORDER_RTOL * np.abs(g1[l]).max(), (l, d, np.abs(g1[l]).max())
    assert np.abs(m1 - m16).max() <= 2e-5 * np.abs(m1).max(), np.abs(m1 - m16).max() / np.abs(m1).max()   # measured 1.8e-6

    # ---- oracle spot check: 4096 samples from the middle of the batch, alone, under the same normalisation
    b, n = 7 * CHUNK + 12345, 4096
    gs, ms, loss_s = accumulated(sx, enc, mlp, x, tgt, [(b, b + n)])
    ocfg = oracle.Config(dim=3, levels=16, table_size=1 << 19, features=2, base_resolution=16, growth=1.5)
    mc = oracle.MlpConfig(32, 64, 2, 3)
    xs = x[b:b + n].cpu().numpy().astype(np.float64)
    ts = tgt[b:b + n].cpu().numpy().astype(np.float64)
    tables = oracle_lib.init_tables(ocfg, 42)
    feats, bad = oracle_lib.encode(ocfg, tables, xs)
    assert bad == -1
    assert np.array_equal(enc.encode(x[b:b + n]).cpu().numpy().view(np.uint32), feats.view(np.uint32))
    params = mlp.parameters()
    pred, acts = oracle_lib.mlp_forward(mc, params, feats)
    err = pred.astype(np.float64) - ts
    want_loss = (err ** 2).sum() / (N * 3.0)
    assert abs(loss_s - want_loss) <= 10 * TC3_RTOL * want_loss, (loss_s, want_loss)
    up = 2.0 * err / (N * 3.0)                                         # src/trainer.cpp:26-27,40-43
    wg, wig = oracle_lib.mlp_backward(mc, params, acts, up)
    og, ot, _ = oracle_lib.encode_backward(ocfg, xs, wig)
    og = np.asarray(og, dtype=np.float64).reshape(16, -1)
    touched = (gs.view(np.int32) != UNTOUCHED).reshape(16, -1, 2).any(axis=2)
    assert np.array_equal(touched, np.asarray(ot).reshape(16, -1).astype(bool))
    bar = 4 * TC3_RTOL * np.abs(wig).max()                            # per contribution (weights <= 1), tests/test_gpu_tc.py
    for l in range(16):
        d = np.abs(np.where(gs[l].view(np.int32) == UNTOUCHED, 0.0, gs[l]) - og[l])
        off = d > 4 * max(bar, 4 * TC3_RTOL * np.abs(og[l]).max())     # (coarse rows add a handful of contributions)
        # a ReLU flip moves one sample's whole input gradient (tests/test_gpu_tc.py): few samples, hence few rows
        assert off.mean() <= 1e-2 * touched[l].mean() + 1e-6, (l, off.mean(), d.max(), np.abs(og[l]).max())
    assert np.abs(ms - wg).max() <= 5e-3 * np.abs(wg).max()            # sanity only: the bars are tests/test_gpu_tc.py's

    # ---- and the step is applied: two whole steps on the batch, the second one starts lower
    mlp.clear_gradient()
    tr = sx.Trainer(enc, mlp)
    ta, ma = sx.AdamConfig(lr=1e-2), sx.AdamConfig(lr=1e-3)
    la = tr.step(x, tgt, ta, ma)
    lb = tr.step(x, tgt, ta, ma)
    assert abs(la - loss1) <= 1e-7 * loss1 and lb < la, (loss1, la, lb)
