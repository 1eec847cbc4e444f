"""CPU: the oracle's analytic gradients against central finite differences of its own loss -- the reference's gradient
integrity checks (tests/test_encoding.cpp:437-480: encode_backward vs FD; tests/test_neural.cpp:192-228: MLP FD at 1e-3;
tests/acceptance_main.cpp:400-509: 20 random parameters of the full pipeline, rel 1e-3).  The GPU tests compare the device
path with these analytic gradients; this test pins the gradients themselves."""
import numpy as np
import pytest

import oracle

FD_RTOL = 1e-3   # the reference's bar (acceptance_main.cpp:489-505)


@pytest.mark.parametrize("dim,backend", [(2, oracle.BACKEND_SIMPLEX), (3, oracle.BACKEND_SIMPLEX), (2, oracle.BACKEND_GRID)])
def test_pipeline_gradients_match_finite_differences(oracle_lib, dim, backend):
    cfg = oracle.Config(dim=dim, levels=4, table_size=1 << 8, features=2, base_resolution=4, growth=1.8, backend=backend)
    mc = oracle.MlpConfig(cfg.encoded_width, 8, 2, 2)
    rng = np.random.default_rng(11 + dim)
    tables = (rng.standard_normal((cfg.levels, cfg.table_size, cfg.features)) * 0.3).astype(np.float32)
    params = oracle_lib.mlp_init(mc, 5)
    params[-2:] = [0.2, -0.1]
    n = 64
    coords = rng.random((n, dim))
    targets = rng.random((n, 2))

    # An independent double-precision pipeline (the reference's own device for this check, acceptance_main.cpp:360-399: no float
    # activations, so differences of the loss are clean): vertex chains from the oracle's lookup, blend, MLP, MSE -- all numpy f64.
    idx, w = oracle_lib.encode_debug(cfg, coords)[:2]

    def loss(tb, pr):
        tb = tb.astype(np.float64)
        feats = np.zeros((n, cfg.levels, cfg.features))
        for l in range(cfg.levels):
            feats[:, l, :] = (w[:, l, :, None] * tb[l][idx[:, l, :]]).sum(axis=1)
        hcur = feats.reshape(n, -1)
        pr = pr.astype(np.float64)
        off = 0
        for layer in range(mc.layer_count):
            i_w, o_w = mc.layer_in(layer), mc.layer_out(layer)
            W = pr[off:off + o_w * i_w].reshape(o_w, i_w)
            off += o_w * i_w
            b = pr[off:off + o_w]
            off += o_w
            hcur = hcur @ W.T + b
            if layer + 1 < mc.layer_count:
                hcur = np.maximum(hcur, 0.0)
        return float(((hcur - targets) ** 2).sum() / (n * mc.output_width))     # src/trainer.cpp:118-120

    base, tg, touched, mg, _ = oracle_lib.train_grads(cfg, mc, tables, params, coords, targets)
    assert abs(loss(tables, params) - base) <= 1e-6 * base        # the two pipelines agree on the loss itself (float activations)
    rows = np.argwhere(touched)
    picks = rows[rng.choice(len(rows), size=12, replace=False)]
    h = 1e-6   # in double: far below any ReLU kink's reach, far above rounding

    def fd_of(perturb):
        return (loss(*perturb(+h)) - loss(*perturb(-h))) / (2 * h)

    for l, r in picks:   # 12 table entries the batch touched
        f = int(rng.integers(cfg.features))

        def perturb(d, l=l, r=r, f=f):
            tb = tables.astype(np.float64)
            tb[l, r, f] += d
            return tb, params
        fd = fd_of(perturb)
        assert abs(fd - tg[l, r, f]) <= FD_RTOL * max(abs(tg[l, r, f]), 1e-6) + 1e-9, (l, r, f, fd, tg[l, r, f])
    for i in rng.choice(params.size, size=8, replace=False):   # 8 MLP parameters

        def perturb(d, i=i):
            pr = params.astype(np.float64)
            pr[i] += d
            return tables, pr
        fd = fd_of(perturb)
        assert abs(fd - mg[i]) <= FD_RTOL * max(abs(mg[i]), 1e-6) + 1e-9, (i, fd, mg[i])
    # untouched rows have exactly zero gradient and stay untouched (lazy Adam relies on it, src/optimizer.cpp:68-81)
    assert not tg[~touched.astype(bool)].any()
