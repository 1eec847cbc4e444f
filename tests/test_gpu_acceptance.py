"""GPU (-m gpu): the reference's acceptance criteria that concern the hot path (/root/reference/proj/tests/acceptance_main.cpp),
run on the device path with the reference's own configurations and pass conditions:

  vertex-count-scaling  (:243-280)  exactly (n+1) simplex vs 2^n grid vertices per lookup, n = 2..7, zero out-of-bounds
  kernel-scaling-trend  (:285-304)  grid / simplex time per lookup: >= 2.0 at n = 7 and larger than at n = 2
  roundtrip-safety      (:540-567)  zero out-of-bounds accesses over 10^6 encodes per n = 2..5, both backends, with coordinates
                                    forced to exactly 0.0 and 1.0 along the way; outputs finite
  gradient-integrity    (:345-509)  analytic backward of the whole pipeline (encoder -> MLP -> MSE) against central finite
                                    differences on 20 random parameters, rel 1e-3; the difference quotient goes through an
                                    independent double-precision pipeline (tests/independent.py) reading the live parameters
(image-fitting-parity: tests/test_gpu_tasks.py and tests/test_gpu_reproducible.py; tests/test_oracle_fd.py runs
gradient-integrity on the oracle as well.)"""
import numpy as np
import pytest

from independent import encode_simplex_level, mlp_forward

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def sx():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2311_15439_b200 as pkg
    return pkg


def test_vertex_count_scaling(sx):
    points, levels = 64, 3
    for n in range(2, 8):
        for backend in (sx.Backend.simplex, sx.Backend.grid):
            enc = sx.HashEncoder(sx.EncoderConfig(dim=n, levels=levels, table_size=1 << 12, features=2, base_resolution=4,
                                                  backend=backend))
            enc.init_tables(1)
            x = torch.empty((points, n), dtype=torch.float64, device="cuda")
            sx.CounterRng(7700 + n).fill_device(x)
            enc.encode(x)
            got = enc.counters()
            per_lookup = n + 1 if backend == sx.Backend.simplex else 1 << n
            assert got.touched_vertices == points * levels * per_lookup and got.out_of_bounds == 0, (n, backend)


def test_kernel_scaling_trend(sx):
    def per_lookup_seconds(n, backend):
        r = sx.bench_kernel(sx.KernelBenchConfig(n=n, cells=1 << 21, samples=1 << 10, reps=1000, backend=backend,
                                                 table_size=1 << 19, features=2, seed=99))
        return r.seconds / (r.reps * r.samples)
    # (1024 samples per launch is far below what fills a B200; the protocol is the reference's, the trend is what is asserted)
    ratio2 = per_lookup_seconds(2, sx.Backend.grid) / per_lookup_seconds(2, sx.Backend.simplex)
    ratio7 = per_lookup_seconds(7, sx.Backend.grid) / per_lookup_seconds(7, sx.Backend.simplex)
    print(f"grid/simplex time per lookup: n=2 -> {ratio2:.3f}, n=7 -> {ratio7:.3f}")
    assert ratio7 >= 2.0 and ratio7 > ratio2


def test_roundtrip_safety(sx):
    N = 1_000_000
    for n in range(2, 6):
        for backend in (sx.Backend.simplex, sx.Backend.grid):
            enc = sx.HashEncoder(sx.EncoderConfig(dim=n, levels=4, table_size=1 << 14, features=2, base_resolution=16,
                                                  growth=1.5, backend=backend))
            enc.init_tables(3)
            gen = torch.Generator(device="cuda").manual_seed(31337 + n)
            x = torch.rand((N, n), dtype=torch.float64, device="cuda", generator=gen)
            k = torch.arange(N, device="cuda")
            axis = torch.randint(0, n, (N,), device="cuda", generator=gen)
            ones, zeros = (k % 97 == 0), (k % 101 == 0)
            x[ones, axis[ones]] = 1.0
            axis2 = torch.randint(0, n, (N,), device="cuda", generator=gen)
            x[zeros, axis2[zeros]] = 0.0
            out = enc.encode(x)
            enc.check()
            assert enc.counters().out_of_bounds == 0, (n, backend)
            assert bool(torch.isfinite(out).all())


def test_gradient_integrity(sx):
    ec = sx.EncoderConfig(dim=2, levels=2, table_size=64, features=2, base_resolution=4)
    enc = sx.HashEncoder(ec)
    T, F, L = ec.table_size, ec.features, ec.levels

    def draws(seed, count, lo=0.0, hi=1.0):
        t = torch.empty(count, dtype=torch.float64, device="cuda")
        sx.CounterRng(seed).fill_device(t, lo, hi)
        return t.cpu().numpy()

    # a generic operating point: tables at activation scale, biases off zero (away from the ReLU kinks, :352-360)
    tables = draws(96, L * T * F, -0.5, 0.5).astype(np.float32).reshape(L, T * F)
    for l in range(L):
        enc.set_table(l, tables[l])
    mc = sx.MlpConfig(ec.encoded_width(), 16, 2, 1)
    mlp = sx.Mlp(mc)
    mlp.init_params(sx.hash_combine(314, 1))
    params = mlp.parameters()
    bias_draws, pos, off = draws(97, 16 + 16 + 1, -0.25, 0.25), 0, 0
    spans = []                                           # (weights slice, bias slice) per layer
    for l in range(mc.layer_count()):
        i, o = mc.layer_input_width(l), mc.layer_output_width(l)
        params[off + i * o:off + i * o + o] += bias_draws[pos:pos + o].astype(np.float32)
        spans.append((slice(off, off + i * o), slice(off + i * o, off + i * o + o), o, i))
        pos, off = pos + o, off + i * o + o
    mlp.set_parameters(params)
    B = 8
    u = draws(2718, 3 * B).reshape(B, 3)
    points, targets = np.ascontiguousarray(u[:, :2]), -0.5 + u[:, 2:3]

    # analytic gradient of the mean squared error over the fixed batch, on the device
    trainer = sx.Trainer(enc, mlp)
    trainer.accumulate(torch.as_tensor(points, device="cuda"), torch.as_tensor(targets, device="cuda"), B)
    torch.cuda.synchronize()
    tgrad = trainer.table_grad_device().cpu().numpy().astype(np.float64).reshape(L, T * F)
    mgrad = mlp.gradient()

    def reference_loss(tab, par):
        feat = np.concatenate([encode_simplex_level(2, enc.resolution(l), T, F, tab[l], points) for l in range(L)], axis=1)
        ws = [par[w].reshape(o, i) for w, _, o, i in spans]
        bs = [par[b] for _, b, _, _ in spans]
        e = mlp_forward(mc, ws, bs, feat)[:, 0] - targets[:, 0]
        return float((e * e).sum() / B)

    candidates = [("t", l, k, tgrad[l, k]) for l in range(L) for k in range(T * F) if abs(tgrad[l, k]) > 1e-6]
    candidates += [("m", 0, k, mgrad[k]) for k in range(mgrad.size) if abs(mgrad[k]) > 1e-6]
    assert len(candidates) >= 20
    order = np.random.default_rng(424242).permutation(len(candidates))
    worst, kinds = 0.0, set()
    for ci in order[:20]:
        kind, l, k, analytic = candidates[ci]
        tab, par = tables.copy(), params.copy()
        arr = tab[l] if kind == "t" else par
        orig = arr[k]
        arr[k] = orig + np.float32(1e-3)
        up, loss_up = float(arr[k]), reference_loss(tab, par)
        arr[k] = orig - np.float32(1e-3)
        down, loss_down = float(arr[k]), reference_loss(tab, par)
        fd = (loss_up - loss_down) / (up - down)
        worst = max(worst, abs(fd - analytic) / abs(analytic))
        kinds.add(kind)
    print(f"gradient-integrity on the device: 20 parameters, max relative error {worst:.3g} (tolerance 1e-3)")
    assert worst <= 1e-3 and kinds == {"t", "m"}
