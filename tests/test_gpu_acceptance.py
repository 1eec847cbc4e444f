"""GPU (-m gpu): the reference's acceptance criteria that concern the hot path (/root/reference/proj/tests/acceptance_main.cpp),
run on the device path with the reference's own configurations and pass conditions:

  vertex-count-scaling  (:243-280)  exactly (n+1) simplex vs 2^n grid vertices per lookup, n = 2..7, zero out-of-bounds
  kernel-scaling-trend  (:285-304)  grid / simplex time per lookup: >= 2.0 at n = 7 and larger than at n = 2
  roundtrip-safety      (:540-567)  zero out-of-bounds accesses over 10^6 encodes per n = 2..5, both backends, with coordinates
                                    forced to exactly 0.0 and 1.0 along the way; outputs finite
(image-fitting-parity: tests/test_gpu_tasks.py and tests/test_gpu_reproducible.py; gradient-integrity: tests/test_oracle_fd.py
pins the oracle, tests/test_gpu_neural.py and tests/test_gpu_fused_step.py compare the device path with it.)"""
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
