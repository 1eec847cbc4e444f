"""CPU: the bench-kernel mirror's host logic (include/sxen/analysis.hpp:56-75, src/analysis.cpp:122,243-257,340-372):
resolution choice, CSV schema and its round trip, rejections."""
import pytest

import paper_2311_15439_b200 as sx
from paper_2311_15439_b200.analysis import KERNEL_HEADER


def test_bench_side_is_the_largest_integer_root():
    for n in range(1, 9):
        for cells in (1, 2, 7, 8, 9, 1000, 2 ** 21, 2 ** 27, 10 ** 12 + 1):
            side = sx.bench_side(n, cells)
            assert side >= 1 and side ** n <= cells < (side + 1) ** n, (n, cells, side)
    # the reference's own protocol sizes: 2^27 cells
    assert [sx.bench_side(n, 1 << 27) for n in (2, 3, 4)] == [11585, 512, 107]


def test_kernel_csv_schema_round_trips_bit_exactly(tmp_path):
    rows = [sx.KernelBenchReport(n=3, backend=sx.Backend.simplex, cells=2 ** 21, samples=1024, reps=1000,
                                 seconds=0.1 + 0.2, vertices_per_sample=4.0),
            sx.KernelBenchReport(n=6, backend=sx.Backend.grid, cells=11390625, samples=7, reps=10,
                                 seconds=1.2345678901234567e-3, vertices_per_sample=64.0)]
    path = str(tmp_path / "kernel.csv")
    sx.write_kernel_csv(path, rows)
    text = open(path).read().split("\n")
    assert text[0] == KERNEL_HEADER == "n,backend,cells,samples,reps,seconds,vertices_per_sample"
    assert text[1].startswith("3,simplex,2097152,1024,1000,0.30000000000000004,4")
    assert sx.read_kernel_csv(path) == rows  # doubles written as %.17g come back bit-identical


def test_kernel_csv_rejections(tmp_path):
    p = tmp_path / "bad.csv"
    p.write_text("n,backend,cells\n")
    with pytest.raises(sx.IoError):
        sx.read_kernel_csv(str(p))
    p.write_text(KERNEL_HEADER + "\n3,simplex,8,1,1,0.5\n")
    with pytest.raises(sx.IoError):
        sx.read_kernel_csv(str(p))
    p.write_text(KERNEL_HEADER + "\n3,hexagonal,8,1,1,0.5,4\n")
    with pytest.raises(sx.IoError):
        sx.read_kernel_csv(str(p))
    with pytest.raises(sx.IoError):
        sx.read_kernel_csv(str(tmp_path / "missing.csv"))
    p.write_text("")
    with pytest.raises(sx.IoError):
        sx.read_kernel_csv(str(p))


def test_bench_kernel_argument_checks():
    for bad in (dict(n=0), dict(n=9), dict(cells=0), dict(samples=0), dict(reps=0)):
        with pytest.raises(ValueError):
            sx.bench_kernel(sx.KernelBenchConfig(**bad))
