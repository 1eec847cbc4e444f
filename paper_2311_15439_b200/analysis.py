"""bench-kernel mirror (include/sxen/analysis.hpp:56-75, src/analysis.cpp:233-313,340-372) over the device encoder.

Same protocol as the reference's ``bench_kernel``: a single-level encoder whose resolution is the largest ``side`` with
``side**n <= cells``, ``samples`` points drawn from ``CounterRng(seed, 1)``, ``reps`` passes over them, setup outside the
timed region, touched vertices from the exact counters -- and the same CSV schema (``write_kernel_csv`` /
``read_kernel_csv``), so reports of the reference CLI and of this library can be concatenated for the n = 2..6 sweep.
Differences: one pass over the batch is ONE kernel launch, and the time is CUDA-event time on the launching stream."""
from __future__ import annotations

from dataclasses import dataclass
from typing import Iterable, List

from .encoding import Backend, EncoderConfig, HashEncoder, LevelScale
from .errors import IoError
from .rng import CounterRng

KERNEL_HEADER = "n,backend,cells,samples,reps,seconds,vertices_per_sample"  # src/analysis.cpp:122
MAX_DIM = 8


@dataclass
class KernelBenchConfig:  # include/sxen/analysis.hpp:56-65, same defaults
    n: int = 3
    cells: int = 1 << 21
    samples: int = 1 << 10
    reps: int = 1000
    backend: int = Backend.simplex
    table_size: int = 1 << 19
    features: int = 2
    seed: int = 99


@dataclass
class KernelBenchReport:  # include/sxen/analysis.hpp:20-29
    n: int = 0
    backend: int = Backend.simplex
    cells: int = 0
    samples: int = 0
    reps: int = 0
    seconds: float = 0.0
    vertices_per_sample: float = 0.0


def bench_side(n: int, cells: int) -> int:
    """Largest integer side with side**n <= cells (src/analysis.cpp:243-257), in exact integer arithmetic."""
    side = max(1, round(cells ** (1.0 / n)))
    while side ** n > cells:
        side -= 1
    while (side + 1) ** n <= cells:
        side += 1
    return side


def bench_kernel(cfg: KernelBenchConfig, device: int = 0) -> KernelBenchReport:
    import torch
    if cfg.n < 1 or cfg.n > MAX_DIM:
        raise ValueError(f"bench: n must be in [1, {MAX_DIM}]")
    if cfg.cells < 1:
        raise ValueError("bench: cells must be >= 1")
    if cfg.samples < 1 or cfg.reps < 1:
        raise ValueError("bench: samples and reps must be >= 1")
    side = bench_side(cfg.n, cfg.cells)
    ec = EncoderConfig(dim=cfg.n, levels=1, table_size=cfg.table_size, features=cfg.features, base_resolution=side,
                       growth=2.0, backend=cfg.backend, level_scale=LevelScale.raw)
    enc = HashEncoder(ec, device=device)
    enc.init_tables(cfg.seed)
    dev = torch.device(f"cuda:{device}")
    x = torch.empty((cfg.samples, cfg.n), dtype=torch.float64, device=dev)
    CounterRng(cfg.seed, 1).fill_device(x)  # src/analysis.cpp:269-271
    out = torch.empty((cfg.samples, ec.encoded_width()), dtype=torch.float32, device=dev)
    stream = torch.cuda.current_stream(dev)
    enc.encode(x, out=out)  # warm-up, outside the timed region
    reps = cfg.reps
    while True:
        enc.reset_counters()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(reps):
            enc.encode(x, out=out)
        e1.record(stream)
        e1.synchronize()
        seconds = e0.elapsed_time(e1) * 1e-3
        if not bool(torch.isfinite(out[:, 0].double().sum())):
            raise RuntimeError("bench: encode produced non-finite values")
        if seconds >= 1e-3:  # src/analysis.cpp:296-301: raise reps until the timer resolves
            break
        reps *= 10
    enc.check()
    lookups = reps * cfg.samples
    return KernelBenchReport(n=cfg.n, backend=cfg.backend, cells=side ** cfg.n, samples=cfg.samples, reps=reps,
                             seconds=seconds, vertices_per_sample=enc.counters().touched_vertices / lookups)


def _backend_name(b: int) -> str:
    return "simplex" if b == Backend.simplex else "grid"


def write_kernel_csv(path: str, rows: Iterable[KernelBenchReport]) -> None:
    """src/analysis.cpp:340-348: stable column order, doubles as %.17g (round-trip bit-exactly)."""
    lines = [KERNEL_HEADER]
    for r in rows:
        lines.append(f"{r.n},{_backend_name(r.backend)},{r.cells},{r.samples},{r.reps},{r.seconds:.17g},"
                     f"{r.vertices_per_sample:.17g}")
    try:
        with open(path, "w") as f:
            f.write("\n".join(lines) + "\n")
    except OSError as exc:
        raise IoError(f"cannot open '{path}' for writing") from exc


def read_kernel_csv(path: str) -> List[KernelBenchReport]:
    """src/analysis.cpp:350-372: rejects unknown headers, wrong column counts and unknown backends."""
    try:
        with open(path) as f:
            lines = f.read().split("\n")
    except OSError as exc:
        raise IoError(f"cannot open '{path}'") from exc
    if not lines or lines[0] == "" and len(lines) == 1:
        raise IoError(f"csv '{path}' is empty")
    if lines[0] != KERNEL_HEADER:
        raise IoError(f"csv '{path}' header mismatch: expected '{KERNEL_HEADER}', got '{lines[0]}'")
    out = []
    for line in lines[1:]:
        if not line:
            continue
        f = line.split(",")
        if len(f) != 7:
            raise IoError(f"csv '{path}': expected 7 columns")
        if f[1] not in ("simplex", "grid"):
            raise IoError(f"csv: unknown backend '{f[1]}'")
        try:
            out.append(KernelBenchReport(n=int(f[0]), backend=Backend.simplex if f[1] == "simplex" else Backend.grid,
                                         cells=int(f[2]), samples=int(f[3]), reps=int(f[4]), seconds=float(f[5]),
                                         vertices_per_sample=float(f[6])))
        except ValueError as exc:
            raise IoError(f"csv '{path}': malformed field") from exc
    return out
