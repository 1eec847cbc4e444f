#!/usr/bin/env python
"""tools/bench_kernel_sweep.py -- the paper's single-level kernel protocol (2^27 cells, n = 2..7,
simplex vs grid) through the bench-kernel mirror, written in the reference's CSV schema.

    python tools/bench_kernel_sweep.py [out.csv]

The reference times 2^10 points x 1000 reps on one CPU thread; here one rep is one launch over 2^20 points."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2311_15439_b200 as sx  # noqa: E402

out = sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/bench_kernel.csv"
rows = []
for backend in (sx.Backend.simplex, sx.Backend.grid):
    for n in range(2, 8):
        r = sx.bench_kernel(sx.KernelBenchConfig(n=n, cells=1 << 27, samples=1 << 20, reps=20, backend=backend,
                                                 table_size=1 << 19, features=2, seed=99))
        rows.append(r)
        print(f"n={n} {'simplex' if backend == sx.Backend.simplex else 'grid':7s} cells={r.cells} "
              f"{r.seconds / r.reps * 1e6:9.1f} us per 2^20 lookups = {r.samples * r.reps / r.seconds / 1e9:7.3f} G lookups/s, "
              f"{r.vertices_per_sample:.0f} vertices/lookup", flush=True)
os.makedirs(os.path.dirname(out) or ".", exist_ok=True)
sx.write_kernel_csv(out, rows)
print("grid/simplex time per lookup, n = 2..7:",
      [round((rows[6 + i].seconds / rows[6 + i].reps) / (rows[i].seconds / rows[i].reps), 2) for i in range(6)])
