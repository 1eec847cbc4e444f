#!/usr/bin/env python
"""tools/chunk_sweep.py -- the chunked fused launch at configs[1] over block size and L2 eviction hints (CUDA events, rotating
inputs): is the library's choice (256 threads, reds evict_first) still the best shape once the levels are walked in ranges?"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2311_15439_b200 as sx  # noqa: E402

n, N, LF, L = 3, 1 << 20, 32, 16
cfg = sx.EncoderConfig(dim=n, levels=L, table_size=1 << 19, features=2, base_resolution=16, growth=1.5)
enc = sx.HashEncoder(cfg)
enc.init_tables(42)
grad = sx.EncoderGradient(enc)
sets = []
for i in range(4):
    x = torch.empty((N, n), dtype=torch.float32, device="cuda")
    r = sx.CounterRng(99, 1)
    r.counter = i * N * n
    r.fill_device(x)
    up = torch.empty((N, LF), dtype=torch.float32, device="cuda")
    r = sx.CounterRng(7, 2)
    r.counter = i * N * LF
    r.fill_device(up, -1e-3, 1e-3)
    sets.append((x, up, torch.empty((N, LF), dtype=torch.float32, device="cuda")))
stream = torch.cuda.current_stream()


def timeit(reps=20):
    def fn(i):
        x, up, out = sets[i % 4]
        enc.encode_forward_backward(x, up, grad, out=out)
    for i in range(3):
        fn(i)
    torch.cuda.synchronize()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(reps)]
    for i, (e0, e1) in enumerate(ev):
        e0.record(stream)
        fn(i)
        e1.record(stream)
    torch.cuda.synchronize()
    ms = sorted(e0.elapsed_time(e1) for e0, e1 in ev)
    return ms[len(ms) // 2]


best = None
for chunk in (8, -1):
    for block in (128, 256, 384, 512):
        for hints in (-1, 0, 8, 9, 4, 5, 12, 13):
            for replicas in (0,):
                enc.set_tuning(sx.Tuning(levels_per_thread=2, block_threads=block, level_major=0, exact_blend=1, level_chunk=chunk,
                                         cache_hints=hints, coarse_replicas=replicas))
                ms = timeit()
                tag = f"level_chunk {chunk:2d} block {block:3d} cache_hints {hints:2d}"
                print(f"{tag}: {ms:.4f} ms  frac {1816 * N / (ms * 1e-3) / 1e9 / 6552:.3f}", flush=True)
                if best is None or ms < best[0]:
                    best = (ms, tag)
print("best:", best)
enc.check()
