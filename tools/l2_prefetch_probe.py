#!/usr/bin/env python
"""tools/l2_prefetch_probe.py -- would a SEQUENTIAL pre-read of a level's table / accumulator slice into L2 pay at T = 2^22?
There every random 8-byte gather or red that misses L2 costs a 32-byte DRAM sector at random-access efficiency; a streaming
read of the same 32 MiB moves at full HBM bandwidth and the random accesses that follow hit L2.  Emulated here with a torch
reduction over the slice before each level range's launch (the library kernels unchanged)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2311_15439_b200 as sx  # noqa: E402

n, N, LF, L, T = 3, 1 << 20, 32, 16, 1 << 22
cfg = sx.EncoderConfig(dim=n, levels=L, table_size=T, features=2, base_resolution=16, growth=1.5)
enc = sx.HashEncoder(cfg)
enc.init_tables(42)
grad = sx.EncoderGradient(enc)
tables = enc.tables_device().view(L, T * 2)
gview = grad.device_view().view(L, T * 2)
sets = []
for i in range(3):
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
sink = torch.zeros(1, device="cuda")


def timeit(fn, reps=8):
    for i in range(2):
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


def run(count, touch_tables, touch_grads, mode):
    def fn(i):
        x, up, out = sets[i % 3]
        for first in range(0, L, count):
            if touch_tables and mode != "bwd":
                sink.add_(tables[first:first + count].sum())
            if touch_grads and mode != "fwd":
                sink.add_(gview[first:first + count].sum())
            if mode == "bwd":
                enc.encode_backward(x, up, grad, levels=(first, count))
            else:
                enc.encode_forward_backward(x, up, grad, out=out, levels=(first, count))
    return fn


touch_only = timeit(lambda i: sink.add_(tables.sum()))
print(f"streaming read of all tables (512 MiB) with torch.sum: {touch_only:.4f} ms", flush=True)
for mode in ("bwd", "both"):
    for count in (16, 4, 2, 1):
        base = timeit(run(count, False, False, mode))
        tt = timeit(run(count, True, True, mode))
        print(f"{mode:4s} level ranges of {count:2d}: plain {base:.4f} ms   with sequential pre-read {tt:.4f} ms "
              f"(pre-read alone costs ~{touch_only * (1 if mode == 'bwd' else 2):.3f} ms)", flush=True)
enc.check()
