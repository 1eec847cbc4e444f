#!/usr/bin/env python
"""tools/fused_step_bench.py -- the training step's gradient pass as ONE kernel (csrc/sxen_train_fused.cu) against the three
kernels it replaces (encode | tcgen05 head | encode_backward), CUDA events, rotating coordinate sets; then the whole step
(+ sparse Adam + Adam) queued.

    python tools/fused_step_bench.py [--dim 3] [--log2n 20] [--reps 20] [--once]"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2311_15439_b200 as sx  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--dim", type=int, default=3)
ap.add_argument("--log2n", type=int, default=20)
ap.add_argument("--log2t", type=int, default=19)
ap.add_argument("--reps", type=int, default=20)
ap.add_argument("--once", action="store_true", help="one fused accumulate after a warm-up (for ncu)")
a = ap.parse_args()
n, N = a.dim, 1 << a.log2n
cfg = sx.EncoderConfig(dim=n, levels=16, table_size=1 << a.log2t, features=2, base_resolution=16, growth={2: 2.0, 3: 1.5}[n])
xs = []
for i in range(4):
    x = torch.empty((N, n), dtype=torch.float32, device="cuda")
    r = sx.CounterRng(99, 1)
    r.counter = i * N * n
    r.fill_device(x)
    xs.append(x)
tgt = torch.rand((N, 3), dtype=torch.float32, device="cuda")
ta, ma = sx.AdamConfig(lr=1e-2), sx.AdamConfig(lr=1e-3)
stream = torch.cuda.current_stream()


def timeit(fn, reps):
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
    return ms[len(ms) // 2], ms[0]


for fused in ((1,) if a.once else (0, 1)):
    enc = sx.HashEncoder(cfg)
    enc.init_tables(42)
    mlp = sx.Mlp(sx.MlpConfig(32, 64, 2, 3))
    mlp.init_params(sx.hash_combine(42, 1))
    mlp.set_precision(1)
    tr = sx.Trainer(enc, mlp)
    tr.set_fused(fused)
    if a.once:
        tr.accumulate(xs[0], tgt, N)
        torch.cuda.synchronize()
        tr.accumulate(xs[1], tgt, N)
        torch.cuda.synchronize()
        print("fused accumulate done")
        break
    med, best = timeit(lambda i: tr.accumulate(xs[i % 4], tgt, N), a.reps)
    name = "ONE fused kernel      " if fused else "three kernels (unfused)"
    print(f"gradient pass, {name}: median {med:.4f} ms  best {best:.4f} ms  = {N / med / 1e6:.3f} G samples/s", flush=True)
    tr.update(ta, ma)

    def step(i):
        tr.step_enqueue(xs[i % 4], tgt, ta, ma)

    med, best = timeit(step, a.reps)
    losses, failed = tr.collect()
    print(f"whole step (+ Adam),  {name}: median {med:.4f} ms  best {best:.4f} ms  = {N / med / 1e6:.3f} G samples/s; "
          f"loss {losses[0]:.5f} -> {losses[-1]:.5f}", flush=True)

# ---- where the roles of the fused kernel spend their cycles (sxen_debug_fused_timing: 16 device counters)
import ctypes as C  # noqa: E402
fn = getattr(sx.lib, "sxen_debug_fused_timing", None)
if fn is not None and not a.once:
    fn.restype = C.c_int
    counters = torch.zeros(16, dtype=torch.int64, device="cuda")
    fn(C.c_void_p(counters.data_ptr()))
    enc = sx.HashEncoder(cfg)
    enc.init_tables(42)
    mlp = sx.Mlp(sx.MlpConfig(32, 64, 2, 3))
    mlp.init_params(sx.hash_combine(42, 1))
    mlp.set_precision(1)
    tr = sx.Trainer(enc, mlp)
    tr.set_fused(1)
    tr.accumulate(xs[0], tgt, N)
    torch.cuda.synchronize()
    counters.zero_()
    tr.accumulate(xs[1], tgt, N)
    torch.cuda.synchronize()
    fn(None)
    c = counters.cpu().numpy().astype(float)
    ctas = min(148, (N + 127) // 128)
    tiles = (N + 127) // 128 / ctas
    names = [("gather", ["x0_empty"]), ("scatter", ["dx_full"]), ("chain-MMA", ["x0_full", "bar_ready", "dx_empty"]),
             ("epilogue", ["chain commits", "layer-1 commit", "wgrad commit"])]
    for r, (name, waits) in enumerate(names):
        total = c[4 * r] / ctas
        line = f"{name:10s}: {total / tiles:9.0f} cycles per tile in the loop"
        for i, wname in enumerate(waits):
            line += f"; waiting on {wname} {c[4 * r + 1 + i] / ctas / tiles:8.0f}"
        print(line, flush=True)
