#!/usr/bin/env python
"""tools/level_drop.py -- upper bound of privatising the coarse levels: time the fused/fwd/bwd launches of the BASELINE
ladder with its first k levels removed (k = 0..4), and pinned-memory PCIe bandwidth (one way and both ways at once)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2311_15439_b200 as sx  # noqa: E402

n = 3
N = 1 << 20
ladder = [16, 24, 36, 54, 81, 121, 182, 273, 410, 615, 922, 1383, 2075, 3113, 4670, 7006]
xs = []
for i in range(4):
    x = torch.empty((N, n), dtype=torch.float32, device="cuda")
    r = sx.CounterRng(99, 1)
    r.counter = i * N * n
    r.fill_device(x)
    xs.append(x)
print("levels  fwd_us  bwd_us  fused_us")
for k in range(0, 5):
    Lk = 16 - k
    cfg = sx.EncoderConfig(dim=n, levels=Lk, table_size=1 << 19, features=2, base_resolution=ladder[k], growth=1.5)
    enc = sx.HashEncoder(cfg)
    enc.init_tables(1)
    grad = sx.EncoderGradient(enc)
    ups = [torch.rand((N, 2 * Lk), dtype=torch.float32, device="cuda") * 1e-3 for _ in range(4)]
    outs = [torch.empty((N, 2 * Lk), dtype=torch.float32, device="cuda") for _ in range(4)]
    enc.set_tuning(sx.Tuning(levels_per_thread=2))
    res_t = []
    for which in ("fwd", "bwd", "fused"):
        fn = {"fwd": lambda i: enc.encode(xs[i % 4], out=outs[i % 4]), "bwd": lambda i: enc.encode_backward(xs[i % 4], ups[i % 4], grad),
              "fused": lambda i: enc.encode_forward_backward(xs[i % 4], ups[i % 4], grad, out=outs[i % 4])}[which]
        for i in range(3):
            fn(i)
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for i in range(12):
            fn(i)
        b.record()
        torch.cuda.synchronize()
        res_t.append(a.elapsed_time(b) / 12 * 1e3)
    print(f"{Lk:4d} (res>={ladder[k]:3d}) {res_t[0]:7.1f} {res_t[1]:7.1f} {res_t[2]:7.1f}", flush=True)
    del enc, grad, ups, outs

# PCIe
nb = 256 << 20
h1 = torch.empty(nb, dtype=torch.uint8, pin_memory=True)
h2 = torch.empty(nb, dtype=torch.uint8, pin_memory=True)
d1 = torch.empty(nb, dtype=torch.uint8, device="cuda")
d2 = torch.empty(nb, dtype=torch.uint8, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
def t(fn, reps=5):
    fn(); torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    torch.cuda.synchronize()
    b.record(); torch.cuda.synchronize()
    return a.elapsed_time(b) / reps
ms = t(lambda: d1.copy_(h1, non_blocking=True)); print(f"H2D {nb / ms / 1e6:.1f} GB/s")
ms = t(lambda: h2.copy_(d2, non_blocking=True)); print(f"D2H {nb / ms / 1e6:.1f} GB/s")
def both():
    with torch.cuda.stream(s1):
        d1.copy_(h1, non_blocking=True)
    with torch.cuda.stream(s2):
        h2.copy_(d2, non_blocking=True)
ms = t(both); print(f"H2D+D2H concurrently: {nb / ms / 1e6:.1f} GB/s each way")
