#!/usr/bin/env python
"""tools/hints.py -- cache-policy knobs on the fused / fwd / bwd launches (sxen_tuning.cache_hints)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2311_15439_b200 as sx  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 3
log2t = int(sys.argv[2]) if len(sys.argv) > 2 else 19
lpt = int(sys.argv[3]) if len(sys.argv) > 3 else 2
lm = int(sys.argv[4]) if len(sys.argv) > 4 else -1
N = 1 << 20
growth = 2.0 if n == 2 else 1.5
cfg = sx.EncoderConfig(dim=n, levels=16, table_size=1 << log2t, features=2, base_resolution=16, growth=growth)
enc = sx.HashEncoder(cfg)
enc.init_tables(42)
grad = sx.EncoderGradient(enc)
xs, ups, outs = [], [], []
for i in range(4):
    x = torch.empty((N, n), dtype=torch.float32, device="cuda")
    r = sx.CounterRng(99, 1); r.counter = i * N * n; r.fill_device(x)
    up = torch.empty((N, 32), dtype=torch.float32, device="cuda")
    r = sx.CounterRng(7, 2); r.counter = i * N * 32; r.fill_device(up, -1e-3, 1e-3)
    xs.append(x); ups.append(up); outs.append(torch.empty((N, 32), dtype=torch.float32, device="cuda"))
print(f"# n={n} T=2^{log2t} lpt={lpt} level_major={lm}; hints = gather policy + 4 * red policy (0 none, 1 evict_last, 2 evict_first, 3 evict_unchanged)\nhints  fwd_us  bwd_us  fused_us")
for h in range(16):
    enc.set_tuning(sx.Tuning(levels_per_thread=lpt, level_major=lm, cache_hints=h))
    res_t = []
    for which in ("fwd", "bwd", "fused"):
        fn = {"fwd": lambda i: enc.encode(xs[i % 4], out=outs[i % 4]), "bwd": lambda i: enc.encode_backward(xs[i % 4], ups[i % 4], grad),
              "fused": lambda i: enc.encode_forward_backward(xs[i % 4], ups[i % 4], grad, out=outs[i % 4])}[which]
        for i in range(4):
            fn(i)
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for i in range(20):
            fn(i)
        b.record()
        torch.cuda.synchronize()
        res_t.append(a.elapsed_time(b) / 20 * 1e3)
    print(f"{h:4d} {res_t[0]:7.1f} {res_t[1]:7.1f} {res_t[2]:7.1f}", flush=True)
