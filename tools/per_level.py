#!/usr/bin/env python
"""tools/per_level.py -- cost of ONE level at each resolution of the BASELINE ladder (L=1 encoders, 2^20 samples).
Shows where forward gathers / backward atomics are cheap (coarse, few hot rows) or dear."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2311_15439_b200 as sx  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 3
N = 1 << 20
x = torch.empty((N, n), dtype=torch.float32, device="cuda")
sx.CounterRng(99, 1).fill_device(x)
up = torch.empty((N, 2), dtype=torch.float32, device="cuda")
sx.CounterRng(7, 2).fill_device(up, -1e-3, 1e-3)
out = torch.empty((N, 2), dtype=torch.float32, device="cuda")
ladder = [16, 24, 36, 54, 81, 121, 182, 273, 410, 615, 922, 1383, 2075, 3113, 4670, 7006] if n == 3 else [16 << l for l in range(16)]
print("res      fwd_us  bwd_us  bwd_nomerge_us fused_us")
for res in ladder:
    cfg = sx.EncoderConfig(dim=n, levels=1, table_size=1 << 19, features=2, base_resolution=res, growth=2.0)
    enc = sx.HashEncoder(cfg)
    enc.init_tables(1)
    grad = sx.EncoderGradient(enc)
    res_t = []
    for merge, which in ((1, "fwd"), (1, "bwd"), (-1, "bwd"), (1, "fused")):
        enc.set_tuning(sx.Tuning(levels_per_thread=1, merge_pairs=merge))
        fn = {"fwd": lambda: enc.encode(x, out=out), "bwd": lambda: enc.encode_backward(x, up, grad),
              "fused": lambda: enc.encode_forward_backward(x, up, grad, out=out)}[which]
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(10):
            fn()
        b.record()
        torch.cuda.synchronize()
        res_t.append(a.elapsed_time(b) * 100)
    print(f"{res:7d} {res_t[0]:7.1f} {res_t[1]:7.1f} {res_t[2]:9.1f} {res_t[3]:10.1f}", flush=True)
