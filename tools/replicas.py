#!/usr/bin/env python
"""tools/replicas.py -- coarse-level side arrays on/off for the fwd / bwd / fused launches of the BASELINE ladders:
replicated gradient accumulators (sxen_tuning.coarse_replicas) and pair-merged 16-byte gathers / reds (merge_pairs)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2311_15439_b200 as sx  # noqa: E402

N = 1 << 20
for n, log2t in ((3, 19), (2, 19), (3, 22), (2, 22)):
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
    print(f"# n={n} T=2^{log2t}\nlm lpt replicas  merge hints  fwd_us  bwd_us  fused_us  fwd+bwd_us")
    for lm, lpt in ((0, 2), (1, 4), (1, 2)):
        for rep, tbl, hints in ((-1, -1, -1), (0, -1, -1), (0, 1, -1)):
            enc.set_tuning(sx.Tuning(levels_per_thread=lpt, level_major=lm, coarse_replicas=rep, merge_pairs=tbl,
                                     cache_hints=hints))
            res_t = []
            for which in ("fwd", "bwd", "fused"):
                fn = {"fwd": lambda i: enc.encode(xs[i % 4], out=outs[i % 4]),
                      "bwd": lambda i: enc.encode_backward(xs[i % 4], ups[i % 4], grad),
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
            print(f"{lm:2d} {lpt:3d} {'on' if rep == 0 else 'off':>8s} {'on' if tbl == 1 else 'off':>6s} {hints:5d} {res_t[0]:7.1f} {res_t[1]:7.1f} {res_t[2]:7.1f} {res_t[0] + res_t[1]:9.1f}", flush=True)
    del enc, grad, xs, ups, outs
    torch.cuda.empty_cache()
