#!/usr/bin/env python
"""tools/prof_run.py -- a short, fixed launch sequence for ncu: warm-up, then forward, backward, fused on 2^20 samples.
    ncu ... -k regex:encode_kernel --launch-skip 6 --launch-count 3 python tools/prof_run.py --dim 3"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2311_15439_b200 as sx  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--dim", type=int, default=3)
ap.add_argument("--lpt", type=int, default=0)
ap.add_argument("--level-major", type=int, default=0)
ap.add_argument("--log2t", type=int, default=19)
ap.add_argument("--level-chunk", type=int, default=0, help="sxen_tuning.level_chunk (0 library default, -1 one grid slice)")
a = ap.parse_args()
n, N = a.dim, 1 << 20
cfg = sx.EncoderConfig(dim=n, levels=16, table_size=1 << a.log2t, features=2, base_resolution=16,
                       growth={2: 2.0, 3: 1.5}.get(n, 1.5))
enc = sx.HashEncoder(cfg)
enc.init_tables(42)
enc.set_tuning(sx.Tuning(levels_per_thread=a.lpt, level_major=a.level_major, level_chunk=a.level_chunk))
grad = sx.EncoderGradient(enc)
x = torch.empty((N, n), dtype=torch.float32, device="cuda")
sx.CounterRng(99, 1).fill_device(x)
up = torch.empty((N, 32), dtype=torch.float32, device="cuda")
sx.CounterRng(7, 2).fill_device(up, -1e-3, 1e-3)
out = torch.empty((N, 32), dtype=torch.float32, device="cuda")
for _ in range(2):  # 6 warm-up encode_kernel launches
    enc.encode(x, out=out)
    enc.encode_backward(x, up, grad)
    enc.encode_forward_backward(x, up, grad, out=out)
torch.cuda.synchronize()
enc.encode(x, out=out)
enc.encode_backward(x, up, grad)
enc.encode_forward_backward(x, up, grad, out=out)
torch.cuda.synchronize()
enc.check()
print("prof_run done")
