#!/usr/bin/env python
"""tools/small_batch_prof.py -- a few queued training steps at the reference's default batch (2048), for an ncu launch
list (which kernels a small-batch step spends its time in)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2311_15439_b200 as sx  # noqa: E402
from paper_2311_15439_b200.tasks import image_sampler  # noqa: E402

B = int(sys.argv[1]) if len(sys.argv) > 1 else 2048
W = H = 1024
img = torch.rand((H, W, 3), dtype=torch.float64, device="cuda")
cfg = sx.EncoderConfig(dim=2, levels=16, table_size=1 << 19, features=2, base_resolution=16, growth=(W / 16) ** (1 / 15))
enc = sx.HashEncoder(cfg)
enc.init_tables(42)
mlp = sx.Mlp(sx.MlpConfig(32, 64, 2, 3))
mlp.init_params(sx.hash_combine(42, 1))
mlp.set_precision(1)
tr = sx.Trainer(enc, mlp)
ta, ma = sx.AdamConfig(lr=1e-2), sx.AdamConfig(lr=1e-3)
sampler = image_sampler(img, W, H, 1234)
for k in range(6):
    tr.step_enqueue(*sampler(k, B), ta, ma)
print(tr.collect())
