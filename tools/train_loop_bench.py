#!/usr/bin/env python
"""tools/train_loop_bench.py -- the training LOOP (train_field's per-step cadence) on one B200: a host round trip per step
(sxen_trainer_step: loss read-back + error words every step) against queued steps (sxen_trainer_step_enqueue, one
collect per window), at the reference's default batch (2048) and the BASELINE batch sizes.  Wall clock around a
synchronised loop, fit_image's device sampler included, 2D L=16 F=2 T=2^19."""
import argparse
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2311_15439_b200 as sx  # noqa: E402
from paper_2311_15439_b200.tasks import image_sampler  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--precision", type=int, default=1)
a = ap.parse_args()
W = H = 1024
img = torch.rand((H, W, 3), dtype=torch.float64, device="cuda")
cfg = sx.EncoderConfig(dim=2, levels=16, table_size=1 << 19, features=2, base_resolution=16, growth=(W / 16) ** (1 / 15))
print(f"# 2D L=16 F=2 T=2^19, head precision {a.precision}, image {W}x{H}")
print("batch    steps  per_step_us  queued_us  speedup  queued_Msamples/s")
for log2b, steps in ((11, 2000), (14, 1000), (16, 600), (18, 300), (20, 100)):
    B = 1 << log2b
    res = {}
    for mode in ("step", "queued"):
        enc = sx.HashEncoder(cfg)
        enc.init_tables(42)
        mlp = sx.Mlp(sx.MlpConfig(32, 64, 2, 3))
        mlp.init_params(sx.hash_combine(42, 1))
        mlp.set_precision(a.precision)
        tr = sx.Trainer(enc, mlp)
        ta, ma = sx.AdamConfig(lr=1e-2), sx.AdamConfig(lr=1e-3)
        sampler = image_sampler(img, W, H, 1234)
        for k in range(5):
            tr.step(*sampler(k, B), ta, ma)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        if mode == "step":
            for k in range(steps):
                tr.step(*sampler(k, B), ta, ma)
        else:
            first = 0
            for k in range(steps):
                tr.step_enqueue(*sampler(k, B), ta, ma)
                if k + 1 - first == 256 or k == steps - 1:
                    losses, failed = tr.collect()
                    assert failed == -1 and np.isfinite(losses).all()
                    first = k + 1
        torch.cuda.synchronize()
        res[mode] = (time.perf_counter() - t0) / steps * 1e6
    print(f"2^{log2b:<2d}  {steps:6d}  {res['step']:11.1f}  {res['queued']:9.1f}  {res['step'] / res['queued']:7.2f}  "
          f"{B / res['queued']:10.1f}", flush=True)
