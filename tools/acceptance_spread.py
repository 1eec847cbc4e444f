#!/usr/bin/env python
"""tools/acceptance_spread.py -- the reference's image-fitting-parity acceptance configuration (tests/acceptance_main.cpp:
315-341: 512 x 512 test image, L=8 T=2^16 F=2 base 4 growth 2 equal-memory, batch 512, 10 000 steps), six launches per
(head precision, backend): how far the final PSNR moves from launch to launch with the order of the fp32 atomics, next to
the reference's own deterministic run (tests/golden/acceptance_image_fitting.npz).  Run from the repo root."""
import sys, os, numpy as np
sys.path.insert(0, os.getcwd())
import paper_2311_15439_b200 as sx
g = np.load("tests/golden/acceptance_image_fitting.npz")
img = sx.make_test_image(512, 512, 7)
for precision in (0, 1):
    for name, backend in (("simplex", 0), ("grid", 1)):
        out = []; worst = []
        for rep in range(6):
            cfg = sx.EncoderConfig(dim=2, levels=8, table_size=1 << 16, features=2, base_resolution=4, growth=2.0, backend=backend, level_scale=1)
            tc = sx.TrainConfig(batch_size=512, steps=10000, seed=1234, threads=1, record_every=1000)
            res = sx.fit_image(img, cfg, tc, sx.FitImageOptions(mlp_precision=precision))
            loss = np.array([v for s, v in res.train.loss_curve if s % 1000 == 0])
            r = loss / g[f"{name}/loss_every_1000"]
            out.append(res.final_psnr); worst.append((r.min(), r.max()))
        print(precision, name, "ref", float(g[f"{name}/final_psnr"]), "psnr", np.round(out, 3), "loss ratio min/max", np.round(np.min(worst, 0)[0], 2), np.round(np.max(worst, 0)[1], 2), flush=True)
