#!/usr/bin/env python
"""tools/fit_field_sweep.py -- fit_field (src/tasks.cpp:139-194) for n = 2..6 on one B200: simplex-lattice noise target,
L=16 F=2 T=2^19, batch 2^18, tcgen05 head; reports time per training step and hold-out MSE against the field variance.
Exercises n > 3 end to end (encode -> MLP -> encode_backward -> sparse Adam) with the device sampler."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2311_15439_b200 as sx  # noqa: E402

steps = int(sys.argv[1]) if len(sys.argv) > 1 else 200
for n in range(2, 7):
    cfg = sx.EncoderConfig(dim=n, levels=16, table_size=1 << 19, features=2, base_resolution=4, growth=1.4)
    spec = sx.NoiseFieldSpec(dim=n, seed=7, kind=sx.NoiseKind.simplex, octaves=2, frequency=4.0)
    tc = sx.TrainConfig(batch_size=1 << 18, steps=steps, record_every=max(1, steps // 4), seed=1234)
    torch.cuda.synchronize()
    t0 = time.time()
    r = sx.fit_field(spec, cfg, tc, sx.FitFieldOptions(mlp_precision=1, holdout_samples=1 << 16))
    torch.cuda.synchronize()
    dt = time.time() - t0
    print(json.dumps({"n": n, "steps": steps, "batch": 1 << 18, "seconds_total": round(dt, 3),
                      "ms_per_step_incl_sampling": round(dt / steps * 1e3, 3),
                      "loss_curve": [(s, round(l, 6)) for s, l in r.train.loss_curve],
                      "holdout_mse": r.holdout_mse, "field_variance": r.field_variance,
                      "explained": 1.0 - r.holdout_mse / r.field_variance}), flush=True)
