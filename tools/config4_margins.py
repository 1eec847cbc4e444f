#!/usr/bin/env python
"""tools/config4_margins.py -- the measured quantities behind the bars of tests/test_gpu_config4_size.py (configs[3] at 2^24
samples: one accumulation vs sixteen worker chunks, and the 4096-sample slice against the CPU checker is left to the test)."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import torch  # noqa: E402

import paper_2311_15439_b200 as sx  # noqa: E402
import test_gpu_config4_size as t  # noqa: E402

enc, mlp = t.make(sx)
x, tgt = t.batch(sx)
g1, m1, l1 = t.accumulated(sx, enc, mlp, x, tgt, [(0, t.N)])
g16, m16, l16 = t.accumulated(sx, enc, mlp, x, tgt, [(c * t.CHUNK, (c + 1) * t.CHUNK) for c in range(t.N // t.CHUNK)])
g1b, m1b, l1b = t.accumulated(sx, enc, mlp, x, tgt, [(0, t.N)])
print(f"loss one launch {l1!r}  sixteen chunks {l16!r}  rel diff {abs(l1 - l16) / l1:.2e}  (same launch again {abs(l1 - l1b) / l1:.2e})")
for l in range(16):
    s = np.abs(g1[l]).max()
    print(f"level {l:2d}: max|g| {s:.3e}  one-vs-sixteen {np.abs(g1[l] - g16[l]).max() / s:.2e}  same launch again {np.abs(g1[l] - g1b[l]).max() / s:.2e}"
          f"  (bar {t.ORDER_RTOL:.0e})")
print(f"MLP gradient: one-vs-sixteen {np.abs(m1 - m16).max() / np.abs(m1).max():.2e}  same launch again {np.abs(m1 - m1b).max() / np.abs(m1).max():.2e}  (bar 1e-4)")
for reps in (3,):
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    tr = sx.Trainer(enc, mlp)
    mlp.clear_gradient()
    ta, ma = sx.AdamConfig(lr=1e-2), sx.AdamConfig(lr=1e-3)
    tr.step(x, tgt, ta, ma)
    e0.record()
    for _ in range(reps):
        tr.step(x, tgt, ta, ma)
    e1.record()
    torch.cuda.synchronize()
    print(f"whole step at 2^24 samples: {e0.elapsed_time(e1) / reps:.2f} ms")
