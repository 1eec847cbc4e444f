#!/usr/bin/env python
"""tools/train_bench.py -- time the fused training step pieces on one B200 (CUDA events):
   tensor-core MLP forward+loss+backward alone, and the whole step (encode -> MLP -> encode_backward -> Adam)."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2311_15439_b200 as sx  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--dim", type=int, default=3)
ap.add_argument("--log2n", type=int, default=20)
ap.add_argument("--reps", type=int, default=10)
ap.add_argument("--once", action="store_true", help="single pass for ncu")
a = ap.parse_args()
n, N = a.dim, 1 << a.log2n
cfg = sx.EncoderConfig(dim=n, levels=16, table_size=1 << 19, features=2, base_resolution=16, growth={2: 2.0, 3: 1.5}[n])
enc = sx.HashEncoder(cfg)
enc.init_tables(42)
x = torch.empty((N, n), dtype=torch.float32, device="cuda")
sx.CounterRng(99, 1).fill_device(x)
tgt = torch.rand((N, 3), dtype=torch.float32, device="cuda")
feats = enc.encode(x)


def timeit(fn, reps):
    for _ in range(2):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


for mode, name in ((1, "tcgen05 bf16x3"), (3, "tcgen05 bf16x4"), (2, "tcgen05 bf16"), (0, "exact fp64")):
    mlp = sx.Mlp(sx.MlpConfig(32, 64, 2, 3))
    mlp.init_params(sx.hash_combine(42, 1))
    mlp.set_precision(mode)
    Nm = N if mode else min(N, 1 << 16)
    reps = 1 if a.once else (a.reps if mode else 2)
    ms = timeit(lambda: mlp.forward_backward(feats[:Nm], tgt[:Nm]), reps)
    fms = timeit(lambda: mlp.forward(feats[:Nm]), reps)
    print(f"MLP {name:16s}: fwd+loss+bwd {ms:8.3f} ms for {Nm} samples = {Nm / ms / 1e6:7.3f} Gsamples/s "
          f"({Nm * 38016 / ms / 1e9:7.1f} TFLOP/s useful); forward only {fms:8.3f} ms = {Nm / fms / 1e6:7.3f} Gsamples/s", flush=True)
    tr = sx.Trainer(enc, mlp)
    ta, ma = sx.AdamConfig(lr=1e-2), sx.AdamConfig(lr=1e-3)
    sms = timeit(lambda: tr.step(x[:Nm], tgt[:Nm], ta, ma), reps)
    print(f"    full training step ({name}): {sms:8.3f} ms for {Nm} samples = {Nm / sms / 1e6:7.3f} Gsamples/s", flush=True)
    if a.once:
        break

# ---- where the stand-alone training kernel's warps spend their cycles (sxen_debug_tc_timing)
if not a.once:
    import ctypes as C
    counters = torch.zeros(8, dtype=torch.int64, device="cuda")
    sx.lib.sxen_debug_tc_timing(C.c_void_p(counters.data_ptr()))
    mlp = sx.Mlp(sx.MlpConfig(32, 64, 2, 3))
    mlp.init_params(sx.hash_combine(42, 1))
    mlp.set_precision(1)
    mlp.forward_backward(feats, tgt)
    torch.cuda.synchronize()
    counters.zero_()
    mlp.forward_backward(feats, tgt)
    torch.cuda.synchronize()
    sx.lib.sxen_debug_tc_timing(None)
    c = counters.cpu().numpy().astype(float)
    ctas = min(148, (N + 127) // 128)
    tiles = (N + 127) // 128 / ctas
    print(f"tcgen05 training kernel, cycles per 128-sample tile: epilogue thread in the loop {c[0] / ctas / tiles:.0f}, of those waiting on "
          f"the chain MMAs {c[1] / ctas / tiles:.0f}, on the weight-gradient MMAs {c[2] / ctas / tiles:.0f}; chain warp in the loop "
          f"{c[4] / ctas / tiles:.0f}, waiting on the epilogue {c[5] / ctas / tiles:.0f}", flush=True)
