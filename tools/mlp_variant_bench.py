#!/usr/bin/env python
"""tools/mlp_variant_bench.py -- A/B of the two stand-alone tcgen05 training kernels (sxen_debug_tc_variant): one tile in
flight per SM (csrc/sxen_mlp_tc.cu) against two (csrc/sxen_mlp_tc2.cu).  CUDA-event time per launch, the kernels' own cycle
counters, and the largest difference between the two kernels' results on the same inputs."""
import argparse
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2311_15439_b200 as sx  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--log2n", type=int, default=20)
ap.add_argument("--width", type=int, default=32)
ap.add_argument("--reps", type=int, default=20)
ap.add_argument("--variant", type=int, default=0, help="1 or 2: only that kernel (for ncu); 0: both and their difference")
a = ap.parse_args()
N = 1 << a.log2n
gen = torch.Generator(device="cuda").manual_seed(5)
feats = torch.rand((N, a.width), dtype=torch.float32, device="cuda", generator=gen) * 2 - 1
tgt = torch.rand((N, 3), dtype=torch.float32, device="cuda", generator=gen)
results = {}
for variant in ((1, 2) if a.variant == 0 else (a.variant,)):
    assert sx.lib.sxen_debug_tc_variant(variant) == 0
    mlp = sx.Mlp(sx.MlpConfig(a.width, 64, 2, 3))
    mlp.init_params(sx.hash_combine(42, 1))
    mlp.set_precision(1)
    for _ in range(3):
        out = mlp.forward_backward(feats, tgt)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(a.reps):
        out = mlp.forward_backward(feats, tgt)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / a.reps
    counters = torch.zeros(8, dtype=torch.int64, device="cuda")
    sx.lib.sxen_debug_tc_timing(C.c_void_p(counters.data_ptr()))
    out = mlp.forward_backward(feats, tgt)
    torch.cuda.synchronize()
    sx.lib.sxen_debug_tc_timing(None)
    mlp.clear_gradient()
    ig, loss, _ = mlp.forward_backward(feats, tgt)
    torch.cuda.synchronize()
    out = (loss, ig, torch.from_numpy(mlp.gradient()))
    c = counters.cpu().numpy().astype(float)
    ctas = min(148, (N + 127) // 128)
    tiles = (N + 127) // 128 / ctas
    per = c / ctas / tiles
    print(f"variant {variant}: {ms:.4f} ms per launch ({N} samples, width {a.width}) = {N / ms / 1e6:.3f} Gsamples/s; cycles per tile of the "
          f"CTA: epilogue loop {per[0]:.0f}, waiting chain {per[1]:.0f}, own wgrad {per[2]:.0f}, other group {per[3]:.0f}; chain warp loop "
          f"{per[4]:.0f}, idle {per[5]:.0f}; gradient flushes per CTA: mid-kernel {c[6] / ctas:.0f} cycles in all, final {c[7] / ctas:.0f}", flush=True)
    results[variant] = out
sx.lib.sxen_debug_tc_variant(2)
if a.variant != 0:
    sys.exit(0)
r1, r2 = results[1], results[2]
names = ("loss", "input_grad", "param_grad")
for k, (x, y) in enumerate(zip(r1, r2)):
    x = torch.as_tensor(x, dtype=torch.float64).flatten().cpu()
    y = torch.as_tensor(y, dtype=torch.float64).flatten().cpu()
    scale = max(float(x.abs().max()), 1e-30)
    print(f"  result {k}: max |v1 - v2| / max |v1| = {float((x - y).abs().max()) / scale:.3e}")
