#!/usr/bin/env python
"""tools/tc_accuracy.py -- errors of the tcgen05 head (split bf16) against the same network in fp64 PyTorch, in the units of
tests/test_gpu_tc.py's bars: predictions and input gradients relative to the largest magnitude of the compared array.  Used to
measure what the fourth product (lo x lo, SXEN_MLP_TENSOR_BF16X4) buys."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2311_15439_b200 as sx  # noqa: E402


def case(n, out_w, in_w, seed, mode):
    mlp = sx.Mlp(sx.MlpConfig(in_w, 64, 2, out_w))
    mlp.init_params(seed)
    rng = np.random.default_rng(seed)
    p = mlp.parameters().copy()
    p[-out_w:] = rng.standard_normal(out_w).astype(np.float32) * 0.1
    p[in_w * 64:in_w * 64 + 64] = rng.standard_normal(64).astype(np.float32) * 0.05
    mlp.set_parameters(p)
    mlp.set_precision(mode)
    x = torch.as_tensor((rng.standard_normal((n, in_w)) * 1e-1).astype(np.float32), device="cuda:0")
    tg = torch.as_tensor(rng.random((n, out_w)), device="cuda:0")
    fwd = mlp.forward(x).double()
    ig, loss, pred = mlp.forward_backward(x, tg, want_pred=True)
    torch.cuda.synchronize()
    g = mlp.gradient()
    pt = torch.from_numpy(p).to("cuda:0").double()
    shapes = [(64, in_w), (64,), (64, 64), (64,), (out_w, 64), (out_w,)]
    parts, off = [], 0
    for shp in shapes:
        k = int(np.prod(shp))
        parts.append(pt[off:off + k].view(*shp).clone().requires_grad_())
        off += k
    W0, b0, W1, b1, W2, b2 = parts
    xd = x.double().requires_grad_()
    out = torch.relu(torch.relu(xd @ W0.T + b0) @ W1.T + b1) @ W2.T + b2
    (((out - tg) ** 2).sum() / (n * out_w)).backward()
    ref_g = torch.cat([t.grad.flatten() for t in parts]).cpu().numpy()
    ep = (pred.double() - out).abs().max().item() / out.abs().max().item()
    d = (ig.double() - xd.grad).abs() / xd.grad.abs().max()
    eg = np.abs(g - ref_g).max() / np.abs(ref_g).max()
    ef = (fwd - out).abs().max().item() / out.abs().max().item()
    print(f"n={n:7d} in={in_w} out={out_w}: forward() {ef:.2e}   predictions {ep:.2e}   input gradients max {d.max().item():.2e}  99.9th pct "
          f"{torch.quantile(d.flatten()[:4_000_000].float(), 0.999).item():.2e}   parameter gradients {eg:.2e}")


for mode, name in ((1, "SXEN_MLP_TENSOR_BF16X3: three products"), (3, "SXEN_MLP_TENSOR_BF16X4: four products")):
  print("#", name)
  for n, out_w, in_w in [(128 * 150 + 37, 3, 32), (500, 1, 32), (128 * 150 + 37, 3, 16), (700, 2, 16), (128 * 148 * 5 + 37, 3, 32),
                         (128 * 148 * 4 + 1, 2, 16), (1 << 20, 3, 32)]:
    case(n, out_w, in_w, 7 + out_w, mode)
