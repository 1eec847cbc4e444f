#!/usr/bin/env python
"""tools/mlp_grad_accuracy.py -- parameter gradients of the tcgen05 head against an fp64 PyTorch reference as the launch grows
(2^16 .. 2^24 samples), for both training kernels (sxen_debug_tc_variant).  The weight-gradient accumulators are fp32 in TMEM:
summed over all tiles of a CTA their error grows with the launch; csrc/sxen_mlp_tc2.cu flushes them every 64 tiles."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2311_15439_b200 as sx  # noqa: E402
torch.manual_seed(0)
for log2n in (16, 20, 22, 24):
    n = 1 << log2n
    gen = torch.Generator(device="cuda").manual_seed(log2n)
    x = torch.randn((n, 32), device="cuda", generator=gen) * 0.3
    tg = torch.rand((n, 3), device="cuda", generator=gen)
    for variant in (1, 2):
        sx.lib.sxen_debug_tc_variant(variant)
        mlp = sx.Mlp(sx.MlpConfig(32, 64, 2, 3)); mlp.init_params(11); mlp.set_precision(1)
        ig, loss, _ = mlp.forward_backward(x, tg); torch.cuda.synchronize()
        g = mlp.gradient()
        if variant == 1:
            # fp64 reference in torch (chunks to bound memory)
            p = torch.from_numpy(mlp.parameters()).cuda().double()
            W0 = p[:2048].view(64, 32).clone().requires_grad_(); b0 = p[2048:2112].clone().requires_grad_()
            W1 = p[2112:2112+4096].view(64, 64).clone().requires_grad_(); b1 = p[6208:6272].clone().requires_grad_()
            W2 = p[6272:6272+192].view(3, 64).clone().requires_grad_(); b2 = p[6464:6467].clone().requires_grad_()
            tot = 0
            for s in range(0, n, 1 << 20):
                xs = x[s:s + (1 << 20)].double(); ts = tg[s:s + (1 << 20)].double()
                h1 = torch.relu(xs @ W0.T + b0); h2 = torch.relu(h1 @ W1.T + b1); out = h2 @ W2.T + b2
                l = ((out - ts) ** 2).sum() / (n * 3)
                l.backward()
            ref = torch.cat([W0.grad.flatten(), b0.grad, W1.grad.flatten(), b1.grad, W2.grad.flatten(), b2.grad]).cpu().numpy()
        err = np.abs(g - ref)
        # per layer relative Frobenius
        offs = [0, 2112, 6272, 6467]
        rel = [np.linalg.norm(g[a:b] - ref[a:b]) / np.linalg.norm(ref[a:b]) for a, b in zip(offs[:-1], offs[1:])]
        print(f"n=2^{log2n} variant {variant}: max|err|/max|ref| = {err.max() / np.abs(ref).max():.2e}; per-layer rel Frobenius {rel[0]:.2e} {rel[1]:.2e} {rel[2]:.2e}", flush=True)
sx.lib.sxen_debug_tc_variant(2)
