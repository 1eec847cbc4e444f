#!/usr/bin/env python
"""tools/mlp_stress.py -- back-to-back launches of the tcgen05 MLP training kernel at awkward batch sizes, no synchronisation
between them: a hand-off bug between its warps (mbarrier parity lapping) shows up as a hang here, not in the parity tests.
    timeout 60 python tools/mlp_stress.py [iterations] [precision]"""
import sys, random
sys.path.insert(0, "/root/repo")
import torch
import paper_2311_15439_b200 as sx
random.seed(1)
iters = int(sys.argv[1]) if len(sys.argv) > 1 else 300
mlp = sx.Mlp(sx.MlpConfig(32, 64, 2, 3)); mlp.init_params(5); mlp.set_precision(int(sys.argv[2]) if len(sys.argv) > 2 else 1)
ref = sx.Mlp(sx.MlpConfig(32, 64, 2, 3)); ref.init_params(5)
big = torch.randn((1 << 21, 32), device="cuda") * 0.1
tg = torch.rand((1 << 21, 3), device="cuda")
for it in range(iters):
    n = random.choice([1, 2, 127, 128, 129, 255, 256, 1000, 18944, 18945, 148 * 128, 148 * 128 + 1, random.randint(1, 1 << 21)])
    import os
    mlp.forward_backward(big[:n], tg[:n])
    if os.environ.get("SYNC", "0") == "1" or it % 50 == 0:
        torch.cuda.synchronize()
        print(it, n, "ok", flush=True)
torch.cuda.synchronize()
print("stress done")
