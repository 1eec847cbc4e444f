#!/usr/bin/env python
"""tools/l2_fetch_granularity.py -- cudaLimitMaxL2FetchGranularity (32 / 64 / 128 bytes) against the encode kernels where the
tables no longer fit L2 (T = 2^22: 512 MiB tables + 512 MiB accumulator; BASELINE configs[4]).  Every gather is an 8-byte row
in a 32-byte sector; a 64-byte fetch granularity (the default) doubles the DRAM bytes of a random gather or red.

    python tools/l2_fetch_granularity.py [--dim 3] [--log2t 22]"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
from cuda.bindings import runtime as rt  # noqa: E402

import paper_2311_15439_b200 as sx  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--dim", type=int, default=3)
ap.add_argument("--log2t", type=int, default=22)
ap.add_argument("--reps", type=int, default=10)
a = ap.parse_args()
n, N, LF = a.dim, 1 << 20, 32
cfg = sx.EncoderConfig(dim=n, levels=16, table_size=1 << a.log2t, features=2, base_resolution=16, growth={2: 2.0}.get(n, 1.5))
enc = sx.HashEncoder(cfg)
enc.init_tables(42)
grad = sx.EncoderGradient(enc)
sets = []
for i in range(3):
    x = torch.empty((N, n), dtype=torch.float32, device="cuda")
    r = sx.CounterRng(99, 1)
    r.counter = i * N * n
    r.fill_device(x)
    up = torch.empty((N, LF), dtype=torch.float32, device="cuda")
    r = sx.CounterRng(7, 2)
    r.counter = i * N * LF
    r.fill_device(up, -1e-3, 1e-3)
    sets.append((x, up, torch.empty((N, LF), dtype=torch.float32, device="cuda")))
stream = torch.cuda.current_stream()


def timeit(fn):
    for i in range(2):
        fn(i)
    torch.cuda.synchronize()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(a.reps)]
    for i, (e0, e1) in enumerate(ev):
        e0.record(stream)
        fn(i)
        e1.record(stream)
    torch.cuda.synchronize()
    ms = sorted(e0.elapsed_time(e1) for e0, e1 in ev)
    return ms[len(ms) // 2]


err, cur = rt.cudaDeviceGetLimit(rt.cudaLimit.cudaLimitMaxL2FetchGranularity)
print("default cudaLimitMaxL2FetchGranularity:", cur, flush=True)
for gran in (cur, 32, 64, 128, 32):
    (err,) = rt.cudaDeviceSetLimit(rt.cudaLimit.cudaLimitMaxL2FetchGranularity, gran)
    err2, got = rt.cudaDeviceGetLimit(rt.cudaLimit.cudaLimitMaxL2FetchGranularity)
    f = timeit(lambda i: enc.encode(sets[i % 3][0], out=sets[i % 3][2]))
    b = timeit(lambda i: enc.encode_backward(sets[i % 3][0], sets[i % 3][1], grad))
    fb = timeit(lambda i: enc.encode_forward_backward(sets[i % 3][0], sets[i % 3][1], grad, out=sets[i % 3][2]))
    bytes_f, bytes_b = 4 * n + 4 * LF * (n + 1) + 4 * LF, 4 * n + 4 * LF + 8 * LF * (n + 1)
    print(f"granularity {gran:3d} (set -> {got}, err {int(err)}): fwd {f:.4f} ms  bwd {b:.4f} ms ({bytes_b * N / b / 1e6 / 6552:.3f} of HBM)  "
          f"fwd+bwd call {fb:.4f} ms = {N / fb / 1e6:.3f} G samples/s ({(bytes_f + bytes_b) * N / fb / 1e6 / 6552:.3f})", flush=True)
enc.check()
