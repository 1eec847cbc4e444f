#!/usr/bin/env python
"""tools/e2e_proto.py -- what the PCIe link allows for the host-buffer fused call: raw pinned copies of one step's bytes
(one way, both ways), and the chunked pipeline prototyped with torch streams around the device entry point
(symmetric streams vs one stream per stage), next to the C entry point."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2311_15439_b200 as sx  # noqa: E402

n, N, LF = 3, 1 << 20, 32
cfg = sx.EncoderConfig(dim=n, levels=16, table_size=1 << 19, features=2, base_resolution=16, growth=1.5)
enc = sx.HashEncoder(cfg)
enc.init_tables(42)
grad = sx.EncoderGradient(enc)
hx = torch.rand((N, n), dtype=torch.float64).pin_memory()
hup = (torch.rand((N, LF), dtype=torch.float32) * 1e-3).pin_memory()
hout = torch.empty((N, LF), dtype=torch.float32).pin_memory()
dx = torch.empty((N, n), dtype=torch.float64, device="cuda")
dup = torch.empty((N, LF), dtype=torch.float32, device="cuda")
dout = torch.empty((N, LF), dtype=torch.float32, device="cuda")


def wall(fn, reps=10):
    for _ in range(2):
        fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps):
        fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / reps * 1e3


s_in, s_out = torch.cuda.Stream(), torch.cuda.Stream()


def h2d():
    with torch.cuda.stream(s_in):
        dx.copy_(hx, non_blocking=True)
        dup.copy_(hup, non_blocking=True)


def d2h():
    with torch.cuda.stream(s_out):
        hout.copy_(dout, non_blocking=True)


def both():
    h2d()
    d2h()


in_b, out_b = hx.numel() * 8 + hup.numel() * 4, hout.numel() * 4
ms = wall(h2d); print(f"H2D only   {ms:.3f} ms  {in_b / ms / 1e6:.1f} GB/s")
ms = wall(d2h); print(f"D2H only   {ms:.3f} ms  {out_b / ms / 1e6:.1f} GB/s")
ms = wall(both); print(f"both ways  {ms:.3f} ms  {in_b / ms / 1e6:.1f} GB/s in, {out_b / ms / 1e6:.1f} GB/s out")


def pipeline(chunk, dedicated):
    k = (N + chunk - 1) // chunk
    if dedicated:
        sc = torch.cuda.Stream()
        ev_in = [torch.cuda.Event() for _ in range(k)]
        ev_k = [torch.cuda.Event() for _ in range(k)]

        def run():
            for c in range(k):
                a, b = c * chunk, min(N, (c + 1) * chunk)
                with torch.cuda.stream(s_in):
                    dx[a:b].copy_(hx[a:b], non_blocking=True)
                    dup[a:b].copy_(hup[a:b], non_blocking=True)
                    ev_in[c].record(s_in)
                with torch.cuda.stream(sc):
                    sc.wait_event(ev_in[c])
                    enc.encode_forward_backward(dx[a:b], dup[a:b], grad, out=dout[a:b], stream=sc.cuda_stream)
                    ev_k[c].record(sc)
                with torch.cuda.stream(s_out):
                    s_out.wait_event(ev_k[c])
                    hout[a:b].copy_(dout[a:b], non_blocking=True)
        return run
    streams = [torch.cuda.Stream() for _ in range(3)]

    def run():
        for c in range(k):
            a, b = c * chunk, min(N, (c + 1) * chunk)
            st = streams[c % 3]
            with torch.cuda.stream(st):
                dx[a:b].copy_(hx[a:b], non_blocking=True)
                dup[a:b].copy_(hup[a:b], non_blocking=True)
                enc.encode_forward_backward(dx[a:b], dup[a:b], grad, out=dout[a:b], stream=st.cuda_stream)
                hout[a:b].copy_(dout[a:b], non_blocking=True)
    return run


for chunk_log2 in (15, 16, 17, 18):
    for dedicated in (False, True):
        ms = wall(pipeline(1 << chunk_log2, dedicated))
        print(f"torch pipeline chunk=2^{chunk_log2} {'stage streams' if dedicated else 'symmetric    '}: {ms:.3f} ms = {N / ms / 1e6:.3f} Gsamples/s")
hxn, hupn, houtn = hx.numpy(), hup.numpy(), hout.numpy()
ms = wall(lambda: enc.encode_forward_backward(hxn, hupn, grad, out=houtn))
print(f"C entry point (torch-pinned buffers): {ms:.3f} ms = {N / ms / 1e6:.3f} Gsamples/s")
