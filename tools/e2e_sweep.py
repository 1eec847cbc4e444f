#!/usr/bin/env python
"""tools/e2e_sweep.py -- the host-buffer fused call (pinned host x/upstream in, features out) at several staging chunk
sizes, next to the PCIe copy times of the same bytes.  One process per chunk size (the staging buffers are sized once)."""
import ctypes as C
import os
import subprocess
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

if len(sys.argv) > 1 and sys.argv[1] == "child":
    import numpy as np
    import torch

    import paper_2311_15439_b200 as sx
    n, N, LF = 3, 1 << 20, 32
    cfg = sx.EncoderConfig(dim=n, levels=16, table_size=1 << 19, features=2, base_resolution=16, growth=1.5)
    enc = sx.HashEncoder(cfg)
    enc.init_tables(42)
    grad = sx.EncoderGradient(enc)
    lib = sx.lib

    def pinned(shape, dtype):
        nbytes = int(np.prod(shape)) * np.dtype(dtype).itemsize
        p = C.c_void_p()
        assert lib.sxen_host_alloc(nbytes, C.byref(p)) == 0
        return np.frombuffer((C.c_char * nbytes).from_address(p.value), dtype=dtype).reshape(shape)

    hx, hup, hout = pinned((N, n), np.float64), pinned((N, LF), np.float32), pinned((N, LF), np.float32)
    hx[:] = np.random.default_rng(0).random((N, n))
    hup[:] = 1e-3
    for _ in range(3):
        enc.encode_forward_backward(hx, hup, grad, out=hout)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(10):
        enc.encode_forward_backward(hx, hup, grad, out=hout)
    torch.cuda.synchronize()
    ms = (time.perf_counter() - t0) / 10 * 1e3
    print(f"chunk_log2={os.environ.get('SXEN_HOST_CHUNK_LOG2', 'default(17)')}: {ms:.3f} ms/step = {N / ms / 1e6:.3f} Gsamples/s "
          f"({(hx.nbytes + hup.nbytes) / ms / 1e6:.1f} GB/s in, {hout.nbytes / ms / 1e6:.1f} GB/s out)", flush=True)
else:
    for v in ("16", "17", "18", "19", "20", "21"):
        env = dict(os.environ, SXEN_HOST_CHUNK_LOG2=v)
        subprocess.run([sys.executable, os.path.abspath(__file__), "child"], env=env, check=False)
