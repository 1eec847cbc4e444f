#!/usr/bin/env python
"""tools/l2_window.py -- does keeping the tables resident in L2 help the fused encode fwd+bwd launch at T=2^19?

VERDICT r1 item 4: in the fused launch the gather hit rate falls to 62 % (93.5 % forward-only) and DRAM traffic is 3.3x the
forward + backward launches', because tables (64 MiB) and accumulator (64 MiB) evict each other in a 126 MB L2.  Variants,
each timed with CUDA events over rotating input sets (> L2), 2^20 samples, n=3:

  base        one fused launch (the library default)
  chunks=k    the fused call over k contiguous level ranges (k launches, live working set 1/k)
  window      cudaStreamAttrAccessPolicyWindow over the 64 MiB tables, hitProp = persisting, hitRatio r (set through
              cuda-python on torch's current stream; the library entry point is unchanged)
  split       forward launch + backward launch

    python tools/l2_window.py [--dim 3] [--reps 20]
"""
from __future__ import annotations

import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_2311_15439_b200 as sx  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--dim", type=int, default=3)
    ap.add_argument("--reps", type=int, default=20)
    ap.add_argument("--log2t", type=int, default=19)
    args = ap.parse_args()
    from cuda.bindings import runtime as rt

    n, N, LF, L = args.dim, 1 << 20, 32, 16
    growth = {2: 2.0, 3: 1.5}.get(n, 1.5)
    cfg = sx.EncoderConfig(dim=n, levels=L, table_size=1 << args.log2t, features=2, base_resolution=16, growth=growth)
    enc = sx.HashEncoder(cfg)
    enc.init_tables(42)
    grad = sx.EncoderGradient(enc)
    sets = []
    for i in range(4):
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
        for i in range(3):
            fn(i)
        torch.cuda.synchronize()
        per = []
        for i in range(args.reps):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            fn(i)
            b.record(stream)
            per.append((a, b))
        torch.cuda.synchronize()
        ms = sorted(a.elapsed_time(b) for a, b in per)
        return sum(ms) / len(ms), ms[0], ms[len(ms) // 2]

    def fused(i):
        x, up, out = sets[i % 4]
        enc.encode_forward_backward(x, up, grad, out=out)

    def chunks(k):
        ranges = sx.level_ranges(L, k)

        def fn(i):
            x, up, out = sets[i % 4]
            for first, count in ranges:
                enc.encode_forward_backward(x, up, grad, out=out, levels=(first, count))
        return fn

    def split(i):
        x, up, out = sets[i % 4]
        enc.encode(x, out=out)
        enc.encode_backward(x, up, grad)

    def show(name, t):
        print(f"{name:40s} mean {t[0]:.4f} ms  best {t[1]:.4f}  median {t[2]:.4f}  -> {N / t[2] / 1e6:.3f} G samples/s "
              f"frac {((652 + 1164) if n == 3 else 1424) * N / (t[2] * 1e-3) / 1e9 / 6552:.3f}", flush=True)

    enc.set_tuning(sx.Tuning(exact_blend=1, level_chunk=-1))
    show("base fused (one grid slice)", timeit(fused))
    for ch in (8, 4):
        for lpt in (2, 1, 4):
            enc.set_tuning(sx.Tuning(exact_blend=1, level_chunk=ch, levels_per_thread=lpt, level_major=0))
            show(f"ONE launch, level_chunk={ch} lpt={lpt}", timeit(fused))
    enc.set_tuning(sx.Tuning(exact_blend=1, level_chunk=-1))
    for k in (2, 4):
        show(f"fused in {k} level chunks", timeit(chunks(k)))

    def splits(bounds):
        def fn(i):
            x, up, out = sets[i % 4]
            for first, count in bounds:
                enc.encode_forward_backward(x, up, grad, out=out, levels=(first, count))
        return fn

    for cut in (4, 6, 10, 12):
        show(f"fused split at level {cut}", timeit(splits([(0, cut), (cut, L - cut)])))
    for b in ([(0, 6), (6, 4), (10, 6)], [(0, 8), (8, 4), (12, 4)], [(0, 6), (6, 6), (12, 4)]):
        show(f"fused ranges {b}", timeit(splits(b)))
    show("split fwd + bwd", timeit(split))
    for lm, lpt in ((1, 8),):
        enc.set_tuning(sx.Tuning(levels_per_thread=lpt, level_major=lm, exact_blend=1))
        try:
            show(f"fused level-major lpt={lpt}", timeit(fused))
        except Exception as exc:
            print("level-major lpt", lpt, "failed:", exc)
    enc.set_tuning(sx.Tuning(exact_blend=1, level_chunk=-1))

    # persisting-L2 window over the tables
    err, prop = rt.cudaGetDeviceProperties(0)
    print("persistingL2CacheMaxSize", prop.persistingL2CacheMaxSize >> 20, "MiB; accessPolicyMaxWindowSize",
          prop.accessPolicyMaxWindowSize >> 20, "MiB; l2CacheSize", prop.l2CacheSize >> 20, "MiB", flush=True)
    ATTR = rt.cudaStreamAttrID.cudaStreamAttributeAccessPolicyWindow if hasattr(rt.cudaStreamAttrID, 'cudaStreamAttributeAccessPolicyWindow') else rt.cudaLaunchAttributeID.cudaLaunchAttributeAccessPolicyWindow
    tables_ptr = enc.tables_device().data_ptr()
    table_bytes = L * (1 << args.log2t) * 2 * 4
    gptr = grad.device_view().data_ptr()
    for carve_mib in (32, 64, prop.persistingL2CacheMaxSize >> 20):
        carve = min(carve_mib << 20, prop.persistingL2CacheMaxSize)
        (err,) = rt.cudaDeviceSetLimit(rt.cudaLimit.cudaLimitPersistingL2CacheSize, carve)
        assert err == rt.cudaError_t.cudaSuccess, err
        for what, base_ptr in (("tables", tables_ptr), ("grads", gptr)):
            for ratio in (1.0, 0.6):
                attr = rt.cudaStreamAttrValue()
                w = rt.cudaAccessPolicyWindow()
                w.base_ptr = base_ptr
                w.num_bytes = min(table_bytes, prop.accessPolicyMaxWindowSize)
                w.hitRatio = ratio
                w.hitProp = rt.cudaAccessProperty.cudaAccessPropertyPersisting
                w.missProp = rt.cudaAccessProperty.cudaAccessPropertyStreaming
                attr.accessPolicyWindow = w
                (err,) = rt.cudaStreamSetAttribute(stream.cuda_stream, ATTR, attr)
                assert err == rt.cudaError_t.cudaSuccess, err
                show(f"window {what} carve {carve >> 20} MiB ratio {ratio}", timeit(fused))
                show(f"window {what} carve {carve >> 20} MiB ratio {ratio} + 2 chunks", timeit(chunks(2)))
        # reset
        attr = rt.cudaStreamAttrValue()
        w = rt.cudaAccessPolicyWindow()
        w.num_bytes = 0
        attr.accessPolicyWindow = w
        rt.cudaStreamSetAttribute(stream.cuda_stream, ATTR, attr)
        rt.cudaCtxResetPersistingL2Cache()
    rt.cudaDeviceSetLimit(rt.cudaLimit.cudaLimitPersistingL2CacheSize, 0)
    show("base fused (again)", timeit(fused))
    enc.check()


if __name__ == "__main__":
    main()
