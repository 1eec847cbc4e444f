#!/usr/bin/env python
"""tools/sweep.py -- time every encode-kernel launch shape on one B200 (CUDA events, rotating inputs > L2).

    python tools/sweep.py [--dim 3] [--reps 10] [--quick]

Prints one line per variant: fwd / bwd / fused milliseconds and samples/s for 2^20 samples.  Used to pick the library
defaults; bench.py stays the contract."""
from __future__ import annotations

import argparse
import itertools
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_2311_15439_b200 as sx  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--dim", type=int, default=3)
    ap.add_argument("--reps", type=int, default=8)
    ap.add_argument("--log2n", type=int, default=20)
    ap.add_argument("--log2t", type=int, default=19)
    ap.add_argument("--quick", action="store_true")
    ap.add_argument("--json", default=None)
    args = ap.parse_args()
    n, N, LF = args.dim, 1 << args.log2n, 32
    growth = {2: 2.0, 3: 1.5}.get(n, 1.5)
    cfg = sx.EncoderConfig(dim=n, levels=16, table_size=1 << args.log2t, features=2, base_resolution=16, growth=growth)
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

    def timeit(fn):
        for i in range(2):
            fn(i)
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for i in range(args.reps):
            fn(i)
        b.record()
        torch.cuda.synchronize()
        return a.elapsed_time(b) / args.reps

    lpts = (1, 2, 4, 16) if n in (2, 3) else (1, 2, 4)
    blocks = (128, 256) if args.quick else (128, 256, 512)
    rows = []
    print(f"# n={n} N=2^{args.log2n} T=2^{args.log2t} L=16 F=2; ms per launch (mean of {args.reps}), rotating 4 input sets")
    print("lpt blk lm ex agg |   fwd_ms   bwd_ms fused_ms | fwd_Gs/s bwd_Gs/s fused_Gs/s")
    for lpt, lm, exact, block, agg in itertools.product(lpts, (0, 1), (1, 0), blocks, (0, -1)):
        if block > 256 and lpt >= 4:
            continue
        if args.quick and (agg or (exact == 0 and lm == 1)):
            continue
        # the "agg" column now toggles the pair-merged red.v4 path: 0 = merged (default), -1 = off
        enc.set_tuning(sx.Tuning(levels_per_thread=lpt, block_threads=block, level_major=lm, exact_blend=exact,
                                 merge_pairs=-1 if agg else 1))
        fwd = timeit(lambda i: enc.encode(sets[i % 4][0], out=sets[i % 4][2])) if agg == 0 else float("nan")
        bwd = timeit(lambda i: enc.encode_backward(sets[i % 4][0], sets[i % 4][1], grad))
        fused = timeit(lambda i: enc.encode_forward_backward(sets[i % 4][0], sets[i % 4][1], grad, out=sets[i % 4][2]))
        rows.append(dict(lpt=lpt, block=block, level_major=lm, exact=exact, agg=agg, fwd_ms=fwd, bwd_ms=bwd, fused_ms=fused))
        print(f"{lpt:3d} {block:3d} {lm:2d} {exact:2d} {agg:5d} | {fwd:8.3f} {bwd:8.3f} {fused:8.3f} | "
              f"{N / fwd / 1e6:8.3f} {N / bwd / 1e6:8.3f} {N / fused / 1e6:8.3f}", flush=True)
    enc.check()
    best = min(rows, key=lambda r: r["fused_ms"])
    print("# best fused:", best)
    best_split = min(rows, key=lambda r: (r["fwd_ms"] if r["fwd_ms"] == r["fwd_ms"] else 1e9) + r["bwd_ms"])
    print("# best split:", best_split)
    if args.json:
        json.dump(rows, open(args.json, "w"))


if __name__ == "__main__":
    main()
