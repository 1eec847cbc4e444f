#!/usr/bin/env python
"""tools/tc_probe.py -- pin tcgen05 descriptor conventions and TMEM lane mapping on hardware (tests/cuda/sxen_tc_probe.cu, the test-only probe library)."""
import ctypes as C
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2311_15439_b200 as sx  # noqa: E402

lib = C.CDLL(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests", "cuda", "_build", "libsxen_tc_probe.so"))
lib.sxen_tc_probe.restype = C.c_int
lib.sxen_tc_probe.argtypes = [C.c_void_p, C.c_void_p, C.c_int32, C.c_int32, C.c_int32, C.c_int32, C.c_int32, C.c_int32, C.c_void_p]
rng = np.random.default_rng(0)
ok_all = True
cases = [(128, 64, 32, 0, 0, 0), (128, 64, 16, 0, 1, 0), (64, 64, 128, 1, 1, 0), (64, 64, 32, 0, 0, 0),
         (128, 64, 32, 0, 0, 1), (128, 64, 64, 0, 0, 1), (128, 32, 64, 0, 0, 1), (128, 64, 32, 0, 1, 1), (128, 32, 64, 0, 1, 1),
         (128, 64, 128, 1, 1, 1), (64, 64, 128, 1, 1, 1), (64, 32, 128, 1, 1, 1), (64, 64, 128, 1, 0, 1), (128, 64, 64, 1, 0, 1)]
for M, N, K, a_mn, b_mn, swz in cases:
    A = rng.integers(-3, 4, size=(M, K)).astype(np.float32)
    B = rng.integers(-3, 4, size=(N, K)).astype(np.float32)
    D = A @ B.T
    a, b = torch.as_tensor(A, device="cuda"), torch.as_tensor(B, device="cuda")
    raw = torch.zeros((128, N), dtype=torch.float32, device="cuda")
    st = lib.sxen_tc_probe(a.data_ptr(), b.data_ptr(), M, N, K, a_mn, b_mn, swz, raw.data_ptr())
    if st != 0:
        print("probe failed: status", st)
        ok_all = False
        continue
    R = raw.cpu().numpy()
    if M == 128:
        ok = np.array_equal(R, D)
        print(f"swz={swz} M={M} N={N} K={K} a_mn={a_mn} b_mn={b_mn}: direct lane=row match: {ok}")
    else:
        lanes = [(i // 16) * 32 + i % 16 for i in range(64)]
        ok = np.array_equal(R[lanes], D)
        ok2 = np.array_equal(R[:64], D)
        print(f"swz={swz} M={M} N={N} K={K} a_mn={a_mn} b_mn={b_mn}: lane=(i/16)*32+i%16 match: {ok}; lanes 0-63 match: {ok2}")
        if not ok and not ok2:
            # find for each D row which lane holds it
            mapping = []
            for i in range(64):
                hit = [l for l in range(128) if np.array_equal(R[l], D[i])]
                mapping.append(hit[:2])
            print("   row->lanes:", mapping[:8], "nonzero frac", float((R != 0).mean()))
    ok_all &= bool(ok if M == 128 else (ok or ok2))
    if not ok and M == 128:
        bad = np.argwhere(R != D)
        print("   first mismatches:", bad[:5].tolist(), R[tuple(bad[0])] if len(bad) else None, D[tuple(bad[0])] if len(bad) else None)
print("---- bf16 (kind::f16), CM16 no-swizzle tiles")
lib.sxen_tc_probe_bf16.restype = C.c_int
lib.sxen_tc_probe_bf16.argtypes = [C.c_void_p, C.c_void_p, C.c_int32, C.c_int32, C.c_int32, C.c_int32, C.c_int32, C.c_void_p]
for M, N, K, a_mn, b_mn in [(128, 64, 32, 0, 0), (128, 64, 64, 0, 0), (128, 16, 64, 0, 0), (128, 64, 16, 0, 1), (128, 32, 64, 0, 1),
                            (128, 64, 128, 1, 1), (64, 64, 128, 1, 1), (64, 40, 128, 1, 1), (64, 16, 128, 1, 1), (64, 72, 128, 1, 1),
                            (64, 64, 32, 0, 0), (128, 64, 64, 1, 0)]:
    A = rng.integers(-3, 4, size=(M, K)).astype(np.float32)
    B = rng.integers(-3, 4, size=(N, K)).astype(np.float32)
    D = A @ B.T
    a, b = torch.as_tensor(A, device="cuda"), torch.as_tensor(B, device="cuda")
    raw = torch.zeros((128, N), dtype=torch.float32, device="cuda")
    st = lib.sxen_tc_probe_bf16(a.data_ptr(), b.data_ptr(), M, N, K, a_mn, b_mn, raw.data_ptr())
    if st != 0:
        print("probe failed: status", st)
        continue
    R = raw.cpu().numpy()
    if M == 128:
        print(f"bf16 M={M} N={N} K={K} a_mn={a_mn} b_mn={b_mn}: match {np.array_equal(R, D)} nonzero {float((R != 0).mean()):.2f}")
    else:
        lanes = [(i // 16) * 32 + i % 16 for i in range(64)]
        print(f"bf16 M={M} N={N} K={K} a_mn={a_mn} b_mn={b_mn}: match {np.array_equal(R[lanes], D)} nonzero {float((R != 0).mean()):.2f}")
print("ALL OK" if ok_all else "SOME FAILED")
