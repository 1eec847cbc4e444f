"""Generate tests/golden/*.npz from the UNMODIFIED reference (oracle/_ref, built from /root/reference).

Run in the build container only (the GPU box has no /root/reference):
    python tests/golden/make_golden.py
The fixtures are committed; tests never regenerate them.
"""
from __future__ import annotations

import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import oracle  # noqa: E402
from oracle import AdamConfig, Config, MlpConfig, Ref  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))
U64 = 2**64 - 1


def points(ref: Ref, n: int, count: int, seed: int) -> np.ndarray:
    """count x n points: reference-RNG uniforms + hand-picked boundary / tie cases."""
    x = ref.rng_doubles(seed, n, count * n).reshape(count, n)
    special = [np.zeros(n), np.ones(n), np.full(n, 0.5), np.full(n, np.nextafter(1.0, 0.0)),
               np.array([1.0 if i % 2 == 0 else 0.0 for i in range(n)]),
               np.array([0.999999999 if i == 0 else 1.0 for i in range(n)]),
               np.full(n, 0.25), np.array([(i + 1) / (n + 1) for i in range(n)])]
    for i, s in enumerate(special):
        x[i] = s
    return x


def vertex_lists(ref: Ref, cfg: Config, x: np.ndarray):
    """(idx, w, count) per (sample, level) recovered through the public API: a features=1 encoder and a
    ones upstream make EncoderGradient hold the interpolation weights in first-touch (= chain) order."""
    c1 = Config(**{**cfg.__dict__, "features": 1})
    enc = ref.encoder(c1)
    V = cfg.vertices
    N = x.shape[0]
    idx = np.zeros((N, cfg.levels, V), dtype=np.uint32)
    w = np.zeros((N, cfg.levels, V), dtype=np.float64)
    cnt = np.zeros((N, cfg.levels), dtype=np.uint8)
    up = np.ones((1, cfg.levels))
    for s in range(N):
        _, _, order, bad, st = enc.encode_backward(x[s:s + 1], up)
        assert st == 0 and bad == -1
        lib = ref.lib
        # re-read values in touch order
        g = lib.sxr_grad_create(c1.levels, c1.table_size, 1)
        import ctypes as C
        b = C.c_long(-1)
        xs = np.ascontiguousarray(x[s:s + 1])
        lib.sxr_encode_backward(enc.h, xs.ctypes.data_as(C.POINTER(C.c_double)),
                                up.ctypes.data_as(C.POINTER(C.c_double)), 1, g, C.byref(b))
        for l in range(cfg.levels):
            k = lib.sxr_grad_touched_count(g, l)
            ii = np.empty(k, dtype=np.uint32)
            vv = np.empty(k, dtype=np.float64)
            lib.sxr_grad_read(g, l, ii.ctypes.data_as(C.POINTER(C.c_uint32)), vv.ctypes.data_as(C.POINTER(C.c_double)))
            idx[s, l, :k] = ii
            w[s, l, :k] = vv
            cnt[s, l] = k
        lib.sxr_grad_destroy(g)
    return idx, w, cnt


def sparse_grad(order, grad):
    """Flatten the reference's per-level touch lists: (level, row) pairs + slices."""
    lv, rows, vals = [], [], []
    for l, idx in enumerate(order):
        lv.append(np.full(idx.size, l, dtype=np.int32))
        rows.append(idx.astype(np.uint32))
        vals.append(grad[l, idx])
    return np.concatenate(lv), np.concatenate(rows), np.concatenate(vals)


def encode_cases(ref: Ref):
    cases = {}
    specs = []
    for backend in (oracle.BACKEND_SIMPLEX, oracle.BACKEND_GRID):
        for n in range(1, 8):  # reference test_encoding.cpp:224-251 sweep (small_config, 3 levels)
            specs.append((f"small_b{backend}_n{n}", Config(dim=n, levels=3, table_size=1 << 10, features=2,
                                                           base_resolution=4, growth=2.0, backend=backend), 40, 77))
    specs += [
        ("c2_n3", Config(dim=3, levels=16, table_size=1 << 19, features=2, base_resolution=16, growth=1.5), 96, 42),
        ("c3_n2", Config(dim=2, levels=16, table_size=1 << 19, features=2, base_resolution=16, growth=2.0), 96, 42),
        ("c1_n2", Config(dim=2, levels=16, table_size=1 << 19, features=2, base_resolution=16,
                         growth=(2048 / 16) ** (1 / 15)), 64, 42),
        ("eqmem_n3", Config(dim=3, levels=6, table_size=1 << 14, features=4, base_resolution=8, growth=1.7,
                            level_scale=oracle.SCALE_EQUAL_MEMORY), 48, 5),
        ("f1_n4", Config(dim=4, levels=5, table_size=1 << 12, features=1, base_resolution=3, growth=1.9), 48, 6),
        ("f8_n2", Config(dim=2, levels=4, table_size=1 << 12, features=8, base_resolution=16, growth=2.0), 48, 7),
        ("f3_n5", Config(dim=5, levels=3, table_size=1 << 11, features=3, base_resolution=5, growth=1.5), 48, 8),
        ("n8", Config(dim=8, levels=2, table_size=1 << 13, features=2, base_resolution=4, growth=2.0), 32, 9),
    ]
    for name, cfg, count, seed in specs:
        assert ref.validate(cfg) == 0, name
        enc = ref.encoder(cfg)
        enc.init_tables(seed)
        x = points(ref, cfg.dim, count, 1000 + seed)
        feats, bad, st = enc.encode(x)
        assert st == 0 and bad == -1
        enc.reset_counters()
        enc.encode(x)
        touched_cnt, oob_cnt = enc.counters()
        idx, w, cnt = vertex_lists(ref, cfg, x)
        up = ref.rng_doubles(7, 2, count * cfg.encoded_width, -1.0, 1.0).reshape(count, -1) * 1e-3
        grad, touched, order, bad, st = enc.encode_backward(x, up)
        assert st == 0
        lv, rows, vals = sparse_grad(order, grad)
        res = np.array([enc.resolution(l) for l in range(cfg.levels)], dtype=np.uint32)
        cases[name] = dict(
            cfg=np.array([cfg.dim, cfg.levels, cfg.table_size, cfg.features, cfg.base_resolution, cfg.backend,
                          cfg.level_scale], dtype=np.int64), growth=np.float64(cfg.growth), seed=np.uint64(seed),
            res=res, x=x, features=feats, idx=idx, w=w, cnt=cnt, upstream=up, g_level=lv, g_row=rows, g_val=vals,
            counters=np.array([touched_cnt, oob_cnt], dtype=np.uint64),
            table_head=np.stack([enc.table(l)[:8].copy() for l in range(cfg.levels)]))
    flat = {}
    for name, d in cases.items():
        for k, v in d.items():
            flat[f"{name}/{k}"] = v
    flat["names"] = np.array(list(cases.keys()))
    np.savez_compressed(os.path.join(OUT, "encode_cases.npz"), **flat)
    print("encode_cases:", len(cases), "cases")


def scalar_cases(ref: Ref):
    d = {}
    zs = np.array([0, 1, 42, 1234, U64, 0x9e3779b97f4a7c15, 2**63], dtype=np.uint64)
    d["mix64_in"] = zs
    d["mix64_out"] = np.array([ref.mix64(int(z)) for z in zs], dtype=np.uint64)
    d["hash_combine_out"] = np.array([ref.hash_combine(int(a), int(b)) for a in zs for b in zs[:4]], dtype=np.uint64)
    d["rng_1234_0_u64"] = ref.rng_u64(1234, 0, 16)
    d["rng_99_u64"] = ref.rng_u64(99, None, 16)
    d["rng_99_double"] = ref.rng_doubles(99, None, 16)
    d["rng_7_2_ranged"] = ref.rng_doubles(7, 2, 16, -1.0, 1.0)
    d["skew"] = np.stack([ref.skew_constants(n) for n in range(1, 9)])
    d["eqmem"] = np.array([ref.equal_memory_multiplier(n) for n in range(1, 9)])
    # hash: reference test_encoding.cpp:47-59 protocol (coords in [-1e6, 1e6))
    coords, hashes = [], []
    draws = ref.rng_u64(21, None, 8 * 64 * 8)
    k = 0
    for n in range(1, 9):
        for _ in range(64):
            c = np.array([int(draws[k + i] % 2000000) - 1000000 for i in range(n)] + [0] * (8 - n), dtype=np.int64)
            k += n
            coords.append(c)
            hashes.append(ref.hash_coords(c[:n]))
    d["hash_coords_in"] = np.stack(coords)
    d["hash_coords_n"] = np.repeat(np.arange(1, 9), 64).astype(np.int32)
    d["hash_coords_out"] = np.array(hashes, dtype=np.uint32)
    # subdivide / barycentric on random + tie inputs
    fr_all, perm_all, srt_all, w_all, n_all = [], [], [], [], []
    for n in range(1, 9):
        fr = ref.rng_doubles(13, n, 32 * n).reshape(32, n)
        fr[0] = 0.5
        fr[1] = 0.0
        if n > 1:
            fr[2, 1] = fr[2, 0]
        for f in fr:
            perm, srt = ref.subdivide(f)
            w = ref.barycentric(srt)
            fr_all.append(np.pad(f, (0, 8 - n)))
            perm_all.append(np.pad(perm, (0, 8 - n)))
            srt_all.append(np.pad(srt, (0, 8 - n)))
            w_all.append(np.pad(w, (0, 8 - n)))
            n_all.append(n)
    d["sub_fracs"], d["sub_perm"], d["sub_sorted"], d["sub_w"], d["sub_n"] = map(
        np.array, (fr_all, perm_all, srt_all, w_all, n_all))
    # resolution ladders
    ladders = {
        "res_b16_g1.5": Config(dim=3, levels=16, base_resolution=16, growth=1.5, table_size=1 << 19),
        "res_b16_g2": Config(dim=2, levels=16, base_resolution=16, growth=2.0, table_size=1 << 19),
        "res_eqmem_n2": Config(dim=2, levels=10, base_resolution=16, growth=1.6, level_scale=oracle.SCALE_EQUAL_MEMORY),
        "res_eqmem_n5": Config(dim=5, levels=10, base_resolution=7, growth=1.37, level_scale=oracle.SCALE_EQUAL_MEMORY),
        "res_grid_eqmem": Config(dim=3, levels=6, base_resolution=16, growth=1.5, backend=oracle.BACKEND_GRID,
                                 level_scale=oracle.SCALE_EQUAL_MEMORY),
    }
    for k_, cfg in ladders.items():
        d[k_] = np.array([ref.level_resolution(cfg, l) for l in range(cfg.levels)], dtype=np.uint32)
    np.savez_compressed(os.path.join(OUT, "scalar_cases.npz"), **d)
    print("scalar_cases written")


def neural_cases(ref: Ref):
    d = {}
    mc = MlpConfig(32, 64, 2, 3)
    mlp = ref.mlp(mc)
    seed = ref.hash_combine(42, 1)
    mlp.init(seed)
    d["mlp_seed"] = np.uint64(seed)
    d["mlp_params"] = mlp.params().copy()
    inp = (ref.rng_doubles(31, 0, 24 * 32, -1.0, 1.0).reshape(24, 32)).astype(np.float32)
    up = ref.rng_doubles(31, 1, 24 * 3, -1.0, 1.0).reshape(24, 3)
    out, grad, ig = mlp.forward_backward(inp, up)
    d["mlp_in"], d["mlp_up"], d["mlp_out"], d["mlp_grad"], d["mlp_input_grad"] = inp, up, out, grad, ig
    # second shape: 0 hidden layers and 1 hidden layer, odd widths
    for tag, mc2 in (("h0", MlpConfig(5, 7, 0, 2)), ("h1", MlpConfig(6, 9, 1, 1))):
        m2 = ref.mlp(mc2)
        m2.init(11)
        i2 = ref.rng_doubles(32, 0, 8 * mc2.input_width, -2.0, 2.0).reshape(8, -1).astype(np.float32)
        u2 = ref.rng_doubles(32, 1, 8 * mc2.output_width, -1.0, 1.0).reshape(8, -1)
        o2, g2, ig2 = m2.forward_backward(i2, u2)
        d[f"mlp_{tag}_params"], d[f"mlp_{tag}_in"], d[f"mlp_{tag}_up"] = m2.params().copy(), i2, u2
        d[f"mlp_{tag}_out"], d[f"mlp_{tag}_grad"], d[f"mlp_{tag}_input_grad"] = o2, g2, ig2

    # dense Adam: 5 steps on 16 params
    import ctypes as C
    lib = ref.lib
    ac = AdamConfig(lr=1e-2, beta1=0.9, beta2=0.99, epsilon=1e-15)
    p = ref.rng_doubles(33, 0, 16, -1.0, 1.0).astype(np.float32)
    d["adam_p0"] = p.copy()
    st = lib.sxr_adam_create(16)
    gs, ps = [], []
    for t in range(5):
        g = ref.rng_doubles(33, 10 + t, 16, -1.0, 1.0)
        if t == 2:
            g[3] = 0.0
        cac = ac.c()
        assert lib.sxr_adam_step(st, p.ctypes.data_as(C.POINTER(C.c_float)), g.ctypes.data_as(C.POINTER(C.c_double)), 16,
                                 C.byref(cac)) == 0
        gs.append(g)
        ps.append(p.copy())
    lib.sxr_adam_destroy(st)
    d["adam_g"], d["adam_p"] = np.stack(gs), np.stack(ps)

    # full train_field on a tiny problem, 1 thread and 3 threads (reference src/trainer.cpp:53)
    cfg = Config(dim=2, levels=4, table_size=1 << 10, features=2, base_resolution=4, growth=2.0)
    mc3 = MlpConfig(8, 16, 2, 3)
    steps, batch = 12, 64
    coords = ref.rng_doubles(1234, 5, steps * batch * 2).reshape(steps, batch, 2)
    targets = 0.5 + 0.5 * np.sin(6.0 * coords[..., :1] + np.array([0.0, 1.0, 2.0])) * np.cos(4.0 * coords[..., 1:2])
    targets = np.ascontiguousarray(targets)
    d["train_cfg"] = np.array([cfg.dim, cfg.levels, cfg.table_size, cfg.features, cfg.base_resolution], dtype=np.int64)
    d["train_mlp"] = np.array([8, 16, 2, 3], dtype=np.int64)
    d["train_coords"], d["train_targets"] = coords, targets
    tadam, madam = AdamConfig(lr=1e-2), AdamConfig(lr=1e-3)
    for threads in (1, 3):
        enc = ref.encoder(cfg)
        enc.init_tables(42)
        mlp3 = ref.mlp(mc3)
        mlp3.init(ref.hash_combine(42, 1))
        loss = np.zeros(steps)
        ta, ma = tadam.c(), madam.c()
        stt = lib.sxr_train_field(enc.h, mlp3.h, coords.ctypes.data_as(C.POINTER(C.c_double)),
                                  targets.ctypes.data_as(C.POINTER(C.c_double)), steps, batch, threads, C.byref(ta),
                                  C.byref(ma), loss.ctypes.data_as(C.POINTER(C.c_double)))
        assert stt == 0, ref.lib.sxr_last_error()
        d[f"train_loss_t{threads}"] = loss
        d[f"train_tables_t{threads}"] = enc.tables()
        d[f"train_mlp_params_t{threads}"] = mlp3.params().copy()
    np.savez_compressed(os.path.join(OUT, "neural_cases.npz"), **d)
    print("neural_cases written; loss t1:", d["train_loss_t1"][:3], "...", d["train_loss_t1"][-1])


def field_cases(ref: Ref):
    """noise_field_value and fit_field straight from the reference (src/noise.cpp:167-188, src/tasks.cpp:139-194)."""
    d = {}
    names = []
    rng = np.random.default_rng(11)
    for dim, kind, octaves, freq, seed in ((2, 0, 1, 4.0, 7), (2, 1, 3, 4.0, 7), (3, 0, 2, 3.0, 19), (3, 1, 1, 5.5, 3),
                                           (5, 1, 2, 2.0, 7), (1, 0, 1, 4.0, 7), (6, 0, 1, 2.0, 5)):
        name = f"d{dim}_k{kind}_o{octaves}"
        x = rng.random((400, dim))
        x[0] = 0.0
        x[1] = 1.0
        x[2] = 0.25  # lattice vertices and cell faces at frequency 4
        d[f"{name}/spec"] = np.array([dim, kind, octaves, seed], dtype=np.int64)
        d[f"{name}/freq"] = np.array([freq])
        d[f"{name}/x"] = x
        d[f"{name}/value"] = ref.noise_field(dim, seed, kind, octaves, freq, x)
        names.append(name)
    d["names"] = np.array(names)
    # one short fit_field run per noise kind: batch 4096, 20 steps, record_every 1
    for kind, dim in ((0, 2), (1, 3)):
        cfg = Config(dim=dim, levels=8, table_size=1 << 14, features=2, base_resolution=4, growth=1.6)
        loss, mse, var = ref.fit_field(dim, 7, kind, 2, 4.0, cfg, batch=4096, steps=20, train_seed=1234, threads=1,
                                       init_seed=42, holdout_samples=4096)
        d[f"fit_k{kind}/loss"] = loss
        d[f"fit_k{kind}/holdout"] = np.array([mse, var])
        d[f"fit_k{kind}/cfg"] = np.array([dim, 8, 1 << 14, 2, 4], dtype=np.int64)
        d[f"fit_k{kind}/growth"] = np.array([1.6])
        print("fit_field kind", kind, "loss", loss[0], "->", loss[-1], "holdout mse", mse, "variance", var)
    np.savez_compressed(os.path.join(OUT, "field_cases.npz"), **d)
    print("field_cases written")


def c1_reference(ref: Ref, steps: int = 30):
    """BASELINE configs[0] at full size, run by the reference itself (the CPU reference's own run): 2048 x 2048 test image,
    L=16 F=2 T=2^19, growth (2048/16)^(1/15), batch 2^18.  tools/config_runs.py puts the device fit next to this."""
    import time
    W = H = 2048
    growth = (2048 / 16) ** (1 / 15)
    cfg = Config(dim=2, levels=16, table_size=1 << 19, features=2, base_resolution=16, growth=growth)
    threads = max(1, min(os.cpu_count() or 1, 32))
    t0 = time.time()
    img = ref.make_test_image(W, H, 7)
    t_img = time.time() - t0
    t0 = time.time()
    psnr, loss, _, _ = ref.fit_image(img, cfg, batch=1 << 18, steps=steps, threads=threads)
    dt = time.time() - t0
    np.savez_compressed(os.path.join(OUT, "c1_reference.npz"), loss=loss, final_psnr=np.float64(psnr), steps=np.int64(steps),
                        threads=np.int64(threads), seconds_incl_final_render=np.float64(dt), image_seconds=np.float64(t_img),
                        growth=np.float64(growth), image_probe=img[::256, ::256].copy())
    print("c1_reference written:", steps, "steps on", threads, "threads in", round(dt, 1), "s; loss", loss[0], "->", loss[-1],
          "final PSNR", psnr)


def task_cases(ref: Ref):
    """fit_image on the reference's own procedural test image (src/image.cpp:68-96, src/tasks.cpp:98-137)."""
    d = {}
    img = ref.make_test_image(64, 64, 7)
    cfg = Config(dim=2, levels=16, table_size=1 << 10, features=2, base_resolution=4, growth=1.25)
    steps, batch = 300, 512
    psnr, loss, tables, params = ref.fit_image(img, cfg, batch=batch, steps=steps, train_seed=1234, threads=1, init_seed=42)
    d["image"] = img
    d["cfg"] = np.array([cfg.dim, cfg.levels, cfg.table_size, cfg.features, cfg.base_resolution], dtype=np.int64)
    d["growth"] = np.float64(cfg.growth)
    d["steps"], d["batch"] = np.int64(steps), np.int64(batch)
    d["final_psnr"], d["loss"], d["tables"], d["mlp_params"] = np.float64(psnr), loss, tables, params
    d["psnr_examples_in"] = np.array([0.0, -1.0, 1e-12, 1e-4, 0.5, 1.0, 4.0])
    d["psnr_examples_out"] = np.array([ref.psnr_from_mse(float(v)) for v in d["psnr_examples_in"]])
    np.savez_compressed(os.path.join(OUT, "task_cases.npz"), **d)
    print("task_cases written; reference final PSNR", psnr, "loss", loss[0], "->", loss[-1])


def aux_cases(ref: Ref):
    """train_field with pass-through inputs appended after the encoding (TrainConfig::aux_dims, src/trainer.cpp:32-35): 12
    steps of 256 samples, 2 aux inputs, run by the reference on 1 thread; also the reference's own width-mismatch case
    (tests/test_neural.cpp:439-462)."""
    import ctypes as C
    lib = ref.lib
    cfg = Config(dim=2, levels=4, table_size=1 << 10, features=2, base_resolution=4, growth=2.0)
    aux_dims = 2
    mc = MlpConfig(cfg.encoded_width + aux_dims, 16, 2, 1)
    steps, batch = 12, 256
    coords = ref.rng_doubles(4321, 5, steps * batch * 2).reshape(steps, batch, 2)
    aux = ref.rng_doubles(4321, 6, steps * batch * aux_dims, -1.0, 1.0).reshape(steps, batch, aux_dims)
    targets = np.ascontiguousarray(0.5 + 0.25 * np.sin(5.0 * coords[..., :1]) + 0.25 * aux[..., :1] * aux[..., 1:2])
    enc = ref.encoder(cfg)
    enc.init_tables(42)
    mlp = ref.mlp(mc)
    mlp.init(ref.hash_combine(42, 1))
    loss = np.zeros(steps)
    ta, ma = AdamConfig(lr=1e-2).c(), AdamConfig(lr=1e-3).c()
    lib.sxr_train_field_aux.restype = C.c_int
    st = lib.sxr_train_field_aux(enc.h, mlp.h, coords.ctypes.data_as(C.POINTER(C.c_double)),
                                 aux.ctypes.data_as(C.POINTER(C.c_double)), aux_dims,
                                 targets.ctypes.data_as(C.POINTER(C.c_double)), steps, batch, 1, C.byref(ta), C.byref(ma),
                                 loss.ctypes.data_as(C.POINTER(C.c_double)))
    assert st == 0, ref.lib.sxr_last_error()
    d = {"cfg": np.array([cfg.dim, cfg.levels, cfg.table_size, cfg.features, cfg.base_resolution], dtype=np.int64),
         "growth": np.float64(cfg.growth), "aux_dims": np.int64(aux_dims), "mlp": np.array([mc.input_width, 16, 2, 1], dtype=np.int64),
         "coords": coords, "aux": aux, "targets": targets, "loss": loss, "tables": enc.tables(),
         "mlp_params": mlp.params().copy()}
    np.savez_compressed(os.path.join(OUT, "aux_cases.npz"), **d)
    print("aux_cases written; loss", loss[:3], "...", loss[-1])


def acceptance_image_fitting(ref: Ref):
    """The reference's own acceptance criterion `image-fitting-parity` (tests/acceptance_main.cpp:315-341), run by the
    reference: make_test_image(512, 512, 7), L=8 T=2^16 F=2 base 4 growth 2 equal-memory, batch 512, 10 000 steps,
    1 thread, both backends.  Stores the two final PSNRs and the recorded loss curves (every 1000th step)."""
    import time
    img = ref.make_test_image(512, 512, 7)
    d = {"image_probe": img[::64, ::64].copy()}
    for name, backend in (("simplex", oracle.BACKEND_SIMPLEX), ("grid", oracle.BACKEND_GRID)):
        cfg = Config(dim=2, levels=8, table_size=1 << 16, features=2, base_resolution=4, growth=2.0, backend=backend,
                     level_scale=oracle.SCALE_EQUAL_MEMORY)
        t0 = time.time()
        psnr, loss, _, _ = ref.fit_image(img, cfg, batch=512, steps=10000, train_seed=1234, threads=1, init_seed=42)
        d[f"{name}/final_psnr"] = np.float64(psnr)
        d[f"{name}/loss_every_1000"] = loss[::1000].copy()
        d[f"{name}/loss_first_20"] = loss[:20].copy()
        d[f"{name}/seconds"] = np.float64(time.time() - t0)
        print(name, "final PSNR", psnr, "in", round(time.time() - t0, 1), "s", flush=True)
    np.savez_compressed(os.path.join(OUT, "acceptance_image_fitting.npz"), **d)
    print("acceptance_image_fitting written")


def acceptance_thread_spread(ref: Ref):
    """How far the REFERENCE's own final PSNR moves when only its worker count changes (threads = 1, 2, 3, 4, 8: the per-worker
    fp64 accumulators are merged in worker order, src/trainer.cpp:125-128, so each count is a different summation order of
    the same gradients) on its image-fitting-parity configuration (tests/acceptance_main.cpp:315-341).  This is the
    reference-side yardstick for the device path's launch-to-launch spread (fp32 atomics); written as JSON."""
    import json
    import time
    img = ref.make_test_image(512, 512, 7)
    out = {"config": "512x512 test image seed 7, L=8 T=2^16 F=2 base 4 growth 2 equal-memory, batch 512, 10000 steps, "
                     "train seed 1234, init seed 42", "runs": []}
    for name, backend, counts in (("simplex", oracle.BACKEND_SIMPLEX, (1, 2, 3, 4, 8)), ("grid", oracle.BACKEND_GRID, (1, 2, 8))):
        cfg = Config(dim=2, levels=8, table_size=1 << 16, features=2, base_resolution=4, growth=2.0, backend=backend,
                     level_scale=oracle.SCALE_EQUAL_MEMORY)
        for th in counts:
            t0 = time.time()
            psnr, loss, _, _ = ref.fit_image(img, cfg, batch=512, steps=10000, train_seed=1234, threads=th, init_seed=42)
            out["runs"].append({"backend": name, "threads": th, "final_psnr": float(psnr),
                                "loss_every_1000": [float(v) for v in loss[::1000]], "seconds": round(time.time() - t0, 1)})
            print(name, "threads", th, "final PSNR", psnr, "in", round(time.time() - t0, 1), "s", flush=True)
            with open(os.path.join(OUT, "acceptance_thread_spread.json"), "w") as f:
                json.dump(out, f, indent=1)
    print("acceptance_thread_spread written")


def gigapixel_sampler(ref: Ref):
    """BASELINE configs[2]: the 32768 x 32768 procedural image is never stored (26 GB as doubles); fit_image's sampler
    (src/tasks.cpp:112-126) draws pixel indices and the target is make_test_image's formula (src/image.cpp:68-96) at that
    pixel centre.  This fixture holds, for steps 0 and 7 of train seed 1234, the first 1024 draws: pixel index, coordinates
    and the RGB target computed by the REFERENCE's noise_field_value (the six lines of make_test_image around it are
    restated here in numpy and first checked against ref.make_test_image on a 64 x 64 image)."""
    def test_image_at(coords, seed):
        shared = ref.noise_field(2, ref.hash_combine(seed, 0xAB), oracle.NOISE_PERLIN if hasattr(oracle, "NOISE_PERLIN") else 0, 4, 4.0, coords)
        out = np.empty((coords.shape[0], 3))
        for c in range(3):
            ch = ref.noise_field(2, ref.hash_combine(seed, c + 1), 0, 5, 8.0, coords)
            out[:, c] = np.clip(0.5 + 0.62 * (0.45 * shared + 0.55 * ch), 0.0, 1.0)
        return out

    small = ref.make_test_image(64, 64, 7)
    yy, xx = np.meshgrid(np.arange(64), np.arange(64), indexing="ij")
    cc = np.stack([(xx.ravel() + 0.5) / 64, (yy.ravel() + 0.5) / 64], axis=1)
    assert np.array_equal(test_image_at(cc, 7).reshape(64, 64, 3), small), "numpy restatement of make_test_image differs"
    W = H = 32768
    d = {"width": np.int64(W), "height": np.int64(H), "image_seed": np.int64(7), "train_seed": np.int64(1234)}
    for step in (0, 7):
        u = ref.rng_u64(1234, step, 1024)
        idx = (u % np.uint64(W * H)).astype(np.int64)
        coords = np.stack([((idx % W) + 0.5) / W, ((idx // W) + 0.5) / H], axis=1)
        d[f"step{step}/idx"] = idx
        d[f"step{step}/coords"] = coords
        d[f"step{step}/targets"] = test_image_at(coords, 7)
    np.savez_compressed(os.path.join(OUT, "gigapixel_sampler.npz"), **d)
    print("gigapixel_sampler written", d["step0/idx"][:4], d["step0/targets"][:2])


if __name__ == "__main__":
    oracle.build(ref=True)
    ref = Ref()
    if len(sys.argv) > 1 and sys.argv[1] == "aux":
        aux_cases(ref)
        sys.exit(0)
    if len(sys.argv) > 1 and sys.argv[1] == "acceptance":
        acceptance_image_fitting(ref)
        sys.exit(0)
    if len(sys.argv) > 1 and sys.argv[1] == "gigapixel":
        gigapixel_sampler(ref)
        sys.exit(0)
    if len(sys.argv) > 1 and sys.argv[1] == "spread":
        acceptance_thread_spread(ref)
        sys.exit(0)
    if len(sys.argv) > 1 and sys.argv[1] == "tasks":
        task_cases(ref)
        sys.exit(0)
    if len(sys.argv) > 1 and sys.argv[1] == "c1":
        c1_reference(ref)
        sys.exit(0)
    if len(sys.argv) > 1 and sys.argv[1] == "fields":
        field_cases(ref)
        sys.exit(0)
    scalar_cases(ref)
    encode_cases(ref)
    neural_cases(ref)
    task_cases(ref)
    field_cases(ref)
    c1_reference(ref)
    for f in sorted(os.listdir(OUT)):
        if f.endswith(".npz"):
            print(f, os.path.getsize(os.path.join(OUT, f)) // 1024, "KiB")
