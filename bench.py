#!/usr/bin/env python
"""bench.py -- simplex-encode forward+backward throughput on B200 (BASELINE.json metric, configs[1]).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--dim 3] [--path fused|split]

One "step" = HashEncoder::encode + encode_backward over one batch of 2^20 synthetic samples per GPU
(n=3, L=16, F=2, T=2^19, base 16, growth 1.5; coords CounterRng(99,1), upstream CounterRng(7,2)*1e-3,
tables init_tables(42) -- SURVEY.md 8d).  Prints ONE JSON line (rank 0).

  value     samples/s, inputs resident in HBM, CUDA-event timed, max over ranks
  e2e       the same metric through the host-buffer C-ABI call (pinned host memory in, features out)
  roofline  dominant kernel's algorithmic bytes / its CUDA-event duration vs MEASURED_PEAKS.json hbm_gbs
  cpu_baseline  the reference's own encode+encode_backward (oracle/_ref) on this box's host cores, bounded sample

--impl reference times the unmodified reference CPU implementation (oracle/_ref, else the oracle port) instead.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

METRIC = "simplex_encode_fwd_bwd_samples_per_s"
UNIT = "samples/s"
L, F, T_LOG2, BASE = 16, 2, 19, 16
GROWTH = {2: 2.0, 3: 1.5, 4: 1.5, 5: 1.5, 6: 1.5}
BATCH_LOG2 = 20


def alg_bytes(n: int, mode: str, verts: int = 0) -> int:
    """SURVEY.md 8d payload accounting per sample (f32 coords/features/upstream/grads, scatter-add = read+write).
    verts = vertices per (sample, level): n+1 for the simplex backend (default), 2^n for the grid backend."""
    verts = verts or (n + 1)
    fwd = 4 * n + 4 * L * F * verts + 4 * L * F
    bwd = 4 * n + 4 * L * F + 8 * L * F * verts
    return {"fwd": fwd, "bwd": bwd, "fused": fwd + bwd}[mode]


def hbm_peak():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        try:
            return float(json.load(open(p))["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
        except Exception:
            pass
    return 6650.0, "fallback (B200_PROFILING.md)"


def workload_name(n: int, t_log2: int = T_LOG2, backend: str = "simplex") -> str:
    return (f"{n}D {backend} encode fwd+bwd microbench, L={L} F={F} T=2^{t_log2} base={BASE} growth={GROWTH[n]}, "
            f"2^{BATCH_LOG2} uniform random samples per GPU")


def workload_config(n: int, t_log2: int, backend: str) -> dict:
    """The workload definition, identical (keys and values) on both arms; everything arm-specific lives elsewhere
    in the line (`launch` on the GPU arm, `cpu_baseline.sample` on the reference arm)."""
    return {"workload": workload_name(n, t_log2, backend), "dim": n, "levels": L, "features": F, "backend": backend,
            "table_size_log2": t_log2, "base_resolution": BASE, "growth": GROWTH[n],
            "samples_per_gpu_per_step": 1 << BATCH_LOG2,
            "inputs": "coords CounterRng(99,1), upstream CounterRng(7,2)*1e-3, tables init_tables(42)"}


class ClockSampler:
    """nvidia-smi clocks/throttle reasons DURING the run (B200_PROFILING.md recipe).  Started before the warm-up and stopped
    after the e2e leg (nvidia-smi needs about a second before its first sample, longer than the timed region itself);
    `mark()` timestamps let the summary say how many samples fell inside the timed region."""

    Q = ("timestamp,index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.idx = gpu_index
        self.proc = None
        self.path = None
        self.marks = {}

    def start(self):
        try:
            fd, self.path = tempfile.mkstemp(suffix=".csv")
            os.close(fd)
            self.proc = subprocess.Popen(["nvidia-smi", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                                          "-lms", "50", "-i", str(self.idx)], stdout=open(self.path, "w"),
                                         stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None

    def mark(self, name: str):
        import datetime
        self.marks[name] = datetime.datetime.now()
        if name in ("timed_region_start", "e2e_region_start"):
            self._nvml_start("timed" if name.startswith("timed") else "e2e")
        elif name in ("timed_region_end", "e2e_region_end"):
            self._nvml_stop()

    # nvidia-smi cannot sample faster than the timed region lasts (tens of milliseconds), so the timed region itself is
    # polled through NVML from a thread of this process: SM clock + clock-event reasons about once a millisecond.
    NVML_REASONS = {0x8: "hw_slowdown", 0x40: "hw_thermal_slowdown", 0x20: "sw_thermal_slowdown", 0x4: "sw_power_cap"}

    def _nvml_start(self, tag: str):
        if not hasattr(self, "nvml"):
            self.nvml = {}
        rec = self.nvml.setdefault(tag, {"sm": [], "bits": 0})
        self._nvml_thread = None
        try:
            import threading
            import pynvml
            pynvml.nvmlInit()
            # NVML enumerates physical devices; CUDA_VISIBLE_DEVICES may renumber them for torch
            vis = os.environ.get("CUDA_VISIBLE_DEVICES", "")
            phys = self.idx
            if vis:
                ids = [v for v in vis.split(",") if v.strip()]
                if self.idx < len(ids) and ids[self.idx].strip().isdigit():
                    phys = int(ids[self.idx])
            h = pynvml.nvmlDeviceGetHandleByIndex(phys)
            self._nvml_run = True

            def poll():
                k = 0
                while self._nvml_run:
                    try:
                        rec["sm"].append(float(pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM)))
                        if k % 3 == 0:   # the reasons word costs a second driver call: every third poll
                            rec["bits"] |= int(pynvml.nvmlDeviceGetCurrentClocksThrottleReasons(h))
                        k += 1
                    except Exception:
                        break
                    time.sleep(0.0005)
                try:
                    rec["bits"] |= int(pynvml.nvmlDeviceGetCurrentClocksThrottleReasons(h))
                except Exception:
                    pass

            self._nvml_thread = threading.Thread(target=poll, daemon=True)
            self._nvml_thread.start()
        except Exception:
            self._nvml_thread = None

    def _nvml_stop(self):
        if getattr(self, "_nvml_thread", None) is not None:
            self._nvml_run = False
            self._nvml_thread.join(timeout=2)
            self._nvml_thread = None

    def stop(self):
        import datetime
        out = {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0, "samples_in_timed_region": 0,
               "window": "warm-up + timed region + separate-launch diagnostics + e2e leg (GPU busy throughout)"}
        if self.proc is None:
            return out
        time.sleep(0.15)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        sm, mx, power, reasons, inside = [], [], [], set(), []
        t0, t1 = self.marks.get("timed_region_start"), self.marks.get("timed_region_end")
        try:
            for line in open(self.path):
                p = [c.strip() for c in line.split(",")]
                if len(p) < 10:
                    continue
                try:
                    sm.append(float(p[2]))
                    mx.append(float(p[3]))
                    power.append(float(p[4]))
                except ValueError:
                    continue
                try:
                    ts = datetime.datetime.strptime(p[0], "%Y/%m/%d %H:%M:%S.%f")
                    if t0 is not None and t1 is not None and t0 <= ts <= t1:
                        inside.append(sm[-1])
                except ValueError:
                    pass
                for name, val in zip(("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"), p[6:10]):
                    if val.lower().startswith("active"):
                        reasons.add(name)
            os.unlink(self.path)
        except Exception:
            pass
        if sm:
            out.update(sm_mhz=statistics.median(sm), sm_min_mhz=min(sm), sm_max_mhz=max(mx), power_w_max=max(power),
                       reasons=sorted(reasons), samples=len(sm), samples_in_timed_region=len(inside))
            if inside:
                out["sm_mhz_timed_region"] = statistics.median(inside)
        all_reasons = set(out.get("reasons", []))
        for tag, key in (("timed", "timed_region"), ("e2e", "e2e_region")):
            rec = getattr(self, "nvml", {}).get(tag)
            if not rec or not rec["sm"]:
                continue
            # the in-process NVML poll of that region proper
            nv = rec["sm"]
            out[f"samples_in_{key}"] = out.get(f"samples_in_{key}", 0) + len(nv)
            out[f"sm_mhz_{key}"] = statistics.median(nv)
            out[f"sm_min_mhz_{key}"] = min(nv)
            out[f"reasons_{key}"] = sorted(nm for bit, nm in self.NVML_REASONS.items() if rec["bits"] & bit)
            all_reasons |= set(out[f"reasons_{key}"])
            out["region_source"] = "NVML polled from a thread of this process while the region runs"
            if out.get("sm_mhz") is None:
                out.update(sm_mhz=statistics.median(nv), sm_min_mhz=min(nv), samples=len(nv))
        out["reasons"] = sorted(all_reasons)
        return out


def traffic_for(kernel_key: str):
    """dram bytes per launch of the dominant kernel from the committed ncu capture (profiles/traffic.json), or None."""
    p = os.path.join(ROOT, "profiles", "traffic.json")
    try:
        return json.load(open(p)).get(kernel_key)
    except Exception:
        return None


# ---------------------------------------------------------------------------------------------- reference arm
def cpu_reference_run(n: int, samples: int, threads: int, t_log2: int = T_LOG2):
    """Times the reference's encode + encode_backward worker pattern on `samples` samples. Returns (samples/s, kind)."""
    import numpy as np

    import oracle
    cfg = oracle.Config(dim=n, levels=L, table_size=1 << t_log2, features=F, base_resolution=BASE, growth=GROWTH[n])
    o = oracle.Oracle()
    x = o.rng_doubles(99, 1, samples * n).reshape(samples, n)
    up = o.rng_doubles(7, 2, samples * L * F, -1e-3, 1e-3).reshape(samples, L * F)
    if oracle.Ref.available():
        ref = oracle.Ref()
        enc = ref.encoder(cfg)
        enc.init_tables(42)
        secs = enc.bench_fwd_bwd(x, up, threads)
        kind = "reference"
    else:
        tables = o.init_tables(cfg, 42)
        secs = o.bench_fwd_bwd(cfg, tables, x, up, threads)
        kind = "port"
    if secs <= 0:
        raise RuntimeError("CPU baseline failed")
    return samples / secs, kind


def cpu_reference_train_step(n: int, batch: int, threads: int, t_log2: int = T_LOG2):
    """The reference's own train_field (src/trainer.cpp:53-139: encode -> Mlp::forward -> MSE -> Mlp::backward ->
    encode_backward -> sparse Adam + Adam) on `threads` workers at `batch` samples per step of the bench workload's shape.
    Seconds per step = (wall clock of a 3-step run - wall clock of a 1-step run) / 2, which leaves out the per-run set-up
    (every worker's dense fp64 accumulator, the moments).  None when the compiled reference is not there."""
    one = _cpu_reference_train_run(n, batch, threads, 1, t_log2)
    three = _cpu_reference_train_run(n, batch, threads, 3, t_log2)
    if one is None or three is None or three <= one:
        return None
    return (three - one) / 2.0


def _cpu_reference_train_run(n: int, batch: int, threads: int, steps: int, t_log2: int):
    import ctypes as C
    import time

    import numpy as np

    import oracle
    if not oracle.Ref.available():
        return None
    cfg = oracle.Config(dim=n, levels=L, table_size=1 << t_log2, features=F, base_resolution=BASE, growth=GROWTH[n])
    ref = oracle.Ref()
    enc = ref.encoder(cfg)
    enc.init_tables(42)
    mlp = ref.mlp(oracle.MlpConfig(L * F, 64, 2, 3))
    mlp.init(ref.hash_combine(42, 1))
    o = oracle.Oracle()
    coords = o.rng_doubles(99, 1, steps * batch * n)
    targets = o.rng_doubles(5, 3, steps * batch * 3)
    loss = np.zeros(steps)
    ta, ma = oracle.AdamConfig(lr=1e-2).c(), oracle.AdamConfig(lr=1e-3).c()
    t0 = time.perf_counter()
    st = ref.lib.sxr_train_field(enc.h, mlp.h, coords.ctypes.data_as(C.POINTER(C.c_double)),
                                 targets.ctypes.data_as(C.POINTER(C.c_double)), steps, batch, threads, C.byref(ta),
                                 C.byref(ma), loss.ctypes.data_as(C.POINTER(C.c_double)))
    dt = time.perf_counter() - t0
    if st != 0 or not np.isfinite(loss).all():
        return None
    return dt


def host_threads() -> int:
    cores = os.cpu_count() or 1
    try:
        cores = len(os.sched_getaffinity(0))
    except Exception:
        pass
    # every worker owns a dense fp64 accumulator (128 MiB at T=2^19) + seen maps, as the reference does
    try:
        import psutil
        by_mem = int(psutil.virtual_memory().available // (220 << 20))
        cores = max(1, min(cores, by_mem))
    except Exception:
        pass
    return cores


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    n = args.dim
    threads = host_threads()
    samples = min(1 << BATCH_LOG2, threads << 16)
    vals = []
    kind = "reference"
    for i in range(args.warmup + args.steps):
        v, kind = cpu_reference_run(n, samples, threads, args.log2t)
        if i >= args.warmup:
            vals.append(v)
    value = statistics.mean(vals)
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": 1e3 * samples / value, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": workload_config(n, args.log2t, args.backend),
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": kind,
                         "sample": f"{samples} samples per step (same RNG streams as the GPU arm), mean of {len(vals)} runs after "
                                   f"{args.warmup} warm-up runs, encode+encode_backward per worker chunk, steady_clock; "
                                   f"unmodified reference sources (oracle/_ref) on host cores only"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "gpu_launches": 0,
    }
    print(json.dumps(line), flush=True)


def quick_dim(sx, torch, dev, device_index, n, t_log2, steps=12):
    """Fused encode fwd+bwd samples/s at another input dimension, same workload shape as the headline line."""
    N, LF = 1 << BATCH_LOG2, L * F
    cfg = sx.EncoderConfig(dim=n, levels=L, table_size=1 << t_log2, features=F, base_resolution=BASE, growth=GROWTH[n])
    enc = sx.HashEncoder(cfg, device=device_index)
    enc.init_tables(42)
    grad = sx.EncoderGradient(enc)
    sets = []
    for i in range(4):
        x = torch.empty((N, n), dtype=torch.float32, device=dev)
        r = sx.CounterRng(99, 1)
        r.counter = i * N * n
        r.fill_device(x)
        up = torch.empty((N, LF), dtype=torch.float32, device=dev)
        r2 = sx.CounterRng(7, 2)
        r2.counter = i * N * LF
        r2.fill_device(up, -1e-3, 1e-3)
        sets.append((x, up, torch.empty((N, LF), dtype=torch.float32, device=dev)))
    stream = torch.cuda.current_stream()
    for i in range(3):
        enc.encode_forward_backward(sets[i % 4][0], sets[i % 4][1], grad, out=sets[i % 4][2])
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for i in range(steps):
        enc.encode_forward_backward(sets[i % 4][0], sets[i % 4][1], grad, out=sets[i % 4][2])
    e1.record(stream)
    torch.cuda.synchronize()
    enc.check()
    ms = e0.elapsed_time(e1) / steps
    peak, _ = hbm_peak()
    return {"workload": workload_name(n, t_log2), "value": N / (ms * 1e-3), "unit": UNIT, "ms_per_step": ms, "steps": steps,
            "roofline_frac": alg_bytes(n, "fused") * N / (ms * 1e-3) / 1e9 / peak, "alg_bytes_per_sample": alg_bytes(n, "fused")}


# ---------------------------------------------------------------------------------------------- our arm
def run_ours(args):
    import torch

    import paper_2311_15439_b200 as sx

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if not torch.cuda.is_available() or sx.device_count() < 1:
        raise SystemExit("bench.py: no sm_100 CUDA device -- the GPU arm has no CPU fallback")
    n_dev = torch.cuda.device_count()
    if "WORLD_SIZE" in os.environ and world != args.gpus:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but the launcher started {world} ranks")
    if world > n_dev and not args.oversubscribe:
        raise SystemExit(f"bench.py: {world} ranks but only {n_dev} CUDA device(s) visible -- one rank per GPU "
                         f"(--oversubscribe shares devices for a functional check; its numbers are not scaling numbers)")
    device_index = local_rank % n_dev if args.oversubscribe else local_rank
    torch.cuda.set_device(device_index)
    dist = None
    if world > 1 or "WORLD_SIZE" in os.environ:  # under torchrun a single rank still drives the NCCL path
        import torch.distributed as dist_mod
        dist = dist_mod
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        if args.oversubscribe and world > n_dev:
            # NCCL refuses two ranks on one device; gloo stages CUDA tensors through the host (functional check only)
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device(f"cuda:{device_index}"))
        print(f"[bench rank {rank}/{world}] pid {os.getpid()} device cuda:{device_index} "
              f"({torch.cuda.get_device_name(device_index)}) backend {dist.get_backend()}", file=sys.stderr, flush=True)
    local_rank = device_index
    sampler = ClockSampler(local_rank)
    if rank == 0:
        sampler.start()   # runs through warm-up, the timed region and the e2e leg

    n = args.dim
    N = 1 << BATCH_LOG2
    LF = L * F
    dev = torch.device(f"cuda:{local_rank}")
    verts = (1 << n) if args.backend == "grid" else n + 1
    cfg = sx.EncoderConfig(dim=n, levels=L, table_size=1 << args.log2t, features=F, base_resolution=BASE, growth=GROWTH[n],
                           backend=1 if args.backend == "grid" else 0)
    enc = sx.HashEncoder(cfg, device=local_rank)
    enc.init_tables(42)
    tune = sx.Tuning(levels_per_thread=args.lpt, block_threads=args.block, level_major=args.level_major,
                     exact_blend=args.exact, warp_aggregate=args.aggregate, level_chunk=args.level_chunk)
    enc.set_tuning(tune)
    grad = sx.EncoderGradient(enc)

    # Rotating input sets larger than L2 in total (126 MB): each set is coords 12 MB + upstream 128 MB + out 128 MB.
    n_sets = 4
    xs, ups, outs = [], [], []
    for i in range(n_sets):
        x = torch.empty((N, n), dtype=torch.float32, device=dev)
        # rank r, set i draws its own slice of the reference bench stream CounterRng(99, 1)
        r = sx.CounterRng(99, 1)
        r.counter = (rank * n_sets + i) * N * n
        r.fill_device(x)
        up = torch.empty((N, LF), dtype=torch.float32, device=dev)
        r2 = sx.CounterRng(7, 2)
        r2.counter = (rank * n_sets + i) * N * LF
        r2.fill_device(up, -1e-3, 1e-3)
        xs.append(x)
        ups.append(up)
        outs.append(torch.empty((N, LF), dtype=torch.float32, device=dev))
    gview = grad.device_view()
    stream = torch.cuda.current_stream()

    autotune = None
    if args.path == "auto":
        # Launch-shape autotune OUTSIDE the timed region: one fused launch vs forward + backward launches, sample-major vs
        # level-major.  Which wins depends on whether tables + gradients of the walked levels fit L2 side by side
        # (profiles/r1_sweep_*.log): time each candidate for a few steps and keep the fastest.
        # (path, level_major, levels per thread, level_chunk: -1 one grid slice, 8 = the grid walks ranges of 8 levels)
        cands = [("fused", 0, 2, -1), ("fused", 0, 2, 8), ("split", 0, 2, -1), ("fused", 1, 4, -1), ("split", 1, 2, -1)]
        autotune = {}
        for path, lm, lpt, chunk in cands:
            enc.set_tuning(sx.Tuning(levels_per_thread=lpt, block_threads=args.block, level_major=lm,
                                     exact_blend=args.exact, warp_aggregate=args.aggregate, level_chunk=chunk))

            def one(i, path=path):
                k = i % n_sets
                if path == "fused":
                    enc.encode_forward_backward(xs[k], ups[k], grad, out=outs[k])
                else:
                    enc.encode(xs[k], out=outs[k])
                    enc.encode_backward(xs[k], ups[k], grad)

            for i in range(2):
                one(i)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            for i in range(8):
                one(i)
            e1.record(stream)
            torch.cuda.synchronize()
            autotune[f"{path}/level_major={lm}/lpt={lpt}/level_chunk={chunk}"] = e0.elapsed_time(e1) / 8
        if dist is not None:  # every rank must take the same path
            t = torch.tensor(list(autotune.values()), dtype=torch.float64, device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            autotune = dict(zip(autotune.keys(), [float(v) for v in t.tolist()]))
        best = min(autotune, key=autotune.get)
        path, lm, lpt, chunk = cands[list(autotune.keys()).index(best)]
        args.path = path
        enc.set_tuning(sx.Tuning(levels_per_thread=lpt, block_threads=args.block, level_major=lm, exact_blend=args.exact,
                                 warp_aggregate=args.aggregate, level_chunk=chunk))

    exchange = dist is not None and not args.no_allreduce
    # Level ranges of the overlapped exchange.  Ranges must start on whole 32-byte sectors of the feature rows (4 levels at F = 2)
    # or the launches pay for partial-sector stores, and the LAST range's all-reduce is the exposed one, so it should be small:
    # 8 + 4 + 4 levels compute in 0.500 ms on one GPU where four equal ranges take 0.518 (profiles/r2_l2_window_n3.log).
    if not exchange:
        ranges = sx.level_ranges(L, 1)
    elif args.level_ranges:
        counts = [int(c) for c in args.level_ranges.split(",")]
        assert sum(counts) == L and all(c > 0 for c in counts), "--level-ranges must add up to the level count"
        ranges, first = [], 0
        for c in counts:
            ranges.append((first, c))
            first += c
    else:
        ranges = sx.level_ranges(L, args.level_chunks)
    per_level = gview.numel() // L
    comm = torch.cuda.Stream(device=dev) if exchange else None
    # the exchange goes through the library's own communicator (sxen_comm_*: NCCL resolved with dlopen, the id carried by the
    # launcher's process group); oversubscribed functional runs (two ranks on one device, which NCCL refuses) use gloo
    abi_comm = sx.Comm.from_torch(local_rank) if exchange and dist.get_backend() == "nccl" else None

    def allreduce(t, on):
        if abi_comm is not None:
            abi_comm.allreduce(t, stream=on.cuda_stream)
        else:
            with torch.cuda.stream(on):
                dist.all_reduce(t)

    def step_overlapped(i, ev=None):
        """Batch-sharded step: the levels are walked in chunks and each chunk's slice of the table-gradient accumulator is
        all-reduced on a second stream while the next chunk computes."""
        k = i % n_sets
        if args.path != "fused":
            enc.encode(xs[k], out=outs[k])
            if ev is not None:
                ev[0].record(stream)
        for first, count in ranges:
            if args.path == "fused":
                enc.encode_forward_backward(xs[k], ups[k], grad, out=outs[k], levels=(first, count))
            else:
                enc.encode_backward(xs[k], ups[k], grad, levels=(first, count))
            done = torch.cuda.Event()
            done.record(stream)
            comm.wait_event(done)
            allreduce(gview[first * per_level:(first + count) * per_level], comm)
        if ev is not None:
            ev[1].record(stream)  # compute done; the tail of the exchange is inside the step but not inside kernel_ms
        stream.wait_stream(comm)

    def step(i, ev=None):
        if exchange and len(ranges) > 1:
            return step_overlapped(i, ev)
        k = i % n_sets
        if args.path == "fused":
            enc.encode_forward_backward(xs[k], ups[k], grad, out=outs[k])
            if ev is not None:
                ev[1].record(stream)
        else:
            enc.encode(xs[k], out=outs[k])
            if ev is not None:
                ev[0].record(stream)
            enc.encode_backward(xs[k], ups[k], grad)
            if ev is not None:
                ev[1].record(stream)
        if dist is not None and not args.no_allreduce:
            allreduce(gview, stream)  # table-gradient exchange of the batch-sharded step

    for i in range(args.warmup):
        step(i)
    grad.clear(stream.cuda_stream)  # accumulator zeroed outside the timed region
    torch.cuda.synchronize()
    enc.check()

    evs = [[torch.cuda.Event(enable_timing=True) for _ in range(3)] for _ in range(args.steps)]
    launches0 = sx.launch_count()
    if dist is not None:
        dist.barrier()
    torch.cuda.synchronize()
    t_start = torch.cuda.Event(enable_timing=True)
    t_end = torch.cuda.Event(enable_timing=True)
    if rank == 0:
        sampler.mark("timed_region_start")
    t_start.record(stream)
    for i in range(args.steps):
        evs[i][2].record(stream)
        step(i, evs[i])
    t_end.record(stream)
    torch.cuda.synchronize()
    if dist is not None:
        dist.barrier()
    launches = sx.launch_count() - launches0
    if rank == 0:
        sampler.mark("timed_region_end")
    enc.check()
    total_ms = t_start.elapsed_time(t_end)
    if dist is not None:
        t = torch.tensor([total_ms], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total_ms = float(t.item())
    ms_per_step = total_ms / args.steps
    value = world * N / (ms_per_step * 1e-3)

    # dominant kernel duration, live, from events on the launching stream
    if args.path == "fused":
        per = [e[2].elapsed_time(e[1]) for e in evs]
        kms = statistics.mean(per)
        dom, dom_bytes = "encode_fwd_bwd_fused", alg_bytes(n, "fused", verts)
        parts = {"fused_ms": kms, "fused_ms_best": min(per), "fused_ms_median": statistics.median(per)}
        if world == 1:
            # forward-only and backward-only reported next to the pair (separate launches of the same
            # kernels on the same rotating inputs, outside the headline's timed region)
            fe = [[torch.cuda.Event(enable_timing=True) for _ in range(3)] for _ in range(10)]
            for i in range(3):
                enc.encode(xs[i % n_sets], out=outs[i % n_sets])
                enc.encode_backward(xs[i % n_sets], ups[i % n_sets], grad)
            torch.cuda.synchronize()
            for i, e in enumerate(fe):
                k = i % n_sets
                e[0].record(stream)
                enc.encode(xs[k], out=outs[k])
                e[1].record(stream)
                enc.encode_backward(xs[k], ups[k], grad)
                e[2].record(stream)
            torch.cuda.synchronize()
            f_ms = [e[0].elapsed_time(e[1]) for e in fe]
            b_ms = [e[1].elapsed_time(e[2]) for e in fe]
            parts["separate_launches"] = {
                "fwd_ms": statistics.mean(f_ms), "fwd_ms_best": min(f_ms), "bwd_ms": statistics.mean(b_ms),
                "bwd_ms_best": min(b_ms),
                "fwd_frac_of_hbm": alg_bytes(n, "fwd", verts) * N / (statistics.mean(f_ms) * 1e-3) / 1e9 / hbm_peak()[0],
                "bwd_frac_of_hbm": alg_bytes(n, "bwd", verts) * N / (statistics.mean(b_ms) * 1e-3) / 1e9 / hbm_peak()[0]}
    else:
        fwd_ms = statistics.mean(e[2].elapsed_time(e[0]) for e in evs)
        bwd_ms = statistics.mean(e[0].elapsed_time(e[1]) for e in evs)
        kms, dom, dom_bytes = bwd_ms, "encode_backward", alg_bytes(n, "bwd", verts)
        parts = {"fwd_ms": fwd_ms, "bwd_ms": bwd_ms,
                 "fwd_frac_of_hbm": alg_bytes(n, "fwd", verts) * N / (fwd_ms * 1e-3) / 1e9 / hbm_peak()[0]}
    peak, peak_src = hbm_peak()
    achieved = dom_bytes * N / (kms * 1e-3) / 1e9
    roofline = {"bound": "hbm", "kernel": dom, "achieved": achieved, "peak": peak, "unit": "GB/s",
                "frac": achieved / peak, "traffic": traffic_for(f"{dom}_n{n}" + ("_grid" if args.backend == "grid" else "")), "peak_source": peak_src,
                "alg_bytes_per_sample": dom_bytes, "kernel_ms": kms, **parts}
    if args.path == "fused" and args.backend == "simplex" and n == 3 and args.log2t == T_LOG2:
        # diagnostic next to the contract's HBM figure: what binds is the request rate at both ends of the crossbar
        # (DESIGN.md 3.2).  From the SMs: ~110 requests per sample (52 gathers + 56 reds + the streamed rows); at the L2:
        # 137 tag lookups (28 reds are forwarded between the dies).  The SM-side ceiling is a pure random-gather kernel's
        # rate on this chip, 0.96 of one request per clock per SM (tools/ubench/tma_path.cu,
        # profiles/r1s3_ubench_tma_path.log).
        rate = N / (kms * 1e-3) / 1e9
        roofline["requests"] = {"sm_requests_per_sample": 110, "sm_request_rate_G_per_s": 110 * rate,
                                "measured_sm_request_peak_G_per_s": 278.6, "sm_frac": 110 * rate / 278.6,
                                "l2_lookups_per_sample": 137, "l2_lookup_rate_G_per_s": 137 * rate}

    rank_info = [{"rank": 0, "device": local_rank, "name": torch.cuda.get_device_name(local_rank), "pid": os.getpid()}]
    if dist is not None:
        gathered = [None] * world
        dist.all_gather_object(gathered, {"rank": rank, "device": local_rank, "name": torch.cuda.get_device_name(local_rank),
                                          "pid": os.getpid()})
        rank_info = gathered
    # ---- e2e: the host-buffer C-ABI call on EVERY rank (each GPU has its own PCIe link), pinned host memory, H2D + D2H inside
    # the timed region; wall clock between two barriers, max over ranks
    import ctypes as C

    import numpy as np
    lib = sx.lib

    def pinned(shape, dtype):
        nbytes = int(np.prod(shape)) * np.dtype(dtype).itemsize
        p = C.c_void_p()
        assert lib.sxen_host_alloc(nbytes, C.byref(p)) == 0, lib.sxen_last_error()
        buf = (C.c_char * nbytes).from_address(p.value)
        return np.frombuffer(buf, dtype=dtype).reshape(shape), p

    hx, px = pinned((N, n), np.float64)
    hup, pup = pinned((N, LF), np.float32)
    hout, pout = pinned((N, LF), np.float32)
    hx[:] = xs[0].double().cpu().numpy()
    hup[:] = ups[0].cpu().numpy()
    e2e_steps = max(3, args.steps)
    for _ in range(max(3, args.warmup)):
        enc.encode_forward_backward(hx, hup, grad, out=hout)
    torch.cuda.synchronize()
    if dist is not None:
        dist.barrier()
    per_step = []
    if rank == 0:
        sampler.mark("e2e_region_start")
    t0 = time.perf_counter()
    for _ in range(e2e_steps):
        t1 = time.perf_counter()
        enc.encode_forward_backward(hx, hup, grad, out=hout)   # synchronous: returns with the features in hout
        per_step.append(time.perf_counter() - t1)
    torch.cuda.synchronize()
    e2e_s = (time.perf_counter() - t0) / e2e_steps              # the mean over exactly e2e_steps calls is the value
    if rank == 0:
        sampler.mark("e2e_region_end")
    if dist is not None:
        t = torch.tensor([e2e_s], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_s = float(t.item())
    e2e = {"value": world * N / e2e_s, "unit": UNIT, "h2d_bytes_per_step": int(hx.nbytes + hup.nbytes) * world,
           "d2h_bytes_per_step": int(hout.nbytes) * world, "ms_per_step": e2e_s * 1e3, "steps": e2e_steps,
           "ms_per_step_median": statistics.median(per_step) * 1e3, "ms_per_step_min": min(per_step) * 1e3, "n_gpus": world,
           "call": "sxen_encoder_encode_forward_backward_host (x f64, upstream f32, features f32; pinned host buffers), "
                   "one call per rank per step"}
    # spot parity of the e2e result against the device path
    assert np.array_equal(hout[:4096], outs[0][:4096].cpu().numpy()) or args.exact == 0
    for p in (px, pup, pout):
        lib.sxen_host_free(p)

    line = None
    if rank == 0:
        clocks = sampler.stop()

        # ---- CPU baseline on this box's host cores (bounded sample), N=1 only
        cpu = None
        if world == 1 and not args.no_cpu and args.backend == "simplex":
            try:
                threads = host_threads()
                samples = min(1 << BATCH_LOG2, threads << 16)  # the whole 2^20 batch on >= 16 threads: ~25 core-seconds
                runs = []
                for i in range(4):   # one warm-up run (page faults of every worker's accumulator), then the mean of three
                    v, kind = cpu_reference_run(n, samples, threads, args.log2t)
                    if i > 0:
                        runs.append(v)
                cpu = {"value": statistics.mean(runs), "unit": UNIT, "cores": threads, "kind": kind, "runs": runs,
                       "sample": f"{samples} samples of the same workload (same RNG streams), mean of 3 runs after 1 warm-up "
                                 f"run, reference worker pattern: encode+encode_backward per contiguous chunk into a "
                                 f"per-thread accumulator"}
                # parity in the same run: the first 2^16 samples of this run's inputs through the device
                # path against the CPU checker -- vertex indices, weights and features bit for bit
                try:
                    import oracle
                    sub = 1 << 16
                    ocfg = oracle.Config(dim=n, levels=L, table_size=1 << args.log2t, features=F, base_resolution=BASE,
                                         growth=GROWTH[n])
                    o = oracle.Oracle()
                    xsub = xs[0][:sub].contiguous()
                    xh = xsub.double().cpu().numpy()
                    oi, ow, _, _, _ = o.encode_debug(ocfg, xh)
                    gi, gw = enc.encode_debug(xsub)
                    want, _bad = o.encode(ocfg, o.init_tables(ocfg, 42), xh[:1 << 14])
                    got = enc.encode(xsub[:1 << 14]).cpu().numpy()
                    cpu["parity"] = {"samples": sub, "indices_bit_exact": bool(np.array_equal(gi, oi)),
                                     "weights_bit_exact": bool(np.array_equal(gw, ow)),
                                     "features_bit_exact": bool(np.array_equal(got.view(np.uint32), want.view(np.uint32)))}
                except Exception as exc:
                    cpu["parity"] = {"error": str(exc)}
            except Exception as exc:  # the GPU numbers stand on their own; say why the baseline is missing
                cpu = {"value": None, "unit": UNIT, "cores": 0, "kind": "unavailable", "sample": str(exc)}

        # ---- extra (not the headline): the metric's other dimension (BASELINE.json quotes n = 2 and 3) on the same
        # protocol -- fused launch, rotating inputs, CUDA events -- with fewer steps
        other = None
        if not args.no_train and world == 1 and n == 3 and args.backend == "simplex" and args.log2t == T_LOG2:
            try:
                other = {"n2": quick_dim(sx, torch, dev, local_rank, 2, args.log2t)}
            except Exception as exc:
                other = {"error": str(exc)}

        # ---- extra (not the headline): the whole training step with the tcgen05 head on the same batch shape
        train = None
        if not args.no_train and n in (2, 3) and args.backend == "simplex":
            try:
                mlp = sx.Mlp(sx.MlpConfig(LF, 64, 2, 3), device=local_rank)
                mlp.init_params(sx.hash_combine(42, 1))
                mlp.set_precision(1)
                tr = sx.Trainer(enc, mlp)
                tgt = torch.rand((N, 3), dtype=torch.float32, device=dev)
                ta, ma = sx.AdamConfig(lr=1e-2), sx.AdamConfig(lr=1e-3)
                for _ in range(3):
                    tr.step(xs[0], tgt, ta, ma)
                torch.cuda.synchronize()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(stream)
                for i in range(8):
                    tr.step(xs[i % n_sets], tgt, ta, ma)
                e1.record(stream)
                torch.cuda.synchronize()
                tms = e0.elapsed_time(e1) / 8
                train = {"what": "encode -> tcgen05 MLP 32-64-64-3 (split bf16) fwd+MSE+bwd -> encode_backward -> sparse Adam "
                                 "+ Adam, one 2^20-sample batch per step, loss read back every step",
                         "ms_per_step": tms, "samples_per_s": N / (tms * 1e-3)}
                # the same step queued (sxen_trainer_step_enqueue, losses collected once), at 2^20 samples and at the
                # reference's default batch of 2048 (include/sxen/trainer.hpp:16)
                for key, nb, reps in (("queued", N, 8), ("queued_batch_2048", 2048, 1000)):
                    for i in range(3):
                        tr.step_enqueue(xs[i % n_sets][:nb], tgt[:nb], ta, ma)
                    tr.collect()
                    torch.cuda.synchronize()
                    e0.record(stream)
                    for i in range(reps):
                        tr.step_enqueue(xs[i % n_sets][:nb], tgt[:nb], ta, ma)
                    e1.record(stream)
                    losses, failed = tr.collect()
                    assert failed == -1 and len(losses) == reps
                    qms = e0.elapsed_time(e1) / reps
                    train[key] = {"batch": nb, "ms_per_step": qms, "samples_per_s": nb / (qms * 1e-3)}
                del tr, mlp
                if rank == 0 and world == 1 and not args.no_cpu:
                    # the reference's own train_field on the host cores, bounded: 2 steps of 2^16 samples
                    th = host_threads()
                    sec = cpu_reference_train_step(n, 1 << 16, th, t_log2=args.log2t)
                    if sec is not None:
                        train["cpu_reference"] = {"batch": 1 << 16, "cores": th, "ms_per_step": sec * 1e3,
                                                  "samples_per_s": (1 << 16) / sec,
                                                  "what": "the unmodified reference's train_field (oracle/_ref): (3-step run - "
                                                          "1-step run) / 2, wall clock"}
            except Exception as exc:
                train = {"error": str(exc)}

        t = enc.tuning()
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": "f64 lattice math / u32 hash / f32 features+grads", "data": "synthetic",
            "config": workload_config(n, args.log2t, args.backend),
            "launch": {"coords": "f32 on device", "path": args.path, "autotune_ms": autotune,
                       "ranks": rank_info,
                       "l2_policy": f"inputs larger than L2: {n_sets} rotating input sets x 268 MB, plus "
                                    f"{L * (1 << args.log2t) * F * 4 >> 20} MiB tables and as much gradient accumulator",
                       "tuning": {"levels_per_thread": t.levels_per_thread, "block_threads": t.block_threads,
                                  "level_major": t.level_major, "exact_blend": t.exact_blend,
                                  "warp_aggregate": t.warp_aggregate, "level_chunk": t.level_chunk},
                       "multi_gpu": (f"batch sharded over {world} ranks, tables replicated, "
                                     f"{'sxen_comm_allreduce (NCCL)' if abi_comm is not None else dist.get_backend()} SUM all-reduce of "
                                     f"the {L * (1 << args.log2t) * F * 4 >> 20} MiB table-gradient accumulator per step in "
                                     f"{len(ranges)} level chunks overlapped with the next chunk's kernel")
                                    if exchange else (f"{world} replicas, no exchange (--no-allreduce)" if world > 1
                                                      else "single GPU"),
                       "oversubscribed": bool(args.oversubscribe and world > n_dev)},
            "clocks": clocks, "e2e": e2e, "gpu_launches": int(launches), "roofline": roofline, "cpu_baseline": cpu,
            "train_step": train, "other_dims": other,
        }
    if dist is not None:
        dist.barrier()
        dist.destroy_process_group()
    if line is not None:
        print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=30)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--dim", type=int, default=3, choices=[2, 3, 4, 5, 6])
    ap.add_argument("--log2t", type=int, default=T_LOG2, help="log2 of the table size (19 = BASELINE configs[1], 22 = the sweep)")
    ap.add_argument("--backend", choices=["simplex", "grid"], default="simplex",
                    help="grid = the paper's comparator (2^n corners, n-linear weights), n = 2 or 3")
    ap.add_argument("--path", choices=["auto", "fused", "split"], default="auto")
    ap.add_argument("--lpt", type=int, default=0)
    ap.add_argument("--block", type=int, default=0)
    ap.add_argument("--level-major", type=int, default=-1)
    ap.add_argument("--level-chunk", type=int, default=0, help="sxen_tuning.level_chunk for --path fused|split (0 = library default)")
    ap.add_argument("--exact", type=int, default=1)
    ap.add_argument("--aggregate", type=int, default=0)
    ap.add_argument("--no-allreduce", action="store_true")
    ap.add_argument("--level-ranges", default="8,4,4",
                    help="multi-GPU: level counts of the ranges whose gradient all-reduce overlaps the next range's kernel "
                         "(empty = --level-chunks equal ranges)")
    ap.add_argument("--level-chunks", type=int, default=4,
                    help="multi-GPU: level chunks whose gradient all-reduce overlaps the next chunk's kernel")
    ap.add_argument("--oversubscribe", action="store_true",
                    help="functional check only: let ranks share devices (rank %% device count) over gloo")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-train", action="store_true")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3) if args.impl == "ours" else args.warmup
    if args.impl == "reference":
        run_reference(args)
    elif args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(spawn_ranks(args))
    else:
        run_ours(args)


def spawn_ranks(args) -> int:
    """`python bench.py --gpus N` outside a launcher: re-run this command line as N ranks, one per GPU, the way the driver
    does (python -m torch.distributed.run --nnodes=1 --nproc-per-node N --master-addr 127.0.0.1 --master-port P).  Fails
    loudly when the box has fewer than N devices (unless --oversubscribe)."""
    import socket

    import torch
    n_dev = torch.cuda.device_count() if torch.cuda.is_available() else 0
    if n_dev < 1:
        raise SystemExit("bench.py: no sm_100 CUDA device -- the GPU arm has no CPU fallback")
    if n_dev < args.gpus and not args.oversubscribe:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but only {n_dev} CUDA device(s) visible on this box")
    with socket.socket() as sock:
        sock.bind(("127.0.0.1", 0))
        port = sock.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__)] + sys.argv[1:]
    env = dict(os.environ)
    env.setdefault("OMP_NUM_THREADS", "1")
    print("[bench] spawning:", " ".join(cmd), file=sys.stderr, flush=True)
    return subprocess.call(cmd, env=env)


if __name__ == "__main__":
    main()
