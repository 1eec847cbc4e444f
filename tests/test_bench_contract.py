"""bench.py's JSON line: the keys the driver reads, for the reference arm (CPU, runs here) and for our arm (GPU)."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BASE_KEYS = {"metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
             "vs_baseline", "dtype", "data", "config", "e2e", "cpu_baseline"}


def run_bench(*flags, timeout=600):
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *flags], capture_output=True, text=True,
                         timeout=timeout, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, out.stdout[-2000:]
    return json.loads(lines[0])


def test_reference_arm_line():
    """--impl reference: the unmodified reference's encode + encode_backward on the host cores (oracle/_ref, else the
    oracle port), same metric / unit / workload as our arm, e2e repeating the line's value with zero copy bytes."""
    d = run_bench("--impl", "reference", "--steps", "1", "--warmup", "0")
    assert BASE_KEYS <= set(d), sorted(BASE_KEYS - set(d))
    assert d["impl"] == "reference" and d["metric"] == "simplex_encode_fwd_bwd_samples_per_s" and d["unit"] == "samples/s"
    assert d["higher_is_better"] is True and d["vs_baseline"] is None and d["value"] > 0
    assert d["cpu_baseline"]["kind"] in ("reference", "port") and d["cpu_baseline"]["cores"] >= 1
    assert d["cpu_baseline"]["value"] == d["value"] and d["cpu_baseline"]["sample"]
    assert d["e2e"] == {"value": d["value"], "unit": d["unit"], "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}
    assert "workload" in d["config"] and "3D simplex encode" in d["config"]["workload"]


@pytest.mark.gpu
def test_our_arm_line():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    d = run_bench("--steps", "5", "--warmup", "3", "--no-train")
    assert BASE_KEYS | {"clocks", "gpu_launches", "roofline"} <= set(d)
    assert d["metric"] == "simplex_encode_fwd_bwd_samples_per_s" and d["unit"] == "samples/s" and d["n_gpus"] == 1
    assert d["steps"] == 5 and d["warmup"] == 3 and d["scaling"] == "weak" and d["data"] == "synthetic"
    assert d["value"] > 1e8 and abs(d["value"] - (1 << 20) / (d["ms_per_step"] * 1e-3)) <= 1e-6 * d["value"]
    assert d["gpu_launches"] >= d["steps"]
    r = d["roofline"]
    assert r["bound"] == "hbm" and r["unit"] == "GB/s" and r["peak"] > 1000
    assert abs(r["frac"] - r["achieved"] / r["peak"]) < 1e-9 and 0.05 < r["frac"] < 1.0
    assert r["alg_bytes_per_sample"] == 1816 and (r["traffic"] is None or r["traffic"] > 0)
    e = d["e2e"]
    assert e["value"] > 0 and e["h2d_bytes_per_step"] == (1 << 20) * (3 * 8 + 32 * 4) and e["d2h_bytes_per_step"] == (1 << 20) * 32 * 4
    assert e["value"] < d["value"]  # PCIe both ways cannot beat the resident-input number
    c = d["cpu_baseline"]
    assert c["kind"] in ("reference", "port") and c["cores"] >= 1 and c["value"] > 0
    assert "workload" in d["config"] and "model" not in d["config"]
    assert set(d["clocks"]) >= {"sm_mhz", "sm_max_mhz", "reasons"}


def test_gpus_flag_without_devices_fails_loudly():
    """`python bench.py --gpus 2` outside a launcher re-runs itself as two ranks (one per GPU); on a box that does not have
    them -- this container has none -- it must say so and exit non-zero, never fall back to fewer ranks or to the CPU."""
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--steps", "1"], capture_output=True,
                         text=True, timeout=300, cwd=ROOT, env=env)
    torch = pytest.importorskip("torch")
    if torch.cuda.is_available() and torch.cuda.device_count() >= 2:
        pytest.skip("this box has the devices")
    assert out.returncode != 0
    assert "CUDA device" in (out.stderr + out.stdout)
    assert not [l for l in out.stdout.splitlines() if l.startswith("{")]   # no bench line of a run that did not happen
