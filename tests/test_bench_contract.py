"""The bench.py JSON line keeps the driver's contract (small run on the GPU; the reference arm on CPU)."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _line(args, timeout=900):
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], capture_output=True, text=True,
                       timeout=timeout, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, r.stdout[-2000:]
    return json.loads(lines[0])


@pytest.mark.gpu
def test_bench_line_has_every_contract_key():
    d = _line(["--steps", "3", "--warmup", "3", "--points", "2000000", "--no-secondary"])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
              "vs_baseline", "dtype", "data", "config", "roofline", "gpu_launches", "clocks", "e2e"):
        assert k in d, k
    assert d["n_gpus"] == 1 and d["steps"] == 3 and d["warmup"] == 3 and d["value"] > 0 and d["ms_per_step"] > 0
    assert d["config"]["workload"] and d["gpu_launches"] == 15
    r = d["roofline"]
    assert r["bound"] == "hbm" and r["unit"] == "GB/s" and 0 < r["frac"] < 1.2 and r["peak"] > 0
    assert abs(r["frac"] - r["achieved"] / r["peak"]) < 1e-9
    st = d["ms_per_step_stats"]
    assert st["frames"] == 3 and st["p10"] <= st["median"] <= st["p90"]
    cb = d["cpu_baseline"]
    assert cb["kind"] == "oracle" and cb["value"] > 0 and cb["cores"] == cb["omp_threads"] >= 1
    assert cb["os_cpu_count"] == os.cpu_count() and cb["single_thread"]["cores"] == 1
    e = d["e2e"]
    assert e["value"] > 0 and e["h2d_bytes_per_step"] > 0 and e["d2h_bytes_per_step"] > 0
    assert e["copy_all"]["value"] > 0 and e["copy_all"]["h2d_bytes_per_step"] > e["h2d_bytes_per_step"]


def test_reference_arm_line():
    d = _line(["--impl", "reference", "--steps", "1", "--warmup", "0", "--points", "300000", "--ref-sample", "50000"])
    assert d["impl"] == "reference" and d["value"] > 0 and d["cpu_baseline"]["kind"] == "oracle"
    assert d["cpu_baseline"]["cores"] >= 1 and d["cpu_baseline"]["os_cpu_count"] == os.cpu_count()
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["unit"] == d["unit"]


@pytest.mark.gpu
def test_bench_view_mode_line():
    """--mode view: the configs[4] training step (fwd+bwd over 16 views), same JSON contract."""
    d = _line(["--mode", "view", "--steps", "2", "--warmup", "3"])
    for k in ("metric", "value", "unit", "n_gpus", "ms_per_step", "roofline", "e2e", "clocks", "gpu_launches"):
        assert k in d, k
    assert d["n_gpus"] == 1 and d["config"]["views_total"] == 16 and d["value"] > 0
    assert 0 < d["roofline"]["frac"] < 1.2 and d["e2e"]["h2d_bytes_per_step"] > 0
