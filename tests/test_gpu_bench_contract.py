"""bench.py's one-line JSON contract (the driver parses it): our arm and the
reference arm at N=1, short runs."""

import json
import subprocess
import sys
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu

ROOT = Path(__file__).resolve().parents[1]


def _bench(*args):
    out = subprocess.run([sys.executable, str(ROOT / "bench.py"), *args], cwd=ROOT, capture_output=True, text=True,
                         timeout=600)
    assert out.returncode == 0, out.stderr[-3000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.strip()]
    assert len(lines) == 1, out.stdout[-2000:]
    return json.loads(lines[0])


def test_bench_line_ours():
    d = _bench("--steps", "2", "--warmup", "3", "--cpu-iters", "300")
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
              "vs_baseline", "dtype", "data", "config", "e2e", "gpu_launches", "roofline", "cpu_baseline", "clocks"):
        assert k in d, k
    assert d["n_gpus"] == 1 and d["steps"] == 2 and d["warmup"] == 3 and d["higher_is_better"] is True
    assert d["value"] > 0 and d["gpu_launches"] >= 2 and "workload" in d["config"]
    e = d["e2e"]
    assert e["value"] > 0 and e["unit"] == d["unit"] and e["h2d_bytes_per_step"] > 0 and e["d2h_bytes_per_step"] > 0
    r = d["roofline"]
    assert r["bound"] in ("hbm", "tensor") and r["unit"] == "GB/s" and r["peak"] > 0
    assert r["frac"] == pytest.approx(r["achieved"] / r["peak"])
    assert r["frac_b_iter"] == pytest.approx(r["achieved_b_iter"] / r["peak"]) and r["b_iter"] > 0
    c = d["cpu_baseline"]
    assert c["value"] > 0 and c["cores"] >= 1 and c["kind"] in ("port", "reference") and c["sample"]
    assert set(d["clocks"]) >= {"sm_mhz", "sm_max_mhz", "reasons"}


def test_bench_line_reference_arm():
    d = _bench("--impl", "reference", "--steps", "1", "--warmup", "1")
    assert d["impl"] == "reference" and d["value"] > 0 and d["unit"] == "iters/s"
    assert d["e2e"]["value"] == d["value"] and d["e2e"]["h2d_bytes_per_step"] == 0
    assert d["cpu_baseline"]["value"] == d["value"] and d["cpu_baseline"]["kind"] in ("port", "reference")


def test_both_arms_time_the_same_window():
    """Same trace, same window, same config dict: the driver's same_config check."""
    ours = _bench("--steps", "2", "--warmup", "3", "--no-e2e", "--no-cpu-baseline")
    ref = _bench("--impl", "reference", "--steps", "2", "--warmup", "3")
    assert ours["config"] == ref["config"]
    c = ours["config"]
    assert c["window_start_iteration"] == 5 + 3 * c["iters_per_step"]
    assert c["window_end_iteration"] == c["window_start_iteration"] + 2 * c["iters_per_step"]
    assert 0 < c["pending_requests_start"] <= 1_000_000
