"""bench.py keeps the driver's JSON-line contract (reference arm on CPU, our arm on a GPU)."""

import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(args, timeout=600):
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], capture_output=True, text=True,
                         timeout=timeout, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [l for l in out.stdout.splitlines() if l.strip().startswith("{")]
    assert len(lines) == 1, out.stdout
    return json.loads(lines[0])


def test_reference_arm_contract():
    d = _run(["--impl", "reference", "--config", "0", "--steps", "1", "--warmup", "0", "--cpu-spins-per-core", "8",
              "--quiet"])
    assert d["impl"] == "reference"
    assert d["metric"] == "isochromat-event updates/s" and d["unit"] == d["metric"]
    assert d["value"] > 0 and d["higher_is_better"] is True
    assert d["cpu_baseline"]["kind"] == "port" and d["cpu_baseline"]["cores"] >= 1
    assert d["e2e"] == {"value": d["value"], "unit": d["unit"], "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}
    assert d["config"]["events_per_spin"] == 4480


@pytest.mark.gpu
def test_gpu_arm_contract():
    d = _run(["--config", "0", "--steps", "3", "--warmup", "3", "--no-cpu-baseline", "--quiet"])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
              "vs_baseline", "dtype", "data", "config", "roofline", "e2e", "gpu_launches", "clocks"):
        assert k in d, k
    assert d["steps"] == 3 and d["warmup"] == 3 and d["n_gpus"] == 1
    assert d["value"] > 0 and d["gpu_launches"] >= 3 * 3
    r = d["roofline"]
    assert r["peak"] > 0 and r["achieved"] > 0 and abs(r["frac"] - r["roofline_ms"] / r["kernel_ms"]) < 1e-9
    e = d["e2e"]
    assert e["value"] > 0 and e["h2d_bytes_per_step"] > 0 and e["d2h_bytes_per_step"] > 0
    assert d["config"]["workload"] == "cfg0_se64"
