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
    assert d["cpu_baseline"]["kind"] in ("port", "reference") and d["cpu_baseline"]["cores"] >= 1
    assert d["e2e"] == {"value": d["value"], "unit": d["unit"], "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}
    assert d["config"]["events_per_spin"] == 4480
    assert d["n_gpus"] == 1 and d["scaling"] == "strong"


def test_spawn_path_runs_one_rank_per_gpu_dry():
    """`python bench.py --gpus 2` (no torchrun env) re-launches itself with 2 ranks; --dry runs the
    plumbing (np.linspace shards, one gloo reduce, max-over-ranks time) without a GPU."""
    d = _run(["--gpus", "2", "--dry", "--config", "0", "--steps", "2", "--warmup", "0", "--quiet"])
    assert d["n_gpus"] == 2 and d["dry"] is True and d["scaling"] == "strong"
    assert d["spins_reduced"] == d["config"]["spins_total"] == 2444  # the two shards cover the config once
    assert d["config"]["parallelism"] == "spin-shards x2"


def test_reference_arm_config_dict_matches_ours():
    """Both arms build their `config` object with the same function from the same workload."""
    ref = _run(["--impl", "reference", "--gpus", "2", "--config", "0", "--steps", "1", "--warmup", "0",
                "--cpu-spins-per-core", "8", "--quiet"])
    ours = _run(["--gpus", "2", "--dry", "--config", "0", "--steps", "1", "--warmup", "0", "--quiet"])
    assert ref["config"] == ours["config"]
    assert ref["n_gpus"] == ours["n_gpus"] == 2


def test_world_size_mismatch_is_an_error():
    env = dict(os.environ, WORLD_SIZE="1", RANK="0", LOCAL_RANK="0")
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--dry", "--quiet"],
                         capture_output=True, text=True, timeout=300, cwd=ROOT, env=env)
    assert out.returncode != 0 and "WORLD_SIZE" in out.stderr


@pytest.mark.gpu
def test_gpu_arm_contract():
    d = _run(["--config", "0", "--steps", "3", "--warmup", "3", "--no-cpu-baseline", "--no-per-config",
              "--no-projection", "--quiet"])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
              "vs_baseline", "dtype", "data", "config", "roofline", "e2e", "gpu_launches", "clocks"):
        assert k in d, k
    assert d["steps"] == 3 and d["warmup"] == 3 and d["n_gpus"] == 1
    assert d["value"] > 0 and d["gpu_launches"] >= 3 * 3
    r = d["roofline"]
    assert r["peak"] > 0 and r["achieved"] > 0 and abs(r["frac"] - r["achieved"] / r["peak"]) < 1e-9
    assert r["bound"] in ("hbm", "tensor") and 0 < r["share_of_step"] <= 1  # the step's dominant kernel
    ri = d["roofline_integrator"]
    assert ri["bound"] == "hbm" and ri["algorithmic_bytes"] > 0 and ri["model_frac"] > 0
    assert ri["kernel"] == "resident_integrate_kernel" and d["integrator_launch"]["resident"] == 1
    rc = d["roofline_contraction"]  # config 0's readouts go through the tensor-core contraction
    assert rc["bound"] == "tensor" and rc["achieved"] > 0 and abs(rc["frac"] - rc["achieved"] / rc["peak"]) < 1e-9
    assert d["phases_ms"]["contract"] > 0 and d["phases_ms"]["integrate"] > 0
    e = d["e2e"]
    assert e["value"] > 0 and e["h2d_bytes_per_step"] > 0 and e["d2h_bytes_per_step"] > 0
    assert d["config"]["workload"] == "cfg0_se64"
