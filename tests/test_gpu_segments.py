"""GPU: program segmentation (bounded partial rows, bloch_last_segments).

With a tiny BLOCH_PARTIAL_BUDGET_MB the op stream runs as many launches, the fp64
state handed over through global memory and each segment's samples folded
before the next; echoes and snapshots must be bit-identical to one launch, for
programs with windows, chirps, generic samples, RF trains and snapshots, in
both precisions and with several coils.  The window contraction is off here: it keeps no partial rows
(its U rows must fit the budget, else the windows stay in the integrator, tested below)."""

import json
import os
import subprocess
import sys

import numpy as np
import pytest

import cases
from conftest import load_golden
from paper_1305_6861_b200 import SpinBlock, compute_block, precompute_sequence_tables

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
NAMES = ["mixed", "mixed_coils", "tse16", "epi16", "se16_box"]

_CHILD = r"""
import json, sys
import numpy as np
sys.path.insert(0, sys.argv[1]); sys.path.insert(0, sys.argv[1] + "/tests"); sys.path.insert(0, sys.argv[1] + "/tests/golden")
import cases
from conftest import load_golden
from paper_1305_6861_b200 import SpinBlock, precompute_sequence_tables
from paper_1305_6861_b200.engine import get_engine
name, precision, out = sys.argv[2], int(sys.argv[3]), sys.argv[4]
rec = load_golden(name)
t = precompute_sequence_tables(cases.small_cases()[name]["sequence"], snapshot_times=tuple(rec["snapshot_times"].tolist()))
eng = get_engine(0, precision)
eng.set_contraction(False)  # the integrator's own window sums: the rows the segments bound
e, s = eng.compute(t, rec["spin_pos"], rec["spin_mx"], rec["spin_my"], rec["spin_mz"], rec["spin_t1"], rec["spin_t2"],
                   rec["spin_m0"], rec["spin_domega"], rec["spin_weight"])
np.savez(out, echoes=e, **{f"snap{i}": x for i, x in enumerate(s) if x is not None})
print(json.dumps({"segments": eng.last_segments()}))
"""


@pytest.mark.parametrize("precision", [32, 64])
@pytest.mark.parametrize("name", NAMES)
def test_segmented_program_bit_identical(name, precision, tmp_path):
    rec = load_golden(name)
    t = precompute_sequence_tables(cases.small_cases()[name]["sequence"],
                                   snapshot_times=tuple(rec["snapshot_times"].tolist()))
    b = SpinBlock(index=0, pos=rec["spin_pos"], mx=rec["spin_mx"], my=rec["spin_my"], mz=rec["spin_mz"],
                  t1=rec["spin_t1"], t2=rec["spin_t2"], m0=rec["spin_m0"], domega=rec["spin_domega"],
                  weight=rec["spin_weight"])
    from paper_1305_6861_b200.engine import get_engine

    eng = get_engine(0, precision)
    eng.set_contraction(False)
    try:
        e1, s1 = compute_block(t, b, precision=precision)
    finally:
        eng.set_contraction(True)
    out = str(tmp_path / "seg.npz")
    env = dict(os.environ, BLOCH_PARTIAL_BUDGET_MB="0.002")  # ~2 KB of partial rows per launch
    r = subprocess.run([sys.executable, "-c", _CHILD, ROOT, name, str(precision), out], capture_output=True,
                       text=True, env=env, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    info = json.loads(r.stdout.strip().splitlines()[-1])
    assert info["segments"] > 1, info
    got = np.load(out)
    assert np.array_equal(got["echoes"], e1)
    for i, x in enumerate(s1):
        if x is not None:
            assert np.array_equal(got[f"snap{i}"], x), i


@pytest.mark.parametrize("name", ["tse16", "mixed_coils"])
def test_contraction_over_budget_falls_back_to_integrator_sums(name, tmp_path):
    """A partial budget too small for the U rows: the call runs without the contraction (every window summed by
    the integrator, in segments) and still matches the reference golden."""
    from oracle.bloch_oracle import rel_l2

    rec = load_golden(name)
    out = str(tmp_path / "seg.npz")
    child = _CHILD.replace("eng.set_contraction(False)  # the integrator's own window sums: the rows the segments bound\n",
                           "")
    child += "print(json.dumps({'groups': eng.last_phases()['groups']}))\n"
    env = dict(os.environ, BLOCH_PARTIAL_BUDGET_MB="0.00001")  # ~10 bytes: below any U array
    r = subprocess.run([sys.executable, "-c", child, ROOT, name, "32", out], capture_output=True, text=True, env=env,
                       timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    info = json.loads(r.stdout.strip().splitlines()[-1])
    assert info["groups"] == 0
    got = np.load(out)
    assert rel_l2(rec["echo_full"], got["echoes"]) <= 1e-4


_CHILD_LARGE = r"""
import json, sys
import numpy as np, torch
sys.path.insert(0, sys.argv[1])
from paper_1305_6861_b200 import configs
from paper_1305_6861_b200.engine import get_engine, precompute_sequence_tables
cfg, precision, n, out = int(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4]), sys.argv[5]
w = configs.make(cfg)
b, C = w.block, w.n_coils
seq = w.sequence
t = precompute_sequence_tables(seq, snapshot_times=(seq.end_time,))
dev = torch.device("cuda", 0)
f = lambda a: torch.from_numpy(np.ascontiguousarray(a[:n], dtype=np.float64)).to(dev)
wt = np.ascontiguousarray(np.asarray(b.weight, dtype=np.complex128).reshape(C, b.n)[:, :n]).view(np.float64)
d = dict(pos=f(b.pos), mx=f(b.mx), my=f(b.my), mz=f(b.mz), t1=f(b.t1), t2=f(b.t2), m0=f(b.m0), domega=f(b.domega),
         weight=torch.from_numpy(wt).to(dev))
ptrs = {k: v.data_ptr() for k, v in d.items()}
eng = get_engine(0, precision)
eng.set_contraction(False)  # the integrator's own window sums: the rows the segments bound
fl = eng.set_tables(t)
echo = torch.zeros(C * fl["n_acq"] * fl["max_ns"] * 2, dtype=torch.float64, device=dev)
snap = torch.zeros(n * 3, dtype=torch.float64, device=dev)
outs = []
for it in range(4):  # identical device-resident calls: the graph is recorded on the second and replayed after
    echo.zero_(); snap.zero_()
    eng.compute_device(t, ptrs, n, C, echo.data_ptr(), snap.data_ptr(), sync=True)
    outs.append((echo.cpu().numpy().copy(), snap.cpu().numpy().copy()))
for e, s in outs[1:]:
    assert np.array_equal(e, outs[0][0]) and np.array_equal(s, outs[0][1]), "replay differs"
np.savez(out, echoes=outs[0][0], snap=outs[0][1])
print(json.dumps({"segments": eng.last_segments(), "launch": eng.last_launch()}))
"""


@pytest.mark.slow
@pytest.mark.parametrize("cfg,precision", [(1, 32), (1, 64), (4, 32), (4, 64)])
def test_segmented_large_block_bit_identical(cfg, precision, tmp_path):
    """A multi-row grid (80,000 spins of config 1, one coil, and of config 4, eight coils), both precisions,
    through compute_device called four times (CUDA-graph capture and replay): a partial budget that cuts the
    program into several segments must reproduce the one-launch result bit for bit."""
    n = 80000
    res = {}
    for tag, budget in (("one", None), ("cut", "64")):
        out = str(tmp_path / f"{tag}.npz")
        env = dict(os.environ)
        if budget:
            env["BLOCH_PARTIAL_BUDGET_MB"] = budget
        r = subprocess.run([sys.executable, "-c", _CHILD_LARGE, ROOT, str(cfg), str(precision), str(n), out],
                           capture_output=True, text=True, env=env, timeout=900)
        assert r.returncode == 0, r.stderr[-2000:]
        res[tag] = (json.loads(r.stdout.strip().splitlines()[-1]), np.load(out))
    # (eight coils in fp64 already need two segments under the default 24 GiB budget)
    assert res["cut"][0]["segments"] > res["one"][0]["segments"] >= 1, (res["one"][0], res["cut"][0])
    assert np.array_equal(res["one"][1]["echoes"], res["cut"][1]["echoes"])
    assert np.array_equal(res["one"][1]["snap"], res["cut"][1]["snap"])
    assert np.abs(res["one"][1]["echoes"]).max() > 0
