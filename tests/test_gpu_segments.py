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
