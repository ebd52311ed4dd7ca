"""GPU: the reference's OWN test suite with its kernel swapped for the B200 engine.

The unmodified reference (``mrsim``, installed into baseline/_ref by tools/install_reference.sh,
git-ignored; it travels to the GPU box with the repository snapshot) runs its own tests with
``mrsim.engine.compute_block`` replaced by ``integration/mrsim_b200.compute_block_b200`` — the
ctypes stub over the C-ABI a reference maintainer would add — in the fp64 mode (the reference's
unit tests compare at 1e-12 .. 1e-14), served by one GPU process (integration/mrsim_b200_pytest.py).
``run`` (engine.py:465-537), its process pool (``_run_pool``, engine.py:540-595, the reference's
own fork workers), ``simulate_spin`` (engine.py:313-335) and the tests' own ``compute_block`` calls
all reach the GPU:
test_engine.py (tables, single-spin physics, partition invariance, worker determinism, linearity,
m0 scaling, worker-panic fault injection, snapshots, split intervals, metrics, files) and the
acceptance criteria (Hahn echo, k-t vs spin engine, head phantom, TSE ghost, CPMG T2 mapping,
parallel determinism, ...).

Deselected: criterion 11 (test_acceptance.py:541-568), a gate on the reference's own CPU process
scaling η(4)/η(1) of run(), which says nothing about the kernel.
"""

import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = os.path.join(ROOT, "baseline", "_ref")
TESTS = os.path.join(REF, "mrsim_tests")


def test_reference_suite_with_b200_compute_block(tmp_path):
    if not (os.path.isdir(os.path.join(REF, "mrsim")) and os.path.isdir(TESTS)):
        pytest.skip("baseline/_ref not installed (tools/install_reference.sh)")
    calls = tmp_path / "calls.txt"
    env = dict(os.environ, PYTHONPATH=os.pathsep.join([REF, os.path.join(ROOT, "integration"), TESTS]),
               MRSIM_B200_PRECISION="64", MRSIM_B200_CALLS_FILE=str(calls),
               MRSIM_B200_LIB=os.path.join(ROOT, "paper_1305_6861_b200", "libbloch_b200.so"),
               OPENBLAS_NUM_THREADS="1", OMP_NUM_THREADS="1")
    cmd = [sys.executable, "-m", "pytest", TESTS, "-q", "-p", "mrsim_b200_pytest", "-p", "no:cacheprovider",
           "-k", "not criterion_11", "-rf"]
    r = subprocess.run(cmd, cwd=TESTS, env=env, capture_output=True, text=True, timeout=1800)
    tail = (r.stdout + r.stderr)[-4000:]
    print(tail)
    assert r.returncode == 0, tail
    assert "passed" in r.stdout and " failed" not in r.stdout
    assert int(calls.read_text()) > 50, "the reference's kernel calls did not reach the B200 engine"
