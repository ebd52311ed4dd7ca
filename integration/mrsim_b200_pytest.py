"""pytest plugin: run the reference's own test suite with its kernel swapped for the B200 engine.

    PYTHONPATH=baseline/_ref:integration MRSIM_B200_PRECISION=64 \
        python -m pytest baseline/_ref/mrsim_tests -p mrsim_b200_pytest

Installs ``mrsim_b200.compute_block_b200`` as ``mrsim.engine.compute_block`` before any test module
imports it (so ``from mrsim.engine import compute_block`` in the tests binds the GPU kernel too), and
switches the reference's process pool (``_run_pool``, engine.py:540-595) to the forkserver start
method with this module preloaded: every worker process gets the patched engine and opens its own
CUDA context (a plain fork after the parent initialised CUDA could not).  At the end it writes the
number of GPU calls made in the main process to $MRSIM_B200_CALLS_FILE.
"""

import multiprocessing as mp
import os

import mrsim_b200

mrsim_b200.install()
if mp.current_process().name == "MainProcess":
    try:
        mp.set_start_method("forkserver", force=True)
        mp.set_forkserver_preload(["mrsim_b200_pytest"])
    except (RuntimeError, ValueError):
        pass


def pytest_sessionfinish(session, exitstatus):
    path = os.environ.get("MRSIM_B200_CALLS_FILE")
    if path:
        with open(path, "w") as fh:
            fh.write(str(mrsim_b200.calls()))
