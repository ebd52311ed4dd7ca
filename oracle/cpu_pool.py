"""Multiprocess CPU run of the oracle — TEST / BASELINE INFRASTRUCTURE ONLY.

Restates the reference's worker pool (``engine._run_pool``, engine.py:540-595):
contiguous blocks (``partition_blocks``, engine.py:229-251; default 4 blocks per
worker, engine.py:478) evolved in forked worker processes, partials folded in
ascending block order (deterministic mode, engine.py:594-595).  BLAS threads
are pinned to one per worker — without that the pool oversubscribes the cores
(3.5x slower).  Used for bench.py's ``cpu_baseline`` and
``--impl reference`` arm; never by the product.
"""

from __future__ import annotations

import multiprocessing as mp
import os
import time
from typing import Dict, Optional

import numpy as np

from . import bloch_oracle as O

_G: Dict = {}


def _init(tables, arrays):
    _G["tables"] = tables
    _G["arrays"] = arrays
    try:
        from threadpoolctl import threadpool_limits

        _G["limits"] = threadpool_limits(1)
    except Exception:  # threadpoolctl missing: rely on the env vars set by the parent
        pass


def _work(bounds):
    lo, hi = bounds
    a = _G["arrays"]
    w = np.asarray(a["weight"])
    echoes, snaps = O.compute_block(
        _G["tables"], a["pos"][lo:hi], a["mx"][lo:hi], a["my"][lo:hi], a["mz"][lo:hi], a["t1"][lo:hi],
        a["t2"][lo:hi], a["m0"][lo:hi], a["domega"][lo:hi], w[..., lo:hi],
    )
    return echoes, snaps


def run_pool(tables, arrays: Dict[str, np.ndarray], workers: Optional[int] = None, blocks: Optional[int] = None):
    """Evolve all spins of ``arrays`` on ``workers`` processes; returns (echo_sum, snapshots, wall_s).

    ``arrays`` holds the SpinBlock fields (pos, mx, my, mz, t1, t2, m0, domega,
    weight).  Snapshots are concatenated in block order (engine.py:497-504).
    """
    workers = workers or os.cpu_count() or 1
    n = int(np.asarray(arrays["mx"]).size)
    blocks = blocks or 4 * workers
    bounds = O.partition_bounds(n, blocks)
    pairs = [(int(bounds[i]), int(bounds[i + 1])) for i in range(len(bounds) - 1)]
    for k in ("OPENBLAS_NUM_THREADS", "OMP_NUM_THREADS", "MKL_NUM_THREADS"):
        os.environ.setdefault(k, "1")
    ctx = mp.get_context("fork")
    t0 = time.perf_counter()
    if workers == 1:
        _init(tables, arrays)
        results = [_work(p) for p in pairs]
    else:
        with ctx.Pool(workers, initializer=_init, initargs=(tables, arrays)) as pool:
            results = pool.map(_work, pairs, chunksize=1)  # returned in block order
    wall = time.perf_counter() - t0
    echo_sum = None
    for e, _ in results:
        echo_sum = e if echo_sum is None else echo_sum + e
    n_snap = len(tables.snapshot_times)
    snaps = []
    for i in range(n_snap):
        parts = [s[i] for _, s in results if s[i] is not None]
        snaps.append(np.vstack(parts) if parts else None)
    return echo_sum, snaps, wall
