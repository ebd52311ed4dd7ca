"""Full-size goldens of configs 1 and 3, computed by the REFERENCE itself (build container only).

    python tests/golden/make_golden_full.py [--ref /root/reference/pkg/src] [--only 1 3] [--workers 8]

Every spin of the config (697,708 for config 1, 732,380 for config 3 — no subset) runs through
the reference's own ``precompute_sequence_tables`` (engine.py:83-164), ``partition_blocks``
(engine.py:229-251) and worker pool ``_run_pool`` (engine.py:540-595, deterministic fold in
ascending block order), i.e. the reference's ``compute_block`` (engine.py:259-310) in
``workers`` processes with one BLAS thread each.  The final magnetisation comes from a snapshot
at the end of the sequence, concatenated in block order (engine.py:497-504).

Stored in ``tests/golden/full_cfg{i}.npz`` (committed):

* the whole k-space (un-normalised partial sum, complex128 (n_acq, max_ns)) — 1 MB / 0.3 MB;
* the final magnetisation of every 64th spin in rasterisation order (full rows, (n/64, 3));
* checksums of the whole final magnetisation: per-component sums, the squared norm, and
  projections on a seeded random vector, so the full array is pinned without storing 17 MB.

The tests never import the reference; this script is the only place that does.
"""

from __future__ import annotations

import argparse
import os
import sys
import time
from types import SimpleNamespace

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
sys.path.insert(0, HERE)

from make_golden import to_ref_sequence  # noqa: E402

from paper_1305_6861_b200 import configs  # noqa: E402

M_STRIDE = 64


def m_projection(n):
    rng = np.random.default_rng(2024)
    return rng.normal(size=(n, 3))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--ref", default="/root/reference/pkg/src")
    ap.add_argument("--only", nargs="*", type=int, default=[1, 3])
    ap.add_argument("--workers", type=int, default=os.cpu_count() or 1)
    args = ap.parse_args()
    for k in ("OPENBLAS_NUM_THREADS", "OMP_NUM_THREADS", "MKL_NUM_THREADS"):
        os.environ[k] = "1"
    sys.path.insert(0, args.ref)
    import mrsim.bloch
    import mrsim.engine
    import mrsim.sequence

    class Ref:
        bloch = mrsim.bloch
        engine = mrsim.engine
        sequence = mrsim.sequence

    for index in args.only:
        t0 = time.time()
        w = configs.make(index)
        b = w.block
        assert w.n_coils == 1
        rseq = to_ref_sequence(w.sequence, Ref)
        t_end = w.sequence.end_time
        tables = Ref.engine.precompute_sequence_tables(rseq, snapshot_times=(t_end,))
        arr = Ref.engine.SpinBlock(index=0, pos=np.asarray(b.pos, float), mx=np.asarray(b.mx, float),
                                   my=np.asarray(b.my, float), mz=np.asarray(b.mz, float),
                                   t1=np.asarray(b.t1, float), t2=np.asarray(b.t2, float),
                                   m0=np.asarray(b.m0, float), domega=np.asarray(b.domega, float),
                                   weight=np.asarray(b.weight, complex).reshape(-1))
        blocks = Ref.engine.partition_blocks(arr, 4 * args.workers)
        exp = SimpleNamespace(workers=args.workers, deterministic=True)
        folds, ordered = Ref.engine._run_pool(exp, tables, blocks, {})
        echo = None
        for e, _ in folds:  # engine.py:493-496
            echo = e if echo is None else echo + e
        m = np.vstack([s[0] for _, s in ordered])  # engine.py:497-504
        assert m.shape == (b.n, 3)
        proj = m_projection(b.n)
        rec = dict(
            n_spins=np.array(b.n), snapshot_time=np.array(t_end), echoes=echo,
            m_stride=np.array(M_STRIDE), m_sub=m[::M_STRIDE], m_sum=m.sum(axis=0), m_sq=np.array((m * m).sum()),
            m_proj=(m * proj).sum(axis=0), events=np.array(sum(int(e.pulse_mat is not None) + e.ev_dt.size
                                                            for e in tables.entries)),
        )
        out = os.path.join(HERE, f"full_cfg{index}.npz")
        np.savez_compressed(out, **rec)
        print(f"config {index}: {b.n} spins x {int(rec['events'])} events, k-space {echo.shape}, "
              f"{time.time() - t0:.0f}s -> {out}", flush=True)


if __name__ == "__main__":
    main()
