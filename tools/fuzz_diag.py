"""Per-acquisition / per-coil error of a fuzz seed (tests/test_gpu_fuzz.py) vs the oracle."""
import sys

import numpy as np

sys.path.insert(0, "tests")
from test_gpu_fuzz import random_sequence, random_spins  # noqa: E402

from oracle import bloch_oracle as O  # noqa: E402
from paper_1305_6861_b200 import compute_block, precompute_sequence_tables  # noqa: E402

seed = int(sys.argv[1])
seq = random_sequence(seed)
b = random_spins(seed)
snaps_t = (0.0, seq.end_time * 0.37, seq.end_time)
t = precompute_sequence_tables(seq, snapshot_times=snaps_t)
ref_e, ref_s = O.compute_block(O.precompute_tables(seq, snapshot_times=snaps_t), b.pos, b.mx, b.my, b.mz, b.t1, b.t2,
                               b.m0, b.domega, b.weight)
acq_es = [i for i, e in enumerate(seq.elements) if e.acquisition.enabled]
for prec in (64, 32):
    e, s = compute_block(t, b, precision=prec)
    print(f"precision {prec}: snapshots", [None if r is None else f"{O.rel_l2(r, a):.1e}" for a, r in zip(s, ref_s)])
    for a in range(ref_e.shape[1]):
        es = seq.elements[acq_es[a]]
        errs = [O.rel_l2(ref_e[c, a], e[c, a]) if np.linalg.norm(ref_e[c, a]) else 0.0 for c in range(ref_e.shape[0])]
        print(f"  acq {a} (ES {acq_es[a]}, n={es.acquisition.n_samples}, grad {es.gradient.shape}, "
              f"pulse {es.pulse is not None}): " + " ".join(f"{x:.1e}" for x in errs))
