"""Would L2-sized spin slabs pay?  Kernel time of one launch over all spins vs sequential launches
over 2 / 4 contiguous slabs (device-resident inputs).  Usage: python tools/slab_probe.py CFG"""
import sys

import numpy as np
import torch

from paper_1305_6861_b200 import configs
from paper_1305_6861_b200.engine import get_engine, precompute_sequence_tables

cfg = int(sys.argv[1])
w = configs.make(cfg)
b = w.block
t = precompute_sequence_tables(w.sequence, snapshot_times=(w.sequence.end_time,))
eng = get_engine(0, 32)
f = eng.set_tables(t)
dev = torch.device("cuda", 0)
d = {k: torch.from_numpy(np.ascontiguousarray(getattr(b, k), dtype=np.float64)).to(dev)
     for k in ("pos", "mx", "my", "mz", "t1", "t2", "m0", "domega")}
d["pos"] = d["pos"].reshape(-1)
C = 1 if np.asarray(b.weight).ndim == 1 else np.asarray(b.weight).shape[0]
wt = torch.from_numpy(np.ascontiguousarray(np.asarray(b.weight, complex).reshape(C, -1)).view(np.float64)).to(dev)
echo = torch.zeros(C * f["n_acq"] * f["max_ns"] * 2, dtype=torch.float64, device=dev)
snap = torch.empty(b.n * 3, dtype=torch.float64, device=dev)


def run(lo, hi):
    n = hi - lo
    p = {k: v[lo * (3 if k == "pos" else 1):].data_ptr() for k, v in d.items()}
    p["weight"] = 0 if C == 1 else 0
    if C > 1:  # slab of a [C][n] array: copy to a contiguous [C][n_slab] buffer
        ws = wt.view(C, -1, 2)[:, lo:hi].contiguous()
        p["weight"] = ws.data_ptr()
        run.keep = ws
    if not all(p[k] for k in d):
        print("null ptr", lo, hi, {k: hex(v) for k, v in p.items()})
    eng.compute_device(t, p, n, C, echo.data_ptr(), snap.data_ptr(), sync=True)
    return eng.last_timing()["kernel_ms"]


for n_slab in (1, 2, 3, 4):
    bounds = np.linspace(0, b.n, n_slab + 1).astype(int)
    for _ in range(2):
        ms = sum(run(bounds[k], bounds[k + 1]) for k in range(n_slab))
    print(f"cfg{cfg} slabs={n_slab} kernel_ms_sum={ms:.3f}")
