"""One device-resident call of a config (for ncu captures): python tools/one_call.py CFG [repeats] [shard N]"""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_1305_6861_b200 import configs  # noqa: E402
from paper_1305_6861_b200.engine import _unit_weight, get_engine, precompute_sequence_tables  # noqa: E402

c = int(sys.argv[1])
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 1
nsh = int(sys.argv[3]) if len(sys.argv) > 3 else 1
w = configs.make(c)
b, n, C = w.block, w.n_spins, w.n_coils
if nsh > 1:  # rank 0's np.linspace shard
    from paper_1305_6861_b200.parallel import shard_block
    b = shard_block(b, nsh, 0)
    n = b.n
t = precompute_sequence_tables(w.sequence)
dev = torch.device("cuda", 0)
f = lambda a: torch.from_numpy(np.ascontiguousarray(a, dtype=np.float64)).to(dev)
wt = np.ascontiguousarray(np.asarray(b.weight, dtype=np.complex128).reshape(C, n)).view(np.float64)
d = dict(pos=f(b.pos), mx=f(b.mx), my=f(b.my), mz=f(b.mz), t1=f(b.t1), t2=f(b.t2), m0=f(b.m0), domega=f(b.domega),
         weight=f(wt))
ptrs = {k: v.data_ptr() for k, v in d.items()}
if C == 1 and _unit_weight(wt.view(np.complex128)):
    ptrs["weight"] = 0
e = get_engine(0, 32)
fl = e.set_tables(t)
echo = torch.zeros(C * fl["n_acq"] * fl["max_ns"] * 2, dtype=torch.float64, device=dev)
for _ in range(reps):
    e.compute_device(t, ptrs, n, C, echo.data_ptr(), 0, sync=True)
print("cfg", c, e.last_timing(), e.last_phases())
