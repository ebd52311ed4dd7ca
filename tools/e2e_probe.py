"""Where does the end-to-end (host-buffer) step spend its time?  Config 1, pinned buffers."""
import time

import numpy as np
import torch

from paper_1305_6861_b200 import configs
from paper_1305_6861_b200.engine import _unit_weight, get_engine, precompute_sequence_tables

w = configs.make(1)
b = w.block
t = precompute_sequence_tables(w.sequence, snapshot_times=(w.sequence.end_time,))
pin = lambda a: torch.from_numpy(np.ascontiguousarray(a, dtype=np.float64)).pin_memory().numpy()
h = {k: pin(getattr(b, k)) for k in ("pos", "mx", "my", "mz", "t1", "t2", "m0", "domega")}
wt = torch.from_numpy(np.ascontiguousarray(b.weight).view(np.float64)).pin_memory().numpy().view(np.complex128)
eng = get_engine(0, 32)
f = eng.set_tables(t)
out_e = torch.zeros(f["n_acq"] * f["max_ns"] * 2, dtype=torch.float64).pin_memory().numpy().view(np.complex128)
out_e = out_e.reshape(1, f["n_acq"], f["max_ns"])
out_s = torch.zeros(b.n * 3, dtype=torch.float64).pin_memory().numpy().reshape(1, b.n, 3)
run = lambda: eng.compute(t, h["pos"], h["mx"], h["my"], h["mz"], h["t1"], h["t2"], h["m0"], h["domega"], wt,
                          out_echoes=out_e, out_snaps=out_s)
run()
for _ in range(3):
    t0 = time.perf_counter(); run(); t1 = time.perf_counter()
    tm = eng.last_timing()
    print(f"compute() {1e3 * (t1 - t0):.2f} ms  device_ms {tm['device_ms']:.2f}  kernel_ms {tm['kernel_ms']:.2f}")
t0 = time.perf_counter()
for _ in range(10):
    _unit_weight(wt.reshape(1, -1))
print(f"_unit_weight {1e2 * (time.perf_counter() - t0):.3f} ms")
x = torch.empty(b.n * 10, dtype=torch.float64, device="cuda")
src = torch.from_numpy(np.zeros(b.n * 10)).pin_memory()
torch.cuda.synchronize()
for _ in range(2):
    t0 = time.perf_counter(); x.copy_(src, non_blocking=True); torch.cuda.synchronize()
    print(f"H2D {src.numel() * 8 / 1e6:.1f} MB pinned: {1e3 * (time.perf_counter() - t0):.2f} ms")
