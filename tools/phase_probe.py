"""Per-config device time split (integrator vs window contraction) with the contraction on and off.

    python tools/phase_probe.py [configs...]     (device-resident inputs, best of 5 after warm-up)"""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_1305_6861_b200 import configs  # noqa: E402
from paper_1305_6861_b200.engine import _unit_weight, get_engine, precompute_sequence_tables  # noqa: E402

cfgs = [int(c) for c in sys.argv[1:]] or [0, 1, 2, 3, 4]
dev = torch.device("cuda", 0)
e = get_engine(0, 32)
for c in cfgs:
    w = configs.make(c)
    b, n, C = w.block, w.n_spins, w.n_coils
    t = precompute_sequence_tables(w.sequence)
    f = lambda a: torch.from_numpy(np.ascontiguousarray(a, dtype=np.float64)).to(dev)
    wt = np.ascontiguousarray(np.asarray(b.weight, dtype=np.complex128).reshape(C, n)).view(np.float64)
    d = dict(pos=f(b.pos), mx=f(b.mx), my=f(b.my), mz=f(b.mz), t1=f(b.t1), t2=f(b.t2), m0=f(b.m0), domega=f(b.domega),
             weight=f(wt))
    ptrs = {k: v.data_ptr() for k, v in d.items()}
    if C == 1 and _unit_weight(wt.view(np.complex128)):
        ptrs["weight"] = 0
    fl = e.set_tables(t)
    outs = {}
    for on in (True, False):
        e.set_contraction(on)
        echo = torch.zeros(C * fl["n_acq"] * fl["max_ns"] * 2, dtype=torch.float64, device=dev)
        ks, ph = [], []
        for it in range(8):
            e.compute_device(t, ptrs, n, C, echo.data_ptr(), 0, sync=True)
            if it >= 3:
                ks.append(e.last_timing()["kernel_ms"])
                ph.append(e.last_phases())
        k = int(np.argmin(ks))
        outs[on] = echo.cpu().numpy()
        p = ph[k]
        print(f"cfg{c} n={n} contraction={'on ' if on else 'off'} kernel_ms {ks[k]:.3f} integrate_ms "
              f"{p['integrate_ms']:.3f} contract_ms {p['contract_ms']:.3f} groups {p['groups']} "
              f"samples {p['contracted_samples']} S={e.last_launch()['spins_per_thread']}", flush=True)
    a, r = outs[True], outs[False]
    print(f"cfg{c} rel L2 (contraction vs integrator sums) {np.linalg.norm(a - r) / np.linalg.norm(r):.3e}", flush=True)
    e.set_contraction(True)
