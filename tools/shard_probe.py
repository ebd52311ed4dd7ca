"""Device time of a 1/N spin shard of a config (multi-GPU strong-scaling sizing, one GPU).

    python tools/shard_probe.py CFG N1 N2 ...      (env SLIST="0 8 4 2 1": 0 = the library's own pick)

Per shard: the integrator kernel time and the whole device time of the call (staging kernels,
integrator, reduction), device-resident inputs, best of 5 after warm-up; and the reduction mode."""
import os
import subprocess
import sys

cfg, shards = sys.argv[1], sys.argv[2:]
for nsh in shards:
    for s in os.environ.get("SLIST", "0").split():
        env = dict(os.environ)
        if s != "0":
            env["BLOCH_F32_SPINS"] = s
        code = f"""
import sys, numpy as np, torch
sys.path.insert(0, '.')
from paper_1305_6861_b200 import configs
from paper_1305_6861_b200.engine import get_engine, precompute_sequence_tables
w = configs.make({cfg})
n = w.n_spins
lo, hi = 0, (n + {nsh} - 1) // {nsh}
b = w.block
C = w.n_coils
t = precompute_sequence_tables(w.sequence)
e = get_engine(0, 32)
dev = torch.device('cuda', 0)
f = lambda a: torch.from_numpy(np.ascontiguousarray(a[..., lo:hi] if a.ndim == 1 else a[lo:hi], dtype=np.float64)).to(dev)
wt = np.ascontiguousarray(np.asarray(b.weight, dtype=np.complex128).reshape(C, n)[:, lo:hi]).view(np.float64)
d = dict(pos=f(b.pos), mx=f(b.mx), my=f(b.my), mz=f(b.mz), t1=f(b.t1), t2=f(b.t2), m0=f(b.m0), domega=f(b.domega),
         weight=torch.from_numpy(wt).to(dev))
ptrs = {{k: v.data_ptr() for k, v in d.items()}}
if C == 1 and np.all(np.asarray(b.weight) == 1): ptrs['weight'] = 0
f2 = e.set_tables(t)
echo = torch.zeros(C * f2['n_acq'] * f2['max_ns'] * 2, dtype=torch.float64, device=dev)
ks, ds = [], []
for it in range(8):
    e.compute_device(t, ptrs, hi - lo, C, echo.data_ptr(), 0, sync=True)
    tm = e.last_timing()
    if it >= 3: ks.append(tm['kernel_ms']); ds.append(tm['device_ms'])
L = e.last_launch()
ph = e.last_phases()
print('cfg{cfg} 1/{nsh} n=%d S=%d grid=%d thr=%d kernel_ms %.3f device_ms %.3f integrate_ms %.3f contract_ms %.3f' % (hi - lo, L['spins_per_thread'], L['grid'], L['threads'], min(ks), min(ds), ph['integrate_ms'], ph['contract_ms']))
"""
        r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True)
        print(r.stdout.strip() or r.stderr[-800:], flush=True)
