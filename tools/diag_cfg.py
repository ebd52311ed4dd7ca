"""Diagnostics: per-part errors of GPU fp32/fp64 vs golden for one config."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests", "golden"))
import numpy as np
from conftest import load_golden
from test_gpu_parity import _tables, _block
from oracle.bloch_oracle import rel_l2
from paper_1305_6861_b200 import compute_block

name = sys.argv[1] if len(sys.argv) > 1 else "cfg4"
rec = load_golden(name)
t = _tables(name, rec)
res = {}
for p in (32, 64):
    e, s = compute_block(t, _block(rec), precision=p)
    res[p] = (e, s)
    shape = tuple(rec["echo_shape"])
    ek = e.reshape((-1,) + shape[-2:])
    if "echo_full" in rec:
        print(p, "full", rel_l2(rec["echo_full"], e))
    else:
        print(p, "head", rel_l2(rec["echo_head"], ek[:, :4]), "tail", rel_l2(rec["echo_tail"], ek[:, -4:]),
              "sum", rel_l2(rec["echo_sum"], ek.sum(-1)), "energy", rel_l2(rec["echo_energy"], (np.abs(ek)**2).sum(-1)))
    print(p, "snap", rel_l2(rec["snap_0"], s[0]))
e32, e64 = res[32][0], res[64][0]
print("fp32 vs fp64 gpu full:", rel_l2(e64, e32), "snap", rel_l2(res[64][1][0], res[32][1][0]))
ek32 = e32.reshape((-1,) + e32.shape[-2:]); ek64 = e64.reshape((-1,) + e64.shape[-2:])
# per acquisition-window error (cfg4: 3 windows per line)
na = ek64.shape[1]
for w in range(min(3, na)):
    print("window", w, rel_l2(ek64[:, w::3], ek32[:, w::3]))
per_coil = [rel_l2(ek64[c], ek32[c]) for c in range(ek64.shape[0])]
print("per coil", np.round(per_coil, 7))
# per-line error trend
lines = [rel_l2(ek64[:, 3*l:3*l+3], ek32[:, 3*l:3*l+3]) for l in range(0, na//3, 16)]
print("per line (every 16th)", np.array(lines))
