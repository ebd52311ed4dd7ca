"""Kernel time of a 1/N shard of a config with each fp32 spins-per-thread variant (multi-GPU sizing)."""
import os
import subprocess
import sys

cfg, shards = sys.argv[1], sys.argv[2:]
for nsh in shards:
    for s in os.environ.get("SLIST", "8 4 2").split():
        env = dict(os.environ, BLOCH_F32_SPINS=s)
        code = (f"import numpy as np; from paper_1305_6861_b200 import configs; "
                f"from paper_1305_6861_b200.engine import get_engine, precompute_sequence_tables; "
                f"w = configs.make({cfg}).subset({nsh}); b = w.block; "
                f"t = precompute_sequence_tables(w.sequence); e = get_engine(0, 32); "
                f"[e.compute(t, b.pos, b.mx, b.my, b.mz, b.t1, b.t2, b.m0, b.domega, b.weight) for _ in range(3)]; "
                f"print('cfg{cfg} 1/{nsh} n=%d S={s} kernel_ms %.3f' % (b.n, e.last_timing()['kernel_ms']))")
        print(subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True).stdout.strip())
