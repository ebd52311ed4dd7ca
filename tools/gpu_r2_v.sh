# register-resident spin state (B) vs shared-memory state (A) in the no-window integrator
CONFIGS="1 2 4" ROUNDS=2 STEPS=6 bash tools/ab.sh > gpurun_out/v_ab.txt 2>&1
for L in A B; do for c in 2 1; do BLOCH_LIB=$PWD/ab/lib$L.so SLIST="8 4 2 1" timeout 900 python tools/shard_probe.py $c 1 2 4 8 | sed "s/^/$L /"; done; done > gpurun_out/v_sweep.txt 2>&1
