# resident integrator: next op record prefetched one op ahead (B) vs loaded at the top of the op (A)
for L in A B A B; do for c in 2 1; do BLOCH_LIB=$PWD/ab/lib$L.so timeout 300 python tools/shard_probe.py $c 1 8 | sed "s/^/$L /"; done; BLOCH_RESIDENT_SPINS=1 BLOCH_LIB=$PWD/ab/lib$L.so timeout 300 python tools/shard_probe.py 2 1 | sed "s/^/$L S1 /"; done > gpurun_out/r3cc_shards.txt 2>&1
