# resident integrator: table loads of an op hoisted above its arithmetic (B) vs loaded where used (A)
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider -k "resident" > gpurun_out/r3n_pytest.txt 2>&1; echo "rc=$?" >> gpurun_out/r3n_pytest.txt
for L in A B; do for c in 2 1 4 3; do
  BLOCH_LIB=$PWD/ab/lib$L.so timeout 300 python tools/shard_probe.py $c 1 8 | sed "s/^/$L /"
done; BLOCH_RESIDENT_SPINS=1 BLOCH_LIB=$PWD/ab/lib$L.so timeout 300 python tools/shard_probe.py 2 1 | sed "s/^/$L forceS1 /"; done > gpurun_out/r3n_shards.txt 2>&1
