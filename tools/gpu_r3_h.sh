# software-pipelined resident integrator: parity, then S=2 at 448 threads (A, spills) vs 384 threads (B) vs S=1 at 768
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider -k "resident" > gpurun_out/r3h_pytest.txt 2>&1; echo "rc=$?" >> gpurun_out/r3h_pytest.txt
for L in A B; do for c in 2 1; do
  for S in 0 1; do BLOCH_RESIDENT_SPINS=$S BLOCH_LIB=$PWD/ab/lib$L.so timeout 600 python tools/shard_probe.py $c 1 8 | sed "s/^/$L force$S /"; done
done; done > gpurun_out/r3h_shards.txt 2>&1
