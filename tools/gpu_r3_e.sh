# resident-table integrator v3 (unified exit, 1 or 2 spins per thread): parity, S sweep, config 3 with short runs deferred
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider -k "resident" > gpurun_out/r3e_pytest.txt 2>&1; echo "rc=$?" >> gpurun_out/r3e_pytest.txt
for c in 2 1 4; do
  for S in 1 2; do BLOCH_RESIDENT_SPINS=$S timeout 600 python tools/shard_probe.py $c 1 2 4 8 | sed "s/^/S$S /"; done
done > gpurun_out/r3e_shards.txt 2>&1
timeout 300 python tools/shard_probe.py 3 1 8 | sed "s/^/plain /" >> gpurun_out/r3e_shards.txt 2>&1
BLOCH_DEFER_SHORT=1 timeout 300 python tools/shard_probe.py 3 1 8 | sed "s/^/defer_short /" >> gpurun_out/r3e_shards.txt 2>&1
