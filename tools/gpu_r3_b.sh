# resident-table integrator: parity (on / off), shard probe on / off, quick bench of every config
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -p no:cacheprovider -k "resident or test_gpu_parity or contraction_runs" > gpurun_out/r3b_pytest.txt 2>&1; echo "rc=$?" >> gpurun_out/r3b_pytest.txt
for c in 2 1 4; do
  timeout 600 python tools/shard_probe.py $c 1 2 4 8 | sed "s/^/resident /"
  BLOCH_NO_RESIDENT=1 timeout 600 python tools/shard_probe.py $c 1 8 | sed "s/^/l2path /"
done > gpurun_out/r3b_shards.txt 2>&1
CONFIGS="0 1 2 3 4" STEPS=5 bash tools/quickbench.sh > gpurun_out/r3b_quickbench.txt 2>&1
