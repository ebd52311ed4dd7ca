# L1 prefetch A/B (A: without) on full configs and shards; segments test
CONFIGS="1 2 4" ROUNDS=2 STEPS=6 bash tools/ab.sh > gpurun_out/y_ab.txt 2>&1
for L in A B; do for c in 2 1 4; do BLOCH_LIB=$PWD/ab/lib$L.so timeout 900 python tools/shard_probe.py $c 1 2 4 8 | sed "s/^/$L /"; done; done > gpurun_out/y_shards.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_segments.py -q -p no:cacheprovider > gpurun_out/y_pytest.txt 2>&1; echo "rc=$?" >> gpurun_out/y_pytest.txt
