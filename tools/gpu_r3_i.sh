# contraction partial slots A vs B builds under ab/ (see profiles/r3i_*, r3j_*)
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider -k "contraction or resident" > gpurun_out/r3i_pytest.txt 2>&1; echo "rc=$?" >> gpurun_out/r3i_pytest.txt
CONFIGS="2 4 1 3" ROUNDS=2 STEPS=6 bash tools/ab.sh > gpurun_out/r3i_ab.txt 2>&1
for L in A B; do BLOCH_LIB=$PWD/ab/lib$L.so timeout 300 python tools/shard_probe.py 2 1 8 | sed "s/^/$L /"; BLOCH_LIB=$PWD/ab/lib$L.so timeout 300 python tools/shard_probe.py 4 1 8 | sed "s/^/$L /"; done > gpurun_out/r3i_shards.txt 2>&1
