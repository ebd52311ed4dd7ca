# contraction generators: per-spin phase tables loaded 2 (A) vs 6 (B) stages ahead
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider -k "contraction or resident" > gpurun_out/r3m_pytest.txt 2>&1; echo "rc=$?" >> gpurun_out/r3m_pytest.txt
for L in A B; do for c in 3 2 4 1; do BLOCH_LIB=$PWD/ab/lib$L.so timeout 300 python tools/shard_probe.py $c 1 8 | sed "s/^/$L /"; done; done > gpurun_out/r3m_shards.txt 2>&1
