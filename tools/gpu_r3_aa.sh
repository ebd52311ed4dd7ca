# contraction generator: bf16 split by packed conversion (B) vs Veltkamp split + byte permutes (A)
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider -k "contraction or resident or short" > gpurun_out/r3aa_pytest.txt 2>&1; echo "rc=$?" >> gpurun_out/r3aa_pytest.txt
for L in A B A B; do for c in 2 4 1 3; do BLOCH_LIB=$PWD/ab/lib$L.so timeout 300 python tools/shard_probe.py $c 1 | sed "s/^/$L /"; done; done > gpurun_out/r3aa_shards.txt 2>&1
