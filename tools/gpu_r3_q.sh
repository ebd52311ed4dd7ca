# chirp generator: rows interleaved over the warps, rows beyond the run skipped (B) vs 8 consecutive rows per warp, all 64 generated (A)
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider -k "short or resident or cfg3 or epi16 or mixed" > gpurun_out/r3q_pytest.txt 2>&1; echo "rc=$?" >> gpurun_out/r3q_pytest.txt
for L in A B; do BLOCH_LIB=$PWD/ab/lib$L.so timeout 300 python tools/shard_probe.py 3 1 2 8 | sed "s/^/$L /"; done > gpurun_out/r3q_shards.txt 2>&1
