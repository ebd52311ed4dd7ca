# contraction generators: per-warp cp.async ring of the per-spin phase tables, 4 stages ahead (B) vs register rotation (A)
timeout 120 python tools/one_call.py 0 2 > gpurun_out/r3t_first.txt 2>&1; echo "rc=$?" >> gpurun_out/r3t_first.txt
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -p no:cacheprovider -k "contraction or resident or short" > gpurun_out/r3t_pytest.txt 2>&1; echo "rc=$?" >> gpurun_out/r3t_pytest.txt
for L in A B; do for c in 3 2 4 1; do BLOCH_LIB=$PWD/ab/lib$L.so timeout 300 python tools/shard_probe.py $c 1 8 | sed "s/^/$L /"; done; done > gpurun_out/r3t_shards.txt 2>&1
