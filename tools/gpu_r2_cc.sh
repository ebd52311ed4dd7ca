# register prefetch (B) vs none (A) at one spin per thread; correctness suites that run S = 1 blocks
for r in 1 2; do for L in A B; do for c in 2 1 4; do BLOCH_LIB=$PWD/ab/lib$L.so timeout 900 python tools/shard_probe.py $c 8 | sed "s/^/$L /"; done; done; done > gpurun_out/cc_shards.txt 2>&1
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fuzz.py tests/test_gpu_acceptance.py tests/test_gpu_segments.py tests/test_engine_restated.py -q -p no:cacheprovider > gpurun_out/cc_pytest.txt 2>&1; echo "rc=$?" >> gpurun_out/cc_pytest.txt
