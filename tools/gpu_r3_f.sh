# full GPU suite on the resident build (short runs deferred automatically), quick bench of every config, config 3 shards
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r3f_pytest.txt 2>&1; echo "rc=$?" >> gpurun_out/r3f_pytest.txt
CONFIGS="0 1 2 3 4" STEPS=5 bash tools/quickbench.sh > gpurun_out/r3f_quickbench.txt 2>&1
timeout 300 python tools/shard_probe.py 3 1 2 4 8 > gpurun_out/r3f_shards.txt 2>&1
