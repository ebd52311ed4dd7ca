# smem running factors (fixed init order): correctness suites + shards + bench quick
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/ee_pytest.txt 2>&1; echo "rc=$?" >> gpurun_out/ee_pytest.txt
timeout 900 python tools/shard_probe.py 2 1 2 4 8 > gpurun_out/ee_shards.txt 2>&1
timeout 900 python tools/shard_probe.py 1 1 2 4 8 >> gpurun_out/ee_shards.txt 2>&1
timeout 900 python tools/shard_probe.py 4 1 2 4 8 >> gpurun_out/ee_shards.txt 2>&1
