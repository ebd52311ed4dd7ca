# deferred chirps and single-sample events (config 3 on the register-state integrator)
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/gg_pytest.txt 2>&1; echo "rc=$?" >> gpurun_out/gg_pytest.txt
timeout 600 python tools/phase_probe.py 3 0 > gpurun_out/gg_phases.txt 2>&1
timeout 900 python tools/shard_probe.py 3 1 2 4 8 > gpurun_out/gg_shards3.txt 2>&1
