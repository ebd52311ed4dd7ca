# no-window integrator variant: 2 (A) vs 3 (B) CTAs/SM; shard probe; phase probe incl. multi-coil contraction; GPU parity
CONFIGS="1 2 3" ROUNDS=2 STEPS=6 bash tools/ab.sh > gpurun_out/s_ab.txt 2>&1
timeout 600 python tools/phase_probe.py 0 1 2 3 4 > gpurun_out/s_phases.txt 2>&1
timeout 600 python tools/shard_probe.py 2 1 2 4 8 > gpurun_out/s_shard2.txt 2>&1
timeout 600 python tools/shard_probe.py 1 1 2 4 8 > gpurun_out/s_shard1.txt 2>&1
timeout 600 python tools/shard_probe.py 4 1 2 4 8 > gpurun_out/s_shard4.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -p no:cacheprovider > gpurun_out/s_parity.txt 2>&1; echo "rc=$?" >> gpurun_out/s_parity.txt
