# spins-per-thread sweep of the no-window integrator at full size and shards
for c in 2 1 4 3; do SLIST="8 4 2 1" timeout 900 python tools/shard_probe.py $c 1 2 4 8; done > gpurun_out/t_sweep.txt 2>&1
