# spins-per-thread sweep for the 8-coil kernel after the coils-in-M change; full-lattice per-config bench
SLIST="4 2 1" python tools/shard_probe.py 4 1 2 4 8 > gpurun_out/j_sweep.txt 2>&1
python bench.py --full-lattice --steps 6 --warmup 3 --no-cpu-baseline > gpurun_out/j_bench_full.json 2> gpurun_out/j_bench_full.err
