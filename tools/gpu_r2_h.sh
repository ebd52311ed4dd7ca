# A/B: L2 evict_last on the progression running factors (B) vs HEAD (A)
CONFIGS="2 1 4" ROUNDS=2 STEPS=6 bash tools/ab.sh > gpurun_out/h_ab.txt 2>&1
for v in A B; do BLOCH_LIB=$PWD/ab/lib$v.so python tools/shard_probe.py 2 8 >> gpurun_out/h_ab.txt 2>&1; BLOCH_LIB=$PWD/ab/lib$v.so python tools/shard_probe.py 1 8 >> gpurun_out/h_ab.txt 2>&1; done
M=dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,smsp__inst_executed.sum
CMD="python bench.py --config 2 --steps 1 --warmup 1 --no-cpu-baseline --no-per-config --no-projection --e2e-steps 1 --quiet"
BLOCH_LIB=$PWD/ab/libB.so BLOCH_NO_GRAPH=1 $CMD > /dev/null 2>&1 && BLOCH_LIB=$PWD/ab/libB.so BLOCH_NO_GRAPH=1 ncu --metrics $M --clock-control none -k regex:integrate -s 1 -c 1 --csv --log-file gpurun_out/h_cfg2_B.csv $CMD > /dev/null 2>&1
