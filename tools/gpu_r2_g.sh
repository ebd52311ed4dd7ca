# ncu counters of the integrator per config (issue floor + DRAM traffic for bench.py) and the launch list
SHA=$(python -c "import hashlib;print(hashlib.sha256(open('paper_1305_6861_b200/libbloch_b200.so','rb').read()).hexdigest()[:16])")
M=smsp__inst_executed.sum,dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,sm__cycles_elapsed.avg.per_second,sm__pipe_tensor_subpipe_hmma_cycles_active.avg.pct_of_peak_sustained_active,sm__inst_issued.avg.pct_of_peak_sustained_active
for c in 0 1 2 3 4; do
  CMD="python bench.py --config $c --steps 1 --warmup 1 --no-cpu-baseline --no-per-config --no-projection --e2e-steps 1 --quiet"
  BLOCH_NO_GRAPH=1 $CMD > gpurun_out/g_plain_cfg$c.json 2>&1 && \
  BLOCH_NO_GRAPH=1 ncu --metrics $M --clock-control none -k regex:integrate -s 1 -c 1 --csv --log-file gpurun_out/g_cfg$c.csv $CMD > /dev/null 2>&1
done
python tools/ncu_counters.py gpurun_out/ncu_counters.json $SHA gpurun_out/g_cfg*.csv > gpurun_out/g_counters.log 2>&1
CMD="python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-per-config --no-projection --e2e-steps 1 --quiet"
$CMD > gpurun_out/g_plain_launch.json 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/g_launches_cfg2.csv $CMD > /dev/null 2>&1
