# resident integrator: dealing unit of 4 spins (config 2 needs 1012 spins per CTA for 5 waves; 1008 fit in units of 8):
# does the 5-wave launch engage, is it correct, is it faster?  Then the evidence command list on this build.
BLOCH_RESIDENT_DEBUG=1 timeout 300 python tools/one_call.py 2 > gpurun_out/r4e_debug.txt 2>&1
for c in 2; do
  for r in 1 2 3; do
    for v in dealt uneven; do
      if [ $v = uneven ]; then export BLOCH_RESIDENT_UNEVEN=1; else unset BLOCH_RESIDENT_UNEVEN; fi
      timeout 300 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline --no-per-config --no-projection --e2e-steps 1 --quiet \
        | python -c "import json,sys; d=json.load(sys.stdin); print('cfg$c $v step_ms %.3f kernel_ms %.3f integrate %.3f contract %.3f grid %s threads %s' % (d['ms_per_step'], d['kernel_ms_per_step'], d['phases_ms']['integrate'], d['phases_ms']['contract'], d['integrator_launch']['grid'], d['integrator_launch']['threads']))"
    done
  done
done > gpurun_out/r4e_ab.txt 2>&1
unset BLOCH_RESIDENT_UNEVEN
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r4e_pytest.txt 2>&1; echo "rc=$?" >> gpurun_out/r4e_pytest.txt
SHA=$(python -c "from paper_1305_6861_b200.build import source_hash; print(source_hash())")
M=smsp__inst_executed.sum,dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,sm__cycles_elapsed.avg.per_second,sm__pipe_tensor_subpipe_hmma_cycles_active.avg.pct_of_peak_sustained_active,sm__inst_issued.avg.pct_of_peak_sustained_active
for c in 0 1 2 3 4; do
  CMD="python bench.py --config $c --steps 1 --warmup 1 --no-cpu-baseline --no-per-config --no-projection --e2e-steps 1 --quiet"
  BLOCH_NO_GRAPH=1 timeout 300 $CMD > gpurun_out/r4e_plain_cfg$c.json 2>&1 && \
  BLOCH_NO_GRAPH=1 timeout 600 ncu --metrics $M --clock-control none -k regex:integrate -s 1 -c 1 --csv --log-file gpurun_out/r4e_cfg$c.csv $CMD > /dev/null 2>&1
  BLOCH_NO_GRAPH=1 timeout 600 ncu --metrics $M --clock-control none -k regex:contract_kernel -s 1 -c 1 --csv --log-file gpurun_out/r4e_contract_cfg$c.csv $CMD > /dev/null 2>&1
done
rm -f gpurun_out/ncu_counters.json
python tools/ncu_counters.py gpurun_out/ncu_counters.json $SHA gpurun_out/r4e_cfg*.csv gpurun_out/r4e_contract_cfg*.csv > gpurun_out/r4e_counters.log 2>&1
cp gpurun_out/ncu_counters.json profiles/ncu_counters.json
CMD="python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-per-config --no-projection --e2e-steps 1 --quiet"
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r4e_launches_cfg2.csv $CMD > /dev/null 2>&1
timeout 900 python bench.py > gpurun_out/r4e_bench.json 2> gpurun_out/r4e_bench.err; echo "rc=$?" >> gpurun_out/r4e_bench.err
BLOCH_NO_GRAPH=1 timeout 600 ncu --set full --import-source on --clock-control none -k regex:resident -c 1 -o gpurun_out/r4e_res_cfg2 python tools/one_call.py 2 > gpurun_out/r4e_ncu2.log 2>&1
BLOCH_NO_GRAPH=1 timeout 600 ncu --set full --import-source on --clock-control none -k regex:contract_kernel -c 1 -o gpurun_out/r4e_con_cfg2 python tools/one_call.py 2 > gpurun_out/r4e_ncu3.log 2>&1
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/r4e_reference.json 2> gpurun_out/r4e_reference.err
for c in 1 2 3 4; do timeout 300 python tools/shard_probe.py $c 1 2 4 8; done > gpurun_out/r4e_shards.txt 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r4e_smoke.txt 2>&1
