# pulse matrices in shared memory (env off = A), contraction with 2-stage table prefetch, config 3 integrator profile
for r in 1 2; do for v in A B; do for c in 1 2; do
  if [ $v = A ]; then export BLOCH_NO_SMEM_MATS=1; else unset BLOCH_NO_SMEM_MATS; fi
  python bench.py --config $c --steps 6 --warmup 3 --no-cpu-baseline --no-per-config --no-projection --e2e-steps 1 --quiet | python -c "import json,sys; d=json.load(sys.stdin); print('cfg$c $v kernel_ms %.3f integ %.3f' % (d['kernel_ms_per_step'], d['phases_ms']['integrate']))"
done; done; done > gpurun_out/bb_ab.txt 2>&1
unset BLOCH_NO_SMEM_MATS
for v in A B; do if [ $v = A ]; then export BLOCH_NO_SMEM_MATS=1; else unset BLOCH_NO_SMEM_MATS; fi; timeout 900 python tools/shard_probe.py 2 2 4 8 | sed "s/^/$v /"; done > gpurun_out/bb_shards.txt 2>&1
unset BLOCH_NO_SMEM_MATS
B=tools/microbench/contract_test
for d in 0 2; do CONTRACT_DBG=$d timeout 120 $B 512 512 748763; CONTRACT_DBG=$d timeout 120 $B 384 256 274145; done > gpurun_out/bb_contract.txt 2>&1
timeout 600 python tools/phase_probe.py 1 2 3 4 > gpurun_out/bb_phases.txt 2>&1
BLOCH_NO_GRAPH=1 timeout 600 ncu --set full --import-source on --clock-control none -k regex:integrate -c 1 -o gpurun_out/bb_integ_cfg3 python tools/one_call.py 3 > gpurun_out/bb_ncu3.log 2>&1
