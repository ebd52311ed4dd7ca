# progression running factors in shared memory (B) vs L2 read-modify-write (A, BLOCH_NO_SMEM_PROG)
for r in 1 2; do for v in A B; do for c in 2 4 1; do
  if [ $v = A ]; then export BLOCH_NO_SMEM_PROG=1; else unset BLOCH_NO_SMEM_PROG; fi
  python bench.py --config $c --steps 6 --warmup 3 --no-cpu-baseline --no-per-config --no-projection --e2e-steps 1 --quiet | python -c "import json,sys; d=json.load(sys.stdin); print('cfg$c $v kernel_ms %.3f integ %.3f' % (d['kernel_ms_per_step'], d['phases_ms']['integrate']))"
done; done; done > gpurun_out/dd_ab.txt 2>&1
for v in A B; do if [ $v = A ]; then export BLOCH_NO_SMEM_PROG=1; else unset BLOCH_NO_SMEM_PROG; fi; timeout 900 python tools/shard_probe.py 2 2 4 8 | sed "s/^/$v /"; done > gpurun_out/dd_shards.txt 2>&1
unset BLOCH_NO_SMEM_PROG
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fuzz.py tests/test_gpu_segments.py tests/test_gpu_fullsize.py -q -p no:cacheprovider > gpurun_out/dd_pytest.txt 2>&1; echo "rc=$?" >> gpurun_out/dd_pytest.txt
