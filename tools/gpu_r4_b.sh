# resident integrator: whole warps dealt evenly over full waves of CTAs (CTA sizes differ by one warp) against
# equal CTAs with a ragged last wave (BLOCH_RESIDENT_UNEVEN=1): parity first, then A/B integrator ms per config
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize_golden.py tests/test_gpu_fullsize.py tests/test_gpu_segments.py tests/test_gpu_fuzz.py tests/test_gpu_multidevice.py -m gpu -q -x -p no:cacheprovider > gpurun_out/r4b_pytest.txt 2>&1; echo "rc=$?" >> gpurun_out/r4b_pytest.txt
for c in 2 1 3 4; do
  for r in 1 2 3; do
    for v in even uneven; do
      if [ $v = uneven ]; then export BLOCH_RESIDENT_UNEVEN=1; else unset BLOCH_RESIDENT_UNEVEN; fi
      timeout 300 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline --no-per-config --no-projection --e2e-steps 1 --quiet \
        | python -c "import json,sys; d=json.load(sys.stdin); print('cfg$c $v step_ms %.3f kernel_ms %.3f integrate %.3f contract %.3f grid %s threads %s' % (d['ms_per_step'], d['kernel_ms_per_step'], d['phases_ms']['integrate'], d['phases_ms']['contract'], d['integrator_launch']['grid'], d['integrator_launch']['threads']))"
    done
  done
done > gpurun_out/r4b_ab.txt 2>&1
unset BLOCH_RESIDENT_UNEVEN
for c in 2 4; do timeout 300 python tools/shard_probe.py $c 1 2 4 8; done > gpurun_out/r4b_shards.txt 2>&1
