# A/B kernel timing on one box: build A = libA.so, B = libB.so under ab/, then
#   CONFIGS="1 2" ROUNDS=3 bash tools/ab.sh
# alternates the two builds ROUNDS times per config and prints kernel ms of each run.
for c in ${CONFIGS:-1}; do
  for r in $(seq ${ROUNDS:-3}); do
    for v in ${VARIANTS:-A B}; do
      BLOCH_LIB=$PWD/ab/lib$v.so python bench.py --config $c --steps ${STEPS:-10} --warmup 3 --no-cpu-baseline --no-per-config --no-projection --e2e-steps 1 --quiet \
        | python -c "import json,sys; d=json.load(sys.stdin); print('cfg$c $v kernel_ms %.3f' % d['kernel_ms_per_step'])"
    done
  done
done
