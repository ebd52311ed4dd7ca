# usage: TAG=r1c CONFIGS="1 3 4" bash tools/prof_multi.sh  — plain runs first, then ncu captures
set -e
TAG=${TAG:-prof}
for c in ${CONFIGS:-1}; do
  python bench.py --config $c --steps 1 --warmup 1 --no-cpu-baseline --e2e-steps 1 --quiet > gpurun_out/${TAG}_c${c}_plain.json
done
for c in ${CONFIGS:-1}; do
  CMD="python bench.py --config $c --steps 1 --warmup 1 --no-cpu-baseline --e2e-steps 1 --quiet"
  ncu --set full --clock-control none --import-source on -k regex:integrate -s 1 -c 1 -o gpurun_out/${TAG}_c${c} $CMD > gpurun_out/${TAG}_c${c}_ncu.log 2>&1
done
