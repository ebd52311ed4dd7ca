# usage: CFG=1 TAG=r1b bash tools/prof_cmd.sh   (plain run, then launch list, then full ncu of the integrator)
set -e
CFG=${CFG:-1}; TAG=${TAG:-prof}
CMD="python bench.py --config $CFG --steps 1 --warmup 1 --no-cpu-baseline --e2e-steps 1 --quiet"
$CMD > gpurun_out/${TAG}_plain.json 2> gpurun_out/${TAG}_plain.err
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${TAG}_launches.csv $CMD > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:integrate -s 1 -c 1 -o gpurun_out/${TAG} $CMD > gpurun_out/${TAG}_ncu.log 2>&1
tail -2 gpurun_out/${TAG}_ncu.log
