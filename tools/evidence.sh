# Round evidence: full bench line (default config) + reference arm + launch list + ncu --set full of the integrator
set -e
TAG=${TAG:-r1}
python bench.py > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err
python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/${TAG}_reference.json 2> gpurun_out/${TAG}_reference.err
CMD="python bench.py --steps 2 --warmup 1 --no-cpu-baseline --e2e-steps 1 --quiet"
$CMD > gpurun_out/${TAG}_plain.json
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${TAG}_launches.csv $CMD > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:integrate -s 1 -c 1 -o gpurun_out/${TAG}_full $CMD > gpurun_out/${TAG}_ncu.log 2>&1
nvidia-smi --query-gpu=name,driver_version,clocks.max.sm,power.limit --format=csv > gpurun_out/${TAG}_gpu.csv
