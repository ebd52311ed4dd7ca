# bench line (config 2, short) + ncu of the integrator with the deferred program (configs 2 and 1)
timeout 600 python bench.py --config 2 --steps 5 --warmup 3 --no-cpu-baseline --no-per-config --no-projection --quiet > gpurun_out/r_bench_cfg2.json 2> gpurun_out/r_bench.err; echo "rc=$?" >> gpurun_out/r_bench.err
BLOCH_NO_GRAPH=1 timeout 600 ncu --set full --import-source on --clock-control none -k regex:integrate -c 1 -o gpurun_out/r_integ_cfg2 python tools/one_call.py 2 > gpurun_out/r_ncu2.log 2>&1
BLOCH_NO_GRAPH=1 timeout 600 ncu --set full --import-source on --clock-control none -k regex:integrate -c 1 -o gpurun_out/r_integ_cfg1 python tools/one_call.py 1 > gpurun_out/r_ncu1.log 2>&1
