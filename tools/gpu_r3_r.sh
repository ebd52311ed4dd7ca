# launch list of one config-3 call (per-group contraction launches)
BLOCH_NO_GRAPH=1 timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r3r_launches_cfg3.csv python tools/one_call.py 3 2 > gpurun_out/r3r.log 2>&1
