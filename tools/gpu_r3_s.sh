# ncu --set full of one chirp-group contraction launch (config 3: 10 samples x 64 windows) and of the single-sample group
BLOCH_NO_GRAPH=1 timeout 600 ncu --set full --import-source on --clock-control none -k regex:contract_kernel -s 1 -c 1 -o gpurun_out/r3s_con_cfg3_chirp python tools/one_call.py 3 > gpurun_out/r3s_ncu1.log 2>&1
BLOCH_NO_GRAPH=1 timeout 600 ncu --set full --import-source on --clock-control none -k regex:contract_kernel -s 0 -c 1 -o gpurun_out/r3s_con_cfg3_single python tools/one_call.py 3 > gpurun_out/r3s_ncu2.log 2>&1
