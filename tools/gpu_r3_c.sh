# resident-table integrator: parity, then ncu --set full of the kernel on config 2 (full and 1/8 shard)
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider -k "resident" > gpurun_out/r3c_pytest.txt 2>&1; echo "rc=$?" >> gpurun_out/r3c_pytest.txt
BLOCH_NO_GRAPH=1 timeout 600 ncu --set full --import-source on --clock-control none -k regex:resident -c 1 -o gpurun_out/r3c_res_cfg2_8 python tools/one_call.py 2 1 8 > gpurun_out/r3c_ncu1.log 2>&1
BLOCH_NO_GRAPH=1 timeout 600 ncu --set full --import-source on --clock-control none -k regex:resident -c 1 -o gpurun_out/r3c_res_cfg2 python tools/one_call.py 2 > gpurun_out/r3c_ncu2.log 2>&1
