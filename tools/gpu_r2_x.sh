# re/im row-block generator layout (microbench), shard phases, previously failing tests
B=tools/microbench/contract_test
for a in "17 70 1000" "200 250 3001 3 5" "64 200 50000" "32 4096 20000"; do timeout 120 $B $a; echo "rc=$?"; done > gpurun_out/x_contract.txt 2>&1
for d in 0 1 2; do CONTRACT_DBG=$d BLOCH_CONTRACT_SEG=100000 timeout 120 $B 512 512 748763; echo "rc=$?"; done >> gpurun_out/x_contract.txt 2>&1
BLOCH_CONTRACT_SEG=128 timeout 120 $B 512 512 748763 >> gpurun_out/x_contract.txt 2>&1
BLOCH_CONTRACT_SEG=128 timeout 120 $B 384 256 274145 >> gpurun_out/x_contract.txt 2>&1
timeout 900 python tools/shard_probe.py 2 1 2 4 8 > gpurun_out/x_shard2.txt 2>&1
timeout 900 python tools/shard_probe.py 4 1 2 4 8 > gpurun_out/x_shard4.txt 2>&1
timeout 1200 python -m pytest tests/test_gpu_segments.py tests/test_gpu_fuzz.py tests/test_gpu_fullsize_golden.py tests/test_gpu_fullsize.py tests/test_gpu_parity.py -q -p no:cacheprovider > gpurun_out/x_pytest.txt 2>&1; echo "rc=$?" >> gpurun_out/x_pytest.txt
