# fp32 generator (prep tables), conflict-free stores: microbench modes, phase probe, parity, ncu
B=tools/microbench/contract_test
for a in "17 70 1000" "200 250 3001 3 5" "64 200 50000" "32 4096 20000"; do timeout 120 $B $a; echo "rc=$?"; done > gpurun_out/q_contract.txt 2>&1
for d in 0 1 2; do CONTRACT_DBG=$d BLOCH_CONTRACT_SEG=100000 timeout 120 $B 512 512 748763; echo "rc=$?"; done >> gpurun_out/q_contract.txt 2>&1
for d in 0 2; do CONTRACT_DBG=$d BLOCH_CONTRACT_SEG=100000 timeout 120 $B 256 256 697712; echo "rc=$?"; done >> gpurun_out/q_contract.txt 2>&1
BLOCH_CONTRACT_SEG=325 timeout 120 $B 512 512 748763 >> gpurun_out/q_contract.txt 2>&1
timeout 600 python tools/phase_probe.py 1 2 3 > gpurun_out/q_phases.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -p no:cacheprovider > gpurun_out/q_parity.txt 2>&1; echo "rc=$?" >> gpurun_out/q_parity.txt
BLOCH_CONTRACT_SEG=325 timeout 300 ncu --set full --import-source on --clock-control none -k regex:contract_kernel -c 1 -o gpurun_out/q_contract_cfg2 $B 512 512 748763 > gpurun_out/q_ncu.log 2>&1
