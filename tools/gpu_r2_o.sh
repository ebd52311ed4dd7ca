# contraction microbench (8 generator warps, prefetch) + engine GPU tests of the contraction path
B=tools/microbench/contract_test
for a in "17 70 1000" "200 250 3001 3 5" "64 200 50000"; do timeout 120 $B $a; echo "rc=$?"; done > gpurun_out/o_contract.txt 2>&1
for d in 0 1 2; do CONTRACT_DBG=$d BLOCH_CONTRACT_SEG=100000 timeout 120 $B 512 512 748763; echo "rc=$?"; done >> gpurun_out/o_contract.txt 2>&1
for d in 0 2; do CONTRACT_DBG=$d BLOCH_CONTRACT_SEG=100000 timeout 120 $B 256 256 697712; echo "rc=$?"; done >> gpurun_out/o_contract.txt 2>&1
for sg in 128 325; do BLOCH_CONTRACT_SEG=$sg timeout 120 $B 512 512 748763; echo "rc=$?"; done >> gpurun_out/o_contract.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -p no:cacheprovider > gpurun_out/o_parity.txt 2>&1; echo "rc=$?" >> gpurun_out/o_parity.txt
