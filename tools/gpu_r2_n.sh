# tcgen05 window contraction, spin-block-major U: bottleneck modes (dbg 1: no A generation, 2: no MMA) and segments
B=tools/microbench/contract_test
for a in "17 70 1000" "200 250 3001 3 5" "64 200 50000"; do timeout 120 $B $a; echo "rc=$?"; done > gpurun_out/n2_contract.txt 2>&1
for d in 0 1 2 3; do CONTRACT_DBG=$d BLOCH_CONTRACT_SEG=100000 timeout 120 $B 512 512 748763; echo "rc=$?"; done >> gpurun_out/n2_contract.txt 2>&1
for d in 0 1 2 3; do CONTRACT_DBG=$d BLOCH_CONTRACT_SEG=100000 timeout 120 $B 256 256 697712; echo "rc=$?"; done >> gpurun_out/n2_contract.txt 2>&1
for sg in 64 128 325; do BLOCH_CONTRACT_SEG=$sg timeout 120 $B 512 512 748763; echo "rc=$?"; done >> gpurun_out/n2_contract.txt 2>&1
