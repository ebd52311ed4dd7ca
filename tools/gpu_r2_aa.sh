# N-subtiles in the contraction: microbench (nsub 2 vs 1) + phase probe + parity
B=tools/microbench/contract_test
for a in "17 70 1000" "200 250 3001 3 5" "300 70 5000 2 7" "512 512 20000"; do timeout 120 $B $a; echo "rc=$?"; done > gpurun_out/aa_contract.txt 2>&1
for ns in 1 2; do for a in "512 512 748763" "384 256 274145" "256 256 697712"; do BLOCH_CONTRACT_NSUB=$ns timeout 120 $B $a; echo "rc=$?"; done; done >> gpurun_out/aa_contract.txt 2>&1
for ns in 1 2; do BLOCH_CONTRACT_NSUB=$ns timeout 600 python tools/phase_probe.py 2 4 | grep -v "contraction=off" | sed "s/^/nsub$ns /"; done > gpurun_out/aa_phases.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider > gpurun_out/aa_parity.txt 2>&1; echo "rc=$?" >> gpurun_out/aa_parity.txt
