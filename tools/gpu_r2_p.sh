# phase split per config (contraction on/off) + ncu of the contraction kernel (config-2 size microbench)
timeout 600 python tools/phase_probe.py 0 1 2 3 4 > gpurun_out/p_phases.txt 2>&1; echo "rc=$?" >> gpurun_out/p_phases.txt
B=tools/microbench/contract_test
BLOCH_CONTRACT_SEG=325 timeout 300 ncu --set full --import-source on --clock-control none -k regex:contract_kernel -c 1 -o gpurun_out/p_contract_cfg2 $B 512 512 748763 > gpurun_out/p_ncu.log 2>&1; echo "rc=$?" >> gpurun_out/p_ncu.log
