# generator warps for one-M-tile contraction CTAs: 4 (default) vs 8 (BLOCH_CONTRACT_GW=8)
for r in 1 2; do for gw in 4 8; do BLOCH_CONTRACT_GW=$gw timeout 600 python tools/phase_probe.py 4 | grep "contraction=on" | sed "s/^/gw$gw /"; done; done > gpurun_out/ff_gw.txt 2>&1
B=tools/microbench/contract_test
for gw in 4 8; do for d in 0 2; do BLOCH_CONTRACT_GW=$gw CONTRACT_DBG=$d timeout 120 $B 384 256 274145 | grep contract | sed "s/^/gw$gw dbg$d /"; done; done >> gpurun_out/ff_gw.txt 2>&1
