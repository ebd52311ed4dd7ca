# pipeline depth 1 / 2 / 4 / 8 on the small tile and 1 / 2 / 3 on the config-2 tile, with and without compute (dbg 3 = neither generation nor MMA)
B=tools/microbench/contract_test
for d in 3 0; do for D in 1 2 4 8; do BLOCH_CONTRACT_DEPTH=$D CONTRACT_DBG=$d timeout 120 $B 64 64 732303 | grep -E "^W=|contract:" | tr '\n' ' ' | sed -E "s/^.*depth=([0-9]+) smem.*contract: ([0-9.]+) ms.*/small dbg$d depth \1: \2 ms/"; echo; done; done > gpurun_out/r3w_depth.txt 2>&1
for d in 3 0; do for D in 1 2 3; do BLOCH_CONTRACT_DEPTH=$D CONTRACT_DBG=$d timeout 120 $B 512 512 732303 | grep -E "^W=|contract:" | tr '\n' ' ' | sed -E "s/^.*depth=([0-9]+) smem.*contract: ([0-9.]+) ms.*/cfg2tile dbg$d depth \1: \2 ms/"; echo; done; done >> gpurun_out/r3w_depth.txt 2>&1
