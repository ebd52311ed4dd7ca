# small-tile contraction floor: W=64 windows, K=64 / 10-ish samples, 732k spins; dbg 1 = no generation, 2 = no MMA, 3 = neither
B=tools/microbench/contract_test
for shape in "64 64" "64 128" "128 64" "512 512"; do for d in 0 1 2 3; do CONTRACT_DBG=$d timeout 120 $B $shape 732303 | grep -E "^W=|contract" | tr '\n' ' ' | sed "s/^/dbg$d /"; echo; done; done > gpurun_out/r3u_small_tiles.txt 2>&1
