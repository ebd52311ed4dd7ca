# does the per-stage floor follow the number of TMA loads?  dbg 3 = no generation, no MMA; dbg 7 = also only one of the two U loads per stage
B=tools/microbench/contract_test
for shape in "64 64" "512 512"; do for d in 3 7 0 4; do CONTRACT_DBG=$d timeout 120 $B $shape 732303 | grep -E "contract:" | sed "s/^/shape $shape dbg$d /"; done; done > gpurun_out/r3v_tma_loads.txt 2>&1
