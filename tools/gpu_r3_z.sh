# full pipeline with the generators' phase-table loads removed (dbg 8): is the load wait the pacer?
B=tools/microbench/contract_test
for shape in "64 64" "512 512" "256 256"; do for d in 0 8 11; do CONTRACT_DBG=$d timeout 120 $B $shape 732303 | grep -E "contract:" | cut -c1-60 | sed "s|^|$shape dbg$d |"; done; done > gpurun_out/r3z_noload.txt 2>&1
