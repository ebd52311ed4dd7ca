# ncu source-level profile of the contraction kernel with neither generation nor MMA (dbg 3), small tile: where do the roles wait?
CONTRACT_DBG=3 timeout 600 ncu --set full --import-source on --clock-control none -k regex:contract_kernel -c 1 -o gpurun_out/r3x_dbg3_small tools/microbench/contract_test 64 64 732303 > gpurun_out/r3x_ncu.log 2>&1
