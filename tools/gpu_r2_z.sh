# U split fp32 (B) vs fp64 (A); ncu of the S=1 integrator on config 2 / 8; ncu of the generator alone (config-4 shape)
CONFIGS="1 2 4" ROUNDS=2 STEPS=6 bash tools/ab.sh > gpurun_out/z_ab.txt 2>&1
for L in A B; do BLOCH_LIB=$PWD/ab/lib$L.so timeout 900 python tools/shard_probe.py 2 2 8 | sed "s/^/$L /"; done > gpurun_out/z_shards.txt 2>&1
BLOCH_NO_GRAPH=1 timeout 600 ncu --set full --import-source on --clock-control none -k regex:integrate -c 1 -o gpurun_out/z_integ_cfg2_8 python tools/one_call.py 2 1 8 > gpurun_out/z_ncu1.log 2>&1
BLOCH_NO_GRAPH=1 timeout 600 ncu --set full --import-source on --clock-control none -k regex:integrate -c 1 -o gpurun_out/z_integ_cfg2 python tools/one_call.py 2 > gpurun_out/z_ncu2.log 2>&1
CONTRACT_DBG=2 BLOCH_CONTRACT_SEG=128 timeout 300 ncu --set full --import-source on --clock-control none -k regex:contract_kernel -c 1 -o gpurun_out/z_gen_only tools/microbench/contract_test 384 256 274145 > gpurun_out/z_ncu3.log 2>&1
