# resident-table integrator v2 (staged records, shared-window addresses, packed bf16 split): parity, shard probe
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider -k "resident" > gpurun_out/r3d_pytest.txt 2>&1; echo "rc=$?" >> gpurun_out/r3d_pytest.txt
for c in 2 1 4; do
  timeout 600 python tools/shard_probe.py $c 1 2 4 8 | sed "s/^/resident /"
done > gpurun_out/r3d_shards.txt 2>&1
BLOCH_NO_GRAPH=1 timeout 600 ncu --set full --import-source on --clock-control none -k regex:resident -c 1 -o gpurun_out/r3d_res_cfg2 python tools/one_call.py 2 > gpurun_out/r3d_ncu2.log 2>&1
