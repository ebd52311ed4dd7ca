# contraction pipeline depth cap (small tiles: config 3's short-run groups, config 0) 4 vs 6 vs 8
for D in 4 6 8; do
  for c in 3 0 1; do BLOCH_CONTRACT_MAXDEPTH=$D timeout 300 python tools/shard_probe.py $c 1 8 | sed "s/^/depth$D /"; done
done > gpurun_out/r3l_depth.txt 2>&1
