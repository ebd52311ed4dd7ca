# accumulation segment length: time and error against the full-size reference goldens (BLOCH_CONTRACT_SEG stages per drain)
for SEG in 128 192 256 384; do
  for c in 2 4; do BLOCH_CONTRACT_SEG=$SEG timeout 300 python tools/shard_probe.py $c 1 | sed "s/^/seg$SEG /"; done
  BLOCH_CONTRACT_SEG=$SEG timeout 600 python -m pytest tests/test_gpu_fullsize_golden.py -m gpu -q -s -p no:cacheprovider -k "True" 2>&1 | grep "^config" | sed "s/^/seg$SEG /"
done > gpurun_out/r3k_seg.txt 2>&1
