# round-2: CTA fold (in-kernel fold of the warp rows from L2) vs plain rows; GPU suite; shards; quickbench
python -m pytest tests -q -m gpu --maxfail=30 -p no:cacheprovider -x > gpurun_out/pytest_c.txt 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_c.txt
{
python tools/shard_probe.py 2 1 2 4 8
python tools/shard_probe.py 1 1 2 4 8
python tools/shard_probe.py 4 1 2 4 8
python tools/shard_probe.py 3 1 8
echo "--- BLOCH_NO_CTA_FOLD=1"
BLOCH_NO_CTA_FOLD=1 python tools/shard_probe.py 2 1 2 4 8
BLOCH_NO_CTA_FOLD=1 python tools/shard_probe.py 1 1 2 4 8
BLOCH_NO_CTA_FOLD=1 python tools/shard_probe.py 4 1 2 4 8
BLOCH_NO_CTA_FOLD=1 python tools/shard_probe.py 3 1 8
} > gpurun_out/shards_c.txt 2>&1
