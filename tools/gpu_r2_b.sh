# round-2 check: GPU suite, shard probes with the fixed-point ring vs partial rows, quickbench
python -m pytest tests -q -m gpu --maxfail=30 -p no:cacheprovider > gpurun_out/pytest_b.txt 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_b.txt
{
python tools/shard_probe.py 2 1 2 4 8
python tools/shard_probe.py 1 1 2 4 8
python tools/shard_probe.py 4 1 2 4 8
echo "--- BLOCH_NO_RING=1"
BLOCH_NO_RING=1 python tools/shard_probe.py 2 2 4 8
BLOCH_NO_RING=1 python tools/shard_probe.py 1 2 4 8
BLOCH_NO_RING=1 python tools/shard_probe.py 4 1 2 4 8
} > gpurun_out/shards_b.txt 2>&1
CONFIGS="0 1 2 3 4" STEPS=5 bash tools/quickbench.sh > gpurun_out/quick_b.txt 2>&1
