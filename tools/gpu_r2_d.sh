{
python tools/shard_probe.py 2 1 8
python tools/shard_probe.py 1 1 8
python tools/shard_probe.py 4 1 8
BLOCH_NO_DISCARD=1 python tools/shard_probe.py 2 1 8
BLOCH_NO_CTA_FOLD=1 python tools/shard_probe.py 2 1 8
BLOCH_NO_CTA_FOLD=1 python tools/shard_probe.py 4 1 8
} > gpurun_out/shards_d.txt 2>&1
python -m pytest tests -q -m gpu --maxfail=10 -p no:cacheprovider -k "fuzz or segments or parity" > gpurun_out/pytest_d.txt 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_d.txt
