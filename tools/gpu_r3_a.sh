# HEAD evidence after container re-creation: full GPU suite, bench line, reference arm, shard probe, smoke
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r3a_pytest.txt 2>&1; echo "rc=$?" >> gpurun_out/r3a_pytest.txt
timeout 900 python bench.py > gpurun_out/r3a_bench.json 2> gpurun_out/r3a_bench.err; echo "rc=$?" >> gpurun_out/r3a_bench.err
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/r3a_reference.json 2> gpurun_out/r3a_reference.err
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r3a_smoke.txt 2>&1
timeout 600 python tools/shard_probe.py 2 1 2 4 8 > gpurun_out/r3a_shards.txt 2>&1
